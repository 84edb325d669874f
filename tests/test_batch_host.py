"""Host logic of the batched decode (no GPU): per-request frontier budget and
the requests one forward can hold (batch.py)."""

from paper_2508_04462_b200.batch import CATCH_UP, MAX_ROWS, batch_config, max_batch
from paper_2508_04462_b200.engine import EngineConfig


def test_batch_config_shares_the_frontier_budget():
    cfg = EngineConfig(K=100, k=3, ratio=7, max_new_tokens=64)
    assert [batch_config(cfg, b).K for b in (1, 2, 3, 8, 32, 64, 500)] == [100, 50, 33, 12, 3, 1, 1]
    b = batch_config(cfg, 8)
    assert (b.k, b.ratio, b.max_new_tokens, b.query_depth, b.max_depth) == (3, 7, 64, 7, 14)


def test_max_batch_keeps_both_forwards_within_one_row_tile():
    for K, r in ((100, 7), (12, 7), (3, 7), (1, 7), (6, 5)):
        cfg = EngineConfig(K=K, k=3, ratio=r)
        B = max_batch(cfg)
        assert B >= 1
        assert B * (K + CATCH_UP) <= MAX_ROWS or B == 1
        assert B * (cfg.query_depth + 1) <= MAX_ROWS
        assert (B + 1) * (K + CATCH_UP) > MAX_ROWS or (B + 1) * (cfg.query_depth + 1) > MAX_ROWS
