"""Tensor-parallel target (BASELINE configs[3]) on CPU: the
product's shard plan and shard weights (paper_2508_04462_b200.tp), run by
the fp32 TP restatement (oracle/tp_ref.py) under gloo with world sizes 2
and 3, reproduce the unsharded oracle's logits.  World 3 exercises the
uneven splits (kv heads 4 -> 2/1/1, FFN units and vocabulary tiles that do
not divide).  The device TP forward is tests/test_gpu_tp.py."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _cfg():
    from paper_2508_04462_b200.llama import LlamaConfig

    # 4 kv heads x GQA 2, FFN of 7 units of 64, a vocabulary of 5 tiles + a partial one
    return LlamaConfig(700, 128, 2, 8, 4, 16, 448, 500000.0, 1e-5, False, False,
                       dict(factor=8.0, low_freq_factor=1.0, high_freq_factor=4.0,
                            original_max_position_embeddings=64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle.tp_ref import tp_forward
    from paper_2508_04462_b200.llama import init_weights
    from paper_2508_04462_b200.tp import TPComm, shard_weights, tp_shards

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_num_threads(1)
        cfg = _cfg()
        w = init_weights(cfg, seed=5)
        w = {k: (v * 8 if k[0] == "l" and "norm" not in k else v) for k, v in w.items()}   # non-trivial mixing
        shards = tp_shards(cfg, world)
        toks = [int(t) for t in torch.randint(0, cfg.vocab_size, (37,), generator=torch.Generator().manual_seed(2))]
        got = tp_forward(cfg, shards, rank, shard_weights(cfg, w, shards[rank]), toks, TPComm())
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tp_sharded_forward_matches_unsharded(world):
    from oracle.llama_ref import RefLlama
    from paper_2508_04462_b200.llama import init_weights

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, lg = q.get(timeout=300)
        got[rank] = lg
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = _cfg()
    w = init_weights(cfg, seed=5)
    w = {k: (v * 8 if k[0] == "l" and "norm" not in k else v) for k, v in w.items()}
    toks = [int(t) for t in torch.randint(0, cfg.vocab_size, (37,), generator=torch.Generator().manual_seed(2))]
    want = RefLlama(cfg, w).full_logits(toks)
    for r in range(world):
        assert got[r].shape == want.shape
        assert torch.allclose(got[r], want, rtol=1e-4, atol=1e-4), (r, (got[r] - want).abs().max())
        assert torch.equal(got[r], got[0])   # every rank holds the same logits


def test_tp_shard_plan_uneven_and_covering():
    """70B over 7 ranks: whole GQA groups (kv 2/1/1/1/1/1/1), FFN and
    128-row vocabulary tiles covering the model exactly once."""
    from paper_2508_04462_b200.errors import ConfigError
    from paper_2508_04462_b200.llama import LlamaConfig
    from paper_2508_04462_b200.tp import shard_config, tp_shards

    c70 = LlamaConfig(128256, 8192, 80, 64, 8, 128, 28672, 500000.0, 1e-5, False, False, None)
    sh = tp_shards(c70, 7)
    assert [s.kv_heads[1] - s.kv_heads[0] for s in sh] == [2, 1, 1, 1, 1, 1, 1]
    assert [s.q_heads[1] - s.q_heads[0] for s in sh] == [16, 8, 8, 8, 8, 8, 8]
    assert sh[0].ffn[0] == 0 and sh[-1].ffn[1] == 28672
    assert all(a.ffn[1] == b.ffn[0] and a.vocab[1] == b.vocab[0] for a, b in zip(sh, sh[1:]))
    assert sh[-1].vocab[1] == 128256 and all(s.vocab_padded % 128 == 0 for s in sh)
    assert sorted({s.vocab_padded // 128 for s in sh}) == [143, 144]
    for s in sh:
        c = shard_config(c70, s)
        assert c.n_heads % c.n_kv_heads == 0 and c.ffn % 64 == 0 and c.vocab_size == s.vocab_padded
    with pytest.raises(ConfigError):
        tp_shards(c70, 9)   # 8 kv heads cannot be split over 9 ranks


def test_streamed_shards_equal_dict_shards():
    """A TP rank builds its shard from the weight stream (never the whole
    model): identical tensors to slicing init_weights, tied heads included."""
    import dataclasses

    from paper_2508_04462_b200.llama import init_weights, iter_weights
    from paper_2508_04462_b200.tp import shard_stream, shard_weights, tp_shards

    for cfg in (_cfg(), dataclasses.replace(_cfg(), vocab_size=768, tie_embeddings=True)):
        w = init_weights(cfg, 5)
        for sh in tp_shards(cfg, 3):
            a, b = shard_weights(cfg, w, sh), shard_stream(cfg, iter_weights(cfg, 5), sh)
            assert set(a) == set(b) and all(torch.equal(a[k], b[k]) for k in a)
