"""Paged KV: every request takes its prefix KV pages from its
runtime's PagePool, and the row builders (card_draft_rows /
card_target_rows), the attention (card_attention_paged) and the draft KV
promotion (card_draft_promote) address the prefix through the request's
page table.  A request placed on scattered, out-of-order pages of a
fragmented pool must decode exactly what it decodes on contiguous pages:
same tokens, same trace (bf16 CARD, both drivers), and AR likewise."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200._device import require_cuda
    from paper_2508_04462_b200.llama import PRESETS, init_weights

    require_cuda()
    bias = card.LogitBias(seed=11, order=2, sharpness=4000.0)
    ct, cd = PRESETS["small-target"], PRESETS["small-draft"]
    t = card.LlamaModel(ct, dtype="bf16", weights=init_weights(ct, 2), spec=card.ModelSpec(8.0, 7.0), bias=bias)
    d = card.LlamaModel(cd, dtype="bf16", weights=init_weights(cd, 1), spec=card.ModelSpec(1.0, 1.0), bias=bias)
    return card, d, t


def _fragment(rt):
    """Take every page of the pool, then give back two of every three: the
    next requests get pages scattered over the pool (stride 3)."""
    from paper_2508_04462_b200.llama import PageTable

    pool = rt.page_pool
    hold = [PageTable(pool, 1, rt.dev) for _ in range(len(pool.free))]
    keep = []
    for i, h in enumerate(hold):
        if i % 3 == 2:
            keep.append(h)    # the others are dropped: their pages return to the pool
    return keep


@pytest.mark.parametrize("use_graphs", [False, True])
def test_fragmented_pages_decode_identically(pair, use_graphs):
    card, d, t = pair
    prompt = [int(x) for x in np.random.default_rng(31).integers(0, t.vocab.size, 150)]
    cfg = card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=120)
    t.__dict__.pop("_card_sessions", None)
    ref = card.run_speculative(d, t, prompt, cfg, use_graphs=use_graphs)
    van_ref = card.run_vanilla(t, prompt, cfg)
    t.__dict__.pop("_card_sessions", None)
    import gc

    gc.collect()
    holders = [_fragment(m._runtime) for m in (d, t)]
    from paper_2508_04462_b200.engine import DeviceRun

    run = DeviceRun(d, t, prompt, cfg)
    for ad in (run.da, run.ta):
        pg = ad.pages.pages
        assert pg != sorted(pg) or any(b - a != 1 for a, b in zip(pg, pg[1:])), pg   # really scattered
    del run
    res = card.run_speculative(d, t, prompt, cfg, use_graphs=use_graphs)
    van = card.run_vanilla(t, prompt, cfg)
    assert res.output == ref.output and van.output == van_ref.output == res.output
    strip = lambda tr: [(e.event, e.hit, e.candidate_len, e.accepted_len, e.lnew) for e in tr]  # noqa: E731
    assert strip(res.trace) == strip(ref.trace)
    del holders


def test_page_pool_accounting(pair):
    """Requests draw disjoint pages; they go back to the pool when a request
    is dropped; a request the pool cannot serve raises instead of aliasing
    another request's KV."""
    import gc

    card, d, t = pair
    from paper_2508_04462_b200.errors import ConfigError
    from paper_2508_04462_b200.llama import PageTable

    rt = t._runtime
    pool = rt.page_pool
    gc.collect()
    n0 = len(pool.free)
    per = rt.prefix_slots // 64
    tabs = [rt.page_table() for _ in range(n0 // per)]
    taken = sorted(p for tb in tabs for p in tb.pages)
    assert len(set(taken)) == len(taken) == (n0 // per) * per          # disjoint pages
    with pytest.raises(ConfigError):
        PageTable(pool, pool.n_pages + 1, rt.dev)
    del tabs, taken
    gc.collect()
    assert len(pool.free) == n0
