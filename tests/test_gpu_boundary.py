"""GPU tests of the drop-in boundary pieces the engine tests do not reach
directly: the operator-level ``extension_pool`` (card_cache_pool,
cache.py:190-222), the verify outcome with KV rollback and uniform counts
(card_verify_result; verify.py:80,104-132), and the tree
mask (mask.py:90-217) on the device tree — including the ancestor lists
the device tree attention reads for every frontier row."""

import numpy as np
import pytest

from oracle import card_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def card():
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200._device import require_cuda

    require_cuda()
    return card


def _kg(seed, V, sharp=8.0):
    return O.OracleKGram(seed=seed, vocab_size=V, order=2, sharpness=sharp)


def _dists(tree, model, base):
    return np.vstack([model.next_distribution(base + [tree.token[x] for x in tree.path_to(h)])
                      for h in tree.expansion_parents()])


@pytest.mark.parametrize("seed", range(6))
def test_extension_pool_matches_oracle(card, seed):
    """Device extension_pool == the reference pool (same tuples, same order,
    bit-exact fp64 weights with the correctly rounded log), including EOS
    parents that are skipped and rows with less support than k."""
    rng = np.random.default_rng(seed)
    V = int(rng.integers(6, 40))
    K, k = int(rng.integers(2, 9)), int(rng.integers(1, 4))
    eos = int(rng.integers(0, V)) if seed % 2 else None
    model = _kg(seed, V, sharp=float(rng.uniform(2, 30)))
    dev = card.TreeCache(1, card.CacheConfig(K, k, 6), eos_token=eos)
    ora = O.SoATree(1, K, k, 6, eos, log_fn=O.cr_log)
    for step in range(4):
        d = _dists(ora, model, [1])
        if step == 2:   # a sparse row: support below k
            d[0] = 0.0
            d[0, 3] = 1.0
        got = dev.extension_pool(d)
        want = ora.pool(d)
        assert [(c.token, c.weight, c.parent_index, c.edge_logp) for c in got] == \
            [(t, w, pi, e) for w, t, pi, e in want]
        dev.expand_layer(d)
        ora.expand(d)
        assert dev.frontier == ora.frontier


def test_extension_pool_rejects_bad_rows(card):
    dev = card.TreeCache(0, card.CacheConfig(4, 2, 4))
    with pytest.raises(card.InputError):
        dev.extension_pool(np.array([[0.5, 0.6]]))
    with pytest.raises(card.InputError):
        dev.extension_pool(np.array([[1.5, -0.5]]))
    with pytest.raises(card.InputError):
        dev.extension_pool(np.ones((2, 2)) / 2)   # one parent (the root), two rows


@pytest.mark.parametrize("temperature", [0.0, 1.0])
def test_verify_result_kv_rollback_and_uniforms(card, temperature):
    """Per target step: kv_keep = C_prev + committed - 1 (= C + n unclipped),
    rolled-back rows = L + 1 - committed, and the uniforms consumed follow
    the reference draw order (miss 1; hit with rejection at n: n + 2; full
    accept: L + 1)."""
    import torch

    from paper_2508_04462_b200._device import ptr, stream_ptr
    from paper_2508_04462_b200._lib import lib
    from paper_2508_04462_b200.engine import DeviceRun

    doc = {"vocab_size": 48, "eos_token": None,
           "draft": {"type": "kgram", "seed": 11, "order": 2, "sharpness": 80.0, "mix_seed": 131,
                     "mix_weight": 0.02, "forward_latency": 1.0},
           "target": {"type": "kgram", "seed": 11, "order": 2, "sharpness": 80.0, "forward_latency": 5.0}}
    d, t = card.models_from_dict(doc)
    cfg = card.EngineConfig(K=8, k=2, ratio=5, max_new_tokens=90, temperature=temperature, seed=4)
    run = DeviceRun(d, t, [3, 9, 27], cfg)
    run.prefill()
    out = torch.zeros(6, dtype=torch.int32, device="cuda")
    for _ in range(cfg.query_depth):
        if run.draft_step_sync() == 0:
            break
    kinds = set()
    n_tok = 0
    while True:
        for _ in range(cfg.ratio):
            if run.draft_step_sync() == 0:
                break
        before = run.read_state()
        E = run.target_step_sync()
        assert lib().card_verify_result(run.E_ptr, ptr(out), stream_ptr()) == 0
        n, corr, used, keep, drop, cnt = out.cpu().tolist()
        L = E.L if E.hit else 0
        assert (n, corr, cnt) == (E.n_acc, E.corr, E.n_commit)
        assert keep == before.C + cnt - 1 and drop == L + 1 - cnt
        if cnt == n + 1:
            assert keep == before.C + n
        if temperature > 0.0:
            want = 1 if not E.hit else (L + 1 if n == L else n + 2)
            assert used == want, (E.hit, L, n, used)
        else:
            assert used == 0
        kinds.add("full" if E.hit and n == L else ("reject" if E.hit else "miss"))
        n_tok += cnt
        if E.done:
            break
        run.correct_sync()
    assert n_tok == cfg.max_new_tokens
    assert {"full", "reject"} <= kinds


def test_device_tree_mask_matches_oracle_and_attention_rows(card):
    """Across expansions and corrections of a device run, every frontier
    row's ancestor list in the draft row block (what the tree attention
    reads, card_engine.cu draft_rows_kernel) is exactly that row's
    MaskBuilder mask over the device tree (incremental chains, epoch
    resyncs after each correction)."""
    from paper_2508_04462_b200.engine import DeviceRun
    from paper_2508_04462_b200.mask import MaskBuilder

    doc = {"vocab_size": 40, "eos_token": None,
           "draft": {"type": "kgram", "seed": 7, "order": 2, "sharpness": 20.0, "forward_latency": 1.0},
           "target": {"type": "kgram", "seed": 7, "order": 2, "sharpness": 20.0, "mix_seed": 3,
                      "mix_weight": 0.2, "forward_latency": 4.0}}
    d, t = card.models_from_dict(doc)
    cfg = card.EngineConfig(K=6, k=3, ratio=4, max_new_tokens=40)
    run = DeviceRun(d, t, [5, 6, 7], cfg)
    run.prefill()
    mb = MaskBuilder(run.cache)
    checked = 0
    for cycle in range(8):
        for _ in range(cfg.ratio):
            st = run.cache.state()
            mask = mb.frontier_mask() if st.n_frontier else None
            front = run.cache.frontier
            w = run.draft_step_sync()
            if mask is not None:
                blk = run.drt.rows
                M, nout = int(blk.M.item()), int(blk.n_out.item())
                assert nout == len(front)
                extra = blk.extra.view(-1, blk.extra_max).cpu().numpy()
                n_extra = blk.n_extra.cpu().numpy()
                out_rows = blk.out_rows.cpu().numpy()
                base = run.da.rt.tree_base if hasattr(run.da, "rt") else 0
                for i, h in enumerate(front):
                    m = int(out_rows[i])
                    got = [int(x) - base for x in extra[m, :n_extra[m]]]
                    want = [mask.columns[c] for c in np.flatnonzero(mask.bits[i])]
                    # chains are root-side first in both; compare as ordered lists
                    assert got == sorted(want, key=lambda x: run.cache.arena[x].layer), (cycle, i)
                checked += 1
            if w == 0:
                break
            mb.note_layer(run.cache.frontier)
        E = run.target_step_sync()
        if E.done:
            break
        run.correct_sync()
    assert checked >= 4


def test_verify_sampling_checks_conditionals_lazily(card):
    """verify.py:104-112: a bad draft conditional raises only when the walk
    reaches it; a rejection before it returns normally, with the generator
    advanced exactly as the reference advances it."""
    V = 5
    p0 = np.array([0.0, 0.0, 0.0, 0.0, 1.0])   # rejects candidate 1 at position 0 (p=0)
    pu = np.full(V, 0.2)
    rng = np.random.default_rng(3)
    out = card.verify_sampling([p0, pu, pu], [1.0, 0.0], [1, 2], rng)
    assert out.accepted == () and out.correction == 4
    ref = np.random.default_rng(3)
    ref.random(2)   # one coin + one residual sample
    assert rng.random() == ref.random()
    p1 = np.array([0.0, 1.0, 0.0, 0.0, 0.0])   # accepts candidate 1 surely, then hits q=0
    rng = np.random.default_rng(4)
    with pytest.raises(card.ProtocolError):
        card.verify_sampling([p1, pu, pu], [1.0, 0.0], [1, 2], rng)
    ref = np.random.default_rng(4)
    ref.random(1)
    assert rng.random() == ref.random()
