"""GPU parity: operator plug-in kernels and the device candidate tree
against the CPU oracle and the reference-generated goldens.

Bit-exactness contract: integer / index / structural state is compared
exactly.  Floating state is compared exactly against the oracle run with
the correctly rounded log/exp the device implements; against the goldens
(glibc math.log/exp, misrounded on ~0.04% of inputs) fp64 fields may
differ by at most 1 ulp and the structure must still match exactly.
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import card_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def card():
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200._device import require_cuda

    require_cuda()
    return card


def ulp_close(a, b, ulps=1):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    ok = (a == b) | (np.abs(a - b) <= ulps * np.spacing(np.maximum(np.abs(a), np.abs(b))))
    return bool(ok.all())


# ------------------------------------------------------------ correctly rounded libm
def test_log_exp_correctly_rounded(card):
    import torch
    from paper_2508_04462_b200._device import ptr, stream_ptr
    from paper_2508_04462_b200._lib import lib

    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.random(3000) ** 3, rng.random(1000) * 1e-200, [1.0, 0.5, 0.25, 1e-300]])
    es = np.concatenate([-rng.random(3000) * 60.0, -rng.random(500) * 740, rng.random(500) * 700, [0.0, -1.0]])
    x = torch.tensor(xs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    assert lib().card_log_cr(ptr(x), ptr(y), x.numel(), stream_ptr()) == 0
    got = y.cpu().numpy()
    want = np.array([O.cr_log(float(v)) for v in xs])
    assert np.array_equal(got, want)
    glibc = np.array([math.log(float(v)) for v in xs])
    assert (got != glibc).mean() < 0.005 and ulp_close(got, glibc)
    e = torch.tensor(es, dtype=torch.float64, device="cuda")
    y = torch.empty_like(e)
    assert lib().card_exp_cr(ptr(e), ptr(y), e.numel(), stream_ptr()) == 0
    got = y.cpu().numpy()
    want = np.array([O.cr_exp(float(v)) for v in es])
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, [(es[i], got[i], want[i]) for i in bad[:8]]


# ------------------------------------------------------------ operator plug-in
def test_kgram_dist_vs_golden(card):
    kern = card.get_kernels()
    mism = total = 0
    for c in load_golden("kernels.json")["kgram"]:
        got = kern.kgram_dist(c["seed"], c["seed2"], c["mix_weight"], tuple(c["tail"]), c["V"],
                              c["sharpness"], c["temperature"])
        want_cr = O.kgram_dist(c["seed"], c["seed2"], c["mix_weight"], tuple(c["tail"]), c["V"],
                               c["sharpness"], c["temperature"], exp_fn=O.cr_exp)
        assert got.tolist() == want_cr.tolist()           # bit-exact vs the CR twin
        assert ulp_close(got, c["out"], ulps=2)            # glibc reference: <= 2 ulp
        mism += int((got != np.array(c["out"])).sum())
        total += got.size
    assert mism / total < 0.01


def test_rows_topk_vs_golden(card):
    kern = card.get_kernels()
    for c in load_golden("kernels.json")["rows_topk"]:
        got = kern.rows_topk(np.array(c["dists"]), c["k"])
        assert [[[t, p] for t, p in r] for r in got] == c["rows"]


def test_rows_topk_large_vocab(card):
    kern = card.get_kernels()
    rng = np.random.default_rng(5)
    d = rng.random((7, 5000))
    d[:, ::3] = 0.25          # ties everywhere
    d = d / d.sum(axis=1, keepdims=True)
    assert kern.rows_topk(d, 5) == O.rows_topk(d, 5)


# ------------------------------------------------------------ device tree
def dev_state(cache):
    s = cache._snapshot()
    st = s["state"]
    return dict(token=s["token"], parent=s["parent"], layer=s["layer"], score=s["score"], edge=s["edge"],
                alive=s["alive"], frontier=s["frontier"], root=s["root"], epoch=s["epoch"], dead=s["dead"])


def oracle_state(t):
    return dict(token=t.token, parent=t.parent, layer=t.layer, score=t.score, edge=t.edge, alive=t.alive,
                frontier=t.frontier, root=t.root, epoch=t.epoch, dead=t.dead)


STRUCT = ("token", "parent", "layer", "alive", "frontier", "root", "epoch", "dead")


@pytest.mark.parametrize("idx", range(24))
def test_cache_replay_vs_reference(card, idx):
    """Replay the reference-recorded op sequence on the device; compare to the
    CR oracle bit-exactly and to the reference's own states (<= 1 ulp)."""
    sc = load_golden("cache_ops.json")[idx]
    cache = card.TreeCache(sc["root"], card.CacheConfig(sc["K"], sc["k"], sc["max_depth"]), eos_token=sc["eos"])
    twin = O.SoATree(sc["root"], sc["K"], sc["k"], sc["max_depth"], sc["eos"], log_fn=O.cr_log)
    for n_op, op in enumerate(sc["ops"]):
        if op["op"] == "expand":
            try:
                new = cache.expand_layer(np.array(op["dists"]))
                res = dict(status="ok", new=new)
            except card.FrontierFull:
                res = dict(status="frontier_full")
            try:
                twin.expand(np.array(op["dists"]))
            except O.OracleFrontierFull:
                pass
            assert res == op["result"], n_op
        elif op["op"] == "query":
            q = cache.query(op["depth"])
            hit, path, toks, edges = twin.query(op["depth"])
            assert (q.hit, q.path, q.tokens, q.edge_logps) == (hit, path, toks, edges), n_op
            r = op["result"]
            assert (q.hit, q.path, q.tokens) == (r["hit"], r["path"], r["tokens"]), n_op
            assert ulp_close(q.edge_logps, r["edges"]), n_op
            continue
        else:
            try:
                nr = cache.correct(op["accepted"], op["correction"])
                res = dict(status="ok", new_root=nr)
            except card.ProtocolError:
                res = dict(status="protocol_error")
            try:
                twin.correct(op["accepted"], op["correction"])
            except O.OracleProtocolError:
                pass
            assert res == op["result"], n_op
        got = dev_state(cache)
        assert got == oracle_state(twin), n_op
        want = op["state"]
        for f in STRUCT:
            assert got[f] == want[f], (n_op, f)
        assert ulp_close(got["score"], want["score"], ulps=2) and ulp_close(got["edge"], want["edge"]), n_op
        assert cache.dump() == want["dump"], n_op


def test_cache_churn_random(card):
    """Long random churn through many compactions, device vs CR oracle."""
    rng = np.random.default_rng(123)
    for trial in range(4):
        V, K, k, D = 40, int(rng.integers(4, 40)), int(rng.integers(1, 4)), int(rng.integers(3, 9))
        model = O.OracleKGram(seed=trial, vocab_size=V, order=2, sharpness=6.0)
        cache = card.TreeCache(3, card.CacheConfig(K, k, D))
        twin = O.SoATree(3, K, k, D, log_fn=O.cr_log)
        base = [1, 3]
        for step in range(120):
            if rng.random() < 0.6:
                paths = [[twin.token[x] for x in twin.path_to(h)] for h in twin.expansion_parents()]
                dists = np.vstack([O.kgram_dist(model.seed, 0, 0.0, tuple((base + p)[-2:]), V, 6.0, 1.0,
                                                exp_fn=O.cr_exp) for p in paths])
                full = False
                try:
                    twin.expand(dists)
                except O.OracleFrontierFull:
                    full = True
                try:
                    cache.expand_layer(dists)
                    assert not full
                except card.FrontierFull:
                    assert full
            else:
                hit, path, toks, _ = twin.query(int(rng.integers(1, D + 1)))
                n = int(rng.integers(0, len(toks) + 1)) if hit else 0
                corr = int(toks[n]) if (hit and n < len(toks) and rng.random() < 0.5) else int(rng.integers(0, V))
                twin.correct(toks[:n], corr)
                cache.correct(toks[:n], corr)
                base = base + list(toks[:n]) + [corr]
            assert dev_state(cache) == oracle_state(twin), (trial, step)
        assert cache.alive_below_root() == twin.alive_below_root()


def test_cache_errors(card):
    cache = card.TreeCache(0, card.CacheConfig(K=2, k=2, max_depth=1))
    with pytest.raises(card.InputError):
        cache.expand_layer(np.array([[0.5, 0.6]]))
    with pytest.raises(card.InputError):
        cache.expand_layer(np.array([[1.1, -0.1]]))
    with pytest.raises(card.InputError):
        cache.expand_layer(np.ones((3, 2)) / 2.0)
    cache.expand_layer(np.array([[0.25, 0.75]]))
    with pytest.raises(card.FrontierFull):
        cache.expand_layer(np.ones((2, 2)) / 2.0)
    with pytest.raises(card.ProtocolError):
        cache.correct([5], 1)
    with pytest.raises(card.InputError):
        cache.correct([], None)
    with pytest.raises(card.InputError):
        card.TreeCache(-1, card.CacheConfig(1, 1, 1))
    with pytest.raises(card.ConfigError):
        card.CacheConfig(0, 1, 1)


def test_advance_root_and_reset(card):
    cache = card.TreeCache(0, card.CacheConfig(K=3, k=2, max_depth=4))
    twin = O.SoATree(0, 3, 2, 4, log_fn=O.cr_log)
    d = np.array([[0.5, 0.3, 0.2]])
    cache.expand_layer(d)
    twin.expand(d)
    d2 = np.array([[0.6, 0.4, 0.0], [0.1, 0.1, 0.8]])
    cache.expand_layer(d2)
    twin.expand(d2)
    assert cache.advance_root([0], 0) == twin.advance_root([0], 0)
    assert dev_state(cache) == oracle_state(twin)
    assert cache.advance_root([], 2) is False and twin.advance_root([], 2) is False
    cache.reset(7)
    twin.reset(7)
    assert dev_state(cache) == oracle_state(twin)
