"""Pin the CPU oracle against fixtures produced by the reference itself
(oracle/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import card_oracle as O
from conftest import load_golden


def test_kgram_dist_bitexact():
    for c in load_golden("kernels.json")["kgram"]:
        got = O.kgram_dist(c["seed"], c["seed2"], c["mix_weight"], tuple(c["tail"]), c["V"],
                           c["sharpness"], c["temperature"])
        assert got.tolist() == c["out"]


def test_rows_topk_bitexact():
    for c in load_golden("kernels.json")["rows_topk"]:
        got = O.rows_topk(np.array(c["dists"]), c["k"])
        assert [[[t, p] for t, p in r] for r in got] == c["rows"]


def _state(tree):
    return dict(token=tree.token, parent=tree.parent, layer=tree.layer, score=tree.score,
                edge=tree.edge, alive=tree.alive, frontier=tree.frontier, root=tree.root,
                epoch=tree.epoch, dead=tree.dead, alive_below=tree.alive_below_root(),
                dump=tree.dump())


@pytest.mark.parametrize("idx", range(24))
def test_cache_ops_replay(idx):
    sc = load_golden("cache_ops.json")[idx]
    tree = O.SoATree(sc["root"], sc["K"], sc["k"], sc["max_depth"], sc["eos"])
    for op in sc["ops"]:
        if op["op"] == "expand":
            try:
                new = tree.expand(np.array(op["dists"]))
                res = dict(status="ok", new=new)
            except O.OracleFrontierFull:
                res = dict(status="frontier_full")
            assert res == op["result"]
            assert _state(tree) == op["state"]
        elif op["op"] == "query":
            hit, path, toks, edges = tree.query(op["depth"])
            assert dict(hit=hit, path=path, tokens=toks, edges=edges) == op["result"]
        else:
            try:
                nr = tree.correct(op["accepted"], op["correction"])
                res = dict(status="ok", new_root=nr)
            except O.OracleProtocolError:
                res = dict(status="protocol_error")
            assert res == op["result"]
            assert _state(tree) == op["state"]   # a rejected walk mutates nothing


def test_verify_cases():
    g = load_golden("verify.json")
    for c in g["cases"]:
        d = [np.array(r) for r in c["dists"]]
        acc, corr = O.verify_greedy(d, c["cand"])
        assert [list(acc), corr] == c["greedy"]
        rng = np.random.default_rng(c["seed"])
        acc, corr = O.verify_sampling(d, [1.0] * len(c["cand"]), c["cand"], rng)
        assert [list(acc), corr] == c["sampling"]
        assert float(rng.random()) == c["next_uniform"]
    for s in g["samples"]:
        assert O.sample_index(np.random.default_rng(s["seed"]), np.array(s["p"])) == s["idx"]


def _events(trace):
    return [[e.step_index, e.sim_time, e.hit, e.candidate_len, e.accepted_len, e.lnew,
             e.cache_alive_nodes, e.event] for e in trace]


@pytest.mark.parametrize("idx", range(16))
def test_engine_runs(idx):
    r = load_golden("engine.json")["runs"][idx]
    d, t = O.load_pair(r["models"])
    out, trace = O.run_serial(d, t, r["prompt"], **r["config"])
    assert out == r["output"]
    assert _events(trace) == r["trace"]
    assert O.finalize(trace, t.params_billions, t.forward_latency, d.params_billions) == r["metrics"]
    vout, vtrace = O.run_vanilla(t, r["prompt"], r["config"]["temperature"],
                                 r["config"]["max_new_tokens"], r["config"]["seed"])
    assert vout == r["vanilla_output"]
    assert O.finalize(vtrace, t.params_billions, t.forward_latency) == r["vanilla_metrics"]


def test_reference_fixture_goldens():
    """The reference's ablation / K-sweep recipe (regen_goldens.py:29-66)."""
    g = load_golden("fixture_goldens.json")
    d, t = O.load_pair(g["models"])
    ab = g["config"]["ablate"]
    van = O.aggregate(O.finalize(O.run_vanilla(t, p, 0.0, ab["max_new_tokens"], ab["seed"])[1],
                                 t.params_billions, t.forward_latency) for p in g["corpus"])
    assert van == pytest.approx(g["ablation"]["vanilla"], rel=1e-12)
    for variant, corrected in (("cache_only", False), ("cache_plus_correct", True)):
        runs = [O.finalize(O.run_serial(d, t, p, correction_enabled=corrected, **ab)[1],
                           t.params_billions, t.forward_latency, d.params_billions)
                for p in g["corpus"]]
        assert O.aggregate(runs) == g["ablation"][variant]


def test_kgram_uniforms_vectorised_equals_scalar():
    """The numpy k-gram uniforms (CPU baselines' logit bias) are the scalar
    restatement's values bit for bit (_kernels_py.py:27-45)."""
    import numpy as np

    from oracle.card_oracle import kgram_uniforms, kgram_uniforms_np

    for seed, tail in [(11, [3, 5]), (131, [0]), (7, [123456, 99]), (0, [])]:
        assert np.array_equal(np.array(kgram_uniforms(seed, tail, 3000)), kgram_uniforms_np(seed, tail, 3000))
