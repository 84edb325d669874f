"""BASELINE configs[0] exactly: the tiny random-init fp32 transformer pair
at the reference's own engine configs (pkg/configs/default.json K=50 r=5
and k100_r7.json K=100 r=7, 512 new tokens, greedy) on pkg/corpus/smoke.jsonl
and 8 seeded 512-token prompts.  The fixtures were produced by the
REFERENCE engine (specache.run_speculative / run_vanilla, imported
read-only) driving the CPU fp32 transformer through its ToyModel protocol
(oracle/make_golden_tiny.py).  The device must emit the same tokens, the
same per-step trace (hits, candidate lengths, accepted prefixes, committed
counts, tree size after every step) and the same metrics."""

import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

CONFIGS = {
    "default.json": dict(K=50, k=3, ratio=5, temperature=0.0, max_new_tokens=512, mode="serial_sim",
                         correction_enabled=True, seed=0),
    "k100_r7.json": dict(K=100, k=3, ratio=7, temperature=0.0, max_new_tokens=512, mode="serial_sim",
                         correction_enabled=True, seed=0),
}


@pytest.fixture(scope="module")
def pair():
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200._device import require_cuda
    from paper_2508_04462_b200.llama import PRESETS, init_weights

    require_cuda()
    g = load_golden("tiny_pair.json")
    models = []
    for preset, seed, b, spec in zip(g["presets"], g["seeds"], (g["bias_draft"], g["bias_target"]),
                                     (g["spec_draft"], g["spec_target"])):
        cfg = PRESETS[preset]
        models.append(card.LlamaModel(cfg, dtype="fp32", weights=init_weights(cfg, seed),
                                      spec=card.ModelSpec(*spec), bias=card.LogitBias(**b)))
    return card, models[0], models[1], g["runs"]


def _ids():
    return [f"{c}-{i}" for c in CONFIGS for i in range(12)]


@pytest.mark.parametrize("which", _ids())
def test_tiny_pair_matches_reference_engine(pair, which):
    card, d, t, runs = pair
    cname, idx = which.rsplit("-", 1)
    r = [x for x in runs if x["config"] == cname][int(idx)]
    cfg = card.EngineConfig.from_dict(CONFIGS[cname])
    res = card.run_speculative(d, t, r["prompt"], cfg, use_graphs=False)
    assert res.output == r["output"]
    got = [[e.event, int(e.hit), e.candidate_len, e.accepted_len, e.lnew, e.cache_alive_nodes] for e in res.trace]
    assert got == r["trace"]
    m = res.metrics.to_dict()
    for k, v in r["metrics"].items():
        assert m[k] == pytest.approx(v, rel=1e-12, abs=1e-12), k
    assert r["output"] == r["vanilla"]   # the reference's own losslessness on this pair


@pytest.mark.parametrize("cname", list(CONFIGS))
def test_tiny_pair_graph_driver_matches_reference(pair, cname):
    """The throughput (CUDA-graph) driver on the same fixtures: tokens and
    the trace minus tree sizes (the graph driver does not read them)."""
    card, d, t, runs = pair
    cfg = card.EngineConfig.from_dict(CONFIGS[cname])
    for r in [x for x in runs if x["config"] == cname][4:7]:
        res = card.run_speculative(d, t, r["prompt"], cfg, use_graphs=True)
        assert res.output == r["output"]
        got = [[e.event, int(e.hit), e.candidate_len, e.accepted_len, e.lnew] for e in res.trace]
        assert got == [x[:5] for x in r["trace"]]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tiny_pair_sampling_matches_oracle_engine(pair, seed):
    """T=1 on the transformer pair (weak spot of round 1): the device fp64
    softmax (card_softmax64) + stochastic accept (card_verify_probs) with the
    host PCG64 uniforms emits the tokens of the oracle engine running the
    CPU fp32 transformer with numpy's sampling (verify.py:43-51, 83-132) —
    same seed, same draws, same committed stream and per-step trace."""
    from oracle import card_oracle as O
    from oracle.llama_ref import RefModel
    from paper_2508_04462_b200.llama import PRESETS, init_weights

    card, d, t, _ = pair
    g = load_golden("tiny_pair.json")
    bd, bt = card.LogitBias(**g["bias_draft"]), card.LogitBias(**g["bias_target"])
    cd, ct = PRESETS[g["presets"][0]], PRESETS[g["presets"][1]]
    rd = RefModel(cd, init_weights(cd, g["seeds"][0]), forward_latency=g["spec_draft"][1], bias=bd)
    rt = RefModel(ct, init_weights(ct, g["seeds"][1]), forward_latency=g["spec_target"][1],
                  params_billions=g["spec_target"][0], bias=bt)
    import numpy as np

    prompt = [int(x) for x in np.random.default_rng(500 + seed).integers(0, ct.vocab_size, 24)]
    cfg = dict(K=12, k=3, ratio=4, temperature=1.0, max_new_tokens=64, seed=seed)
    out, trace = O.run_serial(rd, rt, prompt, **cfg)
    res = card.run_speculative(d, t, prompt, card.EngineConfig(**cfg), use_graphs=False)
    assert res.output == out
    strip = lambda tr: [(e.event, e.hit, e.candidate_len, e.accepted_len, e.lnew) for e in tr]  # noqa: E731
    assert strip(res.trace) == strip(trace)
    van = card.run_vanilla(t, prompt, card.EngineConfig(**cfg))
    assert van.output == O.run_vanilla(rt, prompt, temperature=1.0, max_new_tokens=64, seed=seed)[0]
