"""GPU parity of the full query-and-correct engine on the reference's own
toy models: traces, outputs and metrics against fixtures recorded from the
reference (oracle/make_golden.py), and the reference's ablation / K-sweep
golden recipe (regen_goldens.py:29-66)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def card():
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200._device import require_cuda

    require_cuda()
    return card


def _events(trace):
    return [[e.step_index, e.sim_time, e.hit, e.candidate_len, e.accepted_len, e.lnew, e.cache_alive_nodes, e.event]
            for e in trace]


@pytest.mark.parametrize("idx", range(16))
def test_engine_matches_reference_run(card, idx):
    r = load_golden("engine.json")["runs"][idx]
    draft, target = card.models_from_dict(r["models"])
    cfg = card.EngineConfig.from_dict(r["config"])
    res = card.run_speculative(draft, target, r["prompt"], cfg)
    assert res.output == r["output"]
    assert _events(res.trace) == r["trace"]
    assert res.metrics.to_dict() == r["metrics"]
    van = card.run_vanilla(target, r["prompt"], cfg)
    assert van.output == r["vanilla_output"]
    assert van.metrics.to_dict() == r["vanilla_metrics"]


def test_reference_ablation_and_ksweep_goldens(card):
    g = load_golden("fixture_goldens.json")
    draft, target = card.models_from_dict(g["models"])
    ab = g["config"]["ablate"]
    base = card.EngineConfig.from_dict(ab)
    van = card.aggregate(card.run_vanilla(target, p, base).metrics for p in g["corpus"])
    assert van.to_dict() == pytest.approx(g["ablation"]["vanilla"], rel=1e-9)
    for variant, corrected in (("cache_only", False), ("cache_plus_correct", True)):
        c = card.EngineConfig.from_dict({**ab, "correction_enabled": corrected})
        got = card.aggregate(card.run_speculative(draft, target, p, c).metrics for p in g["corpus"])
        want = g["ablation"][variant]
        for k, v in want.items():
            assert getattr(got, k) == pytest.approx(v, rel=1e-9, abs=1e-12), (variant, k)
    ks = dict(g["config"]["ksweep"])
    for K in ks.pop("K_values"):
        c = card.EngineConfig.from_dict({**ks, "K": K})
        got = card.aggregate(card.run_speculative(draft, target, p, c).metrics for p in g["corpus"])
        for k, v in g["ksweep"][str(K)].items():
            assert getattr(got, k) == pytest.approx(v, rel=1e-9, abs=1e-12), (K, k)


def test_identity_draft_accepts_full_window(card):
    """test_engine.py:97-122 analog: identical draft/target with K=k=1."""
    doc = {"vocab_size": 32, "eos_token": None,
           "draft": {"type": "kgram", "seed": 5, "sharpness": 50.0, "forward_latency": 1.0},
           "target": {"type": "kgram", "seed": 5, "sharpness": 50.0, "forward_latency": 7.0}}
    d, t = card.models_from_dict(doc)
    cfg = card.EngineConfig(K=1, k=1, ratio=7, max_new_tokens=128)
    res = card.run_speculative(d, t, [1, 2, 3], cfg)
    assert res.output == card.run_vanilla(t, [1, 2, 3], cfg).output
    assert res.metrics.mean_acceptance_length == 8.0


def test_verify_api_matches_reference_cases(card):
    g = load_golden("verify.json")
    for c in g["cases"][:40]:
        d = [np.array(r) for r in c["dists"]]
        o = card.verify_greedy(d, c["cand"])
        assert [list(o.accepted), o.correction] == c["greedy"]
        rng = np.random.default_rng(c["seed"])
        o = card.verify_sampling(d, [1.0] * len(c["cand"]), c["cand"], rng)
        assert [list(o.accepted), o.correction] == c["sampling"]
        assert float(rng.random()) == c["next_uniform"]
    for s in g["samples"]:
        assert card.sample_index(np.random.default_rng(s["seed"]), np.array(s["p"])) == s["idx"]
