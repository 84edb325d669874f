"""Front end (cli.py): argument and file handling on CPU; one `run` and one
`ablate` through the device engine on the GPU (k-gram pair of the
reference's pair_70b_1b.json shape)."""

import json

import pytest

PAIR = {"vocab_size": 64, "eos_token": None,
        "draft": {"type": "kgram", "seed": 11, "order": 2, "sharpness": 60.0, "mix_seed": 131, "mix_weight": 0.05,
                  "params_billions": 1.0, "forward_latency": 10.0},
        "target": {"type": "kgram", "seed": 11, "order": 2, "sharpness": 60.0, "params_billions": 70.0,
                   "forward_latency": 70.0}}


def _files(tmp_path, corpus_lines, config=None):
    m = tmp_path / "pair.json"
    m.write_text(json.dumps(PAIR))
    c = tmp_path / "prompts.jsonl"
    c.write_text("\n".join(corpus_lines) + "\n")
    cfg = None
    if config is not None:
        cfg = tmp_path / "cfg.json"
        cfg.write_text(json.dumps(config))
    return str(m), str(c), (str(cfg) if cfg else None)


def test_corpus_errors_carry_file_and_line(tmp_path):
    from paper_2508_04462_b200.cli import read_corpus
    from paper_2508_04462_b200.errors import CorpusFormatError

    _, c, _ = _files(tmp_path, ['{"id": "a", "tokens": [1, 2]}', '{"id": "b", "tokens": [1, 99]}'])
    with pytest.raises(CorpusFormatError) as e:
        read_corpus(c, 64)
    assert e.value.line_no == 2
    _, c, _ = _files(tmp_path, ['{"id": "a", "text": "hi"}'])
    with pytest.raises(CorpusFormatError, match="at least 256"):
        read_corpus(c, 64)
    _, c, _ = _files(tmp_path, [""])
    with pytest.raises(CorpusFormatError, match="empty"):
        read_corpus(c, 64)
    _, c, _ = _files(tmp_path, ['{"id": "a", "tokens": [3, 4], "text": "x"}'])
    with pytest.raises(CorpusFormatError, match="exactly one"):
        read_corpus(c, 64)


def test_ratio_auto_and_unknown_keys(tmp_path):
    from paper_2508_04462_b200.cli import engine_config
    from paper_2508_04462_b200.errors import ConfigError
    from paper_2508_04462_b200.lm import models_from_dict

    draft, target = models_from_dict(PAIR)
    cfg = engine_config({"K": 8, "ratio": "auto"}, draft, target, {"seed": 3})
    assert cfg.ratio == 7 and cfg.query_depth == 7 and cfg.max_depth == 14 and cfg.seed == 3
    with pytest.raises(ConfigError):
        engine_config({"K": 8, "bogus": 1}, draft, target, {})


def test_cli_reports_errors_with_exit_code(tmp_path, capsys):
    from paper_2508_04462_b200.cli import main

    m, c, cfg = _files(tmp_path, ['{"id": "a", "tokens": [1, 200]}'], {"K": 4})
    assert main(["run", "--models", m, "--corpus", c, "--config", cfg]) == 2
    assert "prompts.jsonl:1" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_run_and_ablate_on_device(tmp_path, capsys):
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200.cli import main

    m, c, cfg = _files(tmp_path, ['{"id": "p0", "tokens": [1, 2, 3]}', '{"id": "p1", "tokens": [5, 9]}'],
                       {"K": 16, "k": 3, "ratio": 5, "max_new_tokens": 40})
    out, trace = str(tmp_path / "out.jsonl"), str(tmp_path / "trace.jsonl")
    assert main(["run", "--models", m, "--corpus", c, "--config", cfg, "--out", out, "--trace", trace]) == 0
    recs = [json.loads(x) for x in open(out)]
    assert [r["id"] for r in recs] == ["p0", "p1", "__aggregate__"]
    draft, target = card.load_models_file(m)
    want = card.run_speculative(draft, target, [1, 2, 3], card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=40))
    assert recs[0]["output"] == want.output
    assert sum(1 for _ in open(trace)) == len(want.trace) + len(
        card.run_speculative(draft, target, [5, 9], card.EngineConfig(K=16, k=3, ratio=5, max_new_tokens=40)).trace)
    assert main(["ablate", "--models", m, "--corpus", c, "--config", cfg, "--out", out]) == 0
    recs = [json.loads(x) for x in open(out)]
    # the reference's record shape (cli.py:278-288): per prompt, then an aggregate per variant
    assert [(r["id"], r["variant"]) for r in recs] == [(i, v) for v in ("vanilla", "cache_only", "cache_plus_correct")
                                                         for i in ("p0", "p1", "__aggregate__")]
    ab = {r["variant"]: r["metrics"] for r in recs if r["id"] == "__aggregate__"}
    assert ab["vanilla"]["mean_acceptance_length"] == 1.0
    assert ab["cache_plus_correct"]["mean_acceptance_length"] >= ab["cache_only"]["mean_acceptance_length"] > 1.0


def test_sweep_spec_parsing():
    """--sweep param=v1,v2 (cli.py:235-256 of the reference)."""
    from paper_2508_04462_b200.cli import parse_sweep
    from paper_2508_04462_b200.errors import ConfigError

    assert parse_sweep("K=8, 16,") == ("K", [8, 16])
    assert parse_sweep("temperature=0,1.5") == ("temperature", [0.0, 1.5])
    for bad in ("K", "seed=1,2", "K=a", "ratio="):
        with pytest.raises(ConfigError):
            parse_sweep(bad)


@pytest.mark.gpu
def test_cli_sweep_on_device(tmp_path):
    """sweep: one record per (prompt, value) plus an aggregate per value; each
    record equals a direct run at that value."""
    import paper_2508_04462_b200 as card
    from paper_2508_04462_b200.cli import main

    m, c, cfg = _files(tmp_path, ['{"id": "p0", "tokens": [1, 2, 3]}'], {"K": 16, "k": 3, "ratio": 5, "max_new_tokens": 30})
    out = str(tmp_path / "sweep.jsonl")
    assert main(["sweep", "--models", m, "--corpus", c, "--config", cfg, "--out", out, "--sweep", "K=4,16"]) == 0
    recs = [json.loads(x) for x in open(out)]
    assert [(r["id"], r["K"]) for r in recs] == [("p0", 4), ("__aggregate__", 4), ("p0", 16), ("__aggregate__", 16)]
    draft, target = card.load_models_file(m)
    want = card.run_speculative(draft, target, [1, 2, 3], card.EngineConfig(K=4, k=3, ratio=5, max_new_tokens=30))
    assert recs[0]["metrics"] == want.metrics.to_dict()
