"""Front end (the `run`, `sweep` and `ablate` commands of the reference CLI,
/root/reference/pkg/src/specache/cli.py:174-294), over the device engine.  Inputs and outputs keep the reference formats:

* models JSON (lm.py:438-464, plus ``"type": "llama"`` entries);
* engine config JSON (EngineConfig fields; ``"ratio": "auto"`` resolves from
  the model latencies, cli.py:98-117);
* prompts JSONL, one ``{"id", "tokens" | "text"}`` object per line
  (cli.py:46-95);
* JSONL records with sorted keys and a final ``__aggregate__`` record, and
  an optional per-step trace.

Errors are reported as ``error: ...`` with exit code 2, not a traceback.

    python -m paper_2508_04462_b200 run --models pair.json --corpus prompts.jsonl --config k100_r7.json
"""

from __future__ import annotations

import argparse
import json
import sys
from typing import Sequence

from .engine import EngineConfig, communication_ratio, run_speculative, run_vanilla
from .errors import ConfigError, CorpusFormatError, SpecacheError
from .lm import load_models_file
from .metrics import aggregate

SWEEP_PARAMS = {"K": int, "ratio": int, "k": int, "query_depth": int, "temperature": float}   # cli.py:21
COLUMNS = (("tokens", "tokens_emitted", "{:d}"), ("time", "sim_time", "{:.2f}"),
           ("fwd_t", "target_forwards", "{:d}"), ("fwd_d", "draft_forwards", "{:d}"),
           ("hit%", "cache_hit_rate", "{:.3f}"), ("lnew", "mean_acceptance_length", "{:.3f}"),
           ("tok/t", "tokens_per_time", "{:.4f}"), ("speedup", "speedup_vs_vanilla", "{:.3f}"))


def read_json(path: str):
    try:
        with open(path, "r", encoding="utf-8") as fh:
            return json.load(fh)
    except OSError as e:
        raise ConfigError(f"{path}: {e.strerror or e}") from e
    except json.JSONDecodeError as e:
        raise ConfigError(f"{path}:{e.lineno}: {e.msg}") from e


def _prompt_of(rec, path: str, line_no: int, vocab_size: int) -> list[int]:
    if ("tokens" in rec) == ("text" in rec):
        raise CorpusFormatError(path, line_no, "record needs exactly one of 'tokens' or 'text'")
    if "tokens" in rec:
        toks = rec["tokens"]
        if not isinstance(toks, list) or not toks:
            raise CorpusFormatError(path, line_no, "'tokens' must be a nonempty list")
        bad = [t for t in toks if not isinstance(t, int) or isinstance(t, bool) or not 0 <= t < vocab_size]
        if bad:
            raise CorpusFormatError(path, line_no, f"token {bad[0]!r} outside vocabulary of size {vocab_size}")
        return list(toks)
    text = rec["text"]
    if not isinstance(text, str) or not text:
        raise CorpusFormatError(path, line_no, "'text' must be a nonempty string")
    if vocab_size < 256:
        raise CorpusFormatError(path, line_no, f"byte text needs a vocabulary of at least 256, model has {vocab_size}")
    return list(text.encode("utf-8"))


def read_corpus(path: str, vocab_size: int) -> list[tuple[str, list[int]]]:
    """Prompts JSONL (cli.py:46-95 format)."""
    try:
        lines = open(path, "r", encoding="utf-8").read().splitlines()
    except OSError as e:
        raise CorpusFormatError(path, 0, str(e.strerror or e)) from e
    out = []
    for line_no, line in enumerate(lines, start=1):
        if not line.strip():
            continue
        try:
            rec = json.loads(line)
        except json.JSONDecodeError as e:
            raise CorpusFormatError(path, line_no, e.msg) from e
        if not isinstance(rec, dict) or "id" not in rec:
            raise CorpusFormatError(path, line_no, "record must be an object with an 'id'")
        out.append((str(rec["id"]), _prompt_of(rec, path, line_no, vocab_size)))
    if not out:
        raise CorpusFormatError(path, 0, "corpus is empty")
    return out


def engine_config(raw: dict, draft, target, overrides: dict) -> EngineConfig:
    """EngineConfig from JSON plus overrides; ratio "auto" from the latencies."""
    d = {**raw, **overrides}
    if d.get("ratio") == "auto":
        d["ratio"] = communication_ratio(target.spec.forward_latency, draft.spec.forward_latency)
    return EngineConfig.from_dict(d)


def _table(title: str, rows: list[list[str]], first: str) -> str:
    headers = [first] + [c[0] for c in COLUMNS]
    widths = [max(len(headers[i]), *(len(r[i]) for r in rows)) for i in range(len(headers))]
    fmt = lambda cells: "  ".join(c.ljust(widths[i]) for i, c in enumerate(cells)).rstrip()  # noqa: E731
    return "\n".join([title, fmt(headers), "  ".join("-" * w for w in widths)] + [fmt(r) for r in rows])


def _cells(m) -> list[str]:
    return [f.format(getattr(m, attr)) for _, attr, f in COLUMNS]


def _dump(path: str, records) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for rec in records:
            fh.write(json.dumps(rec, sort_keys=True) + "\n")


def _setup(args):
    draft, target = load_models_file(args.models)
    raw = read_json(args.config) if args.config else {}
    if not isinstance(raw, dict):
        raise ConfigError(f"{args.config}: config must be a JSON object")
    overrides = {k: v for k, v in (("mode", args.mode), ("seed", args.seed)) if v is not None}
    return draft, target, raw, overrides, read_corpus(args.corpus, target.vocab.size)


def cmd_run(args) -> int:
    draft, target, raw, overrides, corpus = _setup(args)
    cfg = engine_config(raw, draft, target, overrides)
    records, rows, metrics, traces = [], [], [], []
    for rid, prompt in corpus:
        res = run_speculative(draft, target, prompt, cfg)
        metrics.append(res.metrics)
        records.append({"id": rid, "config": cfg.to_dict(), "output": res.output, "metrics": res.metrics.to_dict()})
        rows.append([rid] + _cells(res.metrics))
        traces.extend({"id": rid, **ev.to_dict()} for ev in res.trace)
    total = aggregate(metrics)
    records.append({"id": "__aggregate__", "metrics": total.to_dict()})
    rows.append(["all"] + _cells(total))
    if args.out:
        _dump(args.out, records)
    if args.trace:
        _dump(args.trace, traces)
    print(_table(f"run  mode={cfg.mode}  prompts={len(corpus)}", rows, "id"))
    return 0


def parse_sweep(spec: str) -> tuple[str, list]:
    """``param=v1,v2,...`` (cli.py:235-256)."""
    if "=" not in spec:
        raise ConfigError(f"--sweep must look like param=v1,v2,... got {spec!r}")
    name, _, tail = spec.partition("=")
    name = name.strip()
    if name not in SWEEP_PARAMS:
        raise ConfigError(f"cannot sweep {name!r}; choose one of {sorted(SWEEP_PARAMS)}")
    values = []
    for part in (p.strip() for p in tail.split(",")):
        if not part:
            continue
        try:
            values.append(SWEEP_PARAMS[name](part))
        except ValueError as e:
            raise ConfigError(f"bad sweep value {part!r} for {name}: {e}") from e
    if not values:
        raise ConfigError(f"--sweep {name} needs at least one value")
    return name, values


def cmd_sweep(args) -> int:
    """The corpus once per value of one engine parameter (cli.py:206-232)."""
    draft, target, raw, overrides, corpus = _setup(args)
    name, values = parse_sweep(args.sweep)
    records, rows = [], []
    for value in values:
        cfg = engine_config(raw, draft, target, {**overrides, name: value})
        per = []
        for rid, prompt in corpus:
            res = run_speculative(draft, target, prompt, cfg)
            per.append(res.metrics)
            records.append({"id": rid, name: value, "config": cfg.to_dict(), "metrics": res.metrics.to_dict()})
        total = aggregate(per)
        records.append({"id": "__aggregate__", name: value, "metrics": total.to_dict()})
        rows.append([f"{name}={value}"] + _cells(total))
    if args.out:
        _dump(args.out, records)
    print(_table(f"sweep {name}  prompts={len(corpus)}", rows, name))
    return 0


def cmd_ablate(args) -> int:
    """Vanilla AR vs the cache without correction vs the full protocol
    (Table 3; cli.py:259-294)."""
    draft, target, raw, overrides, corpus = _setup(args)
    records, rows = [], []
    for variant in ("vanilla", "cache_only", "cache_plus_correct"):
        cfg = engine_config({**raw, "correction_enabled": variant != "cache_only"}, draft, target, overrides)
        per = []
        for rid, prompt in corpus:
            res = run_vanilla(target, prompt, cfg) if variant == "vanilla" else \
                run_speculative(draft, target, prompt, cfg, use_graphs=False)
            per.append(res.metrics)
            records.append({"id": rid, "variant": variant, "metrics": res.metrics.to_dict()})
        total = aggregate(per)
        records.append({"id": "__aggregate__", "variant": variant, "metrics": total.to_dict()})
        rows.append([variant] + _cells(total))
    if args.out:
        _dump(args.out, records)
    print(_table(f"ablate  prompts={len(corpus)}", rows, "variant"))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2508_04462_b200",
                                 description="CARD query-and-correct decoding on B200 (drop-in for specache).")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, fn, hlp in (("run", cmd_run, "decode every prompt once"),
                          ("sweep", cmd_sweep, "rerun the corpus across parameter values"),
                          ("ablate", cmd_ablate, "vanilla vs cache-only vs cache-plus-correction")):
        p = sub.add_parser(name, help=hlp)
        p.add_argument("--models", required=True, help="models JSON file")
        p.add_argument("--corpus", required=True, help="prompts JSONL file")
        p.add_argument("--config", help="engine config JSON file")
        p.add_argument("--out", help="write records to this JSONL file")
        p.add_argument("--mode", choices=["serial_sim", "concurrent"], help="override the run mode")
        p.add_argument("--seed", type=int, help="override the run seed")
        if name == "run":
            p.add_argument("--trace", help="write per-step trace records to this JSONL file")
        if name == "sweep":
            p.add_argument("--sweep", required=True, metavar="param=v1,v2,...",
                           help=f"one of {sorted(SWEEP_PARAMS)} and its values")
        p.set_defaults(func=fn)
    return ap


def main(argv: Sequence[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except SpecacheError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
