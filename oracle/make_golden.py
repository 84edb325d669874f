"""Generate tests/golden/*.json by running the REFERENCE implementation.

Test infrastructure: run in the build container (where /root/reference
exists), never on the GPU box.  The reference is imported read-only from
/root/reference/pkg/src with its pure-Python kernel backend; nothing is
copied.  Floats are stored through ``repr`` so every fixture round-trips
bit-exactly.

    python oracle/make_golden.py            # rewrites tests/golden/*.json
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_PKG = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, os.pardir, "tests", "golden")


def _import_reference():
    os.environ["SPECACHE_KERNELS"] = "pure"
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import specache  # noqa: F401
    return specache


def _dump(name, obj):
    path = os.path.join(OUT, name)
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(obj, fh, separators=(",", ":"))
        fh.write("\n")
    print(f"wrote {os.path.normpath(path)} ({os.path.getsize(path)} bytes)")


# ---------------------------------------------------------------- kernels
def gen_kernels(sp):
    from specache import _kernels_py as kp

    rng = np.random.default_rng(20250804)
    kg = []
    for i in range(160):
        V = int(rng.integers(2, 80))
        order = int(rng.integers(1, 4))
        tail = [int(x) for x in rng.integers(0, V, size=order)]
        T = [0.0, 1.0, 0.5, 2.0, float(rng.uniform(0.1, 3.0))][i % 5]
        sharp = float([0.0, 1.0, 20.0, 60.0, rng.uniform(0, 200)][(i // 5) % 5])
        mixw = 0.0 if i % 3 == 0 else float(rng.uniform(0, 0.3))
        seed = int(rng.integers(0, 2**63)) if i % 7 == 0 else int(rng.integers(0, 5000))
        seed2 = int(rng.integers(0, 5000))
        out = kp.kgram_dist(seed, seed2, mixw, tuple(tail), V, sharp, T)
        kg.append(dict(seed=seed, seed2=seed2, mix_weight=mixw, tail=tail, V=V,
                       sharpness=sharp, temperature=T, out=[float(x) for x in out]))
    tk = []
    for i in range(60):
        N = int(rng.integers(1, 9))
        V = int(rng.integers(2, 40))
        k = int(rng.integers(1, 6))
        d = rng.random((N, V))
        if i % 2 == 0:          # quantise to force exact ties
            d = np.round(d * 4) / 4
        d[rng.random((N, V)) < 0.3] = 0.0
        rows = kp.rows_topk(d, k)
        tk.append(dict(k=k, dists=d.tolist(), rows=[[[int(t), float(p)] for t, p in r] for r in rows]))
    _dump("kernels.json", dict(kgram=kg, rows_topk=tk))


# ---------------------------------------------------------------- cache ops
def _snap(cache, sp):
    a = cache.arena
    return dict(
        token=[n.token for n in a], parent=[(-1 if n.parent is None else n.parent) for n in a],
        layer=[n.layer for n in a], score=[n.log_score for n in a], edge=[n.edge_logp for n in a],
        alive=[bool(n.alive) for n in a], frontier=list(cache.frontier), root=cache.root,
        epoch=cache.epoch, dead=cache._dead, alive_below=cache.alive_below_root(),
        dump=cache.dump())


def gen_cache(sp):
    from specache import CacheConfig, TreeCache, make_kgram_model, Vocabulary
    from specache.errors import FrontierFull, ProtocolError
    from specache.lm import ModelSpec

    scenarios = []
    rng = np.random.default_rng(4462)
    for sc in range(24):
        V = int(rng.integers(3, 24))
        K = int(rng.integers(1, 12))
        k = int(rng.integers(1, 4))
        depth = int(rng.integers(2, 7))
        eos = int(rng.integers(0, V)) if sc % 5 == 4 else None
        sharp = float(rng.uniform(0.5, 12.0))
        model = make_kgram_model(int(rng.integers(0, 999)), Vocabulary(V), order=2, sharpness=sharp,
                                 spec=ModelSpec(1.0, 1.0), eos_token=eos)
        quant = sc % 3 == 1
        root = int(rng.integers(0, V))
        cache = TreeCache(root, CacheConfig(K=K, k=k, max_depth=depth), eos_token=eos)
        base = [int(rng.integers(0, V)), root]
        ops = []
        n_ops = 40 if sc < 20 else 160      # the long ones churn through compaction
        for _ in range(n_ops):
            r = rng.random()
            if r < 0.55:
                paths = cache.parent_paths()
                dists = np.vstack([model.next_distribution(base + p) for p in paths])
                if quant:   # force exact ties in the pool: snap to quarters, renormalise
                    q = np.round(dists * 4) / 4
                    q[np.arange(q.shape[0]), np.argmax(dists, axis=1)] += 1e-300
                    bad = q.sum(axis=1) <= 0
                    q[bad] = dists[bad]
                    dists = q / q.sum(axis=1, keepdims=True)
                try:
                    new = cache.expand_layer(dists)
                    res = dict(status="ok", new=list(new))
                except FrontierFull:
                    res = dict(status="frontier_full")
                ops.append(dict(op="expand", dists=dists.tolist(), result=res, state=_snap(cache, sp)))
            elif r < 0.75:
                d = int(rng.integers(1, depth + 2))
                q = cache.query(d)
                ops.append(dict(op="query", depth=d, result=dict(hit=q.hit, path=q.path, tokens=q.tokens,
                                                                  edges=q.edge_logps)))
            else:
                q = cache.query(int(rng.integers(1, depth + 1)))
                n = int(rng.integers(0, len(q.tokens) + 1)) if q.hit else 0
                acc = list(q.tokens[:n])
                mode = rng.random()
                if mode < 0.4 and q.hit and n < len(q.tokens):
                    corr = int(q.tokens[n])          # correction lands on a cached child
                elif mode < 0.5 and acc:
                    corr = None
                else:
                    corr = int(rng.integers(0, V))
                if rng.random() < 0.1 and acc:
                    acc = acc[:-1] + [(acc[-1] + 1) % V]   # provoke ProtocolError sometimes
                try:
                    nr = cache.correct(acc, corr)
                    res = dict(status="ok", new_root=nr)
                except ProtocolError:
                    res = dict(status="protocol_error")
                base = base + acc + ([corr] if corr is not None else [])
                ops.append(dict(op="correct", accepted=acc, correction=corr, result=res,
                                state=_snap(cache, sp)))
        scenarios.append(dict(V=V, K=K, k=k, max_depth=depth, eos=eos, root=root, ops=ops))
    _dump("cache_ops.json", scenarios)


# ---------------------------------------------------------------- verify
def gen_verify(sp):
    from specache.verify import verify_greedy, verify_sampling, sample_index

    rng = np.random.default_rng(7)
    cases = []
    for i in range(80):
        V = int(rng.integers(2, 16))
        L = int(rng.integers(0, 8))
        d = rng.random((L + 1, V)) ** 3
        if i % 4 == 0:
            d = np.round(d * 3)
            d[:, 0] += 1
        d = d / d.sum(axis=1, keepdims=True)
        cand = [int(x) for x in rng.integers(0, V, size=L)]
        if i % 2 == 0:   # make a prefix follow the argmax chain
            for j in range(int(rng.integers(0, L + 1))):
                cand[j] = int(np.argmax(d[j]))
        g = verify_greedy(list(d), cand)
        seed = int(rng.integers(0, 10**6))
        r = np.random.default_rng(seed)
        s = verify_sampling(list(d), [1.0] * L, cand, r)
        after = float(r.random())
        cases.append(dict(dists=d.tolist(), cand=cand, seed=seed,
                          greedy=[list(g.accepted), g.correction],
                          sampling=[list(s.accepted), s.correction], next_uniform=after))
    samples = []
    for i in range(40):
        V = int(rng.integers(1, 50))
        p = rng.random(V)
        p[rng.random(V) < 0.4] = 0.0
        if p.sum() == 0:
            p[0] = 1.0
        seed = int(rng.integers(0, 10**6))
        samples.append(dict(p=p.tolist(), seed=seed, idx=sample_index(np.random.default_rng(seed), p)))
    _dump("verify.json", dict(cases=cases, samples=samples))


# ---------------------------------------------------------------- engine
FIXTURE_PAIR = None


def _trace_rows(res):
    return [[e.step_index, e.sim_time, e.hit, e.candidate_len, e.accepted_len, e.lnew,
             e.cache_alive_nodes, e.event] for e in res.trace]


def gen_engine(sp):
    from specache import EngineConfig, run_speculative, run_vanilla, aggregate
    from specache.lm import load_models_file
    from specache.cli import load_corpus

    data = os.path.join(REF_PKG, "tests", "data")
    with open(os.path.join(data, "fixture_models.json")) as fh:
        fixture_doc = json.load(fh)
    with open(os.path.join(data, "fixture_config.json")) as fh:
        fixture_cfg = json.load(fh)
    draft, target = load_models_file(os.path.join(data, "fixture_models.json"))
    corpus = load_corpus(os.path.join(data, "fixture_corpus.jsonl"), target.vocab.size)

    runs = []
    rng = np.random.default_rng(99)
    pairs = []
    for pf in ("pair_70b_1b.json", "pair_70b_7b.json"):
        with open(os.path.join(REF_PKG, "models", pf)) as fh:
            pairs.append((pf, json.load(fh)))
    pairs.append(("fixture_models.json", fixture_doc))
    # an EOS pair and a uniform-draft pair exercise the clipping/absorbing paths
    eos_doc = json.loads(json.dumps(fixture_doc))
    eos_doc["eos_token"] = 5
    pairs.append(("fixture_eos5", eos_doc))
    for name, doc in pairs:
        for variant in range(4):
            cfg = dict(K=int(rng.integers(1, 40)), k=int(rng.integers(1, 4)),
                       ratio=int(rng.integers(1, 8)), max_new_tokens=int(rng.integers(8, 80)),
                       temperature=[0.0, 0.0, 1.0, 0.7][variant], seed=int(rng.integers(0, 1000)),
                       correction_enabled=variant != 1)
            path = os.path.join("/tmp", f"_card_pair_{os.getpid()}.json")
            with open(path, "w") as fh:
                json.dump(doc, fh)
            d, t = load_models_file(path)
            prompt = [int(x) for x in rng.integers(0, doc["vocab_size"], size=int(rng.integers(1, 6)))]
            res = run_speculative(d, t, prompt, EngineConfig.from_dict(cfg))
            van = run_vanilla(t, prompt, EngineConfig.from_dict(cfg))
            runs.append(dict(pair=name, models=doc, config=cfg, prompt=prompt, output=res.output,
                             trace=_trace_rows(res), metrics=res.metrics.to_dict(),
                             vanilla_output=van.output, vanilla_metrics=van.metrics.to_dict()))
    # the reference's own golden recipe (tests/data/regen_goldens.py:29-66), re-run here
    ab_raw = fixture_cfg["ablate"]
    ablation = {}
    base = EngineConfig.from_dict(ab_raw)
    ablation["vanilla"] = aggregate(run_vanilla(target, p, base).metrics for _, p in corpus).to_dict()
    for variant, corrected in (("cache_only", False), ("cache_plus_correct", True)):
        c = EngineConfig.from_dict({**ab_raw, "correction_enabled": corrected})
        ablation[variant] = aggregate(run_speculative(draft, target, p, c).metrics
                                      for _, p in corpus).to_dict()
    ks_raw = dict(fixture_cfg["ksweep"])
    kvals = ks_raw.pop("K_values")
    ksweep = {}
    for K in kvals:
        c = EngineConfig.from_dict({**ks_raw, "K": K})
        ksweep[str(K)] = aggregate(run_speculative(draft, target, p, c).metrics
                                   for _, p in corpus).to_dict()
    _dump("engine.json", dict(runs=runs))
    _dump("fixture_goldens.json", dict(models=fixture_doc, config=fixture_cfg,
                                       corpus=[p for _, p in corpus],
                                       ablation=ablation, ksweep=ksweep))


def main():
    sp = _import_reference()
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["kernels", "cache", "verify", "engine"]
    for w in which:
        globals()[f"gen_{w}"](sp)


if __name__ == "__main__":
    main()
