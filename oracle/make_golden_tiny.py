"""Generate tests/golden/tiny_pair.json: BASELINE configs[0] run by the
REFERENCE engine.

Test infrastructure only (build container; /root/reference must exist).
The reference ``specache.run_speculative`` / ``run_vanilla`` (imported
read-only, pure kernel backend) drive the tiny random-init transformer
pair through the reference's own model protocol: a ``specache.ToyModel``
subclass whose ``_dist`` is the CPU fp32 Llama forward of
``oracle/llama_ref.py`` plus the shared k-gram agreement bias
(lm.py:109-196 is the contract; ``batch_tree_forward`` is the reference's
own).  Engine configs are the reference's ``pkg/configs/default.json``
and ``k100_r7.json`` verbatim (K=50/r=5 and K=100/r=7, 512 new tokens,
greedy); prompts are ``pkg/corpus/smoke.jsonl`` plus 8 seeded 512-token
prompts.  Weights: ``llama.init_weights(tiny-*, seed)``
(target seed 2, draft seed 1), regenerated identically on the GPU box.

    python oracle/make_golden_tiny.py [-j 8]
"""

from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_SRC = "/root/reference/pkg/src"
REF_PKG = "/root/reference/pkg"
OUT = os.path.join(ROOT, "tests", "golden", "tiny_pair.json")

# the agreement knob of pkg/models/pair_70b_1b.json (k-gram seed 11, order 2,
# sharpness 60; the draft mixes stream 131 at weight 0.05)
BIAS_T = dict(seed=11, order=2, sharpness=60.0, mix_seed=0, mix_weight=0.0)
BIAS_D = dict(seed=11, order=2, sharpness=60.0, mix_seed=131, mix_weight=0.05)
SPEC_T = (8.0, 7.0)    # (params_billions, forward_latency)
SPEC_D = (1.0, 1.0)
N_SEEDED = 8


def prompts(V: int) -> list[tuple[str, list[int]]]:
    out = []
    with open(os.path.join(REF_PKG, "corpus", "smoke.jsonl"), encoding="utf-8") as fh:
        for line in fh:
            if line.strip():
                rec = json.loads(line)
                out.append((rec["id"], [int(t) for t in rec["tokens"]]))
    for i in range(N_SEEDED):
        out.append((f"s{i}", [int(x) for x in np.random.default_rng(1000 + i).integers(0, V, 512)]))
    return out


def _models(sp):
    import torch

    sys.path.insert(0, ROOT)
    from oracle.llama_ref import RefLlama
    from oracle.card_oracle import kgram_uniforms
    from paper_2508_04462_b200.llama import PRESETS, init_weights

    torch.set_num_threads(1)

    class RefTiny(sp.ToyModel):
        """Reference ToyModel whose distribution is the fp32 CPU transformer."""

        def __init__(self, preset, seed, bias, spec):
            cfg = PRESETS[preset]
            super().__init__(sp.Vocabulary(cfg.vocab_size), sp.ModelSpec(*spec), None)
            self.llama = RefLlama(cfg, init_weights(cfg, seed))
            self.b = bias

        def _dist(self, ctx, temperature):
            V = self.vocab.size
            lg = self.llama.logits_for(list(ctx)).float().numpy()
            tail = list(ctx)[-self.b["order"]:]
            u = np.array(kgram_uniforms(self.b["seed"], tail, V), dtype=np.float32)
            if self.b["mix_weight"]:
                u = u + np.float32(self.b["mix_weight"]) * np.array(kgram_uniforms(self.b["mix_seed"], tail, V),
                                                                    dtype=np.float32)
            lg = (lg + np.float32(self.b["sharpness"]) * u).astype(np.float64)
            if temperature == 0.0:
                out = np.zeros(V)
                out[int(np.argmax(lg))] = 1.0
                return out
            z = lg / temperature
            e = np.exp(z - z.max())
            return e / e.sum()

    return (RefTiny("tiny-draft", 1, BIAS_D, SPEC_D), RefTiny("tiny-target", 2, BIAS_T, SPEC_T))


def _one(job):
    cfg_name, pid, prompt = job
    os.environ["SPECACHE_KERNELS"] = "pure"
    sys.path.insert(0, REF_SRC)
    import specache as sp

    with open(os.path.join(REF_PKG, "configs", cfg_name), encoding="utf-8") as fh:
        cfg = sp.EngineConfig.from_dict(json.load(fh))
    d, t = _models(sp)
    res = sp.run_speculative(d, t, prompt, cfg)
    van = sp.run_vanilla(t, prompt, cfg)
    trace = [[e.event, int(e.hit), e.candidate_len, e.accepted_len, e.lnew, e.cache_alive_nodes]
             for e in res.trace]
    return dict(config=cfg_name, id=pid, prompt=prompt, output=list(res.output), vanilla=list(van.output),
                trace=trace, metrics=res.metrics.to_dict())


def main():
    jobs = int(sys.argv[sys.argv.index("-j") + 1]) if "-j" in sys.argv else (os.cpu_count() or 1)
    work = [(c, pid, p) for c in ("default.json", "k100_r7.json") for pid, p in prompts(64)]
    with ProcessPoolExecutor(jobs) as ex:
        runs = list(ex.map(_one, work))
    doc = dict(bias_target=BIAS_T, bias_draft=BIAS_D, spec_target=SPEC_T, spec_draft=SPEC_D,
               presets=["tiny-draft", "tiny-target"], seeds=[1, 2], runs=runs)
    with open(OUT, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, separators=(",", ":"))
        fh.write("\n")
    print(f"wrote {OUT}: {len(runs)} runs")


if __name__ == "__main__":
    main()
