"""Does a request that finishes early (EOS) change the others' outputs?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, init_weights
from paper_2508_04462_b200.lm import LogitBias

bias = LogitBias(seed=11, order=2, sharpness=4000.0)
ct, cd = PRESETS["small-target"], PRESETS["small-draft"]
t = card.LlamaModel(ct, dtype="bf16", weights=init_weights(ct, 2), spec=card.ModelSpec(8.0, 7.0), bias=bias)
d = card.LlamaModel(cd, dtype="bf16", weights=init_weights(cd, 1), spec=card.ModelSpec(1.0, 1.0), bias=bias)
prompts = [[int(x) for x in np.random.default_rng(500 + i).integers(0, 512, [32, 50][i % 2])] for i in range(4)]
cfg = card.EngineConfig(K=8, k=3, ratio=4, max_new_tokens=120)
free = card.run_vanilla(t, prompts[0], cfg).output
t.eos_token = d.eos_token = free[len(free) // 3]
ar = [card.run_vanilla(t, p, cfg).output for p in prompts]
print("AR lengths", [len(a) for a in ar], "eos", t.eos_token)
for order in ([0, 2], [2, 0], [2], [1, 2], [0, 1, 2, 3], [2, 3]):
    t.__dict__.pop("_card_batch_sessions", None)
    res, _ = card.run_speculative_batched(d, t, [prompts[i] for i in order], cfg)
    out = []
    for i, r in zip(order, res):
        j = next((j for j in range(min(len(r.output), len(ar[i]))) if r.output[j] != ar[i][j]), None)
        cyc = None
        if j is not None:   # the verify at which it diverged
            n = 0
            for c, ev in enumerate(e for e in r.trace if e.event in ("verify", "miss_step")):
                n += ev.lnew
                if n > j:
                    cyc = c
                    break
        out.append((i, j, len(r.output), cyc))
    print(f"order {order}: (request, first mismatch, length, verify index) {out}", flush=True)
