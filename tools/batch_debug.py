"""Batched decode vs AR on the small bf16 pair: which requests diverge, with
and without EOS, at several horizons / K."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, init_weights
from paper_2508_04462_b200.lm import LogitBias

bias = LogitBias(seed=11, order=2, sharpness=4000.0)
ct, cd = PRESETS["small-target"], PRESETS["small-draft"]
PERS = not (len(sys.argv) > 1 and sys.argv[1] == "nopf")
t = card.LlamaModel(ct, dtype="bf16", weights=init_weights(ct, 2), spec=card.ModelSpec(8.0, 7.0), bias=bias,
                    persistent=PERS)
d = card.LlamaModel(cd, dtype="bf16", weights=init_weights(cd, 1), spec=card.ModelSpec(1.0, 1.0), bias=bias,
                    persistent=PERS)
prompts = [[int(x) for x in np.random.default_rng(500 + i).integers(0, 512, [32, 50][i % 2])] for i in range(4)]
for eos in (False, True):
    for K, new in ((8, 120), (8, 40), (12, 120)):
        cfg = card.EngineConfig(K=K, k=3, ratio=4, max_new_tokens=new)
        t.eos_token = d.eos_token = None
        if eos:
            free = card.run_vanilla(t, prompts[0], cfg).output
            t.eos_token = d.eos_token = free[len(free) // 3]
        for B in (1, 4):
            t.__dict__.pop("_card_batch_sessions", None)
            res, _ = card.run_speculative_batched(d, t, prompts[:B], cfg)
            bad = []
            for i, (p, r) in enumerate(zip(prompts, res)):
                van = card.run_vanilla(t, p, cfg).output
                if r.output != van:
                    j = next((j for j in range(min(len(r.output), len(van))) if r.output[j] != van[j]), None)
                    bad.append((i, j, len(r.output), len(van)))
            single = card.run_speculative(d, t, prompts[0], cfg).output == card.run_vanilla(t, prompts[0], cfg).output
            print(f"persistent={PERS} eos={eos} K={K} new={new} B={B}: mismatches {bad}  (single-run lossless: {single})", flush=True)
