"""Distribution of draft-step widths (frontier rows per draft forward) on the
bench workload: how often a draft forward runs far below its 116-row plan."""
import os
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.lm import LogitBias
from paper_2508_04462_b200.llama import PRESETS

tcfg, dcfg = PRESETS["llama-3.1-8b"], PRESETS["llama-3.2-1b"]
bias = LogitBias(seed=11, order=2, sharpness=1e6, mix_seed=131, mix_weight=0.0)
target = card.LlamaModel(tcfg, seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.0, 7.0))
draft = card.LlamaModel(dcfg, seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.2, 1.0))
cfg = card.EngineConfig(K=100, k=3, ratio=7, temperature=0.0, max_new_tokens=512, seed=0)
hist = Counter()
n_steps = 0
for rep in range(2):
    prompt = [int(x) for x in np.random.default_rng(1000 + rep).integers(0, tcfg.vocab_size, 512)]
    res = card.run_speculative(draft, target, prompt, cfg)
    prev = 1
    for ev in res.trace:
        if ev.event == "draft_expand":
            hist[prev] += 1   # this step forwarded the previous frontier
            prev = ev.candidate_len
            n_steps += 1
        elif ev.event in ("verify", "miss_step"):
            prev = None
    print(f"rep {rep}: {len(res.output)} tokens, acceptance {res.metrics.mean_acceptance_length:.2f}, "
          f"draft steps {res.wall.get('draft_steps')}, target steps {res.wall.get('target_steps')}", flush=True)
buckets = Counter()
for w, c in hist.items():
    b = "after-verify" if w is None else (16 if w <= 16 else 32 if w <= 32 else 64 if w <= 64 else 128)
    buckets[b] += c
print("draft steps by forwarded width bucket:", dict(buckets), "of", n_steps)
print("widths:", sorted(((w if w is not None else -1), c) for w, c in hist.items())[:40])
