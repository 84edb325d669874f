"""Acceptance / speed vs the k-gram logit-bias agreement knob (BASELINE config)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

new = int(os.environ.get("NEW", "128"))
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", spec=card.ModelSpec(8.0, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", spec=card.ModelSpec(1.2, 1.0))
prompt = [int(x) for x in np.random.default_rng(1000).integers(0, 128256, 512)]
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=new)
SWEEP = [(0, 0), (1e5, 0), (3e5, 0), (6e5, 0), (1e6, 0), (2e6, 0), (4e6, 0), (1e7, 0), (2e6, 0.02), (2e6, 0.05)]
if os.environ.get("SWEEP"):
    SWEEP = [tuple(float(v) for v in x.split(":")) for x in os.environ["SWEEP"].split(",")]
for sharp, mix in SWEEP:
    b = LogitBias(11, 2, float(sharp), 131, float(mix))
    target.bias = b
    draft.bias = LogitBias(11, 2, float(sharp), 131, float(mix))
    r = card.run_speculative(draft, target, prompt, cfg)
    r = card.run_speculative(draft, target, prompt, cfg)
    v = card.run_vanilla(target, prompt, cfg)
    print(f"sharp={sharp:6} mix={mix}: acc={r.metrics.mean_acceptance_length:.2f} hit={r.metrics.cache_hit_rate:.2f} "
          f"card={len(r.output)/r.wall['decode_ms']*1e3:.1f} tok/s  ar={len(v.output)/v.wall['decode_ms']*1e3:.1f} tok/s "
          f"draft_steps={r.wall['draft_steps']} target_steps={r.wall['target_steps']} same={r.output == v.output}",
          flush=True)
