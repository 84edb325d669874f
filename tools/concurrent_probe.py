"""mode=concurrent on one B200: per-cycle wall time, draft steps per verify,
acceptance — with the draft stream at high or normal priority."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
import paper_2508_04462_b200.engine as E
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

bias = LogitBias(seed=11, order=2, sharpness=1e6)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
prompt = [int(x) for x in np.random.default_rng(1000).integers(0, 128256, 512)]
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=256, mode="concurrent")
for prio in (-8, 0):
    E._DRAFT_PRIORITY = prio
    for rep in range(2):
        for s_ in list(target.__dict__.get("_card_sessions", {})):
            target._card_sessions.pop(s_)
        r = card.run_speculative(draft, target, prompt, cfg)
        n_v = sum(1 for e in r.trace if e.event in ("verify", "miss_step"))
        n_d = sum(1 for e in r.trace if e.event == "draft_expand")
        ms = r.wall["decode_ms"]
        print(f"draft priority {prio}: {len(r.output) / ms * 1e3:.1f} tokens/s, acceptance "
              f"{r.metrics.mean_acceptance_length:.2f}, {n_v} verifies, {n_d} draft steps "
              f"({n_d / max(1, n_v):.2f}/verify), {ms / max(1, n_v):.2f} ms/cycle", flush=True)
