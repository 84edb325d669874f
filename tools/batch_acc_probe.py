"""Per-request mean acceptance of a batched decode vs the same requests in
smaller batches (same per-request K): a draft-side bug shows up as requests
whose acceptance drops only in the large batch.  Env: B, K, NEW."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

B = int(os.environ.get("B", "32"))
K = int(os.environ.get("K", "3"))
new = int(os.environ.get("NEW", "128"))
bias = LogitBias(seed=11, order=2, sharpness=1e6)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
cfg = card.EngineConfig(K=K, k=3, ratio=7, max_new_tokens=new)
P = [[int(x) for x in np.random.default_rng(1000 + i).integers(0, 128256, 512)] for i in range(B)]
for bs in [int(x) for x in os.environ.get("BSS", f"{B},4,1").split(",")]:
    accs = []
    for j in range(0, min(B, 8) if bs < B else B, bs):
        res, tm = card.run_speculative_batched(draft, target, P[j:j + bs], cfg)
        accs += [round(r.metrics.mean_acceptance_length, 2) for r in res]
    print(f"batch {bs:2d}: acceptance per request {accs}", flush=True)
