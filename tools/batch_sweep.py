"""BASELINE configs[4]-style sweep: B concurrent requests on one B200
(run_speculative_batch), aggregate and per-request tokens/s."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias
T = float(os.environ.get("TEMP", "0"))
new = int(os.environ.get("NEW", "256"))
bias = LogitBias(seed=11, order=2, sharpness=1e6)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=new, temperature=T)
for B in [int(x) for x in os.environ.get("BS", "1,2,4,8").split(",")]:
    P = [[int(x) for x in np.random.default_rng(1000 + i).integers(0, 128256, 512)] for i in range(B)]
    card.run_speculative_batch(draft, target, P[:1], card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=16))
    res, tm = card.run_speculative_batch(draft, target, P, cfg)
    agg = tm["tokens"] / (tm["decode_ms"] / 1e3)
    acc = np.mean([r.metrics.mean_acceptance_length for r in res])
    print(f"B={B}: aggregate {agg:.1f} tokens/s, per request {agg / B:.1f} tokens/s, mean acceptance {acc:.2f}", flush=True)
    del res
    torch.cuda.empty_cache()
