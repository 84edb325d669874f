"""BASELINE configs[4] sweep on one B200: B concurrent requests of the
configs[1] pair (Llama-3.2-1B draft + Llama-3.1-8B target, 512-token
prompts), decoded by BatchRun (shared draft / verify forwards, K = 100 // B
per request) and, for comparison, by the stream-interleaved
run_speculative_batch (K = 100 each).  Env: TEMP, NEW, BS, OLD=1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

T = float(os.environ.get("TEMP", "0"))
new = int(os.environ.get("NEW", "256"))
bias = LogitBias(seed=11, order=2, sharpness=1e6)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=new, temperature=T)
print(f"# T={T}, {new} new tokens per request, 512-token prompts, 1 B200", flush=True)
for B in [int(x) for x in os.environ.get("BS", "1,2,4,8,16,32").split(",")]:
    P = [[int(x) for x in np.random.default_rng(1000 + i).integers(0, 128256, 512)] for i in range(B)]
    bc = card.batch_config(cfg, B)
    card.run_speculative_batched(draft, target, P[:1], card.batch_config(card.EngineConfig(K=100, k=3, ratio=7,
                                                                                          max_new_tokens=16), B))
    res, tm = card.run_speculative_batched(draft, target, P, bc)
    agg = tm["tokens"] / (tm["decode_ms"] / 1e3)
    acc = np.mean([r.metrics.mean_acceptance_length for r in res])
    print(f"batched     B={B:2d} K/request={bc.K:3d}: aggregate {agg:8.1f} tokens/s, per request {agg / B:7.1f},"
          f" mean acceptance {acc:.2f}, draft steps {tm['draft_steps']}, verify steps {tm['target_steps']}",
          flush=True)
    del res
    torch.cuda.empty_cache()
    if os.environ.get("OLD") == "1" and B <= 8:
        res, tm = card.run_speculative_batch(draft, target, P, cfg)
        agg = tm["tokens"] / (tm["decode_ms"] / 1e3)
        acc = np.mean([r.metrics.mean_acceptance_length for r in res])
        print(f"interleaved B={B:2d} K/request={cfg.K:3d}: aggregate {agg:8.1f} tokens/s, per request {agg / B:7.1f},"
              f" mean acceptance {acc:.2f}", flush=True)
        del res
        torch.cuda.empty_cache()
