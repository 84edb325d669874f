"""Quick timing of one CARD request and one AR request on the BASELINE config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

sharp = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
mix = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
new = int(sys.argv[3]) if len(sys.argv) > 3 else 128
t0 = time.time()
bias = LogitBias(seed=11, order=2, sharpness=sharp, mix_seed=131, mix_weight=mix)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias,
                         spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=LogitBias(11, 2, sharp, 131, mix),
                        spec=card.ModelSpec(1.24, 1.0))
torch.cuda.synchronize()
print("init s", time.time() - t0, flush=True)
prompt = [int(x) for x in np.random.default_rng(1000).integers(0, 128256, 512)]
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=new)
for i in range(2):
    t1 = time.time()
    r = card.run_speculative(draft, target, prompt, cfg)
    print("card", i, "wall", time.time() - t1, "decode_ms", r.wall["decode_ms"], "tok", len(r.output),
          "tok/s", len(r.output) / r.wall["decode_ms"] * 1e3, "acc", r.metrics.mean_acceptance_length,
          "hit", r.metrics.cache_hit_rate, r.wall.get("draft_steps"), r.wall.get("target_steps"), flush=True)
for i in range(2):
    v = card.run_vanilla(target, prompt, cfg)
    print("ar", i, "decode_ms", v.wall["decode_ms"], "tok/s", len(v.output) / v.wall["decode_ms"] * 1e3, flush=True)
print("same output:", v.output == r.output)
