"""Short CARD + AR run on the BASELINE config for ncu launch lists / captures.

Model construction (random init, weight packing: torch kernels) and one
warm-up request run outside the profiled range; run ncu with
--profile-from-start off so the launch list holds the requests only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

new = int(os.environ.get("NEW", "16"))
sharp = float(os.environ.get("SHARP", "1e6"))   # the bench's agreement knob
bias = LogitBias(seed=11, order=2, sharpness=sharp)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
prompt = [int(x) for x in np.random.default_rng(1000).integers(0, 128256, 512)]
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=new)
card.run_speculative(draft, target, prompt, cfg)   # warm-up (runtimes, plans)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = card.run_speculative(draft, target, prompt, cfg)
v = card.run_vanilla(target, prompt, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("card", r.wall, "ar", v.wall)
