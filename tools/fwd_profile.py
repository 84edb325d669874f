"""One warm forward of a model at a row budget, for ncu launch lists:
    ncu --metrics gpu__time_duration.sum --csv python tools/fwd_profile.py d116
Prints the number of kernels per forward so the tail can be cut."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200 import _lib
from paper_2508_04462_b200.llama import PRESETS, RowBlock

which = sys.argv[1] if len(sys.argv) > 1 else "d116"
preset, m = {"d116": ("llama-3.2-1b", 116), "t8": ("llama-3.1-8b", 8), "t1": ("llama-3.1-8b", 1)}[which]
cfg = PRESETS[preset]
mdl = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = mdl.runtime(1088, 0, sorted({m, 128}))
rows = RowBlock(m, 16, rt.dev)
rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, m)], 1000 - m,
               out_last_only=False)
for _ in range(2):
    rt.forward(rows, m)
torch.cuda.synchronize()
c0 = _lib.launch_count[0]
rt.forward(rows, m)
torch.cuda.synchronize()
print("kernels per forward:", _lib.launch_count[0] - c0)
