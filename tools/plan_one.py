"""Run one plan linear of a model (ncu target): python tools/plan_one.py d116 o 3"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, RowBlock
which, key, reps = sys.argv[1], sys.argv[2], int(sys.argv[3])
preset, m = {"d116": ("llama-3.2-1b", 116), "t8": ("llama-3.1-8b", 8)}[which]
cfg = PRESETS[preset]
mdl = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = mdl.runtime(1088, 0, sorted({m, 128}))
rows = RowBlock(m, 16, rt.dev)
rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, m)], 1000 - m, out_last_only=False)
rt.forward(rows, m); torch.cuda.synchronize()
lin = rt.plans[m]["lm_head"] if key == "lm_head" else rt.plans[m]["layers"][1][key]
for _ in range(reps):
    lin.run(rows.n_out if key == "lm_head" else rows.M)
torch.cuda.synchronize()
