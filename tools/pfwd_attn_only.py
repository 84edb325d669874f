"""Runs the persistent kernel over the attention step of layer 0 alone (after
one full forward), for profiling the in-kernel attention in isolation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, DeviceLlama, RowBlock

cfg = PRESETS["llama-3.2-1b"]
M, ctx = 116, 1024
m = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = DeviceLlama(cfg, m.packed, max_ctx=ctx + 64, tree_slots=0, row_budgets=(M,), persistent=True)
rows = RowBlock(M, 16, rt.dev)
rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, M)], ctx - M, out_last_only=False)
rt.forward(rows, M)
torch.cuda.synchronize()
pf = rt.plans[M]["pfwd"]
for _ in range(5):
    pf.run(rows.M, 1, 2)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    pf.run(rows.M, 1, 2)
b.record()
b.synchronize()
print(f"attention step alone: {a.elapsed_time(b) / 20 * 1e3:.1f} us per launch")
