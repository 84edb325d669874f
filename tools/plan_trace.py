"""Per-CTA %globaltimer timeline of the real plan linears (fused epilogues) of
layer 0 + lm_head, for a model / row budget (tuning aid; see gemm_trace.py)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.llama import PRESETS, RowBlock

which = sys.argv[1] if len(sys.argv) > 1 else "d116"
preset, m = {"d116": ("llama-3.2-1b", 116), "t8": ("llama-3.1-8b", 8), "t1": ("llama-3.1-8b", 1)}[which]
cfg = PRESETS[preset]
mdl = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = mdl.runtime(1088, 0, sorted({m, 128}))
rows = RowBlock(m, 16, rt.dev)
rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, m)], 1000 - m,
               out_last_only=False)
plan = rt.plans[m]
for _ in range(2):
    rt.forward(rows, m)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["entry", "pdl_wait", "first_kb", "last_mma", "acc_ready", "cbar1", "pushed", "cbar2", "done", "red_ld0", "red_lds0"]
for key in ("qkv", "o", "gu", "d", "lm_head"):
    lin = plan["lm_head"] if key == "lm_head" else plan["layers"][0][key]
    grid = lin.info["grid"]
    tr = torch.zeros(grid * 16, dtype=torch.int64, device="cuda")
    lib().card_linear_trace(lin.h, ctypes.c_void_p(tr.data_ptr()))
    flush.zero_()
    torch.cuda.synchronize()
    lin.run(rows.n_out if key == "lm_head" else rows.M)
    torch.cuda.synchronize()
    lib().card_linear_trace(lin.h, None)
    t = tr.view(grid, 16).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    print(f"{key}: N={lin.N} K={lin.K} {lin.info}")
    for k, nm in enumerate(names):
        col = t[:, k]
        v = col[col > 0] - t0
        if len(v):
            print(f"  {nm:10s} min {v.min()/1e3:7.2f}  med {np.median(v)/1e3:7.2f}  max {v.max()/1e3:7.2f} us")
    end = (t[:, 8].max() - t0) / 1e3
    print(f"  span {end:.2f} us -> {lin.nbytes/end/1e3:.0f} GB/s")
