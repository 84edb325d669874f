"""In-graph timeline of every GEMM of one forward (globaltimer stamps of all
linears set at once, then one graph replay): start/end per GEMM, gaps and
overlaps between consecutive GEMMs."""
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
lins = []
for li, L in enumerate(plan["layers"]):
    for k in ("qkv", "o", "gu", "d"):
        lins.append((f"L{li}.{k}", L[k]))
lins.append(("lm_head", plan["lm_head"]))
bufs = []
for name, lin in lins:
    tr = torch.zeros(lin.info["grid"] * 16, dtype=torch.int64, device="cuda")
    lib().card_linear_trace(lin.h, ctypes.c_void_p(tr.data_ptr()))
    bufs.append(tr)
rt.forward(rows, m)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
    rt.forward(rows, m)
torch.cuda.current_stream().wait_stream(st)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
for b in bufs:
    b.zero_()
g.replay()
torch.cuda.synchronize()
res = []
for (name, lin), b in zip(lins, bufs):
    t = b.view(-1, 16).cpu().numpy().astype(np.float64)
    ent = t[:, 0][t[:, 0] > 0]
    done = t[:, 8][t[:, 8] > 0]
    fk = t[:, 2][t[:, 2] > 0]
    res.append((name, ent.min(), np.median(fk) if len(fk) else np.nan, done.max(), lin.nbytes))
t0 = res[0][1]
prev_end = None
tot_gap = 0.0
for name, s, fk, e, nb in res:
    gap = (s - prev_end) / 1e3 if prev_end is not None else 0.0
    tot_gap += max(0.0, gap)
    if name.startswith("L0.") or name.startswith("L1.") or name == "lm_head" or name.startswith(f"L{len(plan['layers'])-1}."):
        print(f"{name:10s} start {(s-t0)/1e3:8.2f}  first_kb +{(fk-s)/1e3:5.2f}  end {(e-t0)/1e3:8.2f}  dur {(e-s)/1e3:6.2f} us  "
              f"gap_from_prev {gap:6.2f} us  {nb/(e-s):.0f} GB/s")
    prev_end = e
print(f"total span {(res[-1][3]-t0)/1e3:.1f} us; sum of GEMM durations {sum((e-s) for _,s,_,e,_ in res)/1e3:.1f} us; "
      f"sum of positive gaps {tot_gap:.1f} us")
