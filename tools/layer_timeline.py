"""In-graph critical path of the last layer of one forward: per-kernel
%globaltimer stamps of the four GEMMs (card_linear_trace) and of the
attention (card_attention_trace), one CUDA-graph replay.  Times are us from
the layer's QKV GEMM entry.  usage: layer_timeline.py d116|t8|t1"""
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
rt = mdl.runtime(1088, 256, sorted({m, 128}))
rows = RowBlock(m, 16, rt.dev)
R = m
host = torch.zeros(rows.block.numel(), dtype=torch.int32)
n_chain = 16 if m > 16 else m
host[0], host[1] = m, m - n_chain if m > 16 else m
base = 1000
rng = np.random.default_rng(0)
host[2:2 + m] = torch.tensor(rng.integers(0, cfg.vocab_size, m))
for i in range(m):
    if i < n_chain:
        p = base - n_chain + i
        host[2 + R + i], host[2 + 2 * R + i], host[2 + 3 * R + i] = p, p, p + 1
    else:   # tree row at depth 1..14 with a chain of tree slots
        d = 1 + (i % 14)
        host[2 + R + i], host[2 + 2 * R + i], host[2 + 3 * R + i] = base - 1 + d, rt.tree_base + i, base
        host[2 + 4 * R + i] = d
        host[2 + 6 * R + i * 16:2 + 6 * R + i * 16 + d] = torch.arange(rt.tree_base + i - d + 1, rt.tree_base + i + 1)
if m > 16:
    host[2 + 5 * R:2 + 5 * R + m - n_chain] = torch.arange(n_chain, m)
else:
    host[2 + 5 * R:2 + 5 * R + m] = torch.arange(m)
rows.block.copy_(host)
plan = rt.plans[m]
L = plan["layers"][-1]
bufs = {}
for k in ("qkv", "o", "gu", "d"):
    tr = torch.zeros(L[k].info["grid"] * 16, dtype=torch.int64, device="cuda")
    lib().card_linear_trace(L[k].h, ctypes.c_void_p(tr.data_ptr()))
    bufs[k] = tr
at = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
lib().card_attention_trace(ctypes.c_void_p(at.data_ptr()))
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
for b in list(bufs.values()) + [at]:
    b.zero_()
g.replay()
torch.cuda.synchronize()
lib().card_attention_trace(None)
for k in bufs:
    lib().card_linear_trace(L[k].h, None)


def stats(col):
    v = col[col > 0]
    return (v.min(), np.median(v), v.max()) if len(v) else (np.nan,) * 3


q = bufs["qkv"].view(-1, 16).cpu().numpy().astype(np.float64)
t0 = q[:, 0][q[:, 0] > 0].min()
print(f"{which}: last layer, us from its QKV GEMM entry (min / med / max over CTAs)")
gn = ["entry", "pdl_wait", "first_kb", "last_mma", "acc_ready", "cbar1", "pushed", "cbar2", "done"]
an = ["entry", "setup", "pdl", "q_ready", "loop_end", "-", "merged", "end"]
for k in ("qkv", "attn", "o", "gu", "d"):
    if k == "attn":
        t = at.view(-1, 8).cpu().numpy().astype(np.float64)
        names = an
    else:
        t = bufs[k].view(-1, 16).cpu().numpy().astype(np.float64)
        names = gn
    print(f"  {k}")
    for i, nm in enumerate(names):
        if nm == "-":
            continue
        a, b, c = stats(t[:, i])
        if not np.isnan(a):
            print(f"    {nm:10s} {(a-t0)/1e3:7.2f} {(b-t0)/1e3:7.2f} {(c-t0)/1e3:7.2f}")
