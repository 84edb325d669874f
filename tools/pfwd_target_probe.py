"""Persistent forward for the narrow target forwards (verify M=8, AR M=1) of
Llama-3.1-8B vs the per-GEMM fused forward: graph-replay time, logits
agreement, and whether the verify's last row is bit-identical to the AR
forward of the same token (greedy CARD == AR needs it)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, DeviceLlama, RowBlock

preset = sys.argv[1] if len(sys.argv) > 1 else "llama-3.1-8b"
cfg = PRESETS[preset]
m = card.LlamaModel(cfg, seed=2, dtype="bf16")
ctx = 1000
toks = [int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, ctx + 8)]


def graph_time(rt, rows, M):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        rt.forward(rows, M)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            rt.forward(rows, M)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


out = {}
for mode in (True, "all"):
    rt = DeviceLlama(cfg, m.packed, max_ctx=ctx + 72, tree_slots=0, row_budgets=(1, 8, 128), persistent=mode)
    pre = RowBlock(128, 1, rt.dev)
    for s0 in range(0, ctx, 128):   # prefill
        pre.set_chain(toks[s0:min(ctx, s0 + 128)], s0)
        rt.forward(pre, 128)
    r8 = RowBlock(8, 1, rt.dev)
    r8.set_chain(toks[ctx:ctx + 8], ctx, out_last_only=False)
    rt.forward(r8, 8)
    torch.cuda.synchronize()
    l8 = rt.logits[:8].clone()
    r1 = RowBlock(1, 1, rt.dev)
    r1.set_chain(toks[ctx + 7:ctx + 8], ctx + 7)
    rt.forward(r1, 1)
    torch.cuda.synchronize()
    l1 = rt.logits[:1].clone()
    t8 = graph_time(rt, r8, 8)
    t1 = graph_time(rt, r1, 1)
    wb = cfg.stream_params() * 2
    print(f"persistent={mode!s:5s}: verify M=8 {t8:.3f} ms ({wb / t8 / 1e6:.0f} GB/s)  AR M=1 {t1:.3f} ms "
          f"({wb / t1 / 1e6:.0f} GB/s)  verify row 7 == AR bitwise: {torch.equal(l8[7], l1[0])}", flush=True)
    if "info" not in out and "pfwd" in rt.plans[8]:
        print("  pfwd plan M=8:", rt.plans[8]["pfwd"].info())
    out[mode] = l8
    del rt
    torch.cuda.empty_cache()
a, b = out[True], out["all"]
print(f"logits rel diff per-GEMM vs persistent: {float((a - b).norm() / a.norm()):.2e}")
