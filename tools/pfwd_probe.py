"""Persistent wide forward (card_pfwd) vs the per-GEMM fused forward on the
bench draft (Llama-3.2-1B, M rows): logits agreement and CUDA-graph replay
time of both.  Usage: python tools/pfwd_probe.py [preset] [M] [ctx]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, DeviceLlama, RowBlock

preset = sys.argv[1] if len(sys.argv) > 1 else "llama-3.2-1b"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 116
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
cfg = PRESETS[preset]
SWEEP = [(9, 9, 6), (4, 9, 6), (4, 4, 6), (4, 8, 3), (2, 8, 3), (8, 8, 4), (4, 6, 4)] if "sweep" in sys.argv else []
m = card.LlamaModel(cfg, seed=1, dtype="bf16")
toks = [int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, M)]
out = {}
for persistent in (False, True):
    rt = DeviceLlama(cfg, m.packed, max_ctx=ctx + 64, tree_slots=0, row_budgets=(M,), persistent=persistent)
    rows = RowBlock(M, 16, rt.dev)
    rows.set_chain(toks, ctx - M, out_last_only=False)
    if persistent:
        print("pfwd plan:", rt.plans[M]["pfwd"].info())
    rt.forward(rows, M)
    torch.cuda.synchronize()
    out[persistent] = rt.logits[:M].clone()
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
    graph_logits = rt.logits[:M].clone()
    rel_graph = float((graph_logits - out[persistent]).norm() / out[persistent].norm())
    wbytes = cfg.stream_params() * 2
    t = float(np.median(ts))
    print(f"persistent={persistent}: forward {t:.3f} ms (min {min(ts):.3f})  weight stream {wbytes / t / 1e6:.0f} GB/s"
          f"  graph-vs-eager rel {rel_graph:.2e}")
    if persistent:
        from paper_2508_04462_b200._lib import lib as _l
        for so, sd, sq in SWEEP:
            for ph, sp in ((2, so), (4, sd), (0, sq)):
                assert _l().card_pfwd_tune(rt.plans[M]["pfwd"].h, ph, sp) == 0
            with torch.cuda.stream(s):
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2, stream=s):
                    rt.forward(rows, M)
            g2.replay()
            torch.cuda.synchronize()
            tt = []
            for _ in range(10):
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record()
                g2.replay()
                b_.record()
                b_.synchronize()
                tt.append(a_.elapsed_time(b_))
            d = float((rt.logits[:M] - out[True]).norm() / out[True].norm())
            print(f"   splits o={so} d={sd} qkv={sq}: {np.median(tt):.3f} ms  (rel vs default {d:.1e})")
            del g2
    del g, rt
a, b = out[False].double(), out[True].double()
rel = float((a - b).norm() / a.norm())
rows_rel = ((a - b).norm(dim=1) / a.norm(dim=1)).max().item()
top_eq = float((a.argmax(1) == b.argmax(1)).double().mean())
print(f"persistent vs layered: block rel {rel:.3e}  worst row {rows_rel:.3e}  argmax agreement {top_eq:.3f}")
