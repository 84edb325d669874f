"""Draft forward time for a narrow frontier: the 116-row plan running M rows
versus a plan sized for M (graph replay, Llama-3.2-1B, ctx 1024)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, RowBlock

cfg = PRESETS["llama-3.2-1b"]
mdl = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = mdl.runtime(1088, 0, {16, 32, 64, 116})


def graph_time(m_rows, plan_m):
    rows = RowBlock(plan_m, 16, rt.dev)
    rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, m_rows)], 1000 - m_rows,
                   out_last_only=False)
    rt.forward(rows, plan_m)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        rt.forward(rows, plan_m)
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for m in (9, 16, 27, 32, 64, 100):
    own = min(p for p in (16, 32, 64, 116) if p >= m)
    print(f"M={m:3d}: 116-row plan {graph_time(m, 116):.3f} ms   {own}-row plan {graph_time(m, own):.3f} ms", flush=True)
