"""Would splitting the draft tree forward into two row halves on two streams
help?  Times one M=116 forward vs two M=58 forwards (separate runtimes, same
weights) serial and concurrent."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, RowBlock, DeviceLlama

cfg = PRESETS["llama-3.2-1b"]
mdl = card.LlamaModel(cfg, seed=1, dtype="bf16")
def mk(m):
    rt = DeviceLlama(cfg, mdl.packed, max_ctx=1088, tree_slots=0, row_budgets=sorted({m, 128}))
    rows = RowBlock(m, 16, rt.dev)
    rows.set_chain([int(x) for x in np.random.default_rng(m).integers(0, cfg.vocab_size, m)], 1000 - m, out_last_only=False)
    rt.forward(rows, m); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream(); st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        rt.forward(rows, m)
    torch.cuda.current_stream().wait_stream(st); torch.cuda.synchronize()
    return rt, rows, g
k116 = mk(116); ka = mk(58); kb = mk(58)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=7):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
def conc():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): ka[2].replay()
    with torch.cuda.stream(s2): kb[2].replay()
    cur.wait_stream(s1); cur.wait_stream(s2)
print(f"M=116 one forward: {timed(lambda: k116[2].replay()):.3f} ms")
print(f"M=58 one forward: {timed(lambda: ka[2].replay()):.3f} ms")
print(f"2 x M=58 serial: {timed(lambda: (ka[2].replay(), kb[2].replay())):.3f} ms")
print(f"2 x M=58 concurrent: {timed(conc):.3f} ms")
