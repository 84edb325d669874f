"""Does a draft forward (M=116) overlap a target verify forward (M=8) on one
B200?  Times serial vs two-stream concurrent replays of the two graphs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.llama import PRESETS, RowBlock


def build(preset, m, seed):
    cfg = PRESETS[preset]
    mdl = card.LlamaModel(cfg, seed=seed, dtype="bf16")
    rt = mdl.runtime(1088, 0, sorted({m, 128}))
    rows = RowBlock(m, 16, rt.dev)
    rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, m)], 1000 - m,
                   out_last_only=False)
    rt.forward(rows, m)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        rt.forward(rows, m)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    return mdl, rt, rows, g


keep_t = build("llama-3.1-8b", 8, 2)
gt = keep_t[3]
keep_d = build("llama-3.2-1b", 116, 1)
gd = keep_d[3]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for nd in (1, 2, 3):
    def serial():
        gt.replay()
        for _ in range(nd):
            gd.replay()

    def conc():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            gt.replay()
        with torch.cuda.stream(s2):
            for _ in range(nd):
                gd.replay()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    print(f"1 target + {nd} draft: serial {timed(serial):.3f} ms  concurrent {timed(conc):.3f} ms")
print(f"target alone {timed(lambda: gt.replay()):.3f} ms, draft alone {timed(lambda: gd.replay()):.3f} ms")
