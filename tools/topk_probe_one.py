"""(ncu target) Draft lm_head variants at M = 116 rows (Llama-3.2-1B, V = 128256), CUDA
events, L2 flushed: logits + k-gram bias epilogue + top-k reader versus the
fused EPI_TOPK head + record merge."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._device import ptr, stream_ptr
from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.llama import PRESETS, RowBlock

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


cfg = PRESETS["llama-3.2-1b"]
m = 116
mdl = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = mdl.runtime(1088, 0, {m})
rows = RowBlock(m, 16, rt.dev)
rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, m)], 1000 - m, out_last_only=False)
rt.forward(rows, m)
V = cfg.vocab_size
tail = torch.randint(0, V, (m, 2), dtype=torch.int32, device="cuda")
bias = (ptr(tail), 2, 2, 11, 131, 0.0, 1e6)
L = lib()
plan = rt.plans[m]
lm = plan["lm_head"]
head = rt.lm_topk_head(m)
rt._bind_rows(plan, rows)
tok = torch.zeros((m, 3), dtype=torch.int32, device="cuda")
lp = torch.zeros((m, 3), dtype=torch.float64, device="cuda")
cnt = torch.zeros(m, dtype=torch.int32, device="cuda")
wk = torch.zeros(L.card_lmhead_work_floats(m, 3), dtype=torch.float32, device="cuda")
L.card_linear_fuse_topk(head.h, V, 1.0)
L.card_linear_fuse_kgram(head.h, None, 0, 0, 0, 0, 0.0, 0.0)
head.run(rows.n_out)
head.run(rows.n_out)
torch.cuda.synchronize()
print("ok")
