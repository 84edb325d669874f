"""Draft lm_head variants at M = 116 rows (Llama-3.2-1B, V = 128256), CUDA
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
for sharp_on in (False, True):
    b = bias if sharp_on else (None, 0, 0, 0, 0, 0.0, 0.0)
    L.card_linear_fuse_kgram(lm.h, *b)
    L.card_linear_fuse_kgram(head.h, *b)
    L.card_linear_fuse_topk(head.h, V, 1.0)
    t_lm = timeit(lambda: lm.run(rows.n_out))
    t_rd = timeit(lambda: L.card_topk_logits(ptr(rt.logits), ptr(rows.n_out), m, V, 3, 1.0, ptr(tok), ptr(lp), ptr(cnt),
                                             ptr(wk), None, 0, 0, 0, 0, 0.0, 0.0, stream_ptr()))
    t_head = timeit(lambda: head.run(rows.n_out))
    t_mg = timeit(lambda: L.card_lmhead_topk_merge(ptr(head.work), ptr(rows.n_out), m, head.n_tiles, 3, V, ptr(tok),
                                                  ptr(lp), ptr(cnt), stream_ptr()))
    print(f"bias {'on ' if sharp_on else 'off'}: logits lm_head {t_lm:6.1f} us + reader {t_rd:5.1f} us = {t_lm + t_rd:6.1f}   |   "
          f"EPI_TOPK head {t_head:6.1f} us + merge {t_mg:5.1f} us = {t_head + t_mg:6.1f}", flush=True)
L.card_linear_fuse_kgram(lm.h, None, 0, 0, 0, 0, 0.0, 0.0)
