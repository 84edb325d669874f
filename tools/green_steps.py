"""Draft-step and verify-step graph times on SM partitions of one B200
(card_green): each step alone on its partition, then both at once."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes

import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.engine import DeviceRun, _green_partition
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

bias = LogitBias(seed=11, order=2, sharpness=1e6)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
prompt = [int(x) for x in np.random.default_rng(1000).integers(0, 128256, 512)]
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=64, mode="concurrent")   # separate draft state


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return ts


for dsms in [int(x) for x in (sys.argv[1:] or ["0", "48", "64", "80", "96"])]:
    run = DeviceRun(draft, target, prompt, cfg, trace_alive=False)   # fresh state per partition
    run.prefill()
    torch.cuda.synchronize()
    if dsms:
        (pd, pt), (nd, nt) = _green_partition(0, dsms)
        SD, ST = torch.cuda.ExternalStream(pd), torch.cuda.ExternalStream(pt)
    else:
        SD, ST, nd, nt = torch.cuda.Stream(), torch.cuda.Stream(), 148, 148
    pfs = [p["pfwd"] for p in run.da.rt.plans.values() if "pfwd" in p]
    for f in pfs:
        lib().card_pfwd_set_grid(f.h, nd if dsms else 0)
    gd, gt = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    for S, g, fn in ((SD, gd, run.launch_draft_step),
                     (ST, gt, lambda: run.launch_target_step(with_correct=False, readback=False))):
        S.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(S), torch.cuda.graph(g, stream=S):
            fn()
        torch.cuda.current_stream().wait_stream(S)
    for f in pfs:
        lib().card_pfwd_set_grid(f.h, 0)

    def on(S, g):
        def f():
            with torch.cuda.stream(S):
                g.replay()
            torch.cuda.current_stream().wait_stream(S)
        return f

    # draft steps from a fresh tree (real expansions), then verify steps
    td = timed(on(SD, gd), reps=6)
    run.launch_correct   # (the verify below reads the query of the draft state as it stands)
    lib().card_cache_query(run.cache.handle, cfg.query_depth, None)
    torch.cuda.synchronize()
    tt = timed(on(ST, gt), reps=3)
    print(f"draft SMs {nd:3d} / target SMs {nt:3d}: draft steps {[round(x, 3) for x in td]} ms, "
          f"verify steps {[round(x, 3) for x in tt]} ms", flush=True)
    del run, gd, gt
    torch.cuda.empty_cache()
