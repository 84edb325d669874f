"""Where the end-to-end time of one run_speculative call goes (serial graph
driver): DeviceRun setup, prefill, graph capture, decode, output/trace."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200 import engine as E
from paper_2508_04462_b200.lm import LogitBias
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.metrics import finalize

tcfg, dcfg = PRESETS["llama-3.1-8b"], PRESETS["llama-3.2-1b"]
bias = LogitBias(seed=11, order=2, sharpness=1e6, mix_seed=131, mix_weight=0.0)
target = card.LlamaModel(tcfg, seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.0, 7.0))
draft = card.LlamaModel(dcfg, seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.2, 1.0))
cfg = card.EngineConfig(K=100, k=3, ratio=7, temperature=0.0, max_new_tokens=512, seed=0)


def sync_t():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(4):
    prompt = [int(x) for x in np.random.default_rng(1000 + rep).integers(0, tcfg.vocab_size, 512)]
    t = [sync_t()]
    run = E.DeviceRun(draft, target, prompt, cfg, trace_alive=False)
    t.append(sync_t())
    run.prefill()
    t.append(sync_t())
    run.capture()
    t.append(sync_t())
    run.run_graphs()
    t.append(sync_t())
    out = run.output
    res = finalize(run.trace, target.spec, draft.spec)
    t.append(sync_t())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: setup {d[0]:7.1f} ms  prefill {d[1]:7.1f}  capture {d[2]:7.1f}  decode {d[3]:7.1f}  "
          f"output {d[4]:6.1f}   ({len(out)} tokens, acc {res.mean_acceptance_length:.2f})", flush=True)
