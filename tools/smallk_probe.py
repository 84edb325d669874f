"""Acceptance over a 256-token decode at small K: single-request engine vs
BatchRun, with the trees' final state (status, nodes, dead)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2508_04462_b200 as card
from paper_2508_04462_b200.batch import BatchRun
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

K = int(os.environ.get("K", "3"))
new = int(os.environ.get("NEW", "256"))
bias = LogitBias(seed=11, order=2, sharpness=1e6)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
cfg = card.EngineConfig(K=K, k=3, ratio=7, max_new_tokens=new)
P = [[int(x) for x in np.random.default_rng(1000 + i).integers(0, 128256, 512)] for i in range(4)]
for i in range(4):
    r = card.run_speculative(draft, target, P[i], cfg)
    acc = [ev.lnew for ev in r.trace if ev.event in ("verify", "miss_step")]
    print(f"single {i}: acceptance {r.metrics.mean_acceptance_length:.2f}  lnew by cycle {acc}", flush=True)
run = BatchRun(draft, target, P, cfg)
run.prefill()
run.capture()
run.run()
for i in range(4):
    acc = [ev.lnew for ev in run.traces[i] if ev.event in ("verify", "miss_step")]
    st = run.caches[i].state()
    print(f"batch {i}: lnew by cycle {acc}  cache status {st.status} nodes {st.n_nodes} dead {st.dead} cap {run.cap}",
          flush=True)
