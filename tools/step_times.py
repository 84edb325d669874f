"""Per-graph CUDA-event timing of one CARD decode on the BASELINE config:
every draft-step graph and every target-step graph replay timed separately."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._lib import EngineState
from paper_2508_04462_b200.engine import DeviceRun
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

sharp = float(os.environ.get("SHARP", "3000"))
new = int(os.environ.get("NEW", "64"))
K = int(os.environ.get("K", "100"))
bias = LogitBias(seed=11, order=2, sharpness=sharp)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0))
prompt = [int(x) for x in np.random.default_rng(1000).integers(0, 128256, 512)]
cfg = card.EngineConfig(K=K, k=3, ratio=7, max_new_tokens=new)
run = DeviceRun(draft, target, prompt, cfg, trace_alive=False)
run.prefill()
run.capture()
torch.cuda.synchronize()
g_d, g_t = run.graphs
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
d_ms, t_ms = [], []
for _ in range(cfg.query_depth):
    a, b = ev(), ev()
    a.record()
    g_d.replay()
    b.record()
    b.synchronize()
    d_ms.append(a.elapsed_time(b))
run._set_field("n_widths", 0)
run._set_field("stop", 0)
depth = cfg.query_depth
done = False
cycles = 0
accs = []
while not done and cycles < 200:
    n_exp = min(cfg.ratio, max(0, cfg.max_depth - depth))
    for _ in range(n_exp):
        a, b = ev(), ev()
        a.record()
        g_d.replay()
        b.record()
        b.synchronize()
        d_ms.append(a.elapsed_time(b))
    a, b = ev(), ev()
    a.record()
    g_t.replay()
    b.record()
    b.synchronize()
    t_ms.append(a.elapsed_time(b))
    E = EngineState.from_buffer_copy(run._host.numpy().tobytes())
    accs.append(E.n_commit)
    done = bool(E.rec_done)
    depth = E.rec_depth
    cycles += 1
print(f"launches per graph (draft, target): {run.launches_per_graph}")
print(f"draft steps {len(d_ms)}: median {np.median(d_ms):.3f} ms  min {min(d_ms):.3f}  max {max(d_ms):.3f}")
print(f"target steps {len(t_ms)}: median {np.median(t_ms):.3f} ms  min {min(t_ms):.3f}  max {max(t_ms):.3f}")
print(f"committed per cycle: mean {np.mean(accs):.3f}  hist {np.bincount(accs).tolist()}")
print("draft step times (first 20):", [round(x, 3) for x in d_ms[:20]])
