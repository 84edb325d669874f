"""Timeline of mode=concurrent on one B200 (events exchange): device
timestamps of every verify / draft-step / correction graph of a few cycles,
with or without SM partitions.  Usage: concurrent_timeline.py [draft_sms]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._lib import EngineState
from paper_2508_04462_b200.llama import PRESETS
from paper_2508_04462_b200.lm import LogitBias

dsms = int(sys.argv[1]) if len(sys.argv) > 1 else 0
persistent = not (len(sys.argv) > 2 and sys.argv[2] == "nopf")
bias = LogitBias(seed=11, order=2, sharpness=1e6)
target = card.LlamaModel(PRESETS["llama-3.1-8b"], seed=2, dtype="bf16", bias=bias, spec=card.ModelSpec(8.03, 7.0))
draft = card.LlamaModel(PRESETS["llama-3.2-1b"], seed=1, dtype="bf16", bias=bias, spec=card.ModelSpec(1.24, 1.0),
                        persistent=persistent)
prompt = [int(x) for x in np.random.default_rng(1000).integers(0, 128256, 512)]
cfg = card.EngineConfig(K=100, k=3, ratio=7, max_new_tokens=96, mode="concurrent")
card.run_speculative(draft, target, prompt, cfg, draft_sms=dsms or None)   # builds the session + graphs
run = next(iter(target._card_sessions.values()))
drv = run._cdriver
run.rebind(prompt)
run.prefill()
torch.cuda.synchronize()
t_ref = torch.cuda.Event(enable_timing=True)
t_ref.record()
marks = []


def stamp(stream, label):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    marks.append((label, e))


D, T = drv.D, drv.T
D.wait_stream(torch.cuda.current_stream())
T.wait_stream(torch.cuda.current_stream())
for _ in range(cfg.query_depth):
    with torch.cuda.stream(D):
        stamp(D, "d<")
        drv.g_d.replay()
        stamp(D, "d>")
with torch.cuda.stream(D):
    drv.g_q.replay()
    q_ev = torch.cuda.Event()
    q_ev.record(D)
for cyc in range(6):
    T.wait_event(q_ev)
    with torch.cuda.stream(T):
        stamp(T, "V<")
        drv.g_t.replay()
        stamp(T, "V>")
        v_ev = torch.cuda.Event()
        v_ev.record(T)
    n = 0
    while not v_ev.query():
        with torch.cuda.stream(D):
            stamp(D, "d<")
            drv.g_d.replay()
            stamp(D, "d>")
            ev = torch.cuda.Event()
            ev.record(D)
        ev.synchronize()
        n += 1
    E = EngineState.from_buffer_copy(run._host.numpy().tobytes())
    D.wait_event(v_ev)
    with torch.cuda.stream(D):
        stamp(D, "c<")
        drv.g_c.replay()
        stamp(D, "c>")
        q_ev = torch.cuda.Event()
        q_ev.record(D)
torch.cuda.synchronize()
line = []
for label, e in marks:
    line.append(f"{label}{t_ref.elapsed_time(e):.2f}")
print(f"draft_sms={dsms} persistent={persistent}: " + " ".join(line[:60]))
