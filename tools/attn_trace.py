"""Per-CTA timeline of the fused attention in a forward graph (tuning aid)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.llama import PRESETS, RowBlock

which = sys.argv[1] if len(sys.argv) > 1 else "d116"
preset, m = {"d116": ("llama-3.2-1b", 116), "t8": ("llama-3.1-8b", 8)}[which]
cfg = PRESETS[preset]
mdl = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = mdl.runtime(1088, 0, sorted({m, 128}))
rows = RowBlock(m, 16, rt.dev)
rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, m)], 1000 - m,
               out_last_only=False)
rt.forward(rows, m)
torch.cuda.synchronize()
buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
lib().card_attention_trace(ctypes.c_void_p(buf.data_ptr()))
# one attention launch (layer 0 inputs), warm then traced
L = lib()
from paper_2508_04462_b200._device import ptr, stream_ptr
c = cfg
def run():
    L.card_attention(ptr(rt.q), ptr(rows.M), m, ptr(rows.plen), ptr(rows.slot), ptr(rows.n_extra), ptr(rows.extra), rows.extra_max,
                     ptr(rt.k_cache[0]), ptr(rt.v_cache[0]), 0, c.n_heads, c.n_kv_heads, c.head_dim, rt.prefix_slots,
                     ptr(rt.work), ptr(rt.o), 0, stream_ptr())
run(); torch.cuda.synchronize()
buf.zero_(); run(); torch.cuda.synchronize()
lib().card_attention_trace(None)
t = buf.view(-1, 8).cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["entry", "setup", "pdl", "q_ready", "loop_end", "clsync1", "clsync2", "end"]
print(f"{which}: {len(t)} CTAs")
for k, nm in enumerate(names):
    v = t[:, k][t[:, k] > 0] - t0
    if len(v):
        print(f"  {nm:9s} min {v.min()/1e3:7.2f} med {np.median(v)/1e3:7.2f} max {v.max()/1e3:7.2f} us")
