"""Per-step timeline of the persistent wide forward (card_pfwd_trace stamps).

Runs the bench draft forward (Llama-3.2-1B, M=116 chain rows at ctx 1024)
eagerly with one stamp buffer per card_pfwd launch and prints, per launch,
each step's stamps (min / median / max over CTAs, us from the launch's first
CTA start): 0 activations released, 1 first k-block in, 2 accumulator done,
3 outputs published; and the gap between launches (attention + 2 launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._device import ptr, stream_ptr
from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.llama import PRESETS, DeviceLlama, RowBlock

preset = sys.argv[1] if len(sys.argv) > 1 else "llama-3.2-1b"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 116
ctx = 1024
cfg = PRESETS[preset]
m = card.LlamaModel(cfg, seed=1, dtype="bf16")
rt = DeviceLlama(cfg, m.packed, max_ctx=ctx + 64, tree_slots=0, row_budgets=(M,), persistent=True)
rows = RowBlock(M, 16, rt.dev)
rows.set_chain([int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab_size, M)], ctx - M,
               out_last_only=False)
plan = rt.plans[M]
pf = plan["pfwd"]
rt.forward(rows, M)
torch.cuda.synchronize()
G = pf.info()["grid"]
n5 = 5
L_ = lib()
c = cfg
inkernel = False
if inkernel:
    launches = [(0, n5 * c.n_layers)]
else:
    launches = [(0, 1)] + [(n5 * li + 2, min(n5 * (li + 1) + 1, n5 * c.n_layers)) for li in range(c.n_layers)]
bufs = [torch.zeros(G * (2 + 8 * (e - b)), dtype=torch.int64, device="cuda") for b, e in launches]
rt._bind_rows(plan, rows)
dM = rows.M
attn_buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")


assert pf.use_qsw(rows.extra_max)


def sequence():
    for i, (b, e) in enumerate(launches):
        L_.card_pfwd_trace(pf.h, ptr(bufs[i]))
        if i > 0 and not inkernel:
            li = i - 1
            L_.card_attention_tree(ptr(pf.qsw), pf.qsw_tiles, ptr(dM), plan["m_max"], ptr(rows.plen), ptr(rows.n_extra),
                                   ptr(rows.extra), rows.extra_max, ptr(rt.k_cache[li]), ptr(rt.v_cache[li]), None,
                                   c.n_heads, c.n_kv_heads, c.head_dim, rt.prefix_slots, ptr(rt.o), stream_ptr())
        pf.run(dM, b, e)


# in-graph timeline (as the engine replays it): stamps of the last replay;
# the attention stamps are the last layer's (one shared buffer)
L_.card_attention_trace(ptr(attn_buf))
gs = torch.cuda.Stream()
with torch.cuda.stream(gs):
    sequence()
    gs.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=gs):
        sequence()
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
L_.card_pfwd_trace(pf.h, None)
L_.card_attention_trace(None)
names = ["qkv", "attn", "o", "gu", "d"]
t_first = None
prev_end = None
show = {0, 1, 2, c.n_layers} if not inkernel else {0}
for i, (b, e) in enumerate(launches):
    tr = bufs[i].cpu().numpy().reshape(G, 2 + 8 * (e - b)).astype(np.float64)
    t0 = tr[:, 0].min()
    if t_first is None:
        t_first = t0
    gap = (t0 - prev_end) / 1e3 if prev_end is not None else 0.0
    end = tr[:, 1].max()
    if i in show:
        print(f"launch {i} steps [{b},{e}): start +{(t0 - t_first) / 1e3:8.1f} us  (gap from previous end {gap:6.1f})"
              f"  CTA start spread {(tr[:, 0].max() - t0) / 1e3:5.1f}  duration {(end - t0) / 1e3:6.1f} us")
        for j, st in enumerate(range(b, e)):
            if inkernel and 10 <= st < n5 * c.n_layers - 5:
                continue
            cols = tr[:, 2 + 8 * j:10 + 8 * j]
            desc = []
            nms = ("rel", "kb0", "acc", "pub", "drained", "allin", "reduced", "-")
            if st % n5 == 1:
                nms = ("-", "-", "-", "pub", "dep", "meta", "S0", "rounds", "merged_wait", "-", "-", "-") + sum(
                    ((f"S{i}iss", f"PV{i}iss", f"S{i}seen", f"O{i}seen") for i in range(2)), ()) + ("sSeen", "sMax", "sExpA", "sExpB", "sArr", "-", "-", "-") + tuple(
                    f"kv{i}" for i in range(4))
            for k, nm in enumerate(nms[:cols.shape[1]]):
                if nm == "-":
                    continue
                v = cols[:, k]
                v = v[v > 0]
                if len(v):
                    desc.append(f"{nm} {(np.median(v) - t0) / 1e3:5.1f}")
            print(f"   L{st // n5:2d}.{names[st % n5]:4s} " + "  ".join(desc))
    elif i > 0:
        pass
    prev_end = end
total = (prev_end - t_first) / 1e3
print(f"all pfwd launches + attention: {total:.1f} us over {c.n_layers} layers ({total / c.n_layers:.1f} us/layer)")
at = attn_buf.view(-1, 8).cpu().numpy().astype(np.float64)
at = at[at[:, 0] > 0]
last = bufs[-2].cpu().numpy().reshape(G, -1).astype(np.float64)   # launch before the last attention
nxt = bufs[-1].cpu().numpy().reshape(G, -1).astype(np.float64)
pend = last[:, 1].max()
print(f"last attention ({len(at)} CTAs), us after the previous pfwd launch's last CTA exit:")
for k, nm in enumerate(["entry", "setup", "pdl", "q_ready", "loop_end", "-", "merged", "end"]):
    v = at[:, k][at[:, k] > 0] - pend
    if len(v):
        print(f"  {nm:9s} min {v.min() / 1e3:7.2f} med {np.median(v) / 1e3:7.2f} max {v.max() / 1e3:7.2f}")
print(f"  next pfwd launch: first CTA start {(nxt[:, 0].min() - pend) / 1e3:7.2f}  last CTA start {(nxt[:, 0].max() - pend) / 1e3:7.2f}")
