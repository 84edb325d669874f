"""Draft-tree attention at the bench shape (Llama-3.2-1B: hd 64, 32 q / 8 kv
heads; 16 chain rows + 100 tree rows with ancestor extras over a paged
prefix): fp32 torch reference check, CUDA-graph replay time per launch, and
the per-CTA phase stamps of one launch.  Usage: attn_tree_probe.py [P] [depth]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2508_04462_b200._device import ptr, stream_ptr
from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.llama import RowBlock

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 10
hd, nh, nkv, M, n_chain, XM = 64, 32, 8, 116, 16, 16
rng = np.random.default_rng(0)
g = torch.Generator(device="cuda").manual_seed(1)
n_pages = (P + 64 + 63) // 64
perm = rng.permutation(n_pages + 8)[:n_pages]
table = torch.tensor(perm, dtype=torch.int32, device="cuda")
tree_base = (n_pages + 8) * 64
slots = tree_base + 4096
kc = (torch.randn(slots, nkv, hd, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
vc = torch.randn(slots, nkv, hd, device="cuda", generator=g).to(torch.bfloat16)
q = torch.randn(M, nh, hd, device="cuda", generator=g) * (2.0 / hd ** 0.5)
rows = RowBlock(M, XM, "cuda")
R = M
host = torch.zeros(rows.block.numel(), dtype=torch.int32)
host[0] = M
plen = [P - n_chain + i + 1 for i in range(n_chain)] + [P] * (M - n_chain)
nx = [0] * n_chain + [int(rng.integers(1, depth + 1)) for _ in range(M - n_chain)]
extra = np.zeros((M, XM), dtype=np.int32)
for m in range(n_chain, M):
    extra[m, :nx[m]] = tree_base + rng.choice(4096, nx[m], replace=False)
host[2 + 3 * R:2 + 4 * R] = torch.tensor(plen)
host[2 + 4 * R:2 + 5 * R] = torch.tensor(nx)
host[2 + 6 * R:] = torch.from_numpy(extra.reshape(-1))
rows.block.copy_(host)
o = torch.zeros(M, nh * hd, device="cuda", dtype=torch.bfloat16)


def run():
    rc = lib().card_attention_paged(ptr(q), ptr(rows.M), M, ptr(rows.plen), ptr(rows.n_extra), ptr(rows.extra), XM,
                                    ptr(kc), ptr(vc), ptr(table), nh, nkv, hd, P + 64, ptr(o), stream_ptr())
    assert rc == 0, rc


# fp32 reference
run()
torch.cuda.synchronize()
kf, vf = kc.float(), vc.float()
pslots = (table.long().repeat_interleave(64) * 64 + torch.arange(64, device="cuda").repeat(n_pages))
ref = torch.zeros(M, nh, hd, device="cuda")
for m in range(M):
    sl = torch.cat([pslots[:plen[m]], torch.from_numpy(extra[m, :nx[m]]).long().cuda()])
    K = kf[sl].repeat_interleave(nh // nkv, dim=1)   # [n, nh, hd]
    V = vf[sl].repeat_interleave(nh // nkv, dim=1)
    s = torch.einsum("hd,nhd->hn", q[m], K)
    p = torch.softmax(s, dim=-1)
    ref[m] = torch.einsum("hn,nhd->hd", p, V)
err = ((o.float().view(M, nh, hd) - ref).abs().max() / ref.abs().max()).item()
print(f"P={P} depth<={depth}: max abs err / max |ref| = {err:.2e}")
# timing: graph of 20 launches
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    run()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20):
            run()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gr.replay()
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b) / 20 * 1e3)
print(f"graph replay: {np.median(ts):.2f} us per launch (min {min(ts):.2f})")
buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
lib().card_attention_trace(ctypes.c_void_p(buf.data_ptr()))
run()
torch.cuda.synchronize()
buf.zero_()
run()
torch.cuda.synchronize()
lib().card_attention_trace(None)
t = buf.view(-1, 8).cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
print(f"{len(t)} CTAs")
for k, nm in enumerate(["entry", "setup", "pdl", "q_ready", "loop_end", "first_S", "merged", "end"]):
    v = t[:, k][t[:, k] > 0] - t0
    if len(v):
        print(f"  {nm:9s} min {v.min() / 1e3:7.2f} med {np.median(v) / 1e3:7.2f} max {v.max() / 1e3:7.2f} us")
