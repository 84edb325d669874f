"""Time card_attention at the bench's draft-tree and verify shapes (CUDA
events over 50 graph-free launches after warm-up).  GPU only."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_04462_b200._device import ptr, stream_ptr  # noqa: E402
from paper_2508_04462_b200._lib import lib  # noqa: E402
from paper_2508_04462_b200.llama import RowBlock  # noqa: E402


def one(hd, nh, nkv, M, P, n_tree, depth):
    g = torch.Generator(device="cuda").manual_seed(1)
    slots = P + 64 + 4096
    kc = torch.randn(slots, nkv, hd, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn_like(kc)
    q = torch.randn(M, nh, hd, device="cuda", generator=g) / hd ** 0.5
    rows = RowBlock(M, 16, "cuda")
    R = M
    host = torch.zeros(rows.block.numel(), dtype=torch.int32)
    host[0] = M
    n_chain = M - n_tree
    plen = [P - n_chain + i + 1 for i in range(n_chain)] + [P] * n_tree
    nx = [0] * n_chain + [depth] * n_tree
    host[2 + 3 * R:2 + 4 * R] = torch.tensor(plen)
    host[2 + 4 * R:2 + 5 * R] = torch.tensor(nx)
    for m in range(n_chain, M):
        host[2 + 6 * R + m * 16:2 + 6 * R + m * 16 + depth] = torch.arange(P + 64 + m * depth, P + 64 + (m + 1) * depth)
    rows.block.copy_(host)
    o = torch.zeros(M, nh * hd, device="cuda", dtype=torch.bfloat16)
    work = torch.zeros(lib().card_attention_work_floats(((M + 15) // 16) * 16, nh, hd, P + 64), device="cuda")

    def run():
        lib().card_attention(ptr(q), ptr(rows.M), M, ptr(rows.plen), ptr(rows.slot), ptr(rows.n_extra),
                             ptr(rows.extra), 16, ptr(kc), ptr(vc), 0, nh, nkv, hd, P + 64, ptr(work), ptr(o), 0,
                             stream_ptr())
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        run()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) / 50 * 1e3
    print(f"attention hd={hd} M={M} plen~{P} tree_rows={n_tree} depth={depth}: {us:.1f} us/launch")


one(64, 32, 8, 116, 1024, 100, 6)     # draft tree step (Llama-3.2-1B)
one(128, 32, 8, 8, 1024, 0, 0)        # target verify (Llama-3.1-8B)
one(128, 32, 8, 1, 1024, 0, 0)        # AR step
