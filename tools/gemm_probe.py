"""Run one weight-streaming GEMM shape a few times (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2508_04462_b200.llama import _Linear, tile_sw128

N, K, M, epi = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
mpad = ((M + 15) // 16) * 16
X = torch.randn(mpad, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(mpad, N if epi != 3 else N // 2, device="cuda", dtype=torch.float32 if epi < 2 else torch.bfloat16)
dM = torch.tensor([M], dtype=torch.int32, device="cuda")
Wl = W if os.environ.get("ROWMAJOR") else tile_sw128(W)   # production layout: pre-tiled SW128
lin = _Linear(Wl, X, M, epi, out, out.shape[1])
print(lin.info)
for _ in range(reps):
    lin.run(dM)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    lin.run(dM)
b.record()
b.synchronize()
t = a.elapsed_time(b) / 20
print(f"N={N} K={K} M={M}: {t*1e3:.1f} us/launch  {N*K*2/t/1e6:.0f} GB/s (back-to-back, L2-warm for W<126MB)")
