"""Per-CTA %globaltimer timeline of one tc_gemm launch (tuning aid).
stamps: 0 entry, 1 after griddepcontrol.wait, 2 first k-block landed (MMA
thread), 3 last MMA issued, 4 accumulator ready (epilogue), 5 cluster
barrier 1, 6 pushes issued, 7 cluster barrier 2, 8 epilogue done."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.llama import _Linear, tile_sw128

N, K, M, epi = (int(x) for x in sys.argv[1:5])
W = tile_sw128((torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16))
mpad = ((M + 15) // 16) * 16
X = torch.randn(mpad, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(mpad, N if epi != 3 else N // 2, device="cuda", dtype=torch.float32 if epi < 2 else torch.bfloat16)
dM = torch.tensor([M], dtype=torch.int32, device="cuda")
lin = _Linear(W, X, M, epi, out, out.shape[1])
grid = lin.info["grid"]
tr = torch.zeros(grid * 16, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(4):
    lin.run(dM)
torch.cuda.synchronize()
lib().card_linear_trace(lin.h, ctypes.c_void_p(tr.data_ptr()))
res = []
for rep in range(3):
    tr.zero_()
    flush.zero_()
    torch.cuda.synchronize()
    lin.run(dM)
    torch.cuda.synchronize()
    t = tr.view(grid, 16).cpu().numpy().astype(np.float64)
    res.append(t)
lib().card_linear_trace(lin.h, None)
t = res[-1]
t0 = t[:, 0].min()
names = ["entry", "pdl_wait", "first_kb", "last_mma", "acc_ready", "cbar1", "pushed", "cbar2", "done"]
print(lin.info, f"N={N} K={K} M={M} epi={epi}  weight MB {N*K*2/1e6:.1f}")
for k, nm in enumerate(names):
    col = t[:, k]
    v = col[col > 0] - t0
    if len(v):
        print(f"  {nm:10s} min {v.min()/1e3:7.2f}  med {np.median(v)/1e3:7.2f}  max {v.max()/1e3:7.2f} us")
end = (t[:, 8].max() - t0) / 1e3
print(f"  span {end:.2f} us -> {N*K*2/end/1e3:.0f} GB/s")
