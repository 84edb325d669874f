"""Epilogue experiments on the draft gate/up GEMM (M=116): trace with stores
disabled (ldo < 0) vs enabled."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_04462_b200._lib import lib
from paper_2508_04462_b200.llama import _Linear, tile_sw128
N, K, M = 16384, 2048, 116
W = tile_sw128((torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16))
X = torch.randn(128, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(128, N // 2, device="cuda", dtype=torch.bfloat16)
dM = torch.tensor([M], dtype=torch.int32, device="cuda")
for ldo in (N // 2, -1):
    lin = _Linear(W, X, M, 3, out, ldo if ldo > 0 else N // 2)
    if ldo < 0:
        # flip the stored ldo through a second create with negative ldo is not allowed; patch via ctypes is not
        # exposed, so create with ldo=-1 directly
        lin = _Linear(W, X, M, 3, out, -1)
    grid = lin.info["grid"]
    tr = torch.zeros(grid * 16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        lin.run(dM)
    torch.cuda.synchronize()
    lib().card_linear_trace(lin.h, ctypes.c_void_p(tr.data_ptr()))
    lin.run(dM)
    torch.cuda.synchronize()
    lib().card_linear_trace(lin.h, None)
    t = tr.view(grid, 16).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    print(f"ldo={ldo}: acc_ready med {np.median(t[:,4]-t0)/1e3:.2f}  done med {np.median(t[:,8]-t0)/1e3:.2f}  max {np.max(t[:,8]-t0)/1e3:.2f} us")
