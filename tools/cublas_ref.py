"""cuBLAS reference timings (torch.matmul, bf16) of the draft/verify GEMM
shapes, warm L2-flushed, single launches and a 16-layer chain in a graph."""
import torch
shapes = {"d116": [(3072, 2048), (2048, 2048), (16384, 2048), (2048, 8192)], "t8": [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for key, M, L in (("d116", 116, 16), ("t8", 8, 32)):
    Ws = [[(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for (N, K) in shapes[key]] for _ in range(L)]
    X = {K: torch.randn(M, K, device="cuda").to(torch.bfloat16) for (_, K) in shapes[key]}
    for (N, K), W in zip(shapes[key], Ws[0]):
        for _ in range(3):
            y = X[K] @ W.t()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); y = X[K] @ W.t(); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{key} cuBLAS N={N} K={K} M={M}: {ts[len(ts)//2]*1e3:.1f} us  {N*K*2/ts[len(ts)//2]/1e6:.0f} GB/s")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for l in range(L):
            for (N, K), W in zip(shapes[key], Ws[l]):
                y = X[K] @ W.t()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); b.synchronize()
    tot = sum(N * K * 2 for (N, K) in shapes[key]) * L
    print(f"{key} cuBLAS chain of {L} layers x 4 GEMMs (graph): {a.elapsed_time(b):.3f} ms  {tot/a.elapsed_time(b)/1e6:.0f} GB/s")
    del Ws
