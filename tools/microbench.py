"""Per-op CUDA-event timings on the BASELINE models (warm, L2 flushed between reps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200 import _lib
from paper_2508_04462_b200._device import ptr, stream_ptr
from paper_2508_04462_b200.llama import PRESETS, RowBlock

PEAK = 6552.0
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10, flush_l2=True):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush_l2:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def bench_model(name, preset, m_rows, ctx_len):
    cfg = PRESETS[preset]
    m = card.LlamaModel(cfg, seed=1, dtype="bf16")
    rt = m.runtime(ctx_len + 64, 0, sorted({m_rows, 128}))
    rows = RowBlock(m_rows, 16, rt.dev)
    toks = list(np.random.default_rng(0).integers(0, cfg.vocab_size, m_rows))
    rows.set_chain(toks, ctx_len - m_rows, out_last_only=False)
    dM = rows.M
    plan = rt.plans[m_rows]
    if rt.fused:
        rt._bind_rows(plan, rows)
    total_b = total_t = 0.0
    print(f"== {name} M={m_rows} ctx={ctx_len}")
    for key in ("qkv", "o", "gu", "d"):
        lin = plan["layers"][0][key]
        W = lin.keep[0]
        t = timeit(lambda: lin.run(dM))
        b = W.numel() * 2
        total_b += b * cfg.n_layers
        total_t += t * cfg.n_layers
        print(f"  {key:4s} N={lin.N:6d} K={lin.K:6d} {t*1e3:8.1f} us  {b/t/1e6:7.0f} GB/s "
              f"({b/t/1e6/PEAK*100:4.1f}%)  {lin.info}")
    lin = plan["lm_head"]
    W = lin.keep[0]
    t = timeit(lambda: lin.run(rows.n_out))
    b = W.numel() * 2
    total_b += b
    total_t += t
    print(f"  head N={lin.N:6d} K={lin.K:6d} {t*1e3:8.1f} us  {b/t/1e6:7.0f} GB/s ({b/t/1e6/PEAK*100:4.1f}%) {lin.info}")
    print(f"  all GEMMs: {total_t:.3f} ms  {total_b/total_t/1e6:.0f} GB/s")
    L = _lib.lib()
    c = cfg
    t_att = timeit(lambda: L.card_attention(ptr(rt.q), ptr(dM), rt.mpad, ptr(rows.plen), ptr(rows.slot), ptr(rows.n_extra),
                                             ptr(rows.extra), rows.extra_max, ptr(rt.k_cache[0]), ptr(rt.v_cache[0]),
                                             0, c.n_heads, c.n_kv_heads, c.head_dim, rt.prefix_slots, ptr(rt.work),
                                             ptr(rt.o), 0, stream_ptr()))
    t_norm = timeit(lambda: L.card_rmsnorm(ptr(rt.x), ptr(rt.layers[0]["attn_norm"]), c.hidden, c.rms_eps, ptr(dM),
                                            rt.mpad, None, ptr(rt.h), 0, stream_ptr()))
    t_rope = timeit(lambda: L.card_rope_kv(ptr(rt.qkv), ptr(dM), rt.mpad, ptr(rows.pos), ptr(rows.slot), ptr(rt.cos),
                                            ptr(rt.sin), c.n_heads, c.n_kv_heads, c.head_dim, ptr(rt.q),
                                            ptr(rt.k_cache[0]), ptr(rt.v_cache[0]), 0, stream_ptr()))
    tok = torch.zeros((m_rows, 3), dtype=torch.int32, device="cuda")
    lp = torch.zeros((m_rows, 3), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(m_rows, dtype=torch.int32, device="cuda")
    wk = torch.zeros(L.card_lmhead_work_floats(m_rows, 3), dtype=torch.float32, device="cuda")
    t_topk = timeit(lambda: L.card_topk_logits(ptr(rt.logits), ptr(dM), m_rows, c.vocab_size, 3, 1.0, ptr(tok),
                                                ptr(lp), ptr(cnt), ptr(wk), None, 0, 0, 0, 0, 0.0, 0.0, stream_ptr()))
    tail = torch.randint(0, c.vocab_size, (m_rows, 2), dtype=torch.int32, device="cuda")
    t_topk_b = timeit(lambda: L.card_topk_logits(ptr(rt.logits), ptr(dM), m_rows, c.vocab_size, 3, 1.0, ptr(tok),
                                                  ptr(lp), ptr(cnt), ptr(wk), ptr(tail), 2, 2, 11, 131, 0.0, 1e6,
                                                  stream_ptr()))
    am = torch.zeros(m_rows, dtype=torch.int32, device="cuda")
    t_am = timeit(lambda: L.card_argmax_logits(ptr(rt.logits), ptr(dM), m_rows, c.vocab_size, ptr(am), ptr(wk),
                                                None, 0, 0, 0, 0, 0.0, 0.0, stream_ptr()))
    print(f"  attention {t_att*1e3:.1f} us  rmsnorm {t_norm*1e3:.1f} us  rope {t_rope*1e3:.1f} us  "
          f"topk {t_topk*1e3:.1f} us (k-gram biased {t_topk_b*1e3:.1f} us)  argmax {t_am*1e3:.1f} us")
    t_fwd = timeit(lambda: rt.forward(rows, m_rows), reps=5)
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        rt.forward(rows, m_rows)
    torch.cuda.current_stream().wait_stream(st)
    t_g = timeit(lambda: g.replay(), reps=10)
    # GEMM-only graph: the same 4*L+1 linears in forward order, nothing else
    lins = [L[k] for L in plan["layers"] for k in ("qkv", "o", "gu", "d")]
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st), torch.cuda.graph(g2, stream=st):
        for lin in lins:
            lin.run(dM)
        plan["lm_head"].run(rows.n_out)
    torch.cuda.current_stream().wait_stream(st)
    t_g2 = timeit(lambda: g2.replay(), reps=10)
    sb = cfg.stream_params() * 2
    print(f"  GEMM-only graph {t_g2:.3f} ms -> {sb/t_g2/1e6:.0f} GB/s; non-GEMM share of forward {t_g - t_g2:.3f} ms")
    print(f"  full forward {t_fwd:.3f} ms   graph replay {t_g:.3f} ms  -> {sb/t_g/1e6:.0f} GB/s weight stream "
          f"({sb/t_g/1e6/PEAK*100:.1f}% of {PEAK:.0f})")
    del rt, m
    torch.cuda.empty_cache()


which = sys.argv[1:] or ["t1", "t8", "d116"]
for w in which:
    if w == "t1":
        bench_model("target AR", "llama-3.1-8b", 1, 1024)
    if w == "t8":
        bench_model("target verify", "llama-3.1-8b", 8, 1024)
    if w == "d116":
        bench_model("draft tree", "llama-3.2-1b", 116, 1024)
    if w == "d1":
        bench_model("draft flat", "llama-3.2-1b", 1, 1024)
