// card_pfwd.cu — persistent forward of a wide row block (draft tree steps).
//
// A draft tree step runs the 1B draft over M <= 128 rows (the frontier plus
// catch-up rows).  As 80 separate kernels the step is latency-bound: every
// GEMM boundary pays launch, pipeline fill, split-K exchange and epilogue,
// and the small projections (o, down: 16 weight tiles) keep only 64 SMs
// streaming.  Here one CTA per SM walks a static schedule of
// steps, step = (layer, phase), phase in {qkv, attention, o, gate/up, down}
// (attention steps run as their own kernel between launches):
//
//   warp 0   weight producer: streams the pre-tiled 16 KB weight blocks of
//            this CTA's units, step after step, into a ring.  It never waits
//            on activations, so the next step's weights are already in
//            shared memory when the current step's outputs are published.
//   warp 1   activation producer: waits until the previous step is complete
//            (gpu-scope counter), then TMA-loads the activation k-blocks.
//   warp 2   MMA issuer: tcgen05.mma kind::f16, A = weights (128 rows),
//            B = activations (Mpad tokens), accumulator in TMEM (2 buffers).
//   warps 4.. epilogue workers, kGroups groups of four (TMEM lane = weight row).
//
// Units: a step's GEMM is cut into n_tiles x splits units (split-K so that
// ~all SMs stream).  A split unit drains its fp32 partial to an L2-resident
// workspace, bumps its tile's counter, and once all splits of the tile are
// in, reduces a 1/splits token slice of the tile in fixed split order
// (deterministic) and applies the fused epilogue:
//   qkv   RMSNorm scale (norm weight folded into W), bias, RoPE, q * 1/sqrt(hd)
//         -> q (fp32), k / v -> KV-cache slots (bf16)
//   o, d  residual add (fp32) + bf16 copy + per-16-column sums of squares
//   gu    (no split) RMSNorm scale + SwiGLU straight from TMEM -> g (bf16)
// then bumps the step's completion counter.  Every wait is on work of an
// earlier step or on a sibling split of the same step; all CTAs are
// co-resident (cooperative launch, one CTA per SM), so the schedule cannot
// deadlock.
//
// Code size matters: each step's epilogue runs once per layer, so its code is
// cold in the instruction cache every time; the epilogue loops are rolled and
// the kernel is kept small (measured: fully unrolled epilogues ran 2-3x slower
// in the kernel than warm in isolation).
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "card_common.cuh"
#include "card_llm.h"
#include "card_ptx.cuh"

namespace card {
namespace pf {

using namespace ptx;

constexpr int kGroups = 4;                    // epilogue worker groups (4 warps each)
constexpr int kWorkerWarp0 = 4;
constexpr int kWorkers = 128 * kGroups;
constexpr int kThreads = kWorkerWarp0 * 32 + kWorkers;
constexpr int kTileN = 128, kBK = 64;
constexpr int kWBytes = kTileN * kBK * 2;   // one pre-tiled weight block
constexpr int kPhases = 5;
enum { PH_QKV = 0, PH_ATTN = 1, PH_O = 2, PH_GU = 3, PH_D = 4 };
constexpr int kMaxLayers = 64;
constexpr int kMaxSteps = kMaxLayers * kPhases;
constexpr int kTileCtrs = 64;   // split-tile counters per step (n_tiles of a split GEMM <= 64)
constexpr int kMaxMpad = 128;   // TMEM: two 128-column accumulators
constexpr int kMaxSplits = 10;

struct Layer {
    const uint8_t* w[kPhases];   // pre-tiled weights by phase (ATTN: null)
    const float* bqkv;
    __nv_bfloat16* kc;
    __nv_bfloat16* vc;
};

struct Gemm {
    int N, K, n_tiles, kb_total, splits, units;
};

struct Args {
    const Layer* layers;
    Gemm gm[kPhases];
    int step_begin, step_end;
    const int32_t* dM;
    int Mpad, WS, XS;
    float* x;
    __nv_bfloat16* xb;
    float* ssq;
    int ssq_ld, ssq_parts;
    float eps, inv_h;
    float* q;
    __nv_bfloat16* g;
    int F, nh, nkv, hd;
    float qscale;
    // pre-swizzled bf16 Q tiles for card_attention_tree (null: fp32 q):
    // [nkv][qsw_tiles][hd/64][128 query-heads x 64] SWIZZLE_128B blocks,
    // query-head qh = row * (nh/nkv) + head % (nh/nkv) of kv head head / (nh/nkv)
    uint8_t* qsw;
    int qsw_tiles;
    const int32_t* pos;
    const int32_t* slot;
    const float* cos_t;
    const float* sin_t;
    float* ws;   // split-K partials [splits][Mpad][N]
    int* done;   // [kMaxSteps] completed units per step
    int* tctr;   // [kMaxSteps][kTileCtrs] arrived splits per tile
    int* exit_ctr;
    unsigned long long* trace;   // tuning: [grid][2 + 4 * steps] %globaltimer stamps (null: off)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// stamp k of step st: 0 activations released, 1 first k-block in, 2 accumulator done, 3 outputs published,
// 4 partial drained, 5 all splits of the tile in, 6 slice reduced
#define PF_STAMP(st, k)                                                                                        \
    do {                                                                                                       \
        if (a.trace)                                                                                           \
            a.trace[(size_t)blockIdx.x * (2 + 8 * (a.step_end - a.step_begin)) + 2 + 8 * ((st) - a.step_begin) + \
                    (k)] = gtime();                                                                            \
    } while (0)

__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// RMSNorm scale rsqrt(mean x^2 + eps) of tokens [m_lo, m_hi) from the
// per-16-column partials; 8 lanes per token, fixed summation order.
__device__ __forceinline__ void compute_invs(const Args& a, int m_lo, int m_hi, float* invs, int t) {
    const int sub = t & 7;
    const int per = (a.ssq_parts + 7) / 8;
    const int p0 = sub * per, p1 = min(a.ssq_parts, p0 + per);
#pragma unroll 1
    for (int mb = m_lo; mb < m_hi; mb += kWorkers / 8) {
        const int m = mb + t / 8;
        float acc = 0.f;
        if (m < m_hi) {
            const float* src = a.ssq + m;
#pragma unroll 1
            for (int p = p0; p < p1; p += 16) {
                float v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = (p + u < p1) ? src[(int64_t)(p + u) * a.ssq_ld] : 0.f;
#pragma unroll
                for (int u = 0; u < 16; ++u) acc += v[u];
            }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (m < m_hi && sub == 0) invs[m] = rsqrtf(acc * a.inv_h + a.eps);
    }
}

__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}
// sum over the S split partials of one float4 item, every load issued first
// (fixed split order; absent splits add exact zeros)
__device__ __forceinline__ float4 reduce1(const float* pa, int64_t stride, int S) {
    float4 x[kMaxSplits];
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s) x[s] = s < S ? ldcg4(pa + s * stride) : z;
    float4 r = x[0];
#pragma unroll
    for (int s = 1; s < kMaxSplits; ++s) add4(r, x[s]);
    return r;
}
__device__ __forceinline__ uint2 pack4_bf16(float a, float b, float c, float d) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
    return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}
// Operands of one epilogue item that do not depend on the step's partials:
// the residual row (o, down) or the row's KV slot and RoPE cos / sin (qkv).
struct Pre {
    float4 x, cs, sn;
    int slot;
};
__device__ __forceinline__ void pre_item(const Args& a, int p, int N, int tile, int f4, int m, Pre& r) {
    if (p != PH_QKV) {
        r.x = *reinterpret_cast<const float4*>(a.x + (int64_t)m * N + tile * kTileN + 4 * f4);
        return;
    }
    const int half = a.hd >> 1;
    const int fb = 4 * f4;
    const int i0 = fb - (fb / a.hd) * a.hd;
    const int ii = i0 < half ? i0 : i0 - half;
    const int pos = a.pos[m];
    r.slot = a.slot[m];
    r.cs = *reinterpret_cast<const float4*>(a.cos_t + (int64_t)pos * half + ii);
    r.sn = *reinterpret_cast<const float4*>(a.sin_t + (int64_t)pos * half + ii);
}
// o / down epilogue of one float4 item: x += sum, bf16 copy, per-16-column
// sum of squares (a quad of lanes = 16 columns)
__device__ __forceinline__ void resid_item(const Args& a, int N, int ng, int m, const float4& s, float4 xn) {
    add4(xn, s);
    *reinterpret_cast<float4*>(a.x + (int64_t)m * N + ng) = xn;
    *reinterpret_cast<uint2*>(a.xb + (int64_t)m * N + ng) = pack4_bf16(xn.x, xn.y, xn.z, xn.w);
    float sq = xn.x * xn.x + xn.y * xn.y + xn.z * xn.z + xn.w * xn.w;
    sq += __shfl_xor_sync(0xffffffffu, sq, 1);
    sq += __shfl_xor_sync(0xffffffffu, sq, 2);
    if ((threadIdx.x & 3) == 0) a.ssq[(int64_t)(ng >> 4) * a.ssq_ld + m] = sq;
}
// qkv epilogue of one float4 item (features 4 f4 .. of the tile, token m):
// norm scale + bias, RoPE with the partner half of the head via a shuffle
// (the warp holds the whole 128-feature row), q * 1/sqrt(hd) -> q, k / v -> cache
__device__ __forceinline__ void qkv_item(const Args& a, const Layer& L, const float* invs, int tile, int f4, int m,
                                         float4 s, const Pre& pr) {
    const int half = a.hd >> 1;
    const int fb = 4 * f4;   // feature in the tile
    const int hl = fb / a.hd, i0 = fb - hl * a.hd;
    const int head = (tile * kTileN) / a.hd + hl;
    const int ng = tile * kTileN + fb;
    float4 v = s;
    const float iv = invs[m];
    v.x *= iv;
    v.y *= iv;
    v.z *= iv;
    v.w *= iv;
    if (L.bqkv) add4(v, *reinterpret_cast<const float4*>(L.bqkv + ng));
    const int slot = pr.slot;
    const int pl = half >> 2;   // partner lane distance (float4 items)
    float4 o;
    o.x = __shfl_xor_sync(0xffffffffu, v.x, pl);
    o.y = __shfl_xor_sync(0xffffffffu, v.y, pl);
    o.z = __shfl_xor_sync(0xffffffffu, v.z, pl);
    o.w = __shfl_xor_sync(0xffffffffu, v.w, pl);
    if (head >= a.nh + a.nkv) {   // v: no rotation
        *reinterpret_cast<uint2*>(L.vc + ((int64_t)slot * a.nkv + (head - a.nh - a.nkv)) * a.hd + i0) =
            pack4_bf16(v.x, v.y, v.z, v.w);
        return;
    }
    const bool first = i0 < half;
    const float4 cs = pr.cs;
    const float4 sn = pr.sn;
    // first half: x1 = v, x2 = o -> x1 cs - x2 sn; second: x2 = v, x1 = o -> x2 cs + x1 sn
    const float sg = first ? -1.f : 1.f;
    float4 r;
    r.x = v.x * cs.x + sg * (o.x * sn.x);
    r.y = v.y * cs.y + sg * (o.y * sn.y);
    r.z = v.z * cs.z + sg * (o.z * sn.z);
    r.w = v.w * cs.w + sg * (o.w * sn.w);
    if (head < a.nh) {
        r.x *= a.qscale;
        r.y *= a.qscale;
        r.z *= a.qscale;
        r.w *= a.qscale;
        if (a.qsw) {   // the attention's Q operand, already in its shared-memory layout
            const int G = a.nh / a.nkv;
            const int gq = head / G;
            const int qh = m * G + (head - gq * G);
            const int tq = qh & 127, c = (i0 & 63) >> 3;
            uint8_t* dst = a.qsw + ((size_t)((gq * a.qsw_tiles + (qh >> 7)) * (a.hd >> 6) + (i0 >> 6)) << 14) +
                           ((tq >> 3) * 1024 + (tq & 7) * 128 + ((c ^ (tq & 7)) << 4)) + (i0 & 7) * 2;
            *reinterpret_cast<uint2*>(dst) = pack4_bf16(r.x, r.y, r.z, r.w);
        } else {
            *reinterpret_cast<float4*>(a.q + ((int64_t)m * a.nh + head) * a.hd + i0) = r;
        }
    } else {
        *reinterpret_cast<uint2*>(L.kc + ((int64_t)slot * a.nkv + (head - a.nh)) * a.hd + i0) =
            pack4_bf16(r.x, r.y, r.z, r.w);
    }
}

// gate/up epilogue of a whole tile straight from TMEM: rows 32q..32q+15 are the
// gates of features 16q..16q+15, rows 32q+16..32q+31 the ups (interleave_gate_up);
// lanes l and l^16 swap chunk halves with one shuffle per token pair
__device__ __noinline__ void gu_epilogue(const Args& a, const float* invs, uint32_t trow, int tile, int M) {
    const int lane = threadIdx.x & 31;
    const int wi = (threadIdx.x >> 5) - kWorkerWarp0;
    const int wq = wi & 3, grp = wi >> 2;
    const bool up = lane >= 16;
    const int f = tile * 64 + wq * 16 + (lane & 15);
    const int jb = up ? 8 : 0;
#pragma unroll 1
    for (int m0 = 16 * grp; m0 < M; m0 += 16 * kGroups) {
        float v[16];
        tmem_ld16(trow + (uint32_t)m0, v);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const float lo = v[jj] * invs[m0 + jj];
            const float hi = v[8 + jj] * invs[min(m0 + 8 + jj, kMaxMpad - 1)];
            const float mine = up ? hi : lo;
            const float other = __shfl_xor_sync(0xffffffffu, up ? lo : hi, 16);
            const float gg = up ? other : mine;
            const float uu = up ? mine : other;
            if (m0 + jb + jj < M) a.g[(int64_t)(m0 + jb + jj) * a.F + f] = __float2bfloat16(silu(gg) * uu);
        }
    }
}

// split unit: fp32 partial of the tile -> workspace [sp][m][n] (coalesced over n)
__device__ __noinline__ void drain_partial(float* wsp, int N, uint32_t trow, int M) {
    const int wi = (threadIdx.x >> 5) - kWorkerWarp0;
    const int grp = wi >> 2;
#pragma unroll 1
    for (int m0 = 16 * grp; m0 < M; m0 += 16 * kGroups) {
        float v[16];
        tmem_ld16(trow + (uint32_t)m0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (m0 + j < M) __stcg(wsp + (int64_t)(m0 + j) * N, v[j]);
    }
}

// reduce token slice [ma, mb) of a split tile in split order + fused epilogue,
// once all splits of the tile are in (tctr); a warp = one token row of the
// tile (float4 per lane), warp-uniform loop.
__device__ __noinline__ void reduce_slice(const Args& a, const Layer& L, const float* invs, int p, int N, int splits,
                                          int tile, int ma, int mb, int* tctr, int st, bool stamp) {
    const int t = threadIdx.x - kWorkerWarp0 * 32;
    const int f4 = threadIdx.x & 31;
    const int ng = tile * kTileN + 4 * f4;
    const int64_t sstride = (int64_t)a.Mpad * N;
    const int n_items = (mb - ma) * 32;
    if (t == 0) {
        if (stamp) PF_STAMP(st, 4);
        atom_add_acq_rel(tctr, 1);   // release: the CTA's partial stores (bar.sync before the call)
        wait_ge(tctr, splits);
        if (stamp) PF_STAMP(st, 5);
    }
    named_bar(1, kWorkers);
    // (loading the residual / RoPE operands before the wait measured slower:
    // the release waits for them, and at 96 registers they spill)
#pragma unroll 1
    for (int i0 = t; i0 < n_items; i0 += kWorkers) {
        const int m = ma + (i0 >> 5);
        const float4 sm = reduce1(a.ws + (int64_t)m * N + ng, sstride, splits);
        Pre pr;
        pre_item(a, p, N, tile, f4, m, pr);
        if (p == PH_QKV) qkv_item(a, L, invs, tile, f4, m, sm, pr);
        else resid_item(a, N, ng, m, sm, pr.x);
    }
}

__global__ void __launch_bounds__(kThreads, 1)
    pfwd_kernel(const __grid_constant__ CUtensorMap tmXb, const __grid_constant__ CUtensorMap tmO,
                const __grid_constant__ CUtensorMap tmG, const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int xbytes = a.Mpad * kBK * 2;
    uint8_t* sW = smem;
    uint8_t* sX = sW + (size_t)a.WS * kWBytes;
    float* invs = (float*)(sX + (size_t)a.XS * xbytes);   // [kMaxMpad]
    // fixed-count barriers first (constant offsets from one base), then the rings
    uint64_t* bars = (uint64_t*)(invs + kMaxMpad);
    uint64_t* tfull = bars;         // [2]
    uint64_t* tempty = bars + 2;    // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 4);
    uint64_t* wfull = bars + 8;
    uint64_t* wempty = wfull + a.WS;
    uint64_t* xfull = wempty + a.WS;
    uint64_t* xempty = xfull + a.XS;

    // the next kernel (the layer's attention) may launch now: it cannot take
    // an SM before this grid's CTAs leave, and it waits for our results
    // (griddepcontrol.wait) before reading them, so its launch latency hides
    pdl_trigger();
    const int M = *a.dM;   // written before the previous forward's kernels (row builder)
    if (M <= 0) return;   // uniform: nothing to do, no counter touched
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0 && a.trace) a.trace[(size_t)blockIdx.x * (2 + 8 * (a.step_end - a.step_begin))] = gtime();
    if (threadIdx.x == 0) {
        for (int i = 0; i < a.WS; ++i) {
            bar_init(&wfull[i], 1);
            bar_init(&wempty[i], 1);
        }
        for (int i = 0; i < a.XS; ++i) {
            bar_init(&xfull[i], 1);
            bar_init(&xempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            bar_init(&tfull[i], 1);
            bar_init(&tempty[i], kWorkers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem_base = *tmem_slot;
    const int n_mma = ((M + 15) / 16) * 16;
    const int sb = a.step_begin, se = a.step_end;
    const int cta = blockIdx.x, G = gridDim.x;

    if (warp == 0) {
        // ------------------------------------------------ weight producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            for (int st = sb; st < se; ++st) {
                const int p = st % kPhases;
                if (p == PH_ATTN) continue;
                const Gemm& gm = a.gm[p];
                const uint8_t* W = a.layers[st / kPhases].w[p];
                for (int u = cta; u < gm.units; u += G) {
                    const int tile = u / gm.splits, sp = u % gm.splits;
                    const int kb0 = gm.kb_total * sp / gm.splits, kb1 = gm.kb_total * (sp + 1) / gm.splits;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        bar_wait(&wempty[s], ph ^ 1);
                        bar_expect_tx(&wfull[s], kWBytes);
                        bulk_load_hint(sW + (size_t)s * kWBytes, W + ((size_t)tile * gm.kb_total + kb) * kWBytes,
                                       kWBytes, &wfull[s], pol);
                        if (++s == a.WS) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ activation producer
        if (lane == 0) {
            pdl_wait();   // the previous kernel's outputs (attention o, embed x) are visible
            prefetch_map(&tmXb);
            prefetch_map(&tmO);
            prefetch_map(&tmG);
            int s = 0;
            uint32_t ph = 0;
            for (int st = sb; st < se; ++st) {
                const int p = st % kPhases;
                if (p == PH_ATTN) continue;
                const Gemm& gm = a.gm[p];
                if (cta >= gm.units) continue;
                if (st > sb) {
                    wait_ge(&a.done[st - 1], a.gm[(st - 1) % kPhases].units);
                    fence_proxy_async_global();
                }
                PF_STAMP(st, 0);
                const CUtensorMap* map = (p == PH_O) ? &tmO : (p == PH_D) ? &tmG : &tmXb;
                for (int u = cta; u < gm.units; u += G) {
                    const int sp = u % gm.splits;
                    const int kb0 = gm.kb_total * sp / gm.splits, kb1 = gm.kb_total * (sp + 1) / gm.splits;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        bar_wait(&xempty[s], ph ^ 1);
                        bar_expect_tx(&xfull[s], (uint32_t)xbytes);
                        tma_load_2d(sX + (size_t)s * xbytes, map, &xfull[s], kb * kBK, 0);
                        if (++s == a.XS) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 2) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(kTileN, n_mma);
            int ws = 0, xs = 0, acc = 0;
            uint32_t wph = 0, xph = 0, aph = 0;
            for (int st = sb; st < se; ++st) {
                const int p = st % kPhases;
                if (p == PH_ATTN) continue;
                const Gemm& gm = a.gm[p];
                for (int u = cta; u < gm.units; u += G) {
                    const int sp = u % gm.splits;
                    const int kb0 = gm.kb_total * sp / gm.splits, kb1 = gm.kb_total * (sp + 1) / gm.splits;
                    bar_wait(&tempty[acc], aph ^ 1);
                    tc_after();
                    const uint32_t d = tmem_base + (uint32_t)(acc * kMaxMpad);
                    for (int kb = kb0; kb < kb1; ++kb) {
                        bar_wait(&wfull[ws], wph);
                        bar_wait(&xfull[xs], xph);
                        if (kb == kb0 && u == cta) PF_STAMP(st, 1);
                        tc_after();
                        const uint32_t a0 = su32(sW + (size_t)ws * kWBytes);
                        const uint32_t b0 = su32(sX + (size_t)xs * xbytes);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k)
                            tc_mma(d, desc_sw128(a0 + k * 32), desc_sw128(b0 + k * 32), idesc,
                                   (kb > kb0 || k > 0) ? 1u : 0u);
                        tc_commit(&wempty[ws]);
                        tc_commit(&xempty[xs]);
                        if (++ws == a.WS) {
                            ws = 0;
                            wph ^= 1;
                        }
                        if (++xs == a.XS) {
                            xs = 0;
                            xph ^= 1;
                        }
                    }
                    tc_commit(&tfull[acc]);
                    acc ^= 1;
                    if (acc == 0) aph ^= 1;
                }
            }
        }
    } else if (warp >= kWorkerWarp0) {
        // ------------------------------------------------ epilogue workers
        pdl_wait();
        const int t = threadIdx.x - kWorkerWarp0 * 32;
        const int wq = (warp - kWorkerWarp0) & 3;
        const int n_local = wq * 32 + lane;
        int acc = 0;
        uint32_t aph = 0;
        for (int st = sb; st < se; ++st) {
            const int p = st % kPhases;
            if (p == PH_ATTN) continue;
            const Gemm& gm = a.gm[p];
            if (cta >= gm.units) continue;
            const Layer& L = a.layers[st / kPhases];
            if (st > sb) {   // previous step's outputs (x, ssq) visible to every worker
                if (t == 0) wait_ge(&a.done[st - 1], a.gm[(st - 1) % kPhases].units);
                named_bar(1, kWorkers);
            }
            if (p == PH_GU) {
                compute_invs(a, 0, M, invs, t);
                named_bar(1, kWorkers);
            }
            for (int u = cta; u < gm.units; u += G) {
                const int tile = u / gm.splits, sp = u % gm.splits;
                const uint32_t trow = tmem_base + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * kMaxMpad);
                if (gm.splits == 1) {
                    bar_wait_polite(&tfull[acc], aph);
                    if (t == 0 && u == cta) PF_STAMP(st, 2);
                    tc_after();
                    gu_epilogue(a, invs, trow, tile, M);
                    tc_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(&tempty[acc]);
                } else {
                    const int ma = M * sp / gm.splits, mb = M * (sp + 1) / gm.splits;
                    // the qkv norm scale of my slice, while the MMA runs
                    if (p == PH_QKV) compute_invs(a, ma, mb, invs, t);
                    bar_wait_polite(&tfull[acc], aph);
                    if (t == 0 && u == cta) PF_STAMP(st, 2);
                    tc_after();
                    drain_partial(a.ws + (size_t)sp * a.Mpad * gm.N + tile * kTileN + n_local, gm.N, trow, M);
                    tc_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(&tempty[acc]);
                    named_bar(1, kWorkers);
                    reduce_slice(a, L, invs, p, gm.N, gm.splits, tile, ma, mb, &a.tctr[st * kTileCtrs + tile], st,
                                 u == cta);
                    if (t == 0 && u == cta) PF_STAMP(st, 6);
                }
                acc ^= 1;
                if (acc == 0) aph ^= 1;
                // one release per CTA (per-warp arrivals on the step counter
                // measured slower: 16x the same-address atomics)
                named_bar(1, kWorkers);
                if (t == 0) {
                    fence_proxy_async_global();   // xb / g are read by TMA in later steps
                    atom_add_acq_rel(&a.done[st], 1);   // release: the CTA's outputs (bar.sync above)
                    PF_STAMP(st, 3);
                }
            }
        }
    }

    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
    if (threadIdx.x == 0 && a.trace) a.trace[(size_t)blockIdx.x * (2 + 8 * (se - sb)) + 1] = gtime();
    // the last CTA out clears the counters for the next launch
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atom_add_acq_rel(a.exit_ctr, 1) == G - 1;
    }
    __syncthreads();
    if (last) {
        for (int i = threadIdx.x; i < (se - sb) * (kTileCtrs + 1); i += kThreads) {
            const int st = sb + i / (kTileCtrs + 1), j = i % (kTileCtrs + 1);
            if (j == kTileCtrs) a.done[st] = 0;
            else a.tctr[st * kTileCtrs + j] = 0;
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) *a.exit_ctr = 0;
    }
}

}  // namespace pf

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled_pf)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int pf_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    static PFN_encodeTiled_pf enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return CARD_E_CUDA;
        enc = (PFN_encodeTiled_pf)p;
    }
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)pf::kBK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? CARD_OK : CARD_E_CUDA;
}

}  // namespace card

using namespace card;

struct card_pfwd {
    pf::Args args;
    pf::Layer* d_layers;
    CUtensorMap tmXb, tmO, tmG;
    float* ws;
    int* ctr;   // done [kMaxSteps] | tctr [kMaxSteps * kTileCtrs] | exit
    int grid, smem, n_layers;
};

// Split-K ways for a GEMM of n_tiles weight tiles on G SMs: whole tiles when
// they fill half the SMs or more, else the most splits with n_tiles * splits
// <= G (each split >= 2 k-blocks).
static int pf_splits(int n_tiles, int kb_total, int G) {
    if (2 * n_tiles >= G) return 1;
    int s = G / n_tiles;
    if (s > kb_total / 2) s = kb_total / 2;
    if (s > pf::kMaxSplits) s = pf::kMaxSplits;
    return s < 1 ? 1 : s;
}

extern "C" {

int card_pfwd_create(int n_layers, int H, int F, int nh, int nkv, int hd, int m_max, const void* const* layer_w,
                     const float* const* bqkv, void* const* kv, float* x, void* xb, float* ssq, int ssq_ld, float* q,
                     void* o, void* g, int act_rows, const int32_t* pos, const int32_t* slot, const float* cos_t,
                     const float* sin_t, float eps, card_pfwd** out) {
    if (!out || !layer_w || !kv || !x || !xb || !ssq || !q || !o || !g || !pos || !slot || !cos_t || !sin_t)
        return CARD_E_INPUT;
    *out = nullptr;
    if (n_layers <= 0 || n_layers > pf::kMaxLayers || m_max < 1 || m_max > pf::kMaxMpad || act_rows < m_max)
        return CARD_E_CONFIG;
    if ((hd != 64 && hd != 128) || H % pf::kTileN || F % 64 || ((nh + 2 * nkv) * hd) % pf::kTileN ||
        (nh * hd) % pf::kBK || H % pf::kBK)
        return CARD_E_CONFIG;
    const int Mpad = ((m_max + 15) / 16) * 16;
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) return CARD_E_CUDA;

    card_pfwd* h = (card_pfwd*)calloc(1, sizeof(card_pfwd));
    pf::Args& a = h->args;
    const int qkv_n = (nh + 2 * nkv) * hd;
    const int Ns[pf::kPhases] = {qkv_n, 0, H, 2 * F, H};
    const int Ks[pf::kPhases] = {H, 0, nh * hd, H, F};
    size_t ws_floats = 0;
    for (int p = 0; p < pf::kPhases; ++p) {
        pf::Gemm& gm = a.gm[p];
        if (p == pf::PH_ATTN) continue;
        gm.N = Ns[p];
        gm.K = Ks[p];
        gm.n_tiles = gm.N / pf::kTileN;
        gm.kb_total = gm.K / pf::kBK;
        gm.splits = (p == pf::PH_GU) ? 1 : pf_splits(gm.n_tiles, gm.kb_total, sms);
        if (gm.splits > 1 && gm.n_tiles > pf::kTileCtrs) gm.splits = 1;
        gm.units = gm.n_tiles * gm.splits;
        if (p != pf::PH_GU) {   // room for any split count (card_pfwd_tune)
            const size_t need = (size_t)pf::kMaxSplits * Mpad * gm.N;
            if (need > ws_floats) ws_floats = need;
        }
    }
    // the three activation operands the GEMMs read by TMA ([rows, K] bf16)
    int rc = pf_map(&h->tmXb, xb, (uint64_t)act_rows, (uint64_t)H, (uint32_t)Mpad);
    if (!rc) rc = pf_map(&h->tmO, o, (uint64_t)act_rows, (uint64_t)(nh * hd), (uint32_t)Mpad);
    if (!rc) rc = pf_map(&h->tmG, g, (uint64_t)act_rows, (uint64_t)F, (uint32_t)Mpad);
    if (rc) {
        free(h);
        return rc;
    }
    pf::Layer* hl = (pf::Layer*)calloc(n_layers, sizeof(pf::Layer));
    for (int l = 0; l < n_layers; ++l) {
        hl[l].w[pf::PH_QKV] = (const uint8_t*)layer_w[4 * l + 0];
        hl[l].w[pf::PH_O] = (const uint8_t*)layer_w[4 * l + 1];
        hl[l].w[pf::PH_GU] = (const uint8_t*)layer_w[4 * l + 2];
        hl[l].w[pf::PH_D] = (const uint8_t*)layer_w[4 * l + 3];
        hl[l].bqkv = bqkv ? bqkv[l] : nullptr;
        hl[l].kc = (__nv_bfloat16*)kv[2 * l];
        hl[l].vc = (__nv_bfloat16*)kv[2 * l + 1];
    }
    cudaError_t e = cudaMalloc(&h->d_layers, n_layers * sizeof(pf::Layer));
    if (e == cudaSuccess) e = cudaMemcpy(h->d_layers, hl, n_layers * sizeof(pf::Layer), cudaMemcpyHostToDevice);
    free(hl);
    const size_t n_ctr = pf::kMaxSteps + (size_t)pf::kMaxSteps * pf::kTileCtrs + 1;
    if (e == cudaSuccess) e = cudaMalloc(&h->ctr, n_ctr * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(h->ctr, 0, n_ctr * sizeof(int));
    // (the workspace is allocated below, once the attention partials are sized)
    // smem: weight ring + activation ring + invs + barriers
    const int xbytes = Mpad * pf::kBK * 2;
    const int fixed = 1024 + pf::kMaxMpad * 4 + 64 * 8 + 64;
    const int budget = 226 * 1024;   // + the kernel's static shared memory
    // (activation stages: fewer measured slower; weight stages beyond 8 no
    // faster — the gate/up stream is not ring-bound, tools/ab_so.sh)
    a.XS = 6;
    a.WS = (budget - fixed - a.XS * xbytes) / pf::kWBytes;
    if (a.WS > 8) a.WS = 8;
    h->smem = fixed + a.WS * pf::kWBytes + a.XS * xbytes;
    if (e == cudaSuccess && ws_floats) e = cudaMalloc(&h->ws, ws_floats * sizeof(float));
    // one attribute for every instance (the largest any plan can ask for):
    // a per-instance value would be overwritten by the last plan created
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, pf::pfwd_kernel);
    const int dyn_max = optin - (int)fa.sharedSizeBytes;
    if (e == cudaSuccess && h->smem > dyn_max) e = cudaErrorInvalidValue;
    if (e == cudaSuccess) e = cudaFuncSetAttribute(pf::pfwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        if (h->d_layers) cudaFree(h->d_layers);
        if (h->ctr) cudaFree(h->ctr);
        if (h->ws) cudaFree(h->ws);
        free(h);
        return CARD_E_CUDA;
    }
    h->grid = sms;
    h->n_layers = n_layers;
    a.layers = h->d_layers;
    a.Mpad = Mpad;
    a.x = x;
    a.xb = (__nv_bfloat16*)xb;
    a.ssq = ssq;
    a.ssq_ld = ssq_ld;
    a.ssq_parts = H / 16;
    a.eps = eps;
    a.inv_h = 1.0f / (float)H;
    a.q = q;
    a.g = (__nv_bfloat16*)g;
    a.F = F;
    a.nh = nh;
    a.nkv = nkv;
    a.hd = hd;
    a.qscale = 1.0f / sqrtf((float)hd);
    a.pos = pos;
    a.slot = slot;
    a.cos_t = cos_t;
    a.sin_t = sin_t;
    a.ws = h->ws;
    a.done = h->ctr;
    a.tctr = h->ctr + pf::kMaxSteps;
    a.exit_ctr = h->ctr + pf::kMaxSteps + pf::kMaxSteps * pf::kTileCtrs;
    *out = h;
    return CARD_OK;
}

// Steps [step_begin, step_end), step = layer * 5 + phase (0 qkv, 1 attention,
// 2 o, 3 gate/up, 4 down).  Attention steps run outside (card_attention_paged)
// between runs, so a range must not contain one.
int card_pfwd_run(card_pfwd* h, const int32_t* dM, int step_begin, int step_end, void* stream) {
    if (!h || !dM || step_begin < 0 || step_end <= step_begin || step_end > h->n_layers * pf::kPhases)
        return CARD_E_INPUT;
    for (int st = step_begin; st < step_end; ++st)
        if (st % pf::kPhases == pf::PH_ATTN) return CARD_E_CONFIG;
    pf::Args a = h->args;
    a.dM = dM;
    a.step_begin = step_begin;
    a.step_end = step_end;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->grid);
    cfg.blockDim = dim3(pf::kThreads);
    cfg.dynamicSmemBytes = h->smem;
    cfg.stream = (cudaStream_t)stream;
    // cooperative: every CTA co-resident (they wait on each other's steps);
    // programmatic serialization: the weight stream and the prologue start
    // under the previous kernel's tail (the activation producer and the
    // epilogue workers wait for its results)
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, pf::pfwd_kernel, h->tmXb, h->tmO, h->tmG, a);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        int nb = -1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pf::pfwd_kernel, pf::kThreads, h->smem);
        fprintf(stderr, "card_pfwd_run: %s (grid %d, smem %d, blocks/SM %d)\n", cudaGetErrorString(e), h->grid,
                h->smem, nb);
        return CARD_E_CUDA;
    }
    return CARD_OK;
}

// qkv epilogue output for card_attention_tree: pre-swizzled bf16 Q tiles
// (qsw: nkv * tiles * hd/64 * 16 KB; tiles >= ceil(Mpad * nh/nkv / 128));
// NULL restores the fp32 q output
int card_pfwd_set_qsw(card_pfwd* h, void* qsw, int tiles) {
    if (!h) return CARD_E_INPUT;
    const pf::Args& a = h->args;
    if (qsw && (int64_t)tiles * 128 < (int64_t)a.Mpad * (a.nh / a.nkv)) return CARD_E_CONFIG;
    h->args.qsw = (uint8_t*)qsw;
    h->args.qsw_tiles = tiles;
    return CARD_OK;
}

// row-dependent epilogue inputs (the row block the forward runs over)
int card_pfwd_bind(card_pfwd* h, const int32_t* pos, const int32_t* slot) {
    if (!h || !pos || !slot) return CARD_E_INPUT;
    h->args.pos = pos;
    h->args.slot = slot;
    return CARD_OK;
}

// grid of the next launches: G CTAs (one per SM of the partition the forward
// runs on, card_green); split-K ways re-derived for G.  G = 0: the device.
int card_pfwd_set_grid(card_pfwd* h, int G) {
    if (!h || G < 0) return CARD_E_INPUT;
    if (G == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&G, cudaDevAttrMultiProcessorCount, dev);
    }
    pf::Args& a = h->args;
    for (int p = 0; p < pf::kPhases; ++p) {
        if (p == pf::PH_ATTN) continue;
        pf::Gemm& gm = a.gm[p];
        gm.splits = (p == pf::PH_GU) ? 1 : pf_splits(gm.n_tiles, gm.kb_total, G);
        if (gm.splits > 1 && gm.n_tiles > pf::kTileCtrs) gm.splits = 1;
        gm.units = gm.n_tiles * gm.splits;
    }
    h->grid = G;
    return CARD_OK;
}

// tuning: split-K ways of one GEMM phase (0 qkv, 2 o, 3 gate/up, 4 down)
int card_pfwd_tune(card_pfwd* h, int phase, int splits) {
    if (!h || phase < 0 || phase >= pf::kPhases || phase == pf::PH_ATTN || splits < 1 || splits > pf::kMaxSplits)
        return CARD_E_INPUT;
    pf::Gemm& gm = h->args.gm[phase];
    if (splits > 1 && (gm.n_tiles > pf::kTileCtrs || splits > gm.kb_total || phase == pf::PH_GU)) return CARD_E_CONFIG;
    gm.splits = splits;
    gm.units = gm.n_tiles * splits;
    return CARD_OK;
}

int card_pfwd_trace(card_pfwd* h, unsigned long long* trace) {
    if (!h) return CARD_E_INPUT;
    h->args.trace = trace;
    return CARD_OK;
}

int card_pfwd_info(card_pfwd* h, int32_t* info16) {
    if (!h || !info16) return CARD_E_INPUT;
    const pf::Args& a = h->args;
    info16[0] = h->grid;
    info16[1] = h->smem;
    info16[2] = a.WS;
    info16[3] = a.XS;
    info16[4] = a.Mpad;
    for (int p = 0; p < pf::kPhases; ++p) {
        info16[5 + 2 * p] = a.gm[p].splits;
        info16[6 + 2 * p] = a.gm[p].units;
    }
    info16[15] = pf::kGroups;
    return CARD_OK;
}

int card_pfwd_destroy(card_pfwd* h) {
    if (!h) return CARD_OK;
    if (h->d_layers) cudaFree(h->d_layers);
    if (h->ctr) cudaFree(h->ctr);
    if (h->ws) cudaFree(h->ws);
    free(h);
    return CARD_OK;
}

}  // extern "C"
