// card_pfwd.cu — persistent forward of a wide row block (draft tree steps).
//
// A draft tree step runs the 1B draft over M <= 128 rows (the frontier plus
// catch-up rows).  As 80 separate kernels the step is latency-bound: every
// GEMM boundary pays launch, pipeline fill, split-K exchange and epilogue,
// and the small projections (o, down: 16 weight tiles) keep only 64 SMs
// streaming.  Here one CTA per SM walks a static schedule of
// steps, step = (layer, phase), phase in {qkv, attention, o, gate/up, down}:
//
//   warp 0   weight producer: streams the pre-tiled 16 KB weight blocks of
//            this CTA's units, step after step, into a ring.  It never waits
//            on activations, so the next step's weights are already in
//            shared memory when the current step's outputs are published.
//   warp 1   activation producer: waits until the previous step is complete
//            (gpu-scope counter), then TMA-loads the activation k-blocks.
//   warp 2   MMA issuer: tcgen05.mma kind::f16, A = weights (128 rows),
//            B = activations (Mpad tokens), accumulator in TMEM (2 buffers).
//   warps 4-11 epilogue workers (TMEM lane = weight row).
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
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "card_common.cuh"
#include "card_llm.h"
#include "card_ptx.cuh"

namespace card {
namespace pf {

using namespace ptx;

constexpr int kThreads = 256;
constexpr int kWorkerWarp0 = 4;
constexpr int kWorkers = 128;
constexpr int kTileN = 128, kBK = 64;
constexpr int kWBytes = kTileN * kBK * 2;   // one pre-tiled weight block
constexpr int kPhases = 5;
enum { PH_QKV = 0, PH_ATTN = 1, PH_O = 2, PH_GU = 3, PH_D = 4 };
constexpr int kMaxLayers = 64;
constexpr int kMaxSteps = kMaxLayers * kPhases;
constexpr int kTileCtrs = 64;   // split-tile counters per step (n_tiles of a split GEMM <= 64)
constexpr int kMaxMpad = 128;   // TMEM: two 128-column accumulators

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
    const int32_t* pos;
    const int32_t* slot;
    const float* cos_t;
    const float* sin_t;
    float* ws;   // split-K partials [splits][Mpad][N]
    int* done;   // [kMaxSteps] completed units per step
    int* tctr;   // [kMaxSteps][kTileCtrs] arrived splits per tile
    int* exit_ctr;
    unsigned long long* trace;   // tuning: [grid][2 + 32 * steps] %globaltimer stamps (null: off)
    // in-kernel tree attention (hd 64): rows of the forward, paged prefix
    int attn;                    // attention steps run in this kernel
    int n_qt, KS, attn_units;    // query tiles per KV head, key splits per tile, units per step
    __nv_bfloat16* o;            // [rows, nh * hd] attention output (the o-projection's X)
    const int32_t* plen;
    const int32_t* n_extra;
    const int32_t* extra;
    int extra_max;
    const int32_t* page_table;   // null: prefix position p is KV slot p
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// stamp k of step st: 0 activations released, 1 first k-block in, 2 accumulator done, 3 outputs published
#define PF_STAMP(st, k)                                                                                     \
    do {                                                                                                    \
        if (a.trace)                                                                                        \
            a.trace[(size_t)blockIdx.x * (2 + 32 * (a.step_end - a.step_begin)) + 2 + 32 * ((st) - a.step_begin) + \
                    (k)] = gtime();                                                                         \
    } while (0)

__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }
__device__ __forceinline__ float half_warp_sum(float v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int units_of(const Args& a, int st) {
    return st % kPhases == PH_ATTN ? a.attn_units : a.gm[st % kPhases].units;
}

// RMSNorm scale rsqrt(mean x^2 + eps) of tokens [m_lo, m_hi) from the
// per-16-column partials; 8 lanes per token, fixed summation order.
__device__ __forceinline__ void compute_invs(const Args& a, int m_lo, int m_hi, float* invs, int t) {
    const int sub = t & 7;
    const int per = (a.ssq_parts + 7) / 8;
    const int p0 = sub * per, p1 = min(a.ssq_parts, p0 + per);
    for (int mb = m_lo; mb < m_hi; mb += kWorkers / 8) {
        const int m = mb + t / 8;
        float acc = 0.f;
        if (m < m_hi) {
            const float* src = a.ssq + m;
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

template <int MAXS>
__device__ __forceinline__ float sum_splits(const float* p, int64_t stride, int S) {
    float v[MAXS];
#pragma unroll
    for (int s = 0; s < MAXS; ++s) v[s] = s < S ? p[s * stride] : 0.f;
    float acc = v[0];
#pragma unroll
    for (int s = 1; s < MAXS; ++s) acc += v[s];
    return acc;
}
__device__ __forceinline__ float reduce_ws(const float* p, int64_t stride, int S) {
    if (S <= 8) return sum_splits<8>(p, stride, S);
    return sum_splits<8>(p, stride, 8) + sum_splits<8>(p + 8 * stride, stride, S - 8);
}

constexpr int kMaxSplits = 10;

__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}
// sums over the S split partials of two float4 items, every load issued first
// (fixed split order; absent splits add exact zeros)
__device__ __forceinline__ void reduce2(const float* pa, const float* pb, int64_t stride, int S, bool va, bool vb,
                                        float4& sa, float4& sb) {
    float4 x[kMaxSplits], y[kMaxSplits];
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s) {
        x[s] = (s < S && va) ? ldcg4(pa + s * stride) : z;
        y[s] = (s < S && vb) ? ldcg4(pb + s * stride) : z;
    }
    sa = x[0];
    sb = y[0];
#pragma unroll
    for (int s = 1; s < kMaxSplits; ++s) {
        add4(sa, x[s]);
        add4(sb, y[s]);
    }
}
// sum over the S split partials of one float4 item, every load issued first (split order)
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
// o / down epilogue of one float4 item: x += sum, bf16 copy, per-16-column
// sum of squares (a quad of lanes = 16 columns)
__device__ __forceinline__ void resid_item(const Args& a, int N, int ng, int m, bool valid, const float4& s) {
    float4 xn = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
        float4* xp = reinterpret_cast<float4*>(a.x + (int64_t)m * N + ng);
        xn = *xp;
        add4(xn, s);
        *xp = xn;
        *reinterpret_cast<uint2*>(a.xb + (int64_t)m * N + ng) = pack4_bf16(xn.x, xn.y, xn.z, xn.w);
    }
    float sq = xn.x * xn.x + xn.y * xn.y + xn.z * xn.z + xn.w * xn.w;
    sq += __shfl_xor_sync(0xffffffffu, sq, 1);
    sq += __shfl_xor_sync(0xffffffffu, sq, 2);
    if (valid && (threadIdx.x & 3) == 0) a.ssq[(int64_t)(ng >> 4) * a.ssq_ld + m] = sq;
}
// qkv epilogue of one float4 item (features 4 f4 .. of the tile, token m):
// norm scale + bias, RoPE with the partner half of the head via a shuffle
// (the warp holds the whole 128-feature row), q * 1/sqrt(hd) -> q, k / v -> cache
__device__ __forceinline__ void qkv_item(const Args& a, const Layer& L, const float* invs, int tile, int f4, int m,
                                         bool valid, float4 s) {
    const int half = a.hd >> 1;
    const int fb = 4 * f4;                 // feature in the tile
    const int hl = fb / a.hd, i0 = fb - hl * a.hd;
    const int head = (tile * kTileN) / a.hd + hl;
    const int ng = tile * kTileN + fb;
    float4 v = s;
    int pos = 0, slot = 0;
    if (valid) {
        const float iv = invs[m];
        v.x *= iv;
        v.y *= iv;
        v.z *= iv;
        v.w *= iv;
        if (L.bqkv) add4(v, *reinterpret_cast<const float4*>(L.bqkv + ng));
        pos = a.pos[m];
        slot = a.slot[m];
    }
    const int pl = half >> 2;   // partner lane distance (float4 items)
    float4 o;
    o.x = __shfl_xor_sync(0xffffffffu, v.x, pl);
    o.y = __shfl_xor_sync(0xffffffffu, v.y, pl);
    o.z = __shfl_xor_sync(0xffffffffu, v.z, pl);
    o.w = __shfl_xor_sync(0xffffffffu, v.w, pl);
    if (!valid) return;
    if (head >= a.nh + a.nkv) {   // v: no rotation
        *reinterpret_cast<uint2*>(L.vc + ((int64_t)slot * a.nkv + (head - a.nh - a.nkv)) * a.hd + i0) =
            pack4_bf16(v.x, v.y, v.z, v.w);
        return;
    }
    const bool first = i0 < half;
    const int ii = first ? i0 : i0 - half;
    const float4 cs = *reinterpret_cast<const float4*>(a.cos_t + (int64_t)pos * half + ii);
    const float4 sn = *reinterpret_cast<const float4*>(a.sin_t + (int64_t)pos * half + ii);
    // first half: x1 = v, x2 = o -> x1 cs - x2 sn; second: x2 = v, x1 = o -> x2 cs + x1 sn
    float4 r;
    if (first) {
        r.x = v.x * cs.x - o.x * sn.x;
        r.y = v.y * cs.y - o.y * sn.y;
        r.z = v.z * cs.z - o.z * sn.z;
        r.w = v.w * cs.w - o.w * sn.w;
    } else {
        r.x = v.x * cs.x + o.x * sn.x;
        r.y = v.y * cs.y + o.y * sn.y;
        r.z = v.z * cs.z + o.z * sn.z;
        r.w = v.w * cs.w + o.w * sn.w;
    }
    if (head < a.nh) {
        r.x *= a.qscale;
        r.y *= a.qscale;
        r.z *= a.qscale;
        r.w *= a.qscale;
        *reinterpret_cast<float4*>(a.q + ((int64_t)m * a.nh + head) * a.hd + i0) = r;
    } else {
        *reinterpret_cast<uint2*>(L.kc + ((int64_t)slot * a.nkv + (head - a.nh)) * a.hd + i0) =
            pack4_bf16(r.x, r.y, r.z, r.w);
    }
}

// ---------------------------------------------------------------- attention
// Tree attention of mask.py:173-217 without the mask: query-head row (r, h)
// of KV head g sees prefix positions [0, plen[r]) (paged) and the n_extra[r]
// slots extra[r][..] (tree ancestors + itself).  A unit = (g, query tile of
// 128 query-heads, key split ks): its rounds of 128 virtual keys (prefix
// rounds, then the tile rows' extras row after row) run S = Q K^T and O = P V
// on tcgen05 (S, O in TMEM, P bf16 in shared memory); the KS partials
// (m, l, O) of a tile meet in the workspace and each split merges 1/KS of the
// tile's rows in split order.  Head dim 64 only (the draft).
constexpr int kAHD = 64;
constexpr int kAQT = 128;            // query-heads per tile
constexpr int kAKB = 128;            // keys per round
constexpr int kASub = 128 * 64 * 2;  // one [128 x 64] bf16 SW128 block
constexpr int kAMaxRows = 40;        // token rows per tile
constexpr int kAMaxX = 640;          // gathered extra keys per tile
constexpr int kARec = 68;            // partial record: m, l, pad, pad, O[64]
// attention shared memory (aliases the activation ring + aux region)
constexpr int kAoQ = 0, kAoK = kASub, kAoV = 3 * kASub, kAoP = 5 * kASub, kAoMeta = 7 * kASub;
constexpr int kAMetaBytes = kAMaxX * 4 + 3 * kAMaxRows * 4 + 2 * kAQT * 4 + 16 * 4;
constexpr int kAttnBytes = kAoMeta + kAMetaBytes;
constexpr int kLoaders = 64;         // warps 1 and 3 gather K / V during attention steps
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t sw_off(int r, int c) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(kASub >> 4) << 16) | ((uint64_t)64 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// 16-column validity mask of the keys [jc, jc + 16): the prefix range [0, plim),
// then the row's own extras [e0, e1)
__device__ __forceinline__ uint32_t col_mask(int jc, int plim, int e0, int e1) {
    const int lim = plim - jc;
    uint32_t mm = lim >= 16 ? 0xFFFFu : (lim > 0 ? (1u << lim) - 1u : 0u);
    const int x0 = max(0, e0 - jc), x1 = min(16, e1 - jc);
    if (x1 > x0) mm |= ((1u << x1) - 1u) & ~((1u << x0) - 1u);
    return mm;
}

// per-unit tile metadata in shared memory
struct AttnMeta {
    int32_t* ext_slot;   // [kAMaxX]
    int32_t* rplen;      // [kAMaxRows]
    int32_t* rnx;
    int32_t* rxo;
    float* xch;          // [2][kAQT]
    int32_t* info;       // [16]: 0 Kp, 1 Kx, 2 XB, 3 r_begin (round), 4 nr, 5 r_lo, 6 n_rows, 7 live
};
__device__ __forceinline__ AttnMeta attn_meta(uint8_t* sa) {
    AttnMeta m;
    m.ext_slot = (int32_t*)(sa + kAoMeta);
    m.rplen = m.ext_slot + kAMaxX;
    m.rnx = m.rplen + kAMaxRows;
    m.rxo = m.rnx + kAMaxRows;
    m.xch = (float*)(m.rxo + kAMaxRows);
    m.info = (int32_t*)(m.xch + 2 * kAQT);
    return m;
}
__device__ __forceinline__ void attn_decode(const Args& a, int u, int& g, int& qt, int& ks) {
    ks = u % a.KS;
    const int tile = u / a.KS;
    qt = tile % a.n_qt;
    g = tile / a.n_qt;
}

// One attention unit of the worker warps (Q tile, softmax rounds, merge); out
// of line so its register allocation does not compete with the GEMM epilogues.
__device__ __noinline__ void attn_unit_workers(const Args& a, uint8_t* sA, uint64_t* bars, uint32_t tmem_base, int st,
                                               int u, int M, uint32_t& arc_ref) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = threadIdx.x - kWorkerWarp0 * 32;
    const int wq = warp - kWorkerWarp0;   // TMEM lane quarter
    const int cta = blockIdx.x;
    const int GQ = a.nh / a.nkv;
    const int nq = M * GQ;
    const AttnMeta meta = attn_meta(sA);
    const uint32_t tS = tmem_base, tO = tmem_base + 256;
    uint64_t* as_full = bars + 8;
    uint64_t* as_empty = bars + 10;
    uint64_t* ap_full = bars + 12;
    uint64_t* ao_full = bars + 13;
    uint64_t* aq_full = bars + 14;
    uint32_t arc = arc_ref;
    int g, qt, ks;
    attn_decode(a, u, g, qt, ks);
    const int q0 = qt * kAQT;
    const bool live = q0 < nq;
    const int r_lo = q0 / GQ;
    const int r_hi = live ? min(M, (q0 + kAQT - 1) / GQ + 1) : r_lo;
    const int n_rows = r_hi - r_lo;
    for (int i = t; i < n_rows; i += kWorkers) {
        meta.rplen[i] = a.plen[r_lo + i];
        meta.rnx[i] = a.n_extra ? a.n_extra[r_lo + i] : 0;
    }
    named_bar(1, kWorkers);
    if (t == 0) {
        int Kp = 0, x = 0;
        for (int i = 0; i < n_rows; ++i) {
            Kp = max(Kp, meta.rplen[i]);
            meta.rxo[i] = x;
            x += meta.rnx[i];
        }
        const int Kx = min(x, kAMaxX);
        const int n_pr = (Kp + kAKB - 1) / kAKB;
        const int n_tot = live ? n_pr + (Kx + kAKB - 1) / kAKB : 0;
        meta.info[0] = Kp;
        meta.info[1] = Kx;
        meta.info[2] = n_pr * kAKB;
        meta.info[3] = n_tot * ks / a.KS;
        meta.info[4] = n_tot * (ks + 1) / a.KS - n_tot * ks / a.KS;
    }
    named_bar(1, kWorkers);
    const int Kp = meta.info[0], XB = meta.info[2], rb = meta.info[3], nr = meta.info[4];
    for (int i = wq; i < n_rows; i += kWorkers / 32) {
        const int n = meta.rnx[i], xo = meta.rxo[i];
        for (int j = lane; j < n && xo + j < kAMaxX; j += 32)
            meta.ext_slot[xo + j] = a.extra[(int64_t)(r_lo + i) * a.extra_max + j];
    }
    // Q tile: fp32 (pre-scaled) -> bf16, SW128 K-major, query-head row qh = q0 + tr
    if (nr > 0) {
        for (int idx = t; idx < kAQT * 8; idx += kWorkers) {
            const int tr = idx >> 3, c = idx & 7;
            const int qh = q0 + tr;
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            if (qh < nq) {
                const int r = qh / GQ, head = g * GQ + qh % GQ;
                const float4* src = (const float4*)(a.q + ((int64_t)r * a.nh + head) * kAHD + c * 8);
                const float4 x0 = src[0], x1 = src[1];
                w[0] = pack_bf2(x0.x, x0.y);
                w[1] = pack_bf2(x0.z, x0.w);
                w[2] = pack_bf2(x1.x, x1.y);
                w[3] = pack_bf2(x1.z, x1.w);
            }
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(su32(sA + kAoQ) + sw_off(tr, c)),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                         : "memory");
        }
        fence_async_smem();
    }
    named_bar(6, kWorkers + kLoaders);   // metadata (ext_slot) to the loaders
    if (t == 0 && u == cta) PF_STAMP(st, 5);
    tc_before();
    __syncwarp();
    if (lane == 0) bar_arrive(aq_full);
    // softmax: one thread per query-head row (TMEM lane), all 128 key columns
    const int tr = t;
    const int qh = q0 + tr;
    const bool rlive = live && qh < nq;
    const int ri = rlive ? qh / GQ - r_lo : 0;
    const int plim = rlive ? min(meta.rplen[ri], Kp) : 0;
    const int e0 = rlive ? XB + meta.rxo[ri] : 0, e1 = rlive ? XB + meta.rxo[ri] + meta.rnx[ri] : 0;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    for (int li = 0; li < nr; ++li, ++arc) {
        const int j0 = (rb + li) * kAKB;
        const int b = arc & 1;
        bar_wait_polite(&as_full[b], (arc >> 1) & 1);
        tc_after();
        const uint32_t sb_ = tS + b * kAKB + lane_off;
        // row max: one 16-column chunk at a time (rolled: the code stays in the instruction cache)
        float mx = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
            const uint32_t mq = col_mask(j0 + c * 16, plim, e0, e1);
            if (!__any_sync(0xffffffffu, mq != 0u)) continue;
            float v[16];
            tmem_ld16(sb_ + (uint32_t)(c * 16), v);
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) mx = ((mq >> u2) & 1u) ? fmaxf(mx, v[u2]) : mx;
        }
        const float m_cand = fmaxf(m_run, mx);
        // lazy rescale: keep the running max unless the row max grew by more
        // than 2^8 (P stays <= 256, exact enough in bf16 / fp32)
        const bool grow = m_run == -INFINITY ? true : (m_cand - m_run) * kLog2e > 8.f;
        const float m_use = grow ? m_cand : m_run;
        const float alpha = (li == 0 || !grow) ? 1.f : exp2f((m_run - m_use) * kLog2e);
        const float mb = (m_use == -INFINITY) ? 0.f : m_use * kLog2e;
        // P.V of the last round done: P buffer free, O complete
        if (li > 0) {
            bar_wait_polite(ao_full, (arc - 1) & 1);
            tc_after();
            if (__any_sync(0xffffffffu, alpha != 1.f)) {   // rescale my row of O in TMEM
#pragma unroll 1
                for (int c2 = 0; c2 < kAHD / 32; ++c2) {
                    uint32_t ov[2][16];
                    const uint32_t ta = tO + lane_off + (uint32_t)(c2 * 32);
                    tmem_ld16_issue(ta, ov[0]);
                    tmem_ld16_issue(ta + 16, ov[1]);
                    tmem_wait_ld();
#pragma unroll
                    for (int d = 0; d < 16; ++d) {
                        ov[0][d] = __float_as_uint(__uint_as_float(ov[0][d]) * alpha);
                        ov[1][d] = __float_as_uint(__uint_as_float(ov[1][d]) * alpha);
                    }
                    tmem_st16(ta, ov[0]);
                    tmem_st16(ta + 16, ov[1]);
                }
                tmem_wait_st();
            }
        }
        float sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
            const uint32_t mq = col_mask(j0 + c * 16, plim, e0, e1);
            uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            if (__any_sync(0xffffffffu, mq != 0u)) {
                float v[16];
                tmem_ld16(sb_ + (uint32_t)(c * 16), v);
#pragma unroll
                for (int u2 = 0; u2 < 16; u2 += 2) {
                    const float p0 = ((mq >> u2) & 1u) ? exp2f(fmaf(v[u2], kLog2e, -mb)) : 0.f;
                    const float p1 = ((mq >> (u2 + 1)) & 1u) ? exp2f(fmaf(v[u2 + 1], kLog2e, -mb)) : 0.f;
                    w[u2 >> 1] = pack_bf2(p0, p1);
                    const __nv_bfloat162 pr = *reinterpret_cast<__nv_bfloat162*>(&w[u2 >> 1]);
                    sum += __bfloat162float(pr.x) + __bfloat162float(pr.y);   // l sums what P.V uses
                }
            }
            const uint32_t base = su32(sA + kAoP + (c >> 2) * kASub);
            const int ch = (c & 3) * 2;
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(base + sw_off(tr, ch)), "r"(w[0]), "r"(w[1]),
                         "r"(w[2]), "r"(w[3])
                         : "memory");
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(base + sw_off(tr, ch + 1)), "r"(w[4]),
                         "r"(w[5]), "r"(w[6]), "r"(w[7])
                         : "memory");
        }
        fence_async_smem();
        tc_before();
        __syncwarp();
        if (lane == 0) {
            bar_arrive(&as_empty[b]);
            bar_arrive(ap_full);
        }
        l_run = l_run * alpha + sum;
        m_run = m_use;
    }
    if (t == 0 && u == cta) PF_STAMP(st, 7);
    // partial (m, l, O) of my row -> workspace record [tile][ks][row], O straight from TMEM
    const int tile = g * a.n_qt + qt;
    float* rec = a.ws + (((size_t)tile * a.KS + ks) * kAQT + tr) * kARec;
    rec[0] = m_run;
    rec[1] = l_run;
    if (nr > 0) {
        bar_wait_polite(ao_full, (arc - 1) & 1);
        tc_after();
#pragma unroll 1
        for (int c2 = 0; c2 < 4; ++c2) {
            float v[16];
            tmem_ld16(tO + lane_off + (uint32_t)(c2 * 16), v);
#pragma unroll
            for (int d = 0; d < 16; d += 4)
                __stcg(reinterpret_cast<float4*>(rec + 4 + c2 * 16 + d), make_float4(v[d], v[d + 1], v[d + 2], v[d + 3]));
        }
        tc_before();
    } else {
#pragma unroll
        for (int d = 0; d < kAHD; d += 4) __stcg(reinterpret_cast<float4*>(rec + 4 + d), make_float4(0.f, 0.f, 0.f, 0.f));
    }
    named_bar(1, kWorkers);
    int* tc = &a.tctr[st * kTileCtrs + tile];
    if (t == 0) {
        atom_add_acq_rel(tc, 1);
        wait_ge(tc, a.KS);
        if (u == cta) PF_STAMP(st, 8);
    }
    named_bar(1, kWorkers);
    // merge rows [ks * 128 / KS, (ks + 1) * 128 / KS) of the tile over the KS splits
    const int rr0 = kAQT * ks / a.KS, rr1 = kAQT * (ks + 1) / a.KS;
    for (int idx = t; idx < (rr1 - rr0) * (kAHD / 4); idx += kWorkers) {
        const int row = rr0 + idx / (kAHD / 4), d = (idx % (kAHD / 4)) * 4;
        const int qh2 = q0 + row;
        if (qh2 >= nq) continue;
        const float* r0p = a.ws + (((size_t)tile * a.KS) * kAQT + row) * kARec;
        const size_t sstr = (size_t)kAQT * kARec;
        float mm = -INFINITY;
        for (int s2 = 0; s2 < a.KS; ++s2) mm = fmaxf(mm, __ldcg(r0p + s2 * sstr));
        float l = 0.f;
        float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s2 = 0; s2 < a.KS; ++s2) {   // split order: deterministic
            const float* rp = r0p + s2 * sstr;
            const float ms = __ldcg(rp);
            const float w = (ms == -INFINITY) ? 0.f : exp2f((ms - mm) * kLog2e);
            const float4 ov4 = ldcg4(rp + 4 + d);
            l = fmaf(__ldcg(rp + 1), w, l);
            acc4.x = fmaf(ov4.x, w, acc4.x);
            acc4.y = fmaf(ov4.y, w, acc4.y);
            acc4.z = fmaf(ov4.z, w, acc4.z);
            acc4.w = fmaf(ov4.w, w, acc4.w);
        }
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const int r = qh2 / GQ, head = g * GQ + qh2 % GQ;
        *reinterpret_cast<uint2*>(a.o + ((int64_t)r * a.nh + head) * kAHD + d) =
            pack4_bf16(acc4.x * inv, acc4.y * inv, acc4.z * inv, acc4.w * inv);
    }
    named_bar(7, kWorkers + kLoaders);   // the loaders read this unit's info: meta reusable
    if (t == 0) {
        fence_proxy_async_global();   // o is read by TMA in the o step
        atom_add_acq_rel(&a.done[st], 1);
        PF_STAMP(st, 3);
    }
    arc_ref = arc;
}

__global__ void __launch_bounds__(kThreads, 1)
    pfwd_kernel(const __grid_constant__ CUtensorMap tmXb, const __grid_constant__ CUtensorMap tmO,
                const __grid_constant__ CUtensorMap tmG, const __grid_constant__ Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int xbytes = a.Mpad * kBK * 2;
    uint8_t* sW = smem;
    uint8_t* sX = sW + (size_t)a.WS * kWBytes;
    // the attention scratch aliases the activation ring and the aux region behind it
    const int xring = a.XS * xbytes;
    const int aux = kAttnBytes > xring ? kAttnBytes - xring : 0;
    float* invs = (float*)(sX + (size_t)xring + aux);   // [kMaxMpad]
    // fixed-count barriers first (constant offsets from one base), then the rings
    uint64_t* bars = (uint64_t*)(invs + kMaxMpad);
    uint64_t* tfull = bars;            // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint64_t* akv_full = tempty + 2;   // [2] loaders -> MMA
    uint64_t* akv_empty = akv_full + 2;   // [2] MMA commit -> loaders
    uint64_t* as_full = akv_empty + 2;    // [2] S buffer ready
    uint64_t* as_empty = as_full + 2;     // [2] softmax read the S buffer
    uint64_t* ap_full = as_empty + 2;     // P written (and O rescaled)
    uint64_t* ao_full = ap_full + 1;      // P.V of the round accumulated into O
    uint64_t* aq_full = ao_full + 1;      // Q tile + metadata ready
    uint32_t* tmem_slot = (uint32_t*)(aq_full + 1);
    uint64_t* wfull = bars + 16;
    uint64_t* wempty = wfull + a.WS;
    uint64_t* xfull = wempty + a.WS;
    uint64_t* xempty = xfull + a.XS;
    uint8_t* sA = sX;
    const AttnMeta meta = attn_meta(sA);

    const int M = *a.dM;
    if (M <= 0) return;   // uniform: nothing to do, no counter touched
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0 && a.trace) a.trace[(size_t)blockIdx.x * (2 + 32 * (a.step_end - a.step_begin))] = gtime();
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
            bar_init(&akv_full[i], kLoaders);
            bar_init(&akv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            bar_init(&as_full[i], 1);
            bar_init(&as_empty[i], kWorkers / 32);
        }
        bar_init(ap_full, kWorkers / 32);
        bar_init(ao_full, 1);
        bar_init(aq_full, kWorkers / 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem_base = *tmem_slot;
    // attention (the GEMM accumulators are idle during its step): S double-buffered
    // in columns [0, 256), O accumulated over the rounds in [256, 320)
    const uint32_t tS = tmem_base, tO = tmem_base + 256;
    const int n_mma = ((M + 15) / 16) * 16;
    const int sb = a.step_begin, se = a.step_end;
    const int cta = blockIdx.x, G = gridDim.x;
    const int GQ = a.nh / a.nkv;   // query-heads per KV head
    const int nq = M * GQ;

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
    } else if (warp == 1 || warp == 3) {
        // ------------------------------------------------ activation producer (warp 1 lane 0) and
        // attention K / V loaders (warps 1 and 3)
        const int lt = (warp == 1 ? 0 : 32) + lane;
        int s = 0;
        uint32_t ph = 0;
        uint32_t arc = 0;   // attention rounds so far (ring slot / parity)
        if (warp == 1 && lane == 0) {
            prefetch_map(&tmXb);
            prefetch_map(&tmO);
            prefetch_map(&tmG);
        }
        for (int st = sb; st < se; ++st) {
            const int p = st % kPhases;
            if (p == PH_ATTN) {
                const Layer& L = a.layers[st / kPhases];
                for (int u = cta; u < a.attn_units; u += G) {
                    int g, qt, ks;
                    attn_decode(a, u, g, qt, ks);
                    named_bar(6, kWorkers + kLoaders);   // the workers published the tile metadata
                    const int Kp = meta.info[0], Kx = meta.info[1], XB = meta.info[2];
                    const int rb = meta.info[3], nr = meta.info[4];
                    asm volatile("bar.arrive 7, %0;" ::"r"(kWorkers + kLoaders) : "memory");   // info read
                    for (int li = 0; li < nr; ++li, ++arc) {
                        const int b = arc & 1;
                        if (arc >= 2) bar_wait(&akv_empty[b], ((arc >> 1) - 1) & 1);
                        const int j0 = (rb + li) * kAKB;
                        const uint32_t kb = su32(sA + kAoK + b * kASub), vb = su32(sA + kAoV + b * kASub);
                        for (int idx = lt; idx < kAKB * 8; idx += kLoaders) {
                            const int kk = idx >> 3, c = idx & 7;
                            const int j = j0 + kk;
                            const uint32_t off = sw_off(kk, c);
                            int slot = -1;
                            if (j < XB) {
                                if (j < Kp) slot = a.page_table ? a.page_table[j >> 6] * 64 + (j & 63) : j;
                            } else if (j - XB < Kx) {
                                slot = meta.ext_slot[j - XB];
                            }
                            if (slot >= 0) {
                                const int64_t e = ((int64_t)slot * a.nkv + g) * kAHD + c * 8;
                                cp16(kb + off, L.kc + e);
                                cp16(vb + off, L.vc + e);
                            } else {
                                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(kb + off), "r"(0u)
                                             : "memory");
                                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(vb + off), "r"(0u)
                                             : "memory");
                            }
                        }
                        asm volatile("cp.async.wait_all;" ::: "memory");
                        fence_async_smem();
                        bar_arrive(&akv_full[b]);
                        if (lt == 0 && u == cta && li < 4) PF_STAMP(st, 28 + li);
                    }
                }
                continue;
            }
            const Gemm& gm = a.gm[p];
            if (cta >= gm.units) continue;
            if (warp == 1 && lane == 0) {
                if (st > sb) {
                    wait_ge(&a.done[st - 1], units_of(a, st - 1));
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
            __syncwarp();
        }
    } else if (warp == 2) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16(kTileN, n_mma);
            const uint32_t idS = idesc_bf16(kAQT, kAKB);
            const uint32_t idO = idesc_bf16(kAQT, kAHD) | (1u << 16);   // B (V) MN-major
            int ws = 0, xs = 0, acc = 0;
            uint32_t wph = 0, xph = 0, aph = 0, arc = 0, uq = 0;
            for (int st = sb; st < se; ++st) {
                const int p = st % kPhases;
                if (p == PH_ATTN) {
                    for (int u = cta; u < a.attn_units; u += G, ++uq) {
                        bar_wait(aq_full, uq & 1);
                        tc_after();
                        const int nr = meta.info[4];
                        const uint32_t q_s = su32(sA + kAoQ), p_s = su32(sA + kAoP);
                        // S of round c into S buffer c & 1 (global round arc0 + c)
                        const uint32_t arc0 = arc;
                        auto issue_s = [&](int c) {
                            const uint32_t r = arc0 + c;
                            const int b = r & 1;
                            bar_wait(&akv_full[b], (r >> 1) & 1);
                            if (r >= 2) bar_wait(&as_empty[b], ((r >> 1) - 1) & 1);   // softmax read that buffer
                            if (u == cta && c < 4) PF_STAMP(st, 12 + 4 * c);
                            tc_after();
                            const uint32_t k_s = su32(sA + kAoK + b * kASub);
#pragma unroll
                            for (int k = 0; k < kAHD / 16; ++k)
                                tc_mma(tS + b * kAKB, desc_sw128(q_s + k * 32), desc_sw128(k_s + k * 32), idS,
                                       k > 0 ? 1u : 0u);
                            tc_commit(&as_full[b]);
                        };
                        if (nr > 0) issue_s(0);
                        for (int li = 0; li < nr; ++li, ++arc) {
                            const int b = arc & 1;
                            if (li + 1 < nr) issue_s(li + 1);
                            bar_wait(ap_full, arc & 1);   // P written, O rescaled
                            if (u == cta && li < 4) PF_STAMP(st, 13 + 4 * li);
                            tc_after();
                            const uint32_t v_s = su32(sA + kAoV + b * kASub);
#pragma unroll
                            for (int k = 0; k < kAKB / 16; ++k) {
                                const uint32_t pa = p_s + (uint32_t)((k >> 2) * kASub + (k & 3) * 32);
                                tc_mma(tO, desc_sw128(pa), desc_mnmajor(v_s + (uint32_t)(k * 2048)), idO,
                                       (li > 0 || k > 0) ? 1u : 0u);
                            }
                            tc_commit(ao_full);
                            tc_commit(&akv_empty[b]);
                        }
                    }
                    continue;
                }
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
        // ------------------------------------------------ epilogue workers / softmax
        const int t = threadIdx.x - kWorkerWarp0 * 32;
        const int wq = warp - kWorkerWarp0;   // TMEM lane quarter
        const int n_local = wq * 32 + lane;
        int acc = 0;
        uint32_t aph = 0, arc = 0;
        for (int st = sb; st < se; ++st) {
            const int p = st % kPhases;
            const Layer& L = a.layers[st / kPhases];
            const int units = units_of(a, st);
            if (cta >= units) continue;
            if (st > sb) {   // previous step's outputs visible to every worker
                if (t == 0) wait_ge(&a.done[st - 1], units_of(a, st - 1));
                named_bar(1, kWorkers);
            }
            if (p == PH_ATTN) {
                if (t == 0) PF_STAMP(st, 4);
                for (int u = cta; u < units; u += G) attn_unit_workers(a, sA, bars, tmem_base, st, u, M, arc);
                continue;
            }
            const Gemm& gm = a.gm[p];
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
                    // gate/up: rows 32q..32q+15 are the gates of features
                    // 16q..16q+15, rows 32q+16..32q+31 the ups (interleave_gate_up);
                    // lanes l and l^16 swap chunk halves with one shuffle per token pair
                    const bool up = lane >= 16;
                    const int f = tile * 64 + wq * 16 + (lane & 15);
                    const int jb = up ? 8 : 0;
#pragma unroll 1
                    for (int m0 = 0; m0 < M; m0 += 16) {   // rolled: the code stays in the instruction cache
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
                            if (m0 + jb + jj < M)
                                a.g[(int64_t)(m0 + jb + jj) * a.F + f] = __float2bfloat16(silu(gg) * uu);
                        }
                    }
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
                    // split unit: partial -> workspace [sp][m][n] (coalesced over n);
                    // every TMEM chunk of the thread in flight before one wait
                    float* wsp = a.ws + (size_t)sp * a.Mpad * gm.N + tile * kTileN + n_local;
#pragma unroll 1
                    for (int m0 = 0; m0 < M; m0 += 16) {
                        float v[16];
                        tmem_ld16(trow + (uint32_t)m0, v);
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (m0 + j < M) __stcg(wsp + (int64_t)(m0 + j) * gm.N, v[j]);
                    }
                    tc_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(&tempty[acc]);
                    named_bar(1, kWorkers);
                    int* tc = &a.tctr[st * kTileCtrs + tile];
                    if (t == 0) {
                        atom_add_acq_rel(tc, 1);   // release: the CTA's partial stores (bar.sync above)
                        wait_ge(tc, gm.splits);
                    }
                    named_bar(1, kWorkers);
                    // reduce my token slice of the tile in split order: float4
                    // items (token j, features 4 f .. 4 f + 3), one warp per token
                    // row, two items per thread with every load in flight
                    const int nt = mb - ma;
                    const int64_t sstride = (int64_t)a.Mpad * gm.N;
                    const int f4 = lane;   // == (t & 31): a warp covers the tile's 128 features
                    const int ng = tile * kTileN + 4 * f4;
#pragma unroll 1
                    for (int i0 = t; i0 < nt * 32; i0 += kWorkers) {   // a warp = one token row (warp-uniform)
                        const int m = ma + (i0 >> 5);
                        const float4 sm = reduce1(a.ws + (int64_t)m * gm.N + ng, sstride, gm.splits);
                        if (p == PH_QKV) qkv_item(a, L, invs, tile, f4, m, true, sm);
                        else resid_item(a, gm.N, ng, m, true, sm);
                    }
                }
                acc ^= 1;
                if (acc == 0) aph ^= 1;
                named_bar(1, kWorkers);
                if (t == 0) {
                    fence_proxy_async_global();   // xb / g / o are read by TMA in later steps
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
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    if (threadIdx.x == 0 && a.trace) a.trace[(size_t)blockIdx.x * (2 + 32 * (se - sb)) + 1] = gtime();
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
    bool attn_ok;   // attention steps may run in the kernel (bound rows fit its tile limits)
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
                     const float* sin_t, float eps, int attn_inkernel, card_pfwd** out) {
    if (!out || !layer_w || !kv || !x || !xb || !ssq || !q || !o || !g || !pos || !slot || !cos_t || !sin_t)
        return CARD_E_INPUT;
    *out = nullptr;
    if (n_layers <= 0 || n_layers > pf::kMaxLayers || m_max <= 16 || m_max > pf::kMaxMpad || act_rows < m_max)
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
    // smem: weight ring + (activation ring | attention scratch) + invs + barriers
    const int xbytes = Mpad * pf::kBK * 2;
    const int fixed = 1024 + pf::kMaxMpad * 4 + 64 * 8 + 64;
    const int budget = 226 * 1024;   // + the kernel's 1 KB of static shared memory
    a.XS = 6;
    const int region = a.XS * xbytes > pf::kAttnBytes ? a.XS * xbytes : pf::kAttnBytes;
    a.WS = (budget - fixed - region) / pf::kWBytes;
    if (a.WS > 8) a.WS = 8;
    h->smem = fixed + a.WS * pf::kWBytes + region;
    // in-kernel attention: head dim 64, query tiles of 128 query-heads over <= 40 token rows
    const int GQ = nh / nkv;
    a.n_qt = (Mpad * GQ + pf::kAQT - 1) / pf::kAQT;
    a.attn = (attn_inkernel && hd == pf::kAHD && nh % nkv == 0 && pf::kAQT / GQ + 2 <= pf::kAMaxRows) ? 1 : 0;
    a.KS = sms / (nkv * a.n_qt);
    if (a.KS > 8) a.KS = 8;
    if (a.KS < 1) a.KS = 1;
    a.attn_units = nkv * a.n_qt * a.KS;
    if (a.attn && (nkv * a.n_qt > pf::kTileCtrs ||
                   (size_t)nkv * a.n_qt * a.KS * pf::kAQT * pf::kARec > ws_floats))
        a.attn = 0;
    a.o = (__nv_bfloat16*)o;
    if (e == cudaSuccess && ws_floats) e = cudaMalloc(&h->ws, ws_floats * sizeof(float));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(pf::pfwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem);
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
// 2 o, 3 gate/up, 4 down).  Attention steps need the in-kernel attention
// (head dim 64 and bound rows within its tile limits, card_pfwd_info[15]);
// otherwise they run outside (card_attention_paged) between runs.
int card_pfwd_run(card_pfwd* h, const int32_t* dM, int step_begin, int step_end, void* stream) {
    if (!h || !dM || step_begin < 0 || step_end <= step_begin || step_end > h->n_layers * pf::kPhases)
        return CARD_E_INPUT;
    for (int st = step_begin; st < step_end; ++st)
        if (st % pf::kPhases == pf::PH_ATTN && !h->attn_ok) return CARD_E_CONFIG;
    pf::Args a = h->args;
    a.dM = dM;
    a.step_begin = step_begin;
    a.step_end = step_end;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->grid);
    cfg.blockDim = dim3(pf::kThreads);
    cfg.dynamicSmemBytes = h->smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, pf::pfwd_kernel, h->tmXb, h->tmO, h->tmG, a);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return CARD_E_CUDA;
    }
    return CARD_OK;
}

// row-dependent epilogue inputs (the row block the forward runs over)
int card_pfwd_bind(card_pfwd* h, const int32_t* pos, const int32_t* slot, const int32_t* plen,
                   const int32_t* n_extra, const int32_t* extra, int extra_max, const int32_t* page_table) {
    if (!h || !pos || !slot || !plen || (extra_max > 0 && (!n_extra || !extra)) || extra_max < 0) return CARD_E_INPUT;
    pf::Args& a = h->args;
    a.pos = pos;
    a.slot = slot;
    a.plen = plen;
    a.n_extra = extra_max > 0 ? n_extra : nullptr;
    a.extra = extra;
    a.extra_max = extra_max;
    a.page_table = page_table;
    h->attn_ok = a.attn && (pf::kAQT / (a.nh / a.nkv) + 2) * extra_max <= pf::kAMaxX;
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
        info16[5 + 2 * p] = p == pf::PH_ATTN ? a.KS : a.gm[p].splits;
        info16[6 + 2 * p] = p == pf::PH_ATTN ? a.attn_units : a.gm[p].units;
    }
    info16[15] = h->attn_ok ? 1 : 0;
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
