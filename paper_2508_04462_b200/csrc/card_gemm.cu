// card_gemm.cu — decode-phase weight streaming for the draft/target models.
//
//   Y[M, N] = X[M, K] . W[N, K]^T  (+ fused epilogue)
//
// Three kernels, picked per linear layer at plan time:
//   * tc_gemm   (bf16 weights, M >= 2): TMA streams 128x64 weight tiles and
//     the (tiny) activation tile into a multi-stage mbarrier ring; one
//     elected thread issues tcgen05.mma kind::f16 (A = weights, K-major,
//     SWIZZLE_128B; B = activations) into a TMEM accumulator (128 lanes x
//     Mpad fp32 columns, double-buffered); four epilogue warps drain TMEM
//     with tcgen05.ld and apply the fused epilogue.  Either persistent CTAs
//     walk whole tiles (wide N), or the K range of each tile is split over
//     the S ranks of a thread-block cluster whose partial sums are reduced
//     through distributed shared memory in rank order (deterministic).
//   * gemv      (bf16 weights, M == 1): 128-bit vectorised weight loads,
//     one warp per output row group, fp32 accumulation.
//   * f32_gemm  (fp32 weights — the parity mode against the CPU oracle).
//
// Epilogues: STORE_F32, RESID_F32 (out += acc), STORE_BF16, SWIGLU_BF16
// (weight rows interleaved per 128-row tile: 64 gate rows then the 64 up
// rows of the same features; out = silu(gate) * up), optional fp32 bias.
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "card_common.cuh"
#include "card_llm.h"

namespace card {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// 1-D bulk copy (TMA engine, no tensor map): weights are pre-tiled in HBM so
// each pipeline stage is one contiguous 16 KB block already in SW128 order.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// one stage's weight block as `pieces` bulk copies on the same barrier
__device__ __forceinline__ void bulk_load_split(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint64_t* bar,
                                                int pieces) {
    const uint32_t part = bytes / (uint32_t)pieces;
    for (int p = 0; p < pieces; ++p) bulk_load(dst + p * part, src + p * part, part, bar);
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// issue-only TMEM load (no wait): several chunks go in flight before one tmem_wait_ld()
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// address of the same smem variable in cluster CTA `rank` (DSMEM)
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm100 encoding):
// start>>4 | LBO(16B)=1 <<16 | SBO(1024B)=64 <<32 | version 1 <<46 | layout 2 <<61
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TC_STAMP(k) \
    do {            \
        if (a.trace) a.trace[blockIdx.x * 16 + (k)] = gtimer(); \
    } while (0)

__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

struct TcArgs;

// ---------------------------------------------------------------- tcgen05 GEMM
constexpr int kTileN = 128;   // weight rows per tile (MMA M)
constexpr int kBK = 64;       // bf16 K per stage = one 128-byte swizzle atom
// NG epilogue groups of four warps (each group covers the 128 TMEM lanes =
// tile rows; group g drains token chunks g, g+NG, ...), then the TMA
// producer warp and the MMA issuer warp.  Wide tiles (Mpad > 16) use NG = 2:
// their epilogues are bound by the math of 4 warps; narrow ones NG = 1 (two
// CTAs per SM must fit the register file).
constexpr int kGroupThreads = 128;
constexpr int kXchLd = 136;   // row stride (floats) of an epilogue group's [16][128] exchange buffer
template <int NG>
struct Roles {
    static constexpr int kEpiThreads = NG * kGroupThreads;
    static constexpr int kProdWarp = NG * 4, kMmaWarp = NG * 4 + 1;
    static constexpr int kThreads = NG * kGroupThreads + 64;
};

struct TcArgs {
    int N, K, kb_total, n_tiles, splits, items, Mpad, stages, tmem_cols, n_acc_buf;
    const int32_t* dM;
    const uint8_t* w_tiled;   // non-null: [n_tiles][kb_total][128 x 128 B] pre-swizzled blocks
    int epi;
    int bulk_pieces;   // bulk copies per 16 KB weight stage (tuning)
    int cluster;      // == splits: split-K over a thread-block cluster, DSMEM reduction
    float* out_f32;
    __nv_bfloat16* out_bf16;
    const float* bias;
    int ldo;
    unsigned long long* trace;   // optional [grid][16] %globaltimer stamps (tuning)
    // consumer-side RMSNorm (the norm weight is folded into W): out = acc *
    // rsqrt(sum_p ssq_in[p][off + m] * inv_h + eps) + bias, X = bf16 residual
    const float* ssq_in;
    int ssq_parts, ssq_ld;
    float norm_eps, inv_h;
    const int32_t* x_row_off;   // device: first X row of this GEMM (lm_head output rows)
    // producer side (RESID): bf16 copy of the new residual and its per-16-column sum of squares
    float* ssq_out;
    __nv_bfloat16* xb_out;
    // QKV epilogue: RoPE on q/k, q * qscale -> q_out (fp32), k/v -> KV cache slots (bf16)
    const int32_t* pos;
    const int32_t* slot;
    const float* cos_t;
    const float* sin_t;
    float* q_out;
    __nv_bfloat16* k_cache;
    __nv_bfloat16* v_cache;
    int nh, nkv, hd;
    float qscale;
    // lm_head (EPI_STORE_F32 / EPI_TOPK): k-gram logit bias of output row m,
    // vocab id n (card_linear_fuse_kgram); off when kg.sharp == 0
    KgBias kg;
    // EPI_TOPK: vocab size (rows >= V are padding) and 1 / temperature
    int topk_V;
    float inv_temp;
};

// sum over the 16 lanes of a half-warp (all 32 lanes must call)
__device__ __forceinline__ float half_warp_sum(float v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Epilogue for one 16-column chunk (tokens m0..m0+mc) of output row n_glob.
// All loads of a chunk are issued before any store so they overlap.  xch is
// the shared-memory address of a [16][64] fp32 exchange buffer (SwiGLU).
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
template <int EPI>
__device__ __forceinline__ void epi_chunk(const TcArgs& a, int tile, int n_glob, int n_local, int m0, int mc,
                                          float* v, uint32_t xch, const float* invs, const int* tpos,
                                          const int* tslot, float* xch_ptr, int gbar, const uint64_t* kgs) {
    const float b = a.bias ? a.bias[n_glob] : 0.f;
    if (a.ssq_in)
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] *= invs[m0 + j];
    if (EPI == EPI_QKV_ROPE) {
        // pair partner row n_local +- hd/2 of the same head, through xch [16][128]
#pragma unroll
        for (int j = 0; j < 16; ++j) sts_f32(xch + (uint32_t)((j * 128 + n_local) * 4), v[j] + b);
        named_bar(gbar, kGroupThreads);
        const int half = a.hd >> 1;
        const int head = n_glob / a.hd, i = n_glob - head * a.hd;
        if (i < half) {   // the first-half thread of each pair stores both
            float o[16], cs[16], sn[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                o[j] = lds_f32(xch + (uint32_t)((j * 128 + n_local + half) * 4));
                cs[j] = sn[j] = 0.f;
                if (head < a.nh + a.nkv && j < mc) {   // all table loads in flight at once
                    const int64_t pi = (int64_t)tpos[m0 + j] * half + i;
                    cs[j] = a.cos_t[pi];
                    sn[j] = a.sin_t[pi];
                }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j >= mc) break;
                const int m = m0 + j;
                const float x1 = v[j] + b, x2 = o[j];
                if (head < a.nh + a.nkv) {
                    const float o1 = x1 * cs[j] - x2 * sn[j], o2 = x2 * cs[j] + x1 * sn[j];
                    if (head < a.nh) {
                        float* qr = a.q_out + ((int64_t)m * a.nh + head) * a.hd;
                        qr[i] = o1 * a.qscale;
                        qr[i + half] = o2 * a.qscale;
                    } else {
                        __nv_bfloat16* kr = a.k_cache + ((int64_t)tslot[m] * a.nkv + (head - a.nh)) * a.hd;
                        kr[i] = __float2bfloat16(o1);
                        kr[i + half] = __float2bfloat16(o2);
                    }
                } else {
                    __nv_bfloat16* vr = a.v_cache + ((int64_t)tslot[m] * a.nkv + (head - a.nh - a.nkv)) * a.hd;
                    vr[i] = __float2bfloat16(x1);
                    vr[i + half] = __float2bfloat16(x2);
                }
            }
        }
        named_bar(gbar, kGroupThreads);
        return;
    }
    if (EPI == EPI_SWIGLU_BF16) {
        // rows 32q..32q+15 of a tile are the gates of features 16q..16q+15,
        // rows 32q+16..32q+31 the matching ups (interleave_gate_up), so warp q
        // holds both halves of its 16 features: lanes l and l^16 swap halves
        // of the chunk with one shuffle per token pair.  The gate lane
        // finishes tokens 0..7, the up lane tokens 8..15 of feature
        // 16q + (l & 15); each store instruction writes two 32-byte rows.
        const int lane = n_local & 31;
        const bool up = lane >= 16;
        const int f = tile * 64 + (n_local >> 5) * 16 + (lane & 15);
        const int jb = up ? 8 : 0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const float lo = v[jj] + b, hi = v[8 + jj] + b;   // static indices: v stays in registers
            const float mine = up ? hi : lo;
            const float other = __shfl_xor_sync(0xffffffffu, up ? lo : hi, 16);
            const float g = up ? other : mine;
            const float u = up ? mine : other;
            if (jb + jj < mc) a.out_bf16[(int64_t)(m0 + jb + jj) * a.ldo + f] = __float2bfloat16(silu(g) * u);
        }
        return;
    }
    if (EPI == EPI_TOPK) {
        // the group's 16-token x 128-vocab chunk, transposed through xch
        // ([16][128] fp32): 8 threads per token each scan 16 vocab rows
        // (online max / sum-exp and a sorted top-4 by (value desc, token asc)),
        // then merge over the 8 lanes; lane 0 writes the (row, tile) record
        // that card_lmhead_topk_merge combines over the tiles.
        const bool live = n_glob < a.topk_V;
        const uint64_t step = (uint64_t)(n_glob + 1) * kGamma;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            float x = v[j] + b;
            if (a.kg.sharp != 0.f && j < mc)   // (the second stream's state only when it is mixed in)
                x = kg_apply_step(a.kg, x, step, kgs[2 * (m0 + j)], a.kg.mixw != 0.f ? kgs[2 * (m0 + j) + 1] : 0ull);
            sts_f32(xch + (uint32_t)((j * kXchLd + n_local) * 4), (live && j < mc) ? x * a.inv_temp : -INFINITY);
        }
        named_bar(gbar, kGroupThreads);
        const int jt = n_local >> 3, sub = n_local & 7;
        float mx = -INFINITY, sum = 0.f;
        float tv[kTopkKT];
        int tt[kTopkKT];
#pragma unroll
        for (int q = 0; q < kTopkKT; ++q) {
            tv[q] = -INFINITY;
            tt[q] = 0x7fffffff;
        }
        auto insert = [&](float cv, int ci) {   // branch-free sorted insertion
#pragma unroll
            for (int q = 0; q < kTopkKT; ++q) {
                const bool bt = cv > tv[q] || (cv == tv[q] && ci < tt[q]);
                const float ov = tv[q];
                const int oi = tt[q];
                tv[q] = bt ? cv : ov;
                tt[q] = bt ? ci : oi;
                cv = bt ? ov : cv;
                ci = bt ? oi : ci;
            }
        };
        // The tile's top-4 are all >= T, the 4th largest of the 8 lanes'
        // maxima (those are 4 distinct elements), so each lane inserts only
        // its elements >= T (a handful per tile).  The sum-exp is taken
        // against the tile max directly (no rescaling chain).
        // element q of this lane: vocab row sub + 8 q of token jt (rows of
        // kXchLd = 136 floats: the warp's 4 tokens x 8 lanes hit 32 banks)
        const uint32_t rbase = xch + (uint32_t)((jt * kXchLd + sub) * 4);
        float xs[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) xs[q] = lds_f32(rbase + (uint32_t)(q * 32));
        float lm = xs[0];
#pragma unroll
        for (int q = 1; q < 16; ++q) lm = fmaxf(lm, xs[q]);
        float tmx = lm;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) tmx = fmaxf(tmx, __shfl_xor_sync(0xffffffffu, tmx, o));
        // exp(-inf - m) = +0 adds nothing; a chunk of padding rows only (tmx
        // = -inf) subtracts 0 instead, so no element needs the -inf test
        const float tsub = tmx == -INFINITY ? 0.f : tmx;
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) s += __expf(xs[q] - tsub);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        mx = tmx;
        sum = s;
        // rank of this lane's max among the 8 (ties: lower lane first)
        int rnk = 0;
#pragma unroll
        for (int o = 1; o < 8; ++o) {
            const float om = __shfl_xor_sync(0xffffffffu, lm, o);
            rnk += (om > lm || (om == lm && (sub ^ o) < sub)) ? 1 : 0;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, rnk == kTopkKT - 1);
        const int lane_id_ = n_local & 31;
        const unsigned grpmask = 0xffu << (lane_id_ & 24);
        const int src = __ffs(hit & grpmask) - 1;
        const float T = __shfl_sync(0xffffffffu, lm, src);
        // a handful of candidates: walk their mask (a predicated insertion
        // per element would execute all 16)
        unsigned cand = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) cand |= (xs[q] >= T && xs[q] != -INFINITY) ? (1u << q) : 0u;
        while (cand) {
            const int q = __ffs(cand) - 1;
            cand &= cand - 1;
            insert(lds_f32(rbase + (uint32_t)(q * 32)), tile * kTileN + sub + 8 * q);
        }
        // merge the 8 lanes' sorted top-4 lists: per butterfly round a
        // bitonic merge (best of mine[q] vs partner[3-q], then two
        // compare-exchange layers) instead of four insertions
        static_assert(kTopkKT == 4, "bitonic top-4 merge");
        auto better = [](float av, int ai, float bv, int bi) { return av > bv || (av == bv && ai < bi); };
        auto cx = [&](int i, int j) {   // order (i, j) best first
            const bool sw = better(tv[j], tt[j], tv[i], tt[i]);
            const float fi = tv[i], fj = tv[j];
            const int ii = tt[i], ij = tt[j];
            tv[i] = sw ? fj : fi;
            tt[i] = sw ? ij : ii;
            tv[j] = sw ? fi : fj;
            tt[j] = sw ? ii : ij;
        };
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            // (q, 3 - q) pairs: both partner values are read before either
            // slot changes (fewer live registers than four at once)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const float pa = __shfl_xor_sync(0xffffffffu, tv[3 - q], o), pb = __shfl_xor_sync(0xffffffffu, tv[q], o);
                const int ia = __shfl_xor_sync(0xffffffffu, tt[3 - q], o), ib = __shfl_xor_sync(0xffffffffu, tt[q], o);
                if (better(pa, ia, tv[q], tt[q])) {
                    tv[q] = pa;
                    tt[q] = ia;
                }
                if (better(pb, ib, tv[3 - q], tt[3 - q])) {
                    tv[3 - q] = pb;
                    tt[3 - q] = ib;
                }
            }
            cx(0, 2);
            cx(1, 3);
            cx(0, 1);
            cx(2, 3);
        }
        if (sub == 0 && jt < mc) {
            float* rec = a.out_f32 + ((int64_t)(m0 + jt) * a.n_tiles + tile) * kTopkRec;
            rec[0] = mx;
            rec[1] = sum;
#pragma unroll
            for (int q = 0; q < kTopkKT; ++q) {
                rec[2 + 2 * q] = tv[q];
                rec[3 + 2 * q] = __int_as_float(tt[q]);
            }
        }
        named_bar(gbar, kGroupThreads);
        return;
    }
    if (EPI == EPI_RESID_F32) {
        float old[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) old[j] = j < mc ? a.out_f32[(int64_t)(m0 + j) * a.ldo + n_glob] : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float x = old[j] + (v[j] + b);
            if (j < mc) {
                a.out_f32[(int64_t)(m0 + j) * a.ldo + n_glob] = x;
                if (a.xb_out) a.xb_out[(int64_t)(m0 + j) * a.ldo + n_glob] = __float2bfloat16(x);
            }
            if (a.ssq_out) {   // warp-uniform: every lane of the epilogue warps takes this path
                const float sq = half_warp_sum(j < mc ? x * x : 0.f);
                if ((n_local & 15) == 0 && j < mc) a.ssq_out[(int64_t)(n_glob >> 4) * a.ssq_ld + m0 + j] = sq;
            }
        }
        return;
    }
    if (EPI == EPI_STORE_F32 && a.kg.sharp != 0.f) {
        // fused k-gram bias: the top-k / argmax readers then skip the hash
        const uint64_t step = (uint64_t)(n_glob + 1) * kGamma;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (j >= mc) break;
            a.out_f32[(int64_t)(m0 + j) * a.ldo + n_glob] =
                kg_apply_step(a.kg, v[j] + b, step, kgs[2 * (m0 + j)], kgs[2 * (m0 + j) + 1]);
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j >= mc) break;
        if (EPI == EPI_STORE_F32) a.out_f32[(int64_t)(m0 + j) * a.ldo + n_glob] = v[j] + b;
        else a.out_bf16[(int64_t)(m0 + j) * a.ldo + n_glob] = __float2bfloat16(v[j] + b);
    }
}

// CL: split-K cluster variant (one item per CTA, DSMEM reduction); else the
// persistent direct-epilogue variant.  Separate instantiations keep each
// kernel's code small (instruction-cache misses were a measurable cost).
template <int EPI, bool CL, int NG>
__global__ void __launch_bounds__(Roles<NG>::kThreads, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap tmW,
                                                               const __grid_constant__ CUtensorMap tmX, TcArgs a) {
    using R_ = Roles<NG>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B atoms
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int S = a.stages;
    const int bytesA = kTileN * kBK * 2;
    const int bytesB = a.Mpad * kBK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)S * bytesA;
    uint64_t* full = (uint64_t*)(sB + (size_t)S * bytesB);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;    // [2]
    uint64_t* tempty = tfull + 2;   // [2]
    uint64_t* rbar = tempty + 2;    // split-K: every rank's slice of my rows landed (bulk DSMEM copies)
    uint32_t* tmem_slot = (uint32_t*)(rbar + 2);
    float* xch = (float*)(tmem_slot + 4);   // [groups][16][kXchLd] (group 1's only when Mpad > 16)
    float* invs = xch + NG * 16 * kXchLd;   // [256] per-token rsqrt(mean x^2 + eps)
    int* tpos = (int*)(invs + 256);          // [256] QKV: RoPE position of each token row
    int* tslot = tpos + 256;                 // [256] QKV: KV-cache slot of each token row
    uint64_t* kgs = (uint64_t*)(tslot + 256);   // [256][2] lm_head: k-gram stream state of each output row

    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) TC_STAMP(0);
    if (warp == R_::kProdWarp && lane == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], R_::kEpiThreads / 32);
        }
        mbar_init(rbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
    }
    // Weights do not depend on the previous kernel: the producer streams the
    // first pipeline stages of weights before the TMEM allocation (which may
    // wait for a co-resident CTA of the previous GEMM) and the grid dependency.
    int pre = 0;
    if (warp == R_::kProdWarp && lane == 0 && a.w_tiled) {
        const int item = blockIdx.x;
        if (item < a.items) {
            const int tile = item / a.splits, split = item % a.splits;
            const int kb0 = (int)((int64_t)a.kb_total * split / a.splits);
            const int kb1 = (int)((int64_t)a.kb_total * (split + 1) / a.splits);
            pre = (kb1 - kb0) < a.stages ? (kb1 - kb0) : a.stages;
#pragma unroll 1
            for (int i = 0; i < pre; ++i) {
                mbar_expect_tx(&full[i], bytesA + bytesB);
                bulk_load_split(sA + (size_t)i * bytesA, a.w_tiled + ((size_t)tile * a.kb_total + kb0 + i) * (size_t)bytesA,
                                bytesA, &full[i], a.bulk_pieces);
            }
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) TC_STAMP(1);
    const int M = *a.dM;
    const int xoff = a.x_row_off ? *a.x_row_off : 0;   // first X row (contiguous output-row range)
    const int m_rt = M < 1 ? 1 : M;
    const int n_mma = ((m_rt + 15) / 16) * 16;   // runtime MMA N (tokens), <= Mpad

    if (M <= 0) {
        // zero-row replay: drain the prefetched stages, then leave
        if (warp == R_::kProdWarp && lane == 0)
            for (int i = 0; i < pre; ++i) {
                tma_load_2d(sB + (size_t)i * bytesB, &tmX, &full[i], 0, xoff);
                mbar_wait(&full[i], 0);
            }
    } else if (warp == R_::kProdWarp) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            bool first = true;
            for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
                const int tile = item / a.splits, split = item % a.splits;
                const int kb0 = (int)((int64_t)a.kb_total * split / a.splits);
                const int kb1 = (int)((int64_t)a.kb_total * (split + 1) / a.splits);
#pragma unroll 1
                for (int kb = kb0; kb < kb1; ++kb) {
                    if (first && kb - kb0 < pre) {   // weights already in flight
                        tma_load_2d(sB + (size_t)stage * bytesB, &tmX, &full[stage], kb * kBK, xoff);
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], bytesA + bytesB);
                    if (a.w_tiled)
                        bulk_load_split(sA + (size_t)stage * bytesA,
                                        a.w_tiled + ((size_t)tile * a.kb_total + kb) * (size_t)bytesA, bytesA, &full[stage],
                                        a.bulk_pieces);
                    else
                        tma_load_2d(sA + (size_t)stage * bytesA, &tmW, &full[stage], kb * kBK, tile * kTileN);
                    tma_load_2d(sB + (size_t)stage * bytesB, &tmX, &full[stage], kb * kBK, xoff);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                first = false;
            }
        }
    } else if (warp == R_::kMmaWarp) {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n_mma >> 3) << 17) |
                                   ((uint32_t)(kTileN >> 4) << 24);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
                const int split = item % a.splits;
                const int kb0 = (int)((int64_t)a.kb_total * split / a.splits);
                const int kb1 = (int)((int64_t)a.kb_total * (split + 1) / a.splits);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * a.Mpad);
#pragma unroll 1
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    if (kb == kb0) TC_STAMP(2);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + (size_t)stage * bytesA);
                    const uint32_t b0 = smem_u32(sB + (size_t)stage * bytesB);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        tc_mma_bf16(d_tmem, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), idesc,
                                    (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    tc_commit(&empty[stage]);   // frees the smem slot when these MMAs retire
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                TC_STAMP(3);
                tc_commit(&tfull[acc]);   // accumulator ready for the epilogue
                if (a.n_acc_buf == 2) {
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                } else {
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // ---------------- epilogue warps 0..7: TMEM lane = tile row n_local
        const int grp = warp >> 2, wq = warp & 3;
        const int n_local = wq * 32 + lane;
        const int et = threadIdx.x;   // 0..255 over both groups
        if (EPI == EPI_QKV_ROPE) {
            for (int m = et; m < M; m += R_::kEpiThreads) {
                tpos[m] = a.pos[m];
                tslot[m] = a.slot[m];
            }
            if (!a.ssq_in) named_bar(1, R_::kEpiThreads);
        }
        if ((EPI == EPI_STORE_F32 || EPI == EPI_TOPK) && a.kg.sharp != 0.f) {
            for (int m = et; m < M; m += R_::kEpiThreads) kg_row_state(a.kg, m, kgs[2 * m], kgs[2 * m + 1]);
            if (!a.ssq_in) named_bar(1, R_::kEpiThreads);
        }
        if (a.ssq_in) {
            // RMSNorm scale of each token row (overlaps the main loop).  T = 8
            // lanes per token each sum a fixed slice of the partials, then a
            // fixed shuffle tree: the summation order must not depend on M, or
            // the same token would get a different scale in an M=1 AR step
            // than in an M=8 verify step (greedy CARD must equal greedy AR).
            constexpr int T = 8;
            const int t = et & (T - 1);
            const int per = (a.ssq_parts + T - 1) / T;
            const int p0 = t * per, p1 = min(a.ssq_parts, p0 + per);
            for (int mb = 0; mb * (R_::kEpiThreads / T) < M; ++mb) {   // uniform trip count (shuffles)
                const int m = mb * (R_::kEpiThreads / T) + et / T;
                float acc = 0.f;
                if (m < M) {
                    const float* src = a.ssq_in + xoff + m;
                    for (int q = p0; q < p1; q += 32) {
                        float v8[32];
#pragma unroll
                        for (int u = 0; u < 32; ++u) v8[u] = (q + u < p1) ? src[(int64_t)(q + u) * a.ssq_ld] : 0.f;
#pragma unroll
                        for (int u = 0; u < 32; ++u) acc += v8[u];
                    }
                }
                for (int o = T >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (m < M && t == 0) invs[m] = rsqrtf(acc * a.inv_h + a.norm_eps);
            }
            named_bar(1, R_::kEpiThreads);
        }
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
            const int tile = item / a.splits;
            const int n_glob = tile * kTileN + n_local;
            // epilogue warps poll politely: they must not steal issue slots
            // from the producer / MMA threads of this SM
            while (true) {
                uint32_t ok;
                asm volatile(
                    "{\n\t.reg .pred P;\n\t"
                    "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, P;\n\t}"
                    : "=r"(ok)
                    : "r"(smem_u32(&tfull[acc])), "r"(acc_phase)
                    : "memory");
                if (ok) {
                    if (threadIdx.x == 0) TC_STAMP(4);
                    break;
                }
                __nanosleep(128);
            }
            tc_fence_after();
            const uint32_t trow = tmem_base + ((uint32_t)(wq * 32) << 16) + (uint32_t)(acc * a.Mpad);
            // cluster mode (splits > 1): the accumulator stays in TMEM until
            // every rank of the cluster has finished its main loop (below)
            float* gx = xch + grp * 16 * kXchLd;
            for (int m0 = grp * 16; m0 < M && !CL; m0 += NG * 16) {
                float v[16];
                tmem_ld16(trow + (uint32_t)m0, v);
                const int mc = (M - m0) < 16 ? (M - m0) : 16;
                epi_chunk<EPI>(a, tile, n_glob, n_local, m0, mc, v, smem_u32(gx), invs, tpos, tslot, gx, 2 + grp, kgs);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (a.n_acc_buf == 2) {
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            } else {
                acc_phase ^= 1;
            }
        }
    }
    if (CL && EPI != EPI_TOPK) {   // (the top-k lm_head is never split: card_linear_create)
        // split-K over the cluster (S = a.cluster ranks = the K-slices of one
        // tile).  Tile rows are grouped in pair blocks of P rows (P = 128
        // plain, 16 SwiGLU gate/up, hd/2 RoPE): rank r owns Pp = P/S rows of
        // every P-block, so each pair (n, n + P) stays on one owner.  The
        // pipeline smem is free once the accumulator is ready; it holds
        //   recv [S][R][ld]  slice s = rank s's partial of my rows, and
        //   send [S][R][ld]  block o = my partial of owner o's rows (NG = 1).
        // Narrow tiles (NG = 1): each epilogue thread (one tile row) drains
        // TMEM into its send block with local 16-byte stores; after cluster
        // barrier 1 (every rank's recv region is free) S lanes move the
        // blocks with bulk DSMEM copies that complete_tx on the owner's rbar,
        // and the owner waits on rbar alone.  Either way the owner sums its S
        // slices in rank order (deterministic).
        const int S = a.cluster;
        const int R = kTileN / S;
        const int P = (EPI == EPI_SWIGLU_BF16) ? 16 : (EPI == EPI_QKV_ROPE) ? (a.hd >> 1) : kTileN;
        const int Pp = P / S;
        const int ld = a.Mpad + 4;   // padded slice row (floats): spreads banks
        float* buf = reinterpret_cast<float*>(smem);   // recv [S][R][ld] over the stage buffers
        float* snd = buf + kTileN * ld;                // send [S][R][ld]
        if (NG == 2) {
            // wide tiles: each epilogue thread pushes its row's partial sums
            // straight into the owner's recv slice with 16-byte
            // st.shared::cluster (overlaps the TMEM drain; a staged bulk copy
            // measured slower here, DSMEM bandwidth bounds both), then a
            // second cluster barrier publishes them
            cluster_sync_all();   // every rank's main loop done: recv regions free
            if (threadIdx.x == 0) TC_STAMP(5);
            if (warp < R_::kEpiThreads / 32 && M > 0) {
                const int me = (int)cluster_rank();
                const int grp = warp >> 2;
                const int n_local = (warp & 3) * 32 + lane;
                const int i = n_local % P, qd = n_local / P;
                const int owner = i / Pp;
                const int lr = qd * Pp + (i - owner * Pp);
                const uint32_t dst = dsmem_addr(smem_u32(buf), (uint32_t)owner) + (uint32_t)(((me * R + lr) * ld) * 4);
                const uint32_t trow = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
                for (int m0 = grp * 16; m0 < M; m0 += NG * 16) {
                    float v[16];
                    tmem_ld16(trow + (uint32_t)m0, v);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                         dst + (uint32_t)((m0 + 4 * q) * 4)),
                                     "f"(v[4 * q]), "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                                     : "memory");
                }
            }
            if (threadIdx.x == 0) TC_STAMP(6);
            cluster_sync_all();   // all pushes landed; no remote access after this point
            if (threadIdx.x == 0) TC_STAMP(7);
        } else {
            const uint32_t blk_bytes = (uint32_t)(R * ld * 4);
            const int me = (int)cluster_rank();
            if (warp < R_::kEpiThreads / 32 && M > 0) {
                if (threadIdx.x == 0) mbar_expect_tx(rbar, (uint32_t)S * blk_bytes);
                const int grp = warp >> 2;
                const int n_local = (warp & 3) * 32 + lane;
                const int i = n_local % P, qd = n_local / P;
                const int owner = i / Pp;
                const int lr = qd * Pp + (i - owner * Pp);
                const uint32_t dst = smem_u32(snd) + (uint32_t)(((owner * R + lr) * ld) * 4);
                const uint32_t trow = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
                // up to four 16-column chunks in flight per TMEM wait
                constexpr int kStep = NG * 16;
                for (int m0 = grp * 16; m0 < M; m0 += 4 * kStep) {
                    uint32_t r[4][16];
    #pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (m0 + c * kStep < M) tmem_ld16_issue(trow + (uint32_t)(m0 + c * kStep), r[c]);
                    tmem_wait_ld();
    #pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (m0 + c * kStep < M)
    #pragma unroll
                            for (int q = 0; q < 4; ++q)
                                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                                 dst + (uint32_t)((m0 + c * kStep + 4 * q) * 4)),
                                             "r"(r[c][4 * q]), "r"(r[c][4 * q + 1]), "r"(r[c][4 * q + 2]), "r"(r[c][4 * q + 3])
                                             : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // staged rows -> bulk-copy reads
            }
            cluster_sync_all();   // send blocks staged; every rank's recv region free
            if (threadIdx.x == 0) TC_STAMP(5);
            if (warp == 0 && lane < S && M > 0) {
                const uint32_t src = smem_u32(snd) + (uint32_t)lane * blk_bytes;
                const uint32_t dst = dsmem_addr(smem_u32(buf), (uint32_t)lane) + (uint32_t)me * blk_bytes;
                const uint32_t bar = dsmem_addr(smem_u32(rbar), (uint32_t)lane);
                asm volatile(
                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t"
                    "cp.async.bulk.commit_group;" ::"r"(dst),
                    "r"(src), "r"(blk_bytes), "r"(bar)
                    : "memory");
            }
            if (threadIdx.x == 0) TC_STAMP(6);
            if (warp < R_::kEpiThreads / 32 && M > 0) mbar_wait(rbar, 0);   // all S slices of my rows landed
            if (threadIdx.x == 0) TC_STAMP(7);
        }
        if (warp < R_::kEpiThreads / 32 && M > 0) {
            // owner reduction: thread -> (output j, token stripe); RJ outputs per
            // token (R rows, or R/2 pairs), TP token lanes; B tokens per pass
            // with every load issued first.
            const int r = (int)cluster_rank();
            const int tile = blockIdx.x / S;
            const uint32_t sbuf = smem_u32(buf);
            const bool paired = (EPI == EPI_SWIGLU_BF16 || EPI == EPI_QKV_ROPE);
            const int RJ = paired ? R / 2 : R;
            const int TP = R_::kEpiThreads / RJ;
            const int j = threadIdx.x % RJ, m_first = threadIdx.x / RJ;
            // local rows and tile rows of output j (pair: lr0/n0 and lr0 + Pp / n0 + P)
            int lr0, n0;
            if (paired) {
                const int qd2 = j / Pp, jj = j - qd2 * Pp;
                lr0 = 2 * qd2 * Pp + jj;
                n0 = 2 * qd2 * P + r * Pp + jj;
            } else {
                lr0 = j;
                n0 = r * R + j;
            }
            const int ng0 = tile * kTileN + n0;
            const float bias0 = a.bias ? a.bias[ng0] : 0.f;
            const float bias1 = (a.bias && paired) ? a.bias[ng0 + P] : 0.f;
            constexpr int B = 8;
            const int n_it = (M + TP * B - 1) / (TP * B);
            // QKV: this thread's pair is dims (i, i + hd/2) of one head
            const int half = a.hd >> 1;
            const int qhead = (EPI == EPI_QKV_ROPE) ? ng0 / a.hd : 0;
            const int qi = (EPI == EPI_QKV_ROPE) ? ng0 - qhead * a.hd : 0;
            float oldn[B];   // RESID: next pass's residual values, loaded one pass ahead
#pragma unroll
            for (int q = 0; q < B; ++q) {
                const int m = m_first + q * TP;
                oldn[q] = (EPI == EPI_RESID_F32 && m < M) ? a.out_f32[(int64_t)m * a.ldo + ng0] : 0.f;
            }
            for (int it = 0; it < n_it; ++it) {
                const int mb = m_first + it * TP * B;
                float v0[B], v1[B], old[B], cs[B], sn[B];
#pragma unroll
                for (int q = 0; q < B; ++q) {
                    v0[q] = 0.f;
                    v1[q] = 0.f;
                    old[q] = oldn[q];
                    const int mn = mb + TP * B + q * TP;
                    if (EPI == EPI_RESID_F32) oldn[q] = (mn < M) ? a.out_f32[(int64_t)mn * a.ldo + ng0] : 0.f;
                    const int m = mb + q * TP;
                    if (EPI == EPI_QKV_ROPE && qhead < a.nh + a.nkv && m < M) {
                        const int64_t pi = (int64_t)tpos[m] * half + qi;
                        cs[q] = a.cos_t[pi];
                        sn[q] = a.sin_t[pi];
                    }
                }
                if (it == 0 && threadIdx.x == 0) TC_STAMP(9);
                for (int sl = 0; sl < S; ++sl) {
                    const uint32_t row0 = sbuf + (uint32_t)(((sl * R + lr0) * ld) * 4);
                    const uint32_t row1 = sbuf + (uint32_t)(((sl * R + lr0 + Pp) * ld) * 4);
#pragma unroll
                    for (int q = 0; q < B; ++q) {
                        const int m = mb + q * TP;
                        if (m < M) {
                            v0[q] += lds_f32(row0 + (uint32_t)(m * 4));
                            if (paired) v1[q] += lds_f32(row1 + (uint32_t)(m * 4));
                        }
                    }
                }
                if (it == 0 && threadIdx.x == 0) TC_STAMP(10);
#pragma unroll
                for (int q = 0; q < B; ++q) {
                    const int m = mb + q * TP;
                    if (m >= M) continue;
                    const float sc = a.ssq_in ? invs[m] : 1.f;
                    const float x = v0[q] * sc + bias0;
                    if (EPI == EPI_SWIGLU_BF16) {
                        a.out_bf16[(int64_t)m * a.ldo + tile * 64 + (n0 >> 5) * 16 + (n0 & 15)] =
                            __float2bfloat16(silu(x) * (v1[q] * sc + bias1));
                    } else if (EPI == EPI_QKV_ROPE) {
                        const float x2 = v1[q] * sc + bias1;
                        if (qhead < a.nh + a.nkv) {
                            const float o1 = x * cs[q] - x2 * sn[q], o2 = x2 * cs[q] + x * sn[q];
                            if (qhead < a.nh) {
                                float* qr = a.q_out + ((int64_t)m * a.nh + qhead) * a.hd;
                                qr[qi] = o1 * a.qscale;
                                qr[qi + half] = o2 * a.qscale;
                            } else {
                                __nv_bfloat16* kr = a.k_cache + ((int64_t)tslot[m] * a.nkv + (qhead - a.nh)) * a.hd;
                                kr[qi] = __float2bfloat16(o1);
                                kr[qi + half] = __float2bfloat16(o2);
                            }
                        } else {
                            __nv_bfloat16* vr = a.v_cache + ((int64_t)tslot[m] * a.nkv + (qhead - a.nh - a.nkv)) * a.hd;
                            vr[qi] = __float2bfloat16(x);
                            vr[qi + half] = __float2bfloat16(x2);
                        }
                    } else if (EPI == EPI_STORE_F32) {
                        a.out_f32[(int64_t)m * a.ldo + ng0] =
                            a.kg.sharp != 0.f ? kg_apply_step(a.kg, x, (uint64_t)(ng0 + 1) * kGamma, kgs[2 * m], kgs[2 * m + 1])
                                              : x;
                    } else if (EPI == EPI_RESID_F32) {
                        const float xn = old[q] + x;
                        a.out_f32[(int64_t)m * a.ldo + ng0] = xn;
                        if (a.xb_out) a.xb_out[(int64_t)m * a.ldo + ng0] = __float2bfloat16(xn);
                        // x_new^2 in place of this thread's own slice-0 element (read above)
                        if (a.ssq_out) sts_f32(sbuf + (uint32_t)((lr0 * ld + m) * 4), xn * xn);
                    } else {
                        a.out_bf16[(int64_t)m * a.ldo + ng0] = __float2bfloat16(x);
                    }
                }
            }
            if (EPI == EPI_RESID_F32 && a.ssq_out) {
                // per-16-column sums of squares, fixed order, from slice 0
                named_bar(1, R_::kEpiThreads);
                const int G16 = R / 16;
                for (int e = threadIdx.x; e < G16 * M; e += R_::kEpiThreads) {
                    const int gi = e / M, m = e - gi * M;
                    float t = 0.f;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) t += lds_f32(sbuf + (uint32_t)(((gi * 16 + jj) * ld + m) * 4));
                    a.ssq_out[(int64_t)((tile * kTileN + r * R) / 16 + gi) * a.ssq_ld + m] = t;
                }
            }
        }
    }
    if (threadIdx.x == 0) TC_STAMP(8);
    // the send blocks must stay intact until the bulk copies have read them
    if (CL && NG == 1 && warp == 0 && lane < a.cluster && M > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(a.tmem_cols));
    }
}

template <int EPI>
__device__ __forceinline__ void epi_store(const TcArgs& a, int n_glob, int n_local, int m, float v, float* xch) {
    if (a.bias) v += a.bias[n_glob];
    if (EPI == EPI_STORE_F32) {
        a.out_f32[(int64_t)m * a.ldo + n_glob] = v;
    } else if (EPI == EPI_RESID_F32) {
        float* p = a.out_f32 + (int64_t)m * a.ldo + n_glob;
        *p = *p + v;
    } else if (EPI == EPI_STORE_BF16) {
        a.out_bf16[(int64_t)m * a.ldo + n_glob] = __float2bfloat16(v);
    }
}

// ---------------------------------------------------------------- M == 1 GEMV (bf16)
// One warp per 2 output rows; each lane streams 16-byte chunks (8 bf16) of
// the weight rows with ld.global.nc.L1::no_allocate, x cached in smem.
template <int EPI>
__global__ void __launch_bounds__(256) gemv_bf16_kernel(const __nv_bfloat16* __restrict__ W,
                                                        const __nv_bfloat16* __restrict__ X, int N, int K,
                                                        TcArgs a) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    if (*a.dM <= 0) return;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __nv_bfloat16* xs = (__nv_bfloat16*)smem_raw;
    for (int i = threadIdx.x * 8; i < K; i += blockDim.x * 8) *(uint4*)(xs + i) = *(const uint4*)(X + i);
    __syncthreads();
    const int warps = blockDim.x >> 5;
    const int lane = lane_id();
    constexpr int R = 2;
    for (int row0 = (blockIdx.x * warps + warp_id()) * R; row0 < N; row0 += gridDim.x * warps * R) {
        float acc[R] = {0.f, 0.f};
        const uint4* wr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) wr[r] = (const uint4*)(W + (int64_t)min(row0 + r, N - 1) * K);
        const int chunks = K / 8;
#pragma unroll 4
        for (int c = lane; c < chunks; c += 32) {
            const uint4 xv = *(const uint4*)(xs + c * 8);
            const __nv_bfloat162* xp = (const __nv_bfloat162*)&xv;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                uint4 wv;
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(wv.x), "=r"(wv.y), "=r"(wv.z), "=r"(wv.w)
                             : "l"(wr[r] + c));
                const __nv_bfloat162* wp = (const __nv_bfloat162*)&wv;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 wf = __bfloat1622float2(wp[j]);
                    const float2 xf = __bfloat1622float2(xp[j]);
                    acc[r] = fmaf(wf.x, xf.x, acc[r]);
                    acc[r] = fmaf(wf.y, xf.y, acc[r]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float v = acc[r];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[r] = v;
        }
        if (lane == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int n = row0 + r;
                if (n >= N) continue;
                if (EPI == EPI_SWIGLU_BF16) {
                    // interleaved rows: partner of gate row n is n + 16 (same 32-row block)
                    continue;
                }
                epi_store<EPI>(a, n, 0, 0, acc[r], nullptr);
            }
        }
    }
}

// SwiGLU for the GEMV path: rows are computed into a scratch fp32 buffer
// first (EPI_STORE_F32), then combined here.
__global__ void swiglu_from_rows_kernel(const float* __restrict__ rows, const int32_t* dM, int N, __nv_bfloat16* out,
                                        int ldo) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int M = *dM < 1 ? 0 : 1;
    const int F = N / 2;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < M * F; idx += gridDim.x * blockDim.x) {
        const int m = idx / F, f = idx % F;
        const int blk = f / 16, j = f % 16;   // 16 gate rows, then the 16 matching up rows
        const float g = rows[(int64_t)m * N + blk * 32 + j];
        const float u = rows[(int64_t)m * N + blk * 32 + 16 + j];
        out[(int64_t)m * ldo + f] = __float2bfloat16(silu(g) * u);
    }
}

// ---------------------------------------------------------------- fp32 parity GEMM
// One warp per output column n; lanes stride K; rows of X reused from L1.
template <int EPI>
__global__ void __launch_bounds__(256) f32_gemm_kernel(const float* __restrict__ W, const float* __restrict__ X,
                                                       int N, int K, TcArgs a) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int M = *a.dM;
    const int lane = lane_id();
    const int n = blockIdx.x * (blockDim.x >> 5) + warp_id();
    if (n >= N) return;
    const float* w = W + (int64_t)n * K;
    for (int m = 0; m < M; ++m) {
        const float* x = X + (int64_t)m * K;
        float acc = 0.f;
        for (int k = lane; k < K; k += 32) acc = fmaf(w[k], x[k], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            if (EPI == EPI_SWIGLU_BF16 || EPI == EPI_STORE_BF16) {
                a.out_f32[(int64_t)m * a.ldo + n] = acc + (a.bias ? a.bias[n] : 0.f);   // f32 mode stores f32
            } else {
                epi_store<EPI>(a, n, 0, m, acc, nullptr);
            }
        }
    }
}

__global__ void swiglu_f32_kernel(const float* __restrict__ rows, const int32_t* dM, int N, float* out, int ldo) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int M = *dM;
    const int F = N / 2;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < M * F; idx += gridDim.x * blockDim.x) {
        const int m = idx / F, f = idx % F;
        const int blk = f / 16, j = f % 16;   // 16 gate rows, then the 16 matching up rows
        const float g = rows[(int64_t)m * N + blk * 32 + j];
        const float u = rows[(int64_t)m * N + blk * 32 + 16 + j];
        out[(int64_t)m * ldo + f] = (g / (1.0f + expf(-g))) * u;
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

static int make_map_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                         CUtensorMapL2promotion promo) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return CARD_E_CUDA;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? CARD_OK : CARD_E_CUDA;
}

static int g_num_sms = 0;
static int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

}  // namespace card

struct card_linear {
    int kind;   // 0 tc_gemm, 1 gemv, 2 f32
    int epi;
    int N, K, Mpad;
    const void* W;
    const void* X;
    CUtensorMap tmW, tmX;
    card::TcArgs args;
    int grid, smem;
    float* scratch;   // gemv swiglu rows
};

namespace card {

// The attribute is per kernel, not per plan: always allow the full 227 KB so
// plans of different Mpad (hence smem) can share one template instance.
template <int EPI, int NG>
static void set_tc_attr_ng() {
    cudaFuncSetAttribute(tc_gemm_kernel<EPI, true, NG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(tc_gemm_kernel<EPI, true, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(tc_gemm_kernel<EPI, false, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}
template <int EPI>
static cudaError_t set_tc_attr(int smem) {
    (void)smem;
    set_tc_attr_ng<EPI, 1>();
    set_tc_attr_ng<EPI, 2>();
    if constexpr (EPI == EPI_TOPK)
        cudaFuncSetAttribute(tc_gemm_kernel<EPI_TOPK, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
    return cudaGetLastError();
}
// epilogue groups of a plan: the fused top-k lm_head's per-element work
// (bias hash, sum-exp, top-4 insertion) needs four groups to hide under the
// wide tile's weight stream; other wide epilogues two; narrow tiles one
static int epi_groups(int epi, int Mpad) { return Mpad > 16 ? (epi == EPI_TOPK ? 4 : 2) : 1; }

template <int EPI>
static cudaError_t launch_tc(const card_linear* h, const TcArgs& a, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    const int ng = epi_groups(EPI, a.Mpad);
    cfg.gridDim = dim3(h->grid);
    cfg.blockDim = dim3(ng == 4 ? Roles<4>::kThreads : ng == 2 ? Roles<2>::kThreads : Roles<1>::kThreads);
    cfg.dynamicSmemBytes = h->smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    int n = 1;
    if (a.cluster > 1) {
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = a.cluster;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        n = 2;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    if constexpr (EPI == EPI_TOPK)
        if (ng == 4) return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<EPI_TOPK, false, 4>, h->tmW, h->tmX, a);
    if (ng == 2) {
        if (a.cluster > 1) return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<EPI, true, 2>, h->tmW, h->tmX, a);
        return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<EPI, false, 2>, h->tmW, h->tmX, a);
    }
    if (a.cluster > 1) return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<EPI, true, 1>, h->tmW, h->tmX, a);
    return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<EPI, false, 1>, h->tmW, h->tmX, a);
}

// Cluster split-K choice.  Wide N (>= half the resident CTA slots in
// tiles): S = 1, persistent CTAs walk whole tiles.  Otherwise the K range of
// each tile is split over S in {2, 4, 8} cluster ranks (S divides the 128
// tile rows for the DSMEM reduction), the largest S such that every cluster
// is resident at once (one wave) and the [128][Mpad+4] fp32 reduction
// buffer fits in the freed pipeline stages.
template <int EPI>
static int choose_cluster(int n_tiles, int kb_total, int Mpad, int slots, int smem, int stage_smem, int ctas_per_sm) {
    if (2 * n_tiles > slots) return 1;
    int S = 8;
    const size_t red_bytes = (Mpad > 16 ? 1 : 2) * (size_t)kTileN * (Mpad + 4) * 4;   // recv (+ send) regions
    while (S > 1 && (n_tiles * S > slots || S > kb_total || red_bytes > (size_t)stage_smem))
        S >>= 1;
    // cudaOccupancyMaxActiveClusters counts one CTA per SM for this kernel even
    // when two fit (measured: 33 clusters of 4 at 105 KB and at 209 KB); with
    // two CTAs per SM the slot count above is the better bound (the verify
    // forward is 5% faster with S = 4 / 8 than with the API's S = 2 / 4)
    if (ctas_per_sm >= 2) return S;
    while (S > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n_tiles * S);
        cfg.blockDim = dim3(Mpad > 16 ? Roles<2>::kThreads : Roles<1>::kThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = S;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int nc = 0;
        const cudaError_t oe = Mpad > 16 ? cudaOccupancyMaxActiveClusters(&nc, tc_gemm_kernel<EPI, true, 2>, &cfg)
                                         : cudaOccupancyMaxActiveClusters(&nc, tc_gemm_kernel<EPI, true, 1>, &cfg);
        if (oe == cudaSuccess && nc >= n_tiles) break;
        cudaGetLastError();
        S >>= 1;
    }
    return S < 1 ? 1 : S;
}

}  // namespace card

using namespace card;

extern "C" {

int card_linear_create(const void* W, int N, int K, int wdtype, const void* X, int m_max, int epi, void* out,
                       int ldo, const float* bias, card_linear** out_h) {
    if (!out_h || !W || !X || N <= 0 || K <= 0 || m_max <= 0) return CARD_E_INPUT;
    *out_h = nullptr;
    card_linear* h = (card_linear*)calloc(1, sizeof(card_linear));
    h->epi = epi;
    h->N = N;
    h->K = K;
    h->W = W;
    h->X = X;
    TcArgs& a = h->args;
    a.N = N;
    a.K = K;
    a.epi = epi;
    a.bias = bias;
    a.ldo = ldo;
    if (epi == EPI_STORE_BF16 || epi == EPI_SWIGLU_BF16) a.out_bf16 = (__nv_bfloat16*)out;
    else a.out_f32 = (float*)out;
    const bool tiled = (wdtype == 2);
    if (tiled) a.w_tiled = (const uint8_t*)W;
    a.topk_V = N;
    a.inv_temp = 1.f;
    if (epi == EPI_TOPK && !tiled) {   // tcgen05 path only (pre-tiled bf16 weights)
        free(h);
        return CARD_E_CONFIG;
    }
    if (wdtype == 1) {   // fp32 parity path
        h->kind = 2;
        a.out_f32 = (float*)out;
        if (epi == EPI_SWIGLU_BF16) {
            CARD_CUDA_TRY(cudaMalloc(&h->scratch, (size_t)m_max * N * 4));
            a.out_f32 = h->scratch;
            a.ldo = N;
            h->args.out_bf16 = (__nv_bfloat16*)out;   // swiglu target (f32 buffer in f32 mode)
        }
        h->grid = (N + 7) / 8;
        *out_h = h;
        return CARD_OK;
    }
    if (K % kBK != 0 || N % kTileN != 0) {
        free(h);
        return CARD_E_CONFIG;
    }
    if (m_max == 1 && !tiled) {   // decode GEMV over row-major weights
        h->kind = 1;
        if (epi == EPI_SWIGLU_BF16) {
            CARD_CUDA_TRY(cudaMalloc(&h->scratch, (size_t)N * 4));
            a.out_f32 = h->scratch;
            a.ldo = N;
            h->args.out_bf16 = (__nv_bfloat16*)out;
        }
        h->smem = K * 2;
        if (h->smem > 48 * 1024) {
            cudaFuncSetAttribute(gemv_bf16_kernel<EPI_STORE_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            cudaFuncSetAttribute(gemv_bf16_kernel<EPI_RESID_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            cudaFuncSetAttribute(gemv_bf16_kernel<EPI_STORE_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        }
        h->grid = num_sms() * 4;
        *out_h = h;
        return CARD_OK;
    }
    h->kind = 0;
    const int Mpad = ((m_max + 15) / 16) * 16;
    if (Mpad > 256) {
        free(h);
        return CARD_E_CONFIG;
    }
    h->Mpad = Mpad;
    a.Mpad = Mpad;
    a.n_tiles = N / kTileN;
    a.kb_total = K / kBK;
    // TMEM: double-buffered accumulator when two of them fit in 256 columns
    a.n_acc_buf = (2 * Mpad <= 256) ? 2 : 1;
    int cols = 32;
    while (cols < a.n_acc_buf * Mpad) cols <<= 1;
    a.tmem_cols = cols;
    // Mpad >= 64: stages are 32-48 KB (weights + a wide activation tile), so
    // bytes in flight per SM, not CTA count, bound the stream: one CTA per SM
    // with the whole shared memory as its ring (measured 0.3 ms faster per
    // draft forward than two CTAs with half the ring each).
    int ctas_per_sm = (cols <= 256 && Mpad < 64) ? 2 : 1;
    const int stage_bytes = kTileN * kBK * 2 + Mpad * kBK * 2;
    int budget = (ctas_per_sm == 2 ? 110 : 220) * 1024;
    const int extra = 1024 + 64 * 8 + epi_groups(epi, Mpad) * 16 * kXchLd * 4 + 3 * 256 * 4 + 2 * 256 * 8 + 64;
    int stages = (budget - extra) / stage_bytes;
    if (stages > 8) stages = 8;
    if (stages < 2) stages = 2;
    a.stages = stages;
    a.bulk_pieces = 1;   // one 16 KB bulk copy per stage (2-8 pieces measured slower)
    h->smem = stages * stage_bytes + extra;
    const int slots = num_sms() * ctas_per_sm;
    cudaError_t e;
    switch (epi) {
        case EPI_STORE_F32: e = set_tc_attr<EPI_STORE_F32>(h->smem); break;
        case EPI_RESID_F32: e = set_tc_attr<EPI_RESID_F32>(h->smem); break;
        case EPI_STORE_BF16: e = set_tc_attr<EPI_STORE_BF16>(h->smem); break;
        case EPI_SWIGLU_BF16: e = set_tc_attr<EPI_SWIGLU_BF16>(h->smem); break;
        case EPI_QKV_ROPE: e = set_tc_attr<EPI_QKV_ROPE>(h->smem); break;
        case EPI_TOPK: e = set_tc_attr<EPI_TOPK>(h->smem); break;
        default: free(h); return CARD_E_CONFIG;
    }
    if (e != cudaSuccess) {
        set_cuda_error(e);
        free(h);
        return CARD_E_CUDA;
    }
    const int stage_smem = stages * stage_bytes;
    int S = 1;
    switch (epi) {
        case EPI_STORE_F32: S = choose_cluster<EPI_STORE_F32>(a.n_tiles, a.kb_total, Mpad, slots, h->smem, stage_smem, ctas_per_sm); break;
        case EPI_RESID_F32: S = choose_cluster<EPI_RESID_F32>(a.n_tiles, a.kb_total, Mpad, slots, h->smem, stage_smem, ctas_per_sm); break;
        case EPI_STORE_BF16: S = choose_cluster<EPI_STORE_BF16>(a.n_tiles, a.kb_total, Mpad, slots, h->smem, stage_smem, ctas_per_sm); break;
        case EPI_SWIGLU_BF16: S = choose_cluster<EPI_SWIGLU_BF16>(a.n_tiles, a.kb_total, Mpad, slots, h->smem, stage_smem, ctas_per_sm); break;
        case EPI_QKV_ROPE: S = choose_cluster<EPI_QKV_ROPE>(a.n_tiles, a.kb_total, Mpad, slots, h->smem, stage_smem, ctas_per_sm); break;
        case EPI_TOPK: S = 1; break;
    }
    if (S > 1 && (kTileN % S != 0 || (Mpad > 16 ? 1 : 2) * (size_t)kTileN * (Mpad + 4) * 4 > (size_t)stage_smem)) {
        free(h);
        return CARD_E_CONFIG;
    }
    a.splits = S;
    a.cluster = S;
    a.items = a.n_tiles * a.splits;
    h->grid = S > 1 ? a.items : (a.items < slots ? a.items : slots);
    int rc = tiled ? CARD_OK : make_map_bf16(&h->tmW, W, (uint64_t)N, (uint64_t)K, kTileN, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (!rc) rc = make_map_bf16(&h->tmX, X, (uint64_t)Mpad, (uint64_t)K, (uint32_t)Mpad, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
    if (rc) {
        free(h);
        return rc;
    }
    *out_h = h;
    return CARD_OK;
}

int card_linear_run(card_linear* h, const int32_t* dM, void* stream) {
    if (!h) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    TcArgs a = h->args;
    a.dM = dM;
    if (h->kind == 0) {
        cudaError_t e = cudaSuccess;
        switch (h->epi) {
            case EPI_STORE_F32: e = launch_tc<EPI_STORE_F32>(h, a, s); break;
            case EPI_RESID_F32: e = launch_tc<EPI_RESID_F32>(h, a, s); break;
            case EPI_STORE_BF16: e = launch_tc<EPI_STORE_BF16>(h, a, s); break;
            case EPI_SWIGLU_BF16: e = launch_tc<EPI_SWIGLU_BF16>(h, a, s); break;
            case EPI_QKV_ROPE: e = launch_tc<EPI_QKV_ROPE>(h, a, s); break;
            case EPI_TOPK: e = launch_tc<EPI_TOPK>(h, a, s); break;
        }
        if (e != cudaSuccess) {
            set_cuda_error(e);
            return CARD_E_CUDA;
        }
    } else if (h->kind == 1) {
        const __nv_bfloat16* W = (const __nv_bfloat16*)h->W;
        const __nv_bfloat16* X = (const __nv_bfloat16*)h->X;
        switch (h->epi) {
            case EPI_STORE_F32: CARD_PDL((gemv_bf16_kernel<EPI_STORE_F32>), dim3(h->grid), dim3(256), h->smem, s, W, X, h->N, h->K, a); break;
            case EPI_RESID_F32: CARD_PDL((gemv_bf16_kernel<EPI_RESID_F32>), dim3(h->grid), dim3(256), h->smem, s, W, X, h->N, h->K, a); break;
            case EPI_STORE_BF16: CARD_PDL((gemv_bf16_kernel<EPI_STORE_BF16>), dim3(h->grid), dim3(256), h->smem, s, W, X, h->N, h->K, a); break;
            case EPI_SWIGLU_BF16:
                CARD_PDL((gemv_bf16_kernel<EPI_STORE_F32>), dim3(h->grid), dim3(256), h->smem, s, W, X, h->N, h->K, a);
                CARD_PDL((swiglu_from_rows_kernel), dim3((h->N / 2 + 255) / 256), dim3(256), 0, s, h->scratch, dM, h->N, h->args.out_bf16,
                                                                             h->N / 2);
                break;
        }
    } else {
        const float* W = (const float*)h->W;
        const float* X = (const float*)h->X;
        switch (h->epi) {
            case EPI_STORE_F32: CARD_PDL((f32_gemm_kernel<EPI_STORE_F32>), dim3(h->grid), dim3(256), 0, s, W, X, h->N, h->K, a); break;
            case EPI_RESID_F32: CARD_PDL((f32_gemm_kernel<EPI_RESID_F32>), dim3(h->grid), dim3(256), 0, s, W, X, h->N, h->K, a); break;
            case EPI_STORE_BF16: CARD_PDL((f32_gemm_kernel<EPI_STORE_F32>), dim3(h->grid), dim3(256), 0, s, W, X, h->N, h->K, a); break;
            case EPI_SWIGLU_BF16:
                CARD_PDL((f32_gemm_kernel<EPI_STORE_F32>), dim3(h->grid), dim3(256), 0, s, W, X, h->N, h->K, a);
                CARD_PDL((swiglu_f32_kernel), dim3(256), dim3(256), 0, s, h->scratch, dM, h->N, (float*)h->args.out_bf16, h->N / 2);
                break;
        }
    }
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_linear_fuse_norm(card_linear* h, const float* ssq, int parts, int ld, float eps, int H,
                          const int32_t* x_row_off) {
    if (!h || h->kind != 0 || !ssq || parts <= 0 || H <= 0) return CARD_E_INPUT;
    if (h->epi == EPI_RESID_F32) return CARD_E_CONFIG;
    TcArgs& a = h->args;
    a.ssq_in = ssq;
    a.ssq_parts = parts;
    a.ssq_ld = ld;
    a.norm_eps = eps;
    a.inv_h = 1.0f / (float)H;
    a.x_row_off = x_row_off;
    return CARD_OK;
}

int card_linear_fuse_resid(card_linear* h, float* ssq_out, int ld, void* xb_out) {
    if (!h || h->kind != 0 || h->epi != EPI_RESID_F32) return CARD_E_INPUT;
    if (ssq_out && h->args.cluster > 1 && kTileN / h->args.cluster < 16) return CARD_E_CONFIG;
    h->args.ssq_out = ssq_out;
    h->args.ssq_ld = ld;
    h->args.xb_out = (__nv_bfloat16*)xb_out;
    return CARD_OK;
}

int card_linear_fuse_rope(card_linear* h, const int32_t* pos, const int32_t* slot, const float* cos_t,
                          const float* sin_t, int nh, int nkv, int hd, float* q_out, void* k_cache, void* v_cache) {
    if (!h || h->kind != 0 || h->epi != EPI_QKV_ROPE || !pos || !slot || !q_out || !k_cache || !v_cache)
        return CARD_E_INPUT;
    if ((hd != 64 && hd != 128) || (nh + 2 * nkv) * hd != h->N) return CARD_E_CONFIG;
    TcArgs& a = h->args;
    a.pos = pos;
    a.slot = slot;
    a.cos_t = cos_t;
    a.sin_t = sin_t;
    a.nh = nh;
    a.nkv = nkv;
    a.hd = hd;
    a.qscale = 1.0f / sqrtf((float)hd);
    a.q_out = q_out;
    a.k_cache = (__nv_bfloat16*)k_cache;
    a.v_cache = (__nv_bfloat16*)v_cache;
    return CARD_OK;
}

int card_linear_fuse_kgram(card_linear* h, const int32_t* ctx_tail, int order, int stride, uint64_t seed,
                           uint64_t seed2, float mix_weight, float sharpness) {
    if (!h || h->kind != 0 || (h->epi != EPI_STORE_F32 && h->epi != EPI_TOPK)) return CARD_E_INPUT;
    if (ctx_tail && (order < 0 || stride < order)) return CARD_E_INPUT;
    if (h->Mpad > 256) return CARD_E_CONFIG;
    h->args.kg = KgBias{ctx_tail, order, stride, seed, seed2, mix_weight, ctx_tail ? sharpness : 0.f};
    return CARD_OK;
}

int card_linear_fuse_topk(card_linear* h, int V, float inv_temp) {
    if (!h || h->kind != 0 || h->epi != EPI_TOPK || V <= 0 || V > h->N) return CARD_E_INPUT;
    h->args.topk_V = V;
    h->args.inv_temp = inv_temp;
    return CARD_OK;
}

int card_linear_trace(card_linear* h, unsigned long long* trace) {
    if (!h) return CARD_E_INPUT;
    h->args.trace = trace;
    return CARD_OK;
}

int card_linear_info(card_linear* h, int32_t* info8) {
    if (!h || !info8) return CARD_E_INPUT;
    info8[0] = h->kind;
    info8[1] = h->args.splits;
    info8[2] = h->args.stages;
    info8[3] = h->grid;
    info8[4] = h->smem;
    info8[5] = h->Mpad;
    info8[6] = h->args.tmem_cols;
    info8[7] = h->args.cluster > 1 ? -h->args.cluster : h->args.items;
    return CARD_OK;
}

int card_linear_destroy(card_linear* h) {
    if (!h) return CARD_OK;
    if (h->scratch) cudaFree(h->scratch);
    free(h);
    return CARD_OK;
}

}  // extern "C"
