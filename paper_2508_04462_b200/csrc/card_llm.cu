// card_llm.cu — transformer kernels of the draft/target forward (the
// model plug-in of lm.py:109-196, re-designed as a KV-cached GPU forward).
//
//   card_embed         token rows -> fp32 residual stream
//   card_rmsnorm       fp32 rows -> GEMM input (bf16, or fp32 in parity mode),
//                      optionally gathering a subset of rows (lm_head rows)
//   card_rope_kv       fused QKV epilogue: RoPE on q/k, q scaled by 1/sqrt(d),
//                      k/v written to the KV slots of their rows
//   card_attention     one kernel family for every row kind: row r attends
//                      prefix slots [0, plen[r]) plus n_extra[r] listed slots
//                      (tree ancestors + itself).  Causal chains (target
//                      verify, draft catch-up) use plen = pos + 1; draft tree
//                      rows use plen = committed length and list their
//                      ancestors — the tree mask of mask.py:173-217 without
//                      ever materialising it.  Split-KV partials (m, l, o)
//                      are merged by a combine kernel.
//   card_topk_logits   draft lm_head epilogue: per row top-k by (logit desc,
//                      token asc) and log-probs logit/T - logsumexp
//   card_argmax_logits target greedy: first maximum per row
#include <cuda_bf16.h>
#include <math.h>
#include <stdio.h>

#include "card_common.cuh"
#include "card_llm.h"

namespace card {

template <typename T>
__device__ __forceinline__ float ldf(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ldf<float>(const float* p, int64_t i) {
    return p[i];
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
    return __bfloat162float(p[i]);
}
template <typename T>
__device__ __forceinline__ void stf(T* p, int64_t i, float v);
template <>
__device__ __forceinline__ void stf<float>(float* p, int64_t i, float v) {
    p[i] = v;
}
template <>
__device__ __forceinline__ void stf<__nv_bfloat16>(__nv_bfloat16* p, int64_t i, float v) {
    p[i] = __float2bfloat16(v);
}

// ---------------------------------------------------------------- embedding
// xb / ssq (optional): the bf16 copy of the residual row and its per-16-column
// sums of squares, ssq[(col/16)*ssq_ld + r] — the input of the first fused-norm
// GEMM (card_linear_fuse_norm).
template <typename W>
__global__ void embed_kernel(const int32_t* __restrict__ tok, const int32_t* dM, const W* __restrict__ E, int H,
                             float* __restrict__ x, __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq,
                             int ssq_ld) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const int64_t t = tok[r];
    if (!xb) {
        for (int i = threadIdx.x; i < H; i += blockDim.x) x[(int64_t)r * H + i] = ldf(E, t * H + i);
        return;
    }
    if constexpr (sizeof(W) == 2) {   // bf16 table: 32-byte loads, the bf16 copy is the row itself
        for (int g16 = threadIdx.x; g16 < H / 16; g16 += blockDim.x) {
            const uint4* src = reinterpret_cast<const uint4*>(E + t * H + g16 * 16);
            const uint4 a[2] = {src[0], src[1]};
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(a);
            float v[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float2 f = __bfloat1622float2(h2[i]);
                v[2 * i] = f.x;
                v[2 * i + 1] = f.y;
            }
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) acc = fmaf(v[i], v[i], acc);
            float4* xd = reinterpret_cast<float4*>(x + (int64_t)r * H + g16 * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) xd[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            uint4* bd = reinterpret_cast<uint4*>(xb + (int64_t)r * H + g16 * 16);
            bd[0] = a[0];
            bd[1] = a[1];
            ssq[(int64_t)g16 * ssq_ld + r] = acc;
        }
        return;
    }
    for (int g16 = threadIdx.x; g16 < H / 16; g16 += blockDim.x) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int c = g16 * 16 + i;
            const float v = ldf(E, t * H + c);
            x[(int64_t)r * H + c] = v;
            xb[(int64_t)r * H + c] = __float2bfloat16(v);
            acc = fmaf(v, v, acc);
        }
        ssq[(int64_t)g16 * ssq_ld + r] = acc;
    }
}

// ---------------------------------------------------------------- tensor-parallel residual
// x += part (the all-reduced partial of a row-parallel o / down projection),
// then the bf16 copy and the per-16-column sums of squares the next fused
// RMSNorm consumes (what the RESID GEMM epilogue does on one GPU)
__global__ void resid_add_kernel(const int32_t* dM, int H, float* __restrict__ x, const float* __restrict__ part,
                                 __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq, int ssq_ld) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    if (r >= *dM) return;
    for (int g16 = threadIdx.x; g16 < H / 16; g16 += blockDim.x) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int64_t c = (int64_t)r * H + g16 * 16 + i;
            const float v = x[c] + part[c];
            x[c] = v;
            xb[c] = __float2bfloat16(v);
            acc = fmaf(v, v, acc);
        }
        ssq[(int64_t)g16 * ssq_ld + r] = acc;
    }
}

// Output rows of a batched forward -> one contiguous block for the lm_head
// (its activation tile reads rows [0, n_out) contiguously): row out_rows[o]
// of the bf16 residual and its per-16-column sums of squares -> row o.
__global__ void gather_rows_kernel(const int32_t* __restrict__ out_rows, const int32_t* n_out, int H,
                                   const __nv_bfloat16* __restrict__ xb, const float* __restrict__ ssq, int ssq_ld,
                                   __nv_bfloat16* __restrict__ xb_out, float* __restrict__ ssq_out, int ssq_out_ld) {
    pdl_wait();
    pdl_trigger();
    const int o = blockIdx.x;
    if (o >= *n_out) return;
    const int r = out_rows[o];
    const uint4* src = reinterpret_cast<const uint4*>(xb + (int64_t)r * H);
    uint4* dst = reinterpret_cast<uint4*>(xb_out + (int64_t)o * H);
    for (int c = threadIdx.x; c < H / 8; c += blockDim.x) dst[c] = src[c];
    for (int g = threadIdx.x; g < H / 16; g += blockDim.x) ssq_out[(int64_t)g * ssq_out_ld + o] = ssq[(int64_t)g * ssq_ld + r];
}

// ---------------------------------------------------------------- rmsnorm
template <typename Y>
__global__ void rmsnorm_kernel(const float* __restrict__ x, const float* __restrict__ w, int H, float eps,
                               const int32_t* dM, const int32_t* gather, Y* __restrict__ y) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const int src = gather ? gather[r] : r;
    const float* xr = x + (int64_t)src * H;
    __shared__ float red[32];
    float ss = 0.f;
    const bool vec = (H % 4) == 0;
    if (vec) {
        const float4* x4 = reinterpret_cast<const float4*>(xr);
        for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
            const float4 v = x4[i];
            ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
        }
    } else {
        for (int i = threadIdx.x; i < H; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
    }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane_id() == 0) red[warp_id()] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / (float)H + eps);
    if (vec) {
        const float4* x4 = reinterpret_cast<const float4*>(xr);
        const float4* w4 = reinterpret_cast<const float4*>(w);
        for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
            const float4 v = x4[i], g = w4[i];
            const int64_t o = (int64_t)r * H + 4 * i;
            stf(y, o, (v.x * inv) * g.x);
            stf(y, o + 1, (v.y * inv) * g.y);
            stf(y, o + 2, (v.z * inv) * g.z);
            stf(y, o + 3, (v.w * inv) * g.w);
        }
    } else {
        for (int i = threadIdx.x; i < H; i += blockDim.x) stf(y, (int64_t)r * H + i, (xr[i] * inv) * w[i]);
    }
}

// ---------------------------------------------------------------- rope + kv write
template <typename KV>
__global__ void rope_kv_kernel(const float* __restrict__ qkv, const int32_t* dM, const int32_t* __restrict__ pos,
                               const int32_t* __restrict__ slot, const float* __restrict__ cos_t,
                               const float* __restrict__ sin_t, int nh, int nkv, int hd, float qscale,
                               float* __restrict__ q, KV* __restrict__ kc, KV* __restrict__ vc) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const int half = hd / 2;
    const int width = (nh + 2 * nkv) * hd;
    const float* row = qkv + (int64_t)r * width;
    const int p = pos[r];
    const int64_t s = slot[r];
    const float* ct = cos_t + (int64_t)p * half;
    const float* st = sin_t + (int64_t)p * half;
    // q and k heads: rotate pairs (i, i+half) — HF rotate_half convention
    const int n_rot = (nh + nkv) * half;
    for (int idx = threadIdx.x; idx < n_rot; idx += blockDim.x) {
        const int head = idx / half, i = idx % half;
        const float x1 = row[head * hd + i], x2 = row[head * hd + i + half];
        const float c = ct[i], sn = st[i];
        const float o1 = x1 * c - x2 * sn, o2 = x2 * c + x1 * sn;
        if (head < nh) {
            q[((int64_t)r * nh + head) * hd + i] = o1 * qscale;
            q[((int64_t)r * nh + head) * hd + i + half] = o2 * qscale;
        } else {
            const int kh = head - nh;
            stf(kc, (s * nkv + kh) * hd + i, o1);
            stf(kc, (s * nkv + kh) * hd + i + half, o2);
        }
    }
    for (int idx = threadIdx.x; idx < nkv * hd; idx += blockDim.x) {
        stf(vc, s * nkv * hd + idx, row[(nh + nkv) * hd + idx]);
    }
}

// ---------------------------------------------------------------- attention
// Partials: work[((r * nh + h) * (n_splits + 1) + s) * (hd + 2)] = {m, l, o[hd]}
constexpr int kChunk = 64;

template <typename KV>
__global__ void __launch_bounds__(256) attn_prefix_kernel(const float* __restrict__ q, const int32_t* dM,
                                                          const int32_t* __restrict__ plen, const KV* __restrict__ kc,
                                                          const KV* __restrict__ vc, int nh, int nkv, int hd,
                                                          int n_splits, float* __restrict__ work) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    extern __shared__ float sm[];
    const int g = blockIdx.x;          // kv head
    const int sidx = blockIdx.y;       // split
    const int k0 = sidx * kChunk;
    const int M = *dM;
    // any row needing this chunk?
    __shared__ int need;
    if (threadIdx.x == 0) need = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < M; r += blockDim.x)
        if (plen[r] > k0) need = 1;
    __syncthreads();
    if (!need) return;
    const int ld = hd + 1;
    float* Ks = sm;                    // [kChunk][hd+1]
    float* Vs = Ks + kChunk * ld;      // [kChunk][hd+1]
    float* Qw = Vs + kChunk * ld;      // [warps][hd]
    float* Pw = Qw + (blockDim.x >> 5) * hd;   // [warps][kChunk]
    for (int idx = threadIdx.x; idx < kChunk * hd; idx += blockDim.x) {
        const int j = idx / hd, d = idx % hd;
        const int64_t s = k0 + j;
        Ks[j * ld + d] = ldf(kc, (s * nkv + g) * hd + d);
        Vs[j * ld + d] = ldf(vc, (s * nkv + g) * hd + d);
    }
    __syncthreads();
    const int G = nh / nkv;
    const int warp = warp_id(), lane = lane_id(), nw = blockDim.x >> 5;
    float* qw = Qw + warp * hd;
    float* pw = Pw + warp * kChunk;
    for (int item = warp; item < M * G; item += nw) {
        const int r = item / G, h = g * G + item % G;
        const int L = plen[r] - k0;   // valid keys in this chunk
        if (L <= 0) continue;
        const int nvalid = L < kChunk ? L : kChunk;
        const float* qr = q + ((int64_t)r * nh + h) * hd;
        for (int d = lane; d < hd; d += 32) qw[d] = qr[d];
        __syncwarp();
        float mloc = -INFINITY;
        for (int j = lane; j < kChunk; j += 32) {
            float sc = -INFINITY;
            if (j < nvalid) {
                sc = 0.f;
                const float* kr = Ks + j * ld;
                for (int d = 0; d < hd; ++d) sc = fmaf(qw[d], kr[d], sc);
            }
            pw[j] = sc;
            mloc = fmaxf(mloc, sc);
        }
        for (int o = 16; o > 0; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
        float lsum = 0.f;
        for (int j = lane; j < kChunk; j += 32) {
            const float e = (j < nvalid) ? __expf(pw[j] - mloc) : 0.f;
            pw[j] = e;
            lsum += e;
        }
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        __syncwarp();
        float* out = work + (((int64_t)r * nh + h) * (n_splits + 1) + sidx) * (hd + 2);
        for (int d = lane; d < hd; d += 32) {
            float acc = 0.f;
            for (int j = 0; j < nvalid; ++j) acc = fmaf(pw[j], Vs[j * ld + d], acc);
            out[2 + d] = acc;
        }
        if (lane == 0) {
            out[0] = mloc;
            out[1] = lsum;
        }
        __syncwarp();
    }
}


// ---------------------------------------------------------------- tensor-core prefix attention
// CTA = (kv head g, 64-key chunk).  The chunk's K (row-major) and V
// (transposed) are staged once in smem as bf16; every query (row r, head h
// in g's group) with plen[r] > chunk start is processed in tiles of 16 by
// mma.sync.m16n8k16 (bf16 in, fp32 acc): S = Q K^T, masked, exp, O = P V.
// Partials (m, l, o[hd]) go to the same workspace layout as the CUDA-core
// kernel, merged by attn_combine_kernel.
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int HD>
__global__ void __launch_bounds__(128) attn_prefix_tc_kernel(const float* __restrict__ q, const int32_t* dM,
                                                            const int32_t* __restrict__ plen,
                                                            const __nv_bfloat16* __restrict__ kc,
                                                            const __nv_bfloat16* __restrict__ vc, int nh, int nkv,
                                                            int n_splits, float* __restrict__ work) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    constexpr int CH = kChunk;          // 64 keys
    constexpr int KLD = HD + 8;         // padded K row (bf16)
    constexpr int VLD = CH + 8;         // padded V^T row (bf16)
    __shared__ __align__(16) __nv_bfloat16 Ks[CH * KLD];
    __shared__ __align__(16) __nv_bfloat16 Vt[HD * VLD];
    __shared__ int need;
    const int g = blockIdx.x, sidx = blockIdx.y, k0 = sidx * CH;
    const int M = *dM;
    if (threadIdx.x == 0) need = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < M; r += blockDim.x)
        if (plen[r] > k0) need = 1;
    __syncthreads();
    if (!need) return;
    // stage K (16-byte vectors) and V^T
    for (int idx = threadIdx.x; idx < CH * HD / 8; idx += blockDim.x) {
        const int j = idx / (HD / 8), d8 = (idx % (HD / 8)) * 8;
        const int64_t base = (((int64_t)(k0 + j)) * nkv + g) * HD + d8;
        const uint4 kv = *reinterpret_cast<const uint4*>(kc + base);
        *reinterpret_cast<uint4*>(Ks + j * KLD + d8) = kv;
        const uint4 vv = *reinterpret_cast<const uint4*>(vc + base);
        const __nv_bfloat16* ve = reinterpret_cast<const __nv_bfloat16*>(&vv);
#pragma unroll
        for (int e = 0; e < 8; ++e) Vt[(d8 + e) * VLD + j] = ve[e];
    }
    __syncthreads();
    const int G = nh / nkv;
    const int nq = M * G;
    const int lane = lane_id(), warp = warp_id();
    const int gq = lane >> 2, tq = lane & 3;
    for (int tile = warp; tile * 16 < nq; tile += blockDim.x >> 5) {
        // query rows of this tile handled by this thread: gq and gq + 8
        int qa = tile * 16 + gq, qb = qa + 8;
        const int ra = qa < nq ? qa / G : 0, rb = qb < nq ? qb / G : 0;
        const int ha = g * G + (qa % G), hb = g * G + (qb % G);
        const int la = qa < nq ? plen[ra] - k0 : 0, lb = qb < nq ? plen[rb] - k0 : 0;
        const float* qpa = q + ((int64_t)ra * nh + ha) * HD;
        const float* qpb = q + ((int64_t)rb * nh + hb) * HD;
        // S = Q K^T over HD in 16-wide slices
        float s[CH / 8][4];
#pragma unroll
        for (int n = 0; n < CH / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
            const int d0 = ks * 16 + 2 * tq;
            uint32_t a[4];
            const float2 xa0 = qa < nq ? *reinterpret_cast<const float2*>(qpa + d0) : make_float2(0.f, 0.f);
            const float2 xb0 = qb < nq ? *reinterpret_cast<const float2*>(qpb + d0) : make_float2(0.f, 0.f);
            const float2 xa1 = qa < nq ? *reinterpret_cast<const float2*>(qpa + d0 + 8) : make_float2(0.f, 0.f);
            const float2 xb1 = qb < nq ? *reinterpret_cast<const float2*>(qpb + d0 + 8) : make_float2(0.f, 0.f);
            a[0] = pack_bf16(xa0.x, xa0.y);
            a[1] = pack_bf16(xb0.x, xb0.y);
            a[2] = pack_bf16(xa1.x, xa1.y);
            a[3] = pack_bf16(xb1.x, xb1.y);
#pragma unroll
            for (int n = 0; n < CH / 8; ++n) {
                const __nv_bfloat16* kr = Ks + (n * 8 + gq) * KLD + ks * 16 + 2 * tq;
                uint32_t b[2];
                b[0] = *reinterpret_cast<const uint32_t*>(kr);
                b[1] = *reinterpret_cast<const uint32_t*>(kr + 8);
                mma_bf16_16816(s[n], a, b);
            }
        }
        // mask + row max over the 4 threads sharing a row
        float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
        for (int n = 0; n < CH / 8; ++n) {
            const int j0 = n * 8 + 2 * tq;
            if (j0 >= la) s[n][0] = -INFINITY;
            if (j0 + 1 >= la) s[n][1] = -INFINITY;
            if (j0 >= lb) s[n][2] = -INFINITY;
            if (j0 + 1 >= lb) s[n][3] = -INFINITY;
            ma = fmaxf(ma, fmaxf(s[n][0], s[n][1]));
            mb = fmaxf(mb, fmaxf(s[n][2], s[n][3]));
        }
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, 1));
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, 2));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 1));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 2));
        const float sa = ma == -INFINITY ? 0.f : ma, sb = mb == -INFINITY ? 0.f : mb;
        float suma = 0.f, sumb = 0.f;
        uint32_t p[CH / 16][4];
#pragma unroll
        for (int n = 0; n < CH / 8; ++n) {
            const float e0 = __expf(s[n][0] - sa), e1 = __expf(s[n][1] - sa);
            const float e2 = __expf(s[n][2] - sb), e3 = __expf(s[n][3] - sb);
            suma += e0 + e1;
            sumb += e2 + e3;
            // C layout of n-tile n -> A fragment of key slice n/2 (FA2 register reuse)
            if ((n & 1) == 0) {
                p[n >> 1][0] = pack_bf16(e0, e1);
                p[n >> 1][1] = pack_bf16(e2, e3);
            } else {
                p[n >> 1][2] = pack_bf16(e0, e1);
                p[n >> 1][3] = pack_bf16(e2, e3);
            }
        }
        suma += __shfl_xor_sync(0xffffffffu, suma, 1);
        suma += __shfl_xor_sync(0xffffffffu, suma, 2);
        sumb += __shfl_xor_sync(0xffffffffu, sumb, 1);
        sumb += __shfl_xor_sync(0xffffffffu, sumb, 2);
        // O = P V  (B operand from V^T rows: dims x keys)
        float* outa = work + (((int64_t)ra * nh + ha) * (n_splits + 1) + sidx) * (HD + 2);
        float* outb = work + (((int64_t)rb * nh + hb) * (n_splits + 1) + sidx) * (HD + 2);
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk) {
                const __nv_bfloat16* vr = Vt + (nd * 8 + gq) * VLD + kk * 16 + 2 * tq;
                uint32_t b[2];
                b[0] = *reinterpret_cast<const uint32_t*>(vr);
                b[1] = *reinterpret_cast<const uint32_t*>(vr + 8);
                mma_bf16_16816(o, p[kk], b);
            }
            const int dcol = nd * 8 + 2 * tq;
            if (qa < nq && la > 0) {
                outa[2 + dcol] = o[0];
                outa[2 + dcol + 1] = o[1];
            }
            if (qb < nq && lb > 0) {
                outb[2 + dcol] = o[2];
                outb[2 + dcol + 1] = o[3];
            }
        }
        if (tq == 0) {
            if (qa < nq && la > 0) {
                outa[0] = ma;
                outa[1] = suma;
            }
            if (qb < nq && lb > 0) {
                outb[0] = mb;
                outb[1] = sumb;
            }
        }
    }
}

// extra slots (tree ancestors + self): one warp per (row, head)
template <typename KV>
__global__ void attn_extra_kernel(const float* __restrict__ q, const int32_t* dM, const int32_t* __restrict__ n_extra,
                                  const int32_t* __restrict__ extra, int extra_max, const KV* __restrict__ kc,
                                  const KV* __restrict__ vc, int nh, int nkv, int hd, int n_splits,
                                  float* __restrict__ work) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int M = *dM;
    const int gw = blockIdx.x * (blockDim.x >> 5) + warp_id();
    if (gw >= M * nh) return;
    const int r = gw / nh, h = gw % nh, g = h / (nh / nkv);
    const int lane = lane_id();
    const int ne = n_extra[r];
    float* out = work + (((int64_t)r * nh + h) * (n_splits + 1) + n_splits) * (hd + 2);
    if (ne <= 0) {
        if (lane == 0) {
            out[0] = -INFINITY;
            out[1] = 0.f;
        }
        return;
    }
    const float* qr = q + ((int64_t)r * nh + h) * hd;
    float sc[32];
    float m = -INFINITY;
    for (int j = 0; j < ne && j < 32; ++j) {
        const int64_t s = extra[(int64_t)r * extra_max + j];
        float part = 0.f;
        for (int d = lane; d < hd; d += 32) part = fmaf(qr[d], ldf(kc, (s * nkv + g) * hd + d), part);
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        sc[j] = part;
        m = fmaxf(m, part);
    }
    float l = 0.f;
    for (int j = 0; j < ne && j < 32; ++j) {
        sc[j] = __expf(sc[j] - m);
        l += sc[j];
    }
    for (int d = lane; d < hd; d += 32) {
        float acc = 0.f;
        for (int j = 0; j < ne && j < 32; ++j) {
            const int64_t s = extra[(int64_t)r * extra_max + j];
            acc = fmaf(sc[j], ldf(vc, (s * nkv + g) * hd + d), acc);
        }
        out[2 + d] = acc;
    }
    if (lane == 0) {
        out[0] = m;
        out[1] = l;
    }
}

template <typename O>
__global__ void attn_combine_kernel(const int32_t* dM, const int32_t* __restrict__ plen, int nh, int hd, int n_splits,
                                    const float* __restrict__ work, O* __restrict__ o) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x, h = blockIdx.y;
    if (r >= *dM) return;
    const int ns = (plen[r] + kChunk - 1) / kChunk;
    const float* base = work + ((int64_t)r * nh + h) * (n_splits + 1) * (hd + 2);
    float M = -INFINITY;
    for (int s = 0; s < ns; ++s) M = fmaxf(M, base[s * (hd + 2)]);
    M = fmaxf(M, base[n_splits * (hd + 2)]);
    float L = 0.f;
    for (int s = 0; s < ns; ++s) L += __expf(base[s * (hd + 2)] - M) * base[s * (hd + 2) + 1];
    const float me = base[n_splits * (hd + 2)];
    const float we = (me == -INFINITY) ? 0.f : __expf(me - M);
    L += we * base[n_splits * (hd + 2) + 1];
    const float invL = 1.0f / L;
    for (int d = threadIdx.x; d < hd; d += blockDim.x) {
        float acc = 0.f;
        for (int s = 0; s < ns; ++s) acc += __expf(base[s * (hd + 2)] - M) * base[s * (hd + 2) + 2 + d];
        if (we != 0.f) acc += we * base[n_splits * (hd + 2) + 2 + d];
        stf(o, ((int64_t)r * nh + h) * hd + d, acc * invL);
    }
}

// ---------------------------------------------------------------- k-gram logit bias (agreement knob)
// logits[r][i] + sharp * (u1_i + mixw * u2_i): the splitmix64 k-gram stream of
// (seed, context tail of row r), _kernels.pyx:26-41.  Applied on the fly by
// the top-k / argmax readers (one read of the logits instead of a separate
// read-modify-write pass); same fp32 arithmetic as logit_bias_kernel.
// KgBias, kg_row_state and kg_apply live in card_common.cuh (shared with the
// lm_head GEMM epilogue, card_linear_fuse_kgram).

// ---------------------------------------------------------------- lm_head epilogues (split over the vocab)
// Stage 1: CTA (row, split) scans a vocab slice: online max / sum-exp and a
// register-resident sorted top-KT (static indices, bubble insertion).
// Stage 2: one warp per row merges the splits: fp64 log-sum-exp and top-k.
__device__ __forceinline__ bool lbefore(float a, int ta, float b, int tb) { return a > b || (a == b && ta < tb); }

template <int KT>
__global__ void __launch_bounds__(256) topk_partial_kernel(const float* __restrict__ logits, const int32_t* dM, int V,
                                                           int S, float inv_temp, float* __restrict__ work, KgBias kb) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x, sp = blockIdx.y;
    if (r >= *dM) return;
    const bool biased = kb.sharp != 0.f;
    uint64_t ks1 = 0, ks2 = 0;
    if (biased) kg_row_state(kb, r, ks1, ks2);
    auto lg = [&](float v, int i) { return biased ? kg_apply(kb, v, i, ks1, ks2) : v; };
    // split boundaries on 4-element multiples so slices stay float4-aligned
    const int lo = (int)(((int64_t)V * sp / S) & ~3LL);
    const int hi = sp == S - 1 ? V : (int)(((int64_t)V * (sp + 1) / S) & ~3LL);
    const float* lr = logits + (int64_t)r * V;
    float tv[KT];
    int tt[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        tv[j] = -INFINITY;
        tt[j] = 0x7fffffff;
    }
    float mx = -INFINITY, sum = 0.f;
    auto consume = [&](float v, int i) {
        if (v > mx) {
            sum = sum * __expf(mx - v) + 1.f;
            mx = v;
        } else {
            sum += __expf(v - mx);
        }
        if (lbefore(v, i, tv[KT - 1], tt[KT - 1])) {
            float cv = v;
            int ci = i;
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                const bool b = lbefore(cv, ci, tv[j], tt[j]);
                const float ov = tv[j];
                const int oi = tt[j];
                tv[j] = b ? cv : ov;
                tt[j] = b ? ci : oi;
                cv = b ? ov : cv;
                ci = b ? oi : ci;
            }
        }
    };
    // aligned float4 body (4 vectors in flight per thread), scalar head/tail
    int a0 = lo, a1 = hi;
    if (((uintptr_t)(lr + lo) & 15) == 0 && ((int64_t)r * V) % 4 == 0) {
        const int nv = (hi - lo) / 4;
        const float4* l4 = reinterpret_cast<const float4*>(lr + lo);
        int vi = threadIdx.x;
        for (; vi + 3 * (int)blockDim.x < nv; vi += 4 * blockDim.x) {
            float4 q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = __ldg(l4 + vi + u * blockDim.x);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = lo + 4 * (vi + u * blockDim.x);
                if (biased) {   // consecutive tokens: the stream offset steps by kGamma
                    const uint64_t st = (uint64_t)(i + 1) * kGamma;
                    consume(kg_apply_step(kb, q[u].x, st, ks1, ks2) * inv_temp, i);
                    consume(kg_apply_step(kb, q[u].y, st + kGamma, ks1, ks2) * inv_temp, i + 1);
                    consume(kg_apply_step(kb, q[u].z, st + 2 * kGamma, ks1, ks2) * inv_temp, i + 2);
                    consume(kg_apply_step(kb, q[u].w, st + 3 * kGamma, ks1, ks2) * inv_temp, i + 3);
                }
            }
            if (!biased) {
                // batch of 16: one max-rescale per batch, independent exps,
                // insertion only for values that beat the current k-th best
                float xs[16];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    xs[4 * u] = q[u].x * inv_temp;
                    xs[4 * u + 1] = q[u].y * inv_temp;
                    xs[4 * u + 2] = q[u].z * inv_temp;
                    xs[4 * u + 3] = q[u].w * inv_temp;
                }
                float bm = xs[0];
#pragma unroll
                for (int e = 1; e < 16; ++e) bm = fmaxf(bm, xs[e]);
                if (bm > mx) {
                    sum = mx == -INFINITY ? 0.f : sum * __expf(mx - bm);
                    mx = bm;
                }
                float part = 0.f;
#pragma unroll
                for (int e = 0; e < 16; ++e) part += xs[e] == -INFINITY ? 0.f : __expf(xs[e] - mx);
                sum += part;
                if (bm >= tv[KT - 1]) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int i = lo + 4 * (vi + (e >> 2) * blockDim.x) + (e & 3);
                        if (lbefore(xs[e], i, tv[KT - 1], tt[KT - 1])) {
                            float cv = xs[e];
                            int ci = i;
#pragma unroll
                            for (int j = 0; j < KT; ++j) {
                                const bool b = lbefore(cv, ci, tv[j], tt[j]);
                                const float ov = tv[j];
                                const int oi = tt[j];
                                tv[j] = b ? cv : ov;
                                tt[j] = b ? ci : oi;
                                cv = b ? ov : cv;
                                ci = b ? oi : ci;
                            }
                        }
                    }
                }
            }
        }
        for (; vi < nv; vi += blockDim.x) {
            const float4 q = __ldg(l4 + vi);
            const int i = lo + 4 * vi;
            consume(lg(q.x, i) * inv_temp, i);
            consume(lg(q.y, i + 1) * inv_temp, i + 1);
            consume(lg(q.z, i + 2) * inv_temp, i + 2);
            consume(lg(q.w, i + 3) * inv_temp, i + 3);
        }
        a0 = lo + 4 * nv;
        a1 = hi;
    }
    for (int i = a0 + threadIdx.x; i < a1; i += blockDim.x) consume(lg(lr[i], i) * inv_temp, i);
    // block reduction: max/sum then KT rounds of arg-best
    __shared__ float sm_m[8], sm_s[8], bv[8];
    __shared__ int bt[8], bw[8];
    float wm = mx;
    for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    if (lane_id() == 0) sm_m[warp_id()] = wm;
    __syncthreads();
    float gm = sm_m[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) gm = fmaxf(gm, sm_m[w]);
    float ss = mx == -INFINITY ? 0.f : sum * __expf(mx - gm);
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane_id() == 0) sm_s[warp_id()] = ss;
    __syncthreads();
    float* out = work + ((int64_t)r * S + sp) * (2 + 2 * KT);
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm_s[w];
        out[0] = gm;
        out[1] = t;
    }
    int head = 0;
    for (int round = 0; round < KT; ++round) {
        float v = -INFINITY;
        int t = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < KT; ++j)
            if (j == head) {
                v = tv[j];
                t = tt[j];
            }
        int who = threadIdx.x;
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int ot = __shfl_xor_sync(0xffffffffu, t, o);
            const int ow = __shfl_xor_sync(0xffffffffu, who, o);
            if (lbefore(ov, ot, v, t)) {
                v = ov;
                t = ot;
                who = ow;
            }
        }
        if (lane_id() == 0) {
            bv[warp_id()] = v;
            bt[warp_id()] = t;
            bw[warp_id()] = who;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (lbefore(bv[w], bt[w], bv[0], bt[0])) {
                    bv[0] = bv[w];
                    bt[0] = bt[w];
                    bw[0] = bw[w];
                }
            out[2 + 2 * round] = bv[0];
            out[3 + 2 * round] = __int_as_float(bt[0]);
        }
        __syncthreads();
        if (threadIdx.x == bw[0]) ++head;
        __syncthreads();
    }
}

template <int KT>
__global__ void topk_merge_kernel(const int32_t* dM, int S, int k, int V, const float* __restrict__ work,
                                  int32_t* __restrict__ out_tok, double* __restrict__ out_logp,
                                  int32_t* __restrict__ out_cnt) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x * (blockDim.x >> 5) + warp_id();
    if (r >= *dM) return;
    const int lane = lane_id();
    const float* base = work + (int64_t)r * S * (2 + 2 * KT);
    double gm = -INFINITY;
    for (int s = lane; s < S; s += 32) gm = fmax(gm, (double)base[s * (2 + 2 * KT)]);
    for (int o = 16; o > 0; o >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    double tot = 0.0;
    for (int s = lane; s < S; s += 32) {
        const float* p = base + s * (2 + 2 * KT);
        if (p[1] > 0.f) tot += (double)p[1] * exp((double)p[0] - gm);
    }
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const double lse = gm + log(tot);
    // candidates: S * KT, lane-strided; k rounds of warp arg-best with exclusion
    int last_t = -1;
    float last_v = INFINITY;
    for (int round = 0; round < k; ++round) {
        float v = -INFINITY;
        int t = 0x7fffffff;
        for (int c = lane; c < S * KT; c += 32) {
            const float* p = base + (c / KT) * (2 + 2 * KT) + 2 + 2 * (c % KT);
            const float cv = p[0];
            const int ct = __float_as_int(p[1]);
            // strictly after the previous pick in (value desc, token asc) order
            if (lbefore(last_v, last_t, cv, ct) && lbefore(cv, ct, v, t)) {
                v = cv;
                t = ct;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int ot = __shfl_xor_sync(0xffffffffu, t, o);
            if (lbefore(ov, ot, v, t)) {
                v = ov;
                t = ot;
            }
        }
        if (lane == 0) {
            out_tok[(int64_t)r * k + round] = t;
            out_logp[(int64_t)r * k + round] = (double)v - lse;
        }
        last_v = v;
        last_t = t;
    }
    if (lane == 0) out_cnt[r] = k < V ? k : V;
}

// greedy: first maximum per row, split over the vocab then merged
__global__ void __launch_bounds__(256) argmax_partial_kernel(const float* __restrict__ logits, const int32_t* dM,
                                                             int V, int S, float* __restrict__ work, KgBias kb) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x, sp = blockIdx.y;
    if (r >= *dM) return;
    const bool biased = kb.sharp != 0.f;
    uint64_t ks1 = 0, ks2 = 0;
    if (biased) kg_row_state(kb, r, ks1, ks2);
    // split boundaries on 4-element multiples so slices stay float4-aligned
    const int lo = (int)(((int64_t)V * sp / S) & ~3LL);
    const int hi = sp == S - 1 ? V : (int)(((int64_t)V * (sp + 1) / S) & ~3LL);
    const float* lr = logits + (int64_t)r * V;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    auto take = [&](float v, int i) {
        if (biased) v = kg_apply(kb, v, i, ks1, ks2);
        if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    };
    int a0 = lo;
    if (((uintptr_t)(lr + lo) & 15) == 0) {
        const int nv = (hi - lo) / 4;
        const float4* l4 = reinterpret_cast<const float4*>(lr + lo);
        int vi = threadIdx.x;
        for (; vi + 3 * (int)blockDim.x < nv; vi += 4 * blockDim.x) {
            float4 q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = __ldg(l4 + vi + u * blockDim.x);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = lo + 4 * (vi + u * blockDim.x);
                take(q[u].x, i);
                take(q[u].y, i + 1);
                take(q[u].z, i + 2);
                take(q[u].w, i + 3);
            }
        }
        for (; vi < nv; vi += blockDim.x) {
            const float4 q = __ldg(l4 + vi);
            const int i = lo + 4 * vi;
            take(q.x, i);
            take(q.y, i + 1);
            take(q.z, i + 2);
            take(q.w, i + 3);
        }
        a0 = lo + 4 * nv;
    }
    for (int i = a0 + threadIdx.x; i < hi; i += blockDim.x) take(lr[i], i);
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    __shared__ float sv[8];
    __shared__ int si[8];
    if (lane_id() == 0) {
        sv[warp_id()] = bv;
        si[warp_id()] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) {
                bv = sv[w];
                bi = si[w];
            }
        work[((int64_t)r * S + sp) * 2] = bv;
        work[((int64_t)r * S + sp) * 2 + 1] = __int_as_float(bi);
    }
}

__global__ void argmax_merge_kernel(const int32_t* dM, int S, const float* __restrict__ work, int32_t* __restrict__ out) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x * (blockDim.x >> 5) + warp_id();
    if (r >= *dM) return;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int s = lane_id(); s < S; s += 32) {
        const float v = work[((int64_t)r * S + s) * 2];
        const int i = __float_as_int(work[((int64_t)r * S + s) * 2 + 1]);
        if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    if (lane_id() == 0) out[r] = bi;
}

// softmax(logits / T) in fp64, for the stochastic verify path
__global__ void __launch_bounds__(512) softmax64_kernel(const float* __restrict__ logits, const int32_t* dM, int V,
                                                        double inv_temp, double* __restrict__ out) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const float* lr = logits + (int64_t)r * V;
    double* o = out + (int64_t)r * V;
    __shared__ double red[32];
    double mx = -INFINITY;
    for (int i = threadIdx.x; i < V; i += blockDim.x) mx = fmax(mx, (double)lr[i] * inv_temp);
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (lane_id() == 0) red[warp_id()] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) red[0] = fmax(red[0], red[w]);
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    double s = 0.0;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const double e = exp((double)lr[i] * inv_temp - mx);
        o[i] = e;
        s += e;
    }
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane_id() == 0) red[warp_id()] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        red[0] = t;
    }
    __syncthreads();
    const double inv = 1.0 / red[0];
    for (int i = threadIdx.x; i < V; i += blockDim.x) o[i] *= inv;
}

__global__ void logit_bias_kernel(float* __restrict__ logits, const int32_t* dM, int V,
                                  const int32_t* __restrict__ tail, int order, int stride, uint64_t seed,
                                  uint64_t seed2, float mixw, float sharp) {
    pdl_wait();     // predecessor outputs visible from here
    pdl_trigger();  // let the next kernel start its prologue
    const int r = blockIdx.x;
    if (r >= *dM) return;
    __shared__ uint64_t st[2];
    if (threadIdx.x == 0) {
        uint64_t s = mix64(seed + kSeedSalt), s2 = mix64(seed2 + kSeedSalt);
        for (int j = 0; j < order; ++j) {
            const int t = tail[(int64_t)r * stride + j];
            if (t < 0) continue;
            s = mix64(s ^ mix64((uint64_t)t + 1));
            s2 = mix64(s2 ^ mix64((uint64_t)t + 1));
        }
        st[0] = s;
        st[1] = s2;
    }
    __syncthreads();
    float* lr = logits + (int64_t)r * V;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const uint64_t step = (uint64_t)(i + 1) * kGamma;
        float u = to_unit_f(mix64(st[0] + step));
        if (mixw != 0.f) u += mixw * to_unit_f(mix64(st[1] + step));
        lr[i] += sharp * u;
    }
}

}  // namespace card

using namespace card;

extern "C" {

int card_logit_bias(float* logits, const int32_t* dM, int m_max, int V, const int32_t* ctx_tail, int order,
                    int stride, uint64_t seed, uint64_t seed2, float mix_weight, float sharpness, void* stream) {
    if (sharpness == 0.f || m_max <= 0) return CARD_OK;
    if (stride < order) return CARD_E_INPUT;
    CARD_PDL((logit_bias_kernel), dim3(m_max), dim3(512), 0, (cudaStream_t)stream, logits, dM, V, ctx_tail, order, stride, seed, seed2,
                                                               mix_weight, sharpness);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_embed(const int32_t* tok, const int32_t* dM, int m_max, const void* E, int wdtype, int H, float* x,
               void* xb, float* ssq, int ssq_ld, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (xb && (H % 16 != 0 || !ssq)) return CARD_E_INPUT;
    __nv_bfloat16* xbb = (__nv_bfloat16*)xb;
    if (wdtype == 0)
        CARD_PDL((embed_kernel<__nv_bfloat16>), dim3(m_max), dim3(256), 0, s, tok, dM, (const __nv_bfloat16*)E, H, x, xbb,
                 ssq, ssq_ld);
    else CARD_PDL((embed_kernel<float>), dim3(m_max), dim3(256), 0, s, tok, dM, (const float*)E, H, x, xbb, ssq, ssq_ld);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_resid_add(const int32_t* dM, int m_max, int H, float* x, const float* part, void* xb, float* ssq, int ssq_ld,
                   void* stream) {
    if (!dM || !x || !part || !xb || !ssq || H % 16 != 0 || m_max <= 0) return CARD_E_INPUT;
    CARD_PDL(resid_add_kernel, dim3(m_max), dim3(128), 0, (cudaStream_t)stream, dM, H, x, part, (__nv_bfloat16*)xb,
             ssq, ssq_ld);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_gather_rows(const int32_t* out_rows, const int32_t* n_out, int m_max, int H, const void* xb, const float* ssq,
                     int ssq_ld, void* xb_out, float* ssq_out, int ssq_out_ld, void* stream) {
    if (!out_rows || !n_out || !xb || !ssq || !xb_out || !ssq_out || H % 16 != 0 || m_max <= 0) return CARD_E_INPUT;
    CARD_PDL(gather_rows_kernel, dim3(m_max), dim3(128), 0, (cudaStream_t)stream, out_rows, n_out, H,
             (const __nv_bfloat16*)xb, ssq, ssq_ld, (__nv_bfloat16*)xb_out, ssq_out, ssq_out_ld);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_rmsnorm(const float* x, const float* w, int H, float eps, const int32_t* dM, int m_max, const int32_t* gather,
                 void* y, int ydtype, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (ydtype == 0) CARD_PDL((rmsnorm_kernel<__nv_bfloat16>), dim3(m_max), dim3(256), 0, s, x, w, H, eps, dM, gather, (__nv_bfloat16*)y);
    else CARD_PDL((rmsnorm_kernel<float>), dim3(m_max), dim3(256), 0, s, x, w, H, eps, dM, gather, (float*)y);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_rope_kv(const float* qkv, const int32_t* dM, int m_max, const int32_t* pos, const int32_t* slot,
                 const float* cos_t, const float* sin_t, int nh, int nkv, int hd, float* q, void* kc, void* vc,
                 int kvdtype, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const float qscale = 1.0f / sqrtf((float)hd);
    if (kvdtype == 0)
        CARD_PDL((rope_kv_kernel<__nv_bfloat16>), dim3(m_max), dim3(256), 0, s, qkv, dM, pos, slot, cos_t, sin_t, nh, nkv, hd, qscale, q,
                                             (__nv_bfloat16*)kc, (__nv_bfloat16*)vc);
    else
        CARD_PDL((rope_kv_kernel<float>), dim3(m_max), dim3(256), 0, s, qkv, dM, pos, slot, cos_t, sin_t, nh, nkv, hd, qscale, q, (float*)kc,
                                             (float*)vc);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_attention_trace(unsigned long long* buf) {
    const int rc = attn_set_trace(buf);
    return rc != CARD_OK ? rc : attn_tc_set_trace(buf);
}

int card_attention_work_floats(int m_max, int nh, int hd, int max_plen) {
    const int n_splits = (max_plen + kChunk - 1) / kChunk;
    return m_max * nh * (n_splits + 1) * (hd + 2);
}

int card_attention(const float* q, const int32_t* dM, int m_max, const int32_t* plen, const int32_t* slot,
                   const int32_t* n_extra,
                   const int32_t* extra, int extra_max, const void* kc, const void* vc, int kvdtype, int nh, int nkv,
                   int hd, int max_plen, float* work, void* o, int odtype, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int n_splits = (max_plen + kChunk - 1) / kChunk;
    const int threads = 256;
    const size_t smem = (size_t)(2 * kChunk * (hd + 1) + (threads / 32) * (hd + kChunk)) * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_prefix_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(attn_prefix_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr = true;
    }
    // Wide forwards (draft tree rows, prefill chunks: >= 256 query-heads per KV
    // head) run the tcgen05 kernel.  Narrow ones (verify chains, AR steps) keep
    // the register-resident mma.sync kernel: at 60 KB of shared memory it
    // co-resides with the QKV GEMM's tail and starts under it, which the
    // 200 KB tcgen05 kernel cannot; same-box A/B: 3.25 / 3.33 ms vs 3.49 /
    // 3.62 ms per AR / verify forward of Llama-3.1-8B, equal draft forwards
    // (tools/ab_lib.sh, profiles/r02_attention.txt).
    if (kvdtype == 0 && odtype == 0 && m_max * (nh / nkv) >= 256 && attn_tc_fits(m_max, nh, nkv, hd, extra_max))
        return launch_attn_tc(q, dM, m_max, plen, n_extra, extra, extra_max, kc, vc, nullptr, nh, nkv, hd, max_plen,
                              o, s);
    if (kvdtype == 0 && odtype == 0 && (hd == 64 || hd == 128) &&
        attn_fused_fits(m_max, nh, nkv, extra_max))
        if (slot) return launch_attn_fused(q, dM, m_max, plen, slot, nullptr, n_extra, extra, extra_max, kc, vc, nh, nkv, hd,
                                           max_plen, o, s);
    dim3 g1(nkv, n_splits);
    const int ew = (m_max * nh + 7) / 8;
    if (kvdtype == 0) {
        if (hd == 64)
            CARD_PDL((attn_prefix_tc_kernel<64>), dim3(g1), dim3(128), 0, s, q, dM, plen, (const __nv_bfloat16*)kc,
                                                         (const __nv_bfloat16*)vc, nh, nkv, n_splits, work);
        else if (hd == 128)
            CARD_PDL((attn_prefix_tc_kernel<128>), dim3(g1), dim3(128), 0, s, q, dM, plen, (const __nv_bfloat16*)kc,
                                                          (const __nv_bfloat16*)vc, nh, nkv, n_splits, work);
        else
            CARD_PDL((attn_prefix_kernel<__nv_bfloat16>), dim3(g1), dim3(threads), smem, s, q, dM, plen, (const __nv_bfloat16*)kc,
                                                         (const __nv_bfloat16*)vc, nh, nkv, hd, n_splits, work);
        CARD_PDL((attn_extra_kernel<__nv_bfloat16>), dim3(ew), dim3(256), 0, s, q, dM, n_extra, extra, extra_max, (const __nv_bfloat16*)kc,
                                             (const __nv_bfloat16*)vc, nh, nkv, hd, n_splits, work);
    } else {
        CARD_PDL((attn_prefix_kernel<float>), dim3(g1), dim3(threads), smem, s, q, dM, plen, (const float*)kc, (const float*)vc, nh, nkv, hd,
                                                     n_splits, work);
        CARD_PDL((attn_extra_kernel<float>), dim3(ew), dim3(256), 0, s, q, dM, n_extra, extra, extra_max, (const float*)kc, (const float*)vc, nh,
                                             nkv, hd, n_splits, work);
    }
    dim3 g3(m_max, nh);
    if (odtype == 0) CARD_PDL((attn_combine_kernel<__nv_bfloat16>), dim3(g3), dim3(64), 0, s, dM, plen, nh, hd, n_splits, work, (__nv_bfloat16*)o);
    else CARD_PDL((attn_combine_kernel<float>), dim3(g3), dim3(64), 0, s, dM, plen, nh, hd, n_splits, work, (float*)o);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_attention_paged(const float* q, const int32_t* dM, int m_max, const int32_t* plen,
                         const int32_t* n_extra, const int32_t* extra, int extra_max, const void* kc,
                         const void* vc, const int32_t* page_table, int nh, int nkv, int hd, int max_plen,
                         void* o, void* stream) {
    if (!q || !dM || !plen || !kc || !vc || !o || m_max <= 0 || nkv <= 0 || nh % nkv) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    // same shape dispatch as card_attention (wide -> tcgen05, narrow -> mma.sync)
    if (m_max * (nh / nkv) >= 256 && attn_tc_fits(m_max, nh, nkv, hd, extra_max))
        rc = launch_attn_tc(q, dM, m_max, plen, n_extra, extra, extra_max, kc, vc, page_table, nh, nkv, hd, max_plen,
                            o, s);
    else if ((hd == 64 || hd == 128) && attn_fused_fits(m_max, nh, nkv, extra_max))
        rc = launch_attn_fused(q, dM, m_max, plen, nullptr, page_table, n_extra, extra, extra_max, kc, vc, nh, nkv, hd,
                               max_plen, o, s);
    else if (attn_tc_fits(m_max, nh, nkv, hd, extra_max))
        rc = launch_attn_tc(q, dM, m_max, plen, n_extra, extra, extra_max, kc, vc, page_table, nh, nkv, hd, max_plen,
                            o, s);
    else
        return CARD_E_CONFIG;
    if (rc == CARD_OK) CARD_LAUNCH_CHECK();
    return rc;
}

int card_attention_tree(const void* qsw, int qsw_tiles, const int32_t* dM, int m_max, const int32_t* plen,
                        const int32_t* n_extra, const int32_t* extra, int extra_max, const void* kc, const void* vc,
                        const int32_t* page_table, int nh, int nkv, int hd, int max_plen, void* o, void* stream) {
    if (!qsw || !dM || !plen || !kc || !vc || !o || m_max <= 0 || nkv <= 0 || nh % nkv) return CARD_E_INPUT;
    if (!attn_tc_fits(m_max, nh, nkv, hd, extra_max)) return CARD_E_CONFIG;
    const int rc = launch_attn_tc(nullptr, dM, m_max, plen, n_extra, extra, extra_max, kc, vc, page_table, nh, nkv, hd,
                                  max_plen, o, (cudaStream_t)stream, qsw, qsw_tiles);
    if (rc == CARD_OK) CARD_LAUNCH_CHECK();
    return rc;
}

int card_attention_batch(const float* q, const void* qsw, int qsw_tiles, const int32_t* dM, int m_max,
                         const int32_t* plen, const int32_t* n_extra, const int32_t* extra, int extra_max,
                         const void* kc, const void* vc, const int32_t* page_tables, int pt_stride, int seg_rows,
                         int nh, int nkv, int hd, int max_plen, void* o, void* stream) {
    if ((!q && !qsw) || !dM || !plen || !kc || !vc || !o || !page_tables || m_max <= 0 || nkv <= 0 || nh % nkv ||
        seg_rows <= 0 || pt_stride <= 0)
        return CARD_E_INPUT;
    const int G = nh / nkv;
    // segments one tile of 128 query-heads can span
    if (!attn_tc_fits(m_max, nh, nkv, hd, extra_max) || (128 / G + 2 + seg_rows - 1) / seg_rows + 1 > attn_tc_max_segments())
        return CARD_E_CONFIG;
    const int rc = launch_attn_tc(q, dM, m_max, plen, n_extra, extra, extra_max, kc, vc, page_tables, nh, nkv, hd,
                                  max_plen, o, (cudaStream_t)stream, qsw, qsw_tiles, seg_rows, pt_stride);
    if (rc == CARD_OK) CARD_LAUNCH_CHECK();
    return rc;
}

// vocab splits of the lm_head readers: about six CTAs per SM (the logits are
// L2-warm right after the lm_head; more parallel reads win in-graph, +0.6 %
// bench tokens/s against two per SM, same-box A/B)
static int vocab_splits(int m_max) {
    int s = (6 * 148 + m_max - 1) / (m_max > 0 ? m_max : 1);
    return s < 1 ? 1 : (s > 64 ? 64 : s);
}

}  // extern "C"

namespace card {
// Merge of the EPI_TOPK lm_head records of one row (one CTA per row; the
// ~1000 records of a row are spread over the threads so every load is
// independent): fp64 log-sum-exp, then k rounds of block arg-best over the
// per-thread sorted top-4 lists.
__global__ void __launch_bounds__(256) tiles_merge_kernel(const int32_t* dM, int S, int k, int V,
                                                          const float* __restrict__ work, int32_t* __restrict__ out_tok,
                                                          double* __restrict__ out_logp, int32_t* __restrict__ out_cnt) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const float* base = work + (int64_t)r * S * kTopkRec;
    __shared__ double sh_d[8];
    __shared__ float sh_v[8];
    __shared__ int sh_t[8], sh_w[8];
    float tv[kTopkKT];
    int tt[kTopkKT];
#pragma unroll
    for (int q = 0; q < kTopkKT; ++q) {
        tv[q] = -INFINITY;
        tt[q] = 0x7fffffff;
    }
    float lm = -INFINITY;
    constexpr int kKeep = 8;   // records' (max, sum) kept in registers for the second pass
    float rm[kKeep], rs[kKeep];
    int j = 0;
    static_assert(kTopkKT == 4 && kTopkRec % 2 == 0, "bitonic top-4 merge of 8-byte aligned records");
    auto cx = [&](int i, int k) {   // order slots (i, k) best first
        const bool sw = lbefore(tv[k], tt[k], tv[i], tt[i]);
        const float fi = tv[i], fk = tv[k];
        const int ii = tt[i], ik = tt[k];
        tv[i] = sw ? fk : fi;
        tt[i] = sw ? ik : ii;
        tv[k] = sw ? fi : fk;
        tt[k] = sw ? ii : ik;
    };
    for (int s = threadIdx.x; s < S; s += blockDim.x, ++j) {
        const float2* p2 = reinterpret_cast<const float2*>(base + (int64_t)s * kTopkRec);
        const float2 h = p2[0];   // (max, sum-exp)
        float2 c[kTopkKT];        // the record's sorted top-4 (value, token bits)
#pragma unroll
        for (int q = 0; q < kTopkKT; ++q) c[q] = p2[1 + q];
        lm = fmaxf(lm, h.x);
        if (j < kKeep) {
#pragma unroll
            for (int q = 0; q < kKeep; ++q)
                if (q == j) {
                    rm[q] = h.x;
                    rs[q] = h.y;
                }
        }
        // both lists sorted: best of mine[q] / theirs[3 - q], then a bitonic
        // sort of the four (8 compare-selects instead of 4 insertions)
#pragma unroll
        for (int q = 0; q < kTopkKT; ++q) {
            const float ov = c[3 - q].x;
            const int oi = __float_as_int(c[3 - q].y);
            const bool tk = lbefore(ov, oi, tv[q], tt[q]);
            tv[q] = tk ? ov : tv[q];
            tt[q] = tk ? oi : tt[q];
        }
        cx(0, 2);
        cx(1, 3);
        cx(0, 1);
        cx(2, 3);
    }
    // block max of the record maxima
    for (int o = 16; o > 0; o >>= 1) lm = fmaxf(lm, __shfl_xor_sync(0xffffffffu, lm, o));
    if (lane_id() == 0) sh_v[warp_id()] = lm;
    __syncthreads();
    float gmf = sh_v[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) gmf = fmaxf(gmf, sh_v[w]);
    const double gm = (double)gmf;
    double tot = 0.0;
    j = 0;
    for (int s = threadIdx.x; s < S; s += blockDim.x, ++j) {
        float m0, s0;
        if (j < kKeep) {
#pragma unroll
            for (int q = 0; q < kKeep; ++q)
                if (q == j) {
                    m0 = rm[q];
                    s0 = rs[q];
                }
        } else {
            const float* p = base + (int64_t)s * kTopkRec;
            m0 = p[0];
            s0 = p[1];
        }
        if (s0 > 0.f) tot += (double)s0 * exp((double)m0 - gm);
    }
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane_id() == 0) sh_d[warp_id()] = tot;
    __syncthreads();
    double T = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) T += sh_d[w];
    const double lse = gm + log(T);
    int head = 0;
    for (int round = 0; round < k; ++round) {
        float v = -INFINITY;
        int t = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < kTopkKT; ++q)
            if (q == head) {
                v = tv[q];
                t = tt[q];
            }
        int who = threadIdx.x;
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int ot = __shfl_xor_sync(0xffffffffu, t, o);
            const int ow = __shfl_xor_sync(0xffffffffu, who, o);
            if (lbefore(ov, ot, v, t)) {
                v = ov;
                t = ot;
                who = ow;
            }
        }
        __syncthreads();
        if (lane_id() == 0) {
            sh_v[warp_id()] = v;
            sh_t[warp_id()] = t;
            sh_w[warp_id()] = who;
        }
        __syncthreads();
        float bv = sh_v[0];
        int bt = sh_t[0], bw = sh_w[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (lbefore(sh_v[w], sh_t[w], bv, bt)) {
                bv = sh_v[w];
                bt = sh_t[w];
                bw = sh_w[w];
            }
        if (threadIdx.x == bw) ++head;
        if (threadIdx.x == 0) {
            out_tok[(int64_t)r * k + round] = bt;
            out_logp[(int64_t)r * k + round] = (double)bv - lse;
        }
    }
    if (threadIdx.x == 0) out_cnt[r] = k < V ? k : V;
}
}  // namespace card

extern "C" {

int card_lmhead_work_floats(int m_max, int k) { return m_max * vocab_splits(m_max) * (2 + 2 * 8); }

int card_topk_logits(const float* logits, const int32_t* dM, int m_max, int V, int k, double inv_temp,
                     int32_t* out_tok, double* out_logp, int32_t* out_cnt, float* work, const int32_t* ctx_tail,
                     int order, int stride, uint64_t seed, uint64_t seed2, float mix_weight, float sharpness,
                     void* stream) {
    if (k < 1 || k > 8) return CARD_E_CONFIG;
    const KgBias kb{ctx_tail, order, stride, seed, seed2, mix_weight, ctx_tail ? sharpness : 0.f};
    cudaStream_t s = (cudaStream_t)stream;
    const int S = vocab_splits(m_max);
    dim3 g(m_max, S);
    const float it = (float)inv_temp;
    switch (k) {
#define CARD_TOPK_CASE(KT)                                                                                   \
    case KT:                                                                                                 \
        CARD_PDL((topk_partial_kernel<KT>), dim3(g), dim3(256), 0, s, logits, dM, V, S, it, work, kb);                                \
        CARD_PDL((topk_merge_kernel<KT>), dim3((m_max + 7) / 8), dim3(256), 0, s, dM, S, k, V, work, out_tok, out_logp, out_cnt); \
        break;
        CARD_TOPK_CASE(1)
        CARD_TOPK_CASE(2)
        CARD_TOPK_CASE(3)
        CARD_TOPK_CASE(4)
        CARD_TOPK_CASE(5)
        CARD_TOPK_CASE(6)
        CARD_TOPK_CASE(7)
        CARD_TOPK_CASE(8)
#undef CARD_TOPK_CASE
    }
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_lmhead_topk_merge(const float* work, const int32_t* dM, int m_max, int n_tiles, int k, int V,
                           int32_t* out_tok, double* out_logp, int32_t* out_cnt, void* stream) {
    if (k < 1 || k > kTopkKT || n_tiles < 1) return CARD_E_CONFIG;
    CARD_PDL((tiles_merge_kernel), dim3(m_max), dim3(256), 0, (cudaStream_t)stream, dM, n_tiles, k, V, work, out_tok,
             out_logp, out_cnt);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_argmax_logits(const float* logits, const int32_t* dM, int m_max, int V, int32_t* out, float* work,
                       const int32_t* ctx_tail, int order, int stride, uint64_t seed, uint64_t seed2, float mix_weight,
                       float sharpness, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int S = vocab_splits(m_max);
    const KgBias kb{ctx_tail, order, stride, seed, seed2, mix_weight, ctx_tail ? sharpness : 0.f};
    CARD_PDL((argmax_partial_kernel), dim3(m_max, S), dim3(256), 0, s, logits, dM, V, S, work, kb);
    CARD_PDL((argmax_merge_kernel), dim3((m_max + 7) / 8), dim3(256), 0, s, dM, S, work, out);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_softmax64(const float* logits, const int32_t* dM, int m_max, int V, double inv_temp, double* out,
                   void* stream) {
    CARD_PDL((softmax64_kernel), dim3(m_max), dim3(512), 0, (cudaStream_t)stream, logits, dM, V, inv_temp, out);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

}  // extern "C"
