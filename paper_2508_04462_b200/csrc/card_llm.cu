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
template <typename W>
__global__ void embed_kernel(const int32_t* __restrict__ tok, const int32_t* dM, const W* __restrict__ E, int H,
                             float* __restrict__ x) {
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const int64_t t = tok[r];
    for (int i = threadIdx.x; i < H; i += blockDim.x) x[(int64_t)r * H + i] = ldf(E, t * H + i);
}

// ---------------------------------------------------------------- rmsnorm
template <typename Y>
__global__ void rmsnorm_kernel(const float* __restrict__ x, const float* __restrict__ w, int H, float eps,
                               const int32_t* dM, const int32_t* gather, Y* __restrict__ y) {
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const int src = gather ? gather[r] : r;
    const float* xr = x + (int64_t)src * H;
    float ss = 0.f;
    for (int i = threadIdx.x; i < H; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
    __shared__ float red[32];
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
    for (int i = threadIdx.x; i < H; i += blockDim.x) stf(y, (int64_t)r * H + i, (xr[i] * inv) * w[i]);
}

// ---------------------------------------------------------------- rope + kv write
template <typename KV>
__global__ void rope_kv_kernel(const float* __restrict__ qkv, const int32_t* dM, const int32_t* __restrict__ pos,
                               const int32_t* __restrict__ slot, const float* __restrict__ cos_t,
                               const float* __restrict__ sin_t, int nh, int nkv, int hd, float qscale,
                               float* __restrict__ q, KV* __restrict__ kc, KV* __restrict__ vc) {
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

// extra slots (tree ancestors + self): one warp per (row, head)
template <typename KV>
__global__ void attn_extra_kernel(const float* __restrict__ q, const int32_t* dM, const int32_t* __restrict__ n_extra,
                                  const int32_t* __restrict__ extra, int extra_max, const KV* __restrict__ kc,
                                  const KV* __restrict__ vc, int nh, int nkv, int hd, int n_splits,
                                  float* __restrict__ work) {
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

// ---------------------------------------------------------------- lm_head epilogues
constexpr int kTopkRegs = 8;

__device__ __forceinline__ bool lbefore(float a, int ta, float b, int tb) { return a > b || (a == b && ta < tb); }

// One CTA per row: online max / sum-exp (fp32 per thread, fp64 merge) and
// per-thread sorted top-k, merged by k rounds of block arg-best.
__global__ void __launch_bounds__(512) topk_logits_kernel(const float* __restrict__ logits, const int32_t* dM, int V,
                                                          int k, float inv_temp, int32_t* __restrict__ out_tok,
                                                          double* __restrict__ out_logp, int32_t* __restrict__ out_cnt) {
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const float* lr = logits + (int64_t)r * V;
    float tv[kTopkRegs];
    int tt[kTopkRegs];
    int m = 0;
    float mx = -INFINITY, sum = 0.f;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const float v = lr[i] * inv_temp;
        if (v > mx) {
            sum = sum * __expf(mx - v) + 1.f;
            mx = v;
        } else {
            sum += __expf(v - mx);
        }
        int p = m;
        while (p > 0 && lbefore(v, i, tv[p - 1], tt[p - 1])) --p;
        if (p < k) {
            int end = m < k ? m : k - 1;
            for (int j = end; j > p; --j) {
                tv[j] = tv[j - 1];
                tt[j] = tt[j - 1];
            }
            tv[p] = v;
            tt[p] = i;
            if (m < k) ++m;
        }
    }
    __shared__ double sh_m[32], sh_s[32];
    __shared__ float bv[32];
    __shared__ int bt[32], bl[32];
    __shared__ double lse_sh;
    // block max
    float wm = mx;
    for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    if (lane_id() == 0) sh_m[warp_id()] = wm;
    __syncthreads();
    if (threadIdx.x == 0) {
        double g = -INFINITY;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) g = fmax(g, sh_m[w]);
        sh_m[0] = g;
    }
    __syncthreads();
    const double gmax = sh_m[0];
    double ds = (mx == -INFINITY) ? 0.0 : (double)sum * exp((double)mx - gmax);
    for (int o = 16; o > 0; o >>= 1) ds += __shfl_xor_sync(0xffffffffu, ds, o);
    __syncthreads();
    if (lane_id() == 0) sh_s[warp_id()] = ds;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh_s[w];
        lse_sh = gmax + log(t);
    }
    __syncthreads();
    const double lse = lse_sh;
    int head = 0;
    for (int round = 0; round < k; ++round) {
        float v = head < m ? tv[head] : -INFINITY;
        int t = head < m ? tt[head] : 0x7fffffff;
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
            bl[warp_id()] = who;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (lbefore(bv[w], bt[w], bv[0], bt[0])) {
                    bv[0] = bv[w];
                    bt[0] = bt[w];
                    bl[0] = bl[w];
                }
            out_tok[(int64_t)r * k + round] = bt[0];
            out_logp[(int64_t)r * k + round] = (double)bv[0] - lse;
        }
        __syncthreads();
        if (threadIdx.x == bl[0]) ++head;
        __syncthreads();
    }
    if (threadIdx.x == 0) out_cnt[r] = k < V ? k : V;
}

__global__ void __launch_bounds__(512) argmax_logits_kernel(const float* __restrict__ logits, const int32_t* dM, int V,
                                                            int32_t* __restrict__ out) {
    const int r = blockIdx.x;
    if (r >= *dM) return;
    const float* lr = logits + (int64_t)r * V;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        const float v = lr[i];
        if (v > bv) {   // strided ascending scan: first max per thread
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
    __shared__ float sv[32];
    __shared__ int si[32];
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
        out[r] = bi;
    }
}

// softmax(logits / T) in fp64, for the stochastic verify path
__global__ void __launch_bounds__(512) softmax64_kernel(const float* __restrict__ logits, const int32_t* dM, int V,
                                                        double inv_temp, double* __restrict__ out) {
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
        float u = (float)to_unit(mix64(st[0] + step));
        if (mixw != 0.f) u += mixw * (float)to_unit(mix64(st[1] + step));
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
    logit_bias_kernel<<<m_max, 512, 0, (cudaStream_t)stream>>>(logits, dM, V, ctx_tail, order, stride, seed, seed2,
                                                               mix_weight, sharpness);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_embed(const int32_t* tok, const int32_t* dM, int m_max, const void* E, int wdtype, int H, float* x,
               void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (wdtype == 0) embed_kernel<<<m_max, 256, 0, s>>>(tok, dM, (const __nv_bfloat16*)E, H, x);
    else embed_kernel<<<m_max, 256, 0, s>>>(tok, dM, (const float*)E, H, x);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_rmsnorm(const float* x, const float* w, int H, float eps, const int32_t* dM, int m_max, const int32_t* gather,
                 void* y, int ydtype, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (ydtype == 0) rmsnorm_kernel<<<m_max, 256, 0, s>>>(x, w, H, eps, dM, gather, (__nv_bfloat16*)y);
    else rmsnorm_kernel<<<m_max, 256, 0, s>>>(x, w, H, eps, dM, gather, (float*)y);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_rope_kv(const float* qkv, const int32_t* dM, int m_max, const int32_t* pos, const int32_t* slot,
                 const float* cos_t, const float* sin_t, int nh, int nkv, int hd, float* q, void* kc, void* vc,
                 int kvdtype, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const float qscale = 1.0f / sqrtf((float)hd);
    if (kvdtype == 0)
        rope_kv_kernel<<<m_max, 256, 0, s>>>(qkv, dM, pos, slot, cos_t, sin_t, nh, nkv, hd, qscale, q,
                                             (__nv_bfloat16*)kc, (__nv_bfloat16*)vc);
    else
        rope_kv_kernel<<<m_max, 256, 0, s>>>(qkv, dM, pos, slot, cos_t, sin_t, nh, nkv, hd, qscale, q, (float*)kc,
                                             (float*)vc);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_attention_work_floats(int m_max, int nh, int hd, int max_plen) {
    const int n_splits = (max_plen + kChunk - 1) / kChunk;
    return m_max * nh * (n_splits + 1) * (hd + 2);
}

int card_attention(const float* q, const int32_t* dM, int m_max, const int32_t* plen, const int32_t* n_extra,
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
    dim3 g1(nkv, n_splits);
    const int ew = (m_max * nh + 7) / 8;
    if (kvdtype == 0) {
        attn_prefix_kernel<<<g1, threads, smem, s>>>(q, dM, plen, (const __nv_bfloat16*)kc, (const __nv_bfloat16*)vc,
                                                     nh, nkv, hd, n_splits, work);
        attn_extra_kernel<<<ew, 256, 0, s>>>(q, dM, n_extra, extra, extra_max, (const __nv_bfloat16*)kc,
                                             (const __nv_bfloat16*)vc, nh, nkv, hd, n_splits, work);
    } else {
        attn_prefix_kernel<<<g1, threads, smem, s>>>(q, dM, plen, (const float*)kc, (const float*)vc, nh, nkv, hd,
                                                     n_splits, work);
        attn_extra_kernel<<<ew, 256, 0, s>>>(q, dM, n_extra, extra, extra_max, (const float*)kc, (const float*)vc, nh,
                                             nkv, hd, n_splits, work);
    }
    dim3 g3(m_max, nh);
    if (odtype == 0) attn_combine_kernel<<<g3, 64, 0, s>>>(dM, plen, nh, hd, n_splits, work, (__nv_bfloat16*)o);
    else attn_combine_kernel<<<g3, 64, 0, s>>>(dM, plen, nh, hd, n_splits, work, (float*)o);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_topk_logits(const float* logits, const int32_t* dM, int m_max, int V, int k, double inv_temp,
                     int32_t* out_tok, double* out_logp, int32_t* out_cnt, void* stream) {
    if (k < 1 || k > kTopkRegs) return CARD_E_CONFIG;
    topk_logits_kernel<<<m_max, 512, 0, (cudaStream_t)stream>>>(logits, dM, V, k, (float)inv_temp, out_tok, out_logp,
                                                                out_cnt);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_argmax_logits(const float* logits, const int32_t* dM, int m_max, int V, int32_t* out, void* stream) {
    argmax_logits_kernel<<<m_max, 512, 0, (cudaStream_t)stream>>>(logits, dM, V, out);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_softmax64(const float* logits, const int32_t* dM, int m_max, int V, double inv_temp, double* out,
                   void* stream) {
    softmax64_kernel<<<m_max, 512, 0, (cudaStream_t)stream>>>(logits, dM, V, inv_temp, out);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

}  // extern "C"
