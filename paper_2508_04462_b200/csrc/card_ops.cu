// card_ops.cu — the reference's operator plug-in, on the device.
//
//   card_kgram_dist  <- _kernels.pyx:44-93   (hashed k-gram "forward")
//   card_rows_topk   <- _kernels.pyx:96-145  (per-row top-k by (p desc, token asc))
//
// Compiled with --fmad=false (see card_common.cuh).  These kernels serve
// the toy-model parity path and the drop-in TreeCache.expand_layer; the
// transformer path produces candidates from logits in card_llm.cu.
#include <stdio.h>
#include <stdlib.h>

#include "card_common.cuh"

namespace card {

static thread_local char g_cuda_err[256] = {0};
bool pdl_enabled() { return true; }   // programmatic dependent launch on every chained kernel
void set_cuda_error(cudaError_t e) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

// One CTA per row.  The uniform stream and the mix are integer / two-op
// fp64 work spread over the block; the softmax sum is sequential in token
// order (as the reference) and runs on one thread — V is toy-sized here.
__global__ void kgram_dist_kernel(uint64_t s1_seed, uint64_t s2_seed, double mix_weight,
                                  const int32_t* __restrict__ tails, int tail_len, int tail_stride, int vocab,
                                  double sharpness, double temperature, double* __restrict__ out) {
    const int row = blockIdx.x;
    __shared__ uint64_t st[2];
    __shared__ double red_m;
    if (threadIdx.x == 0) {
        // _stream_state (_kernels.pyx:36-41)
        uint64_t s = mix64(s1_seed + kSeedSalt);
        uint64_t s2 = mix64(s2_seed + kSeedSalt);
        for (int j = 0; j < tail_len; ++j) {
            const int32_t tv = tails[(int64_t)row * tail_stride + j];
            if (tv < 0) continue;   // context shorter than the model order (lm.py:235)
            uint64_t t = (uint64_t)(tv + 1);
            s = mix64(s ^ mix64(t));
            s2 = mix64(s2 ^ mix64(t));
        }
        st[0] = s;
        st[1] = s2;
    }
    __syncthreads();
    double* o = out + (int64_t)row * vocab;
    // u_i (+ w * u2_i), then the logits b_i = (sharpness*u_i)/T stored in `o`
    for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
        uint64_t step = (uint64_t)(i + 1) * kGamma;
        double u = to_unit(mix64(st[0] + step));
        if (mix_weight != 0.0) u = __dadd_rn(u, __dmul_rn(mix_weight, to_unit(mix64(st[1] + step))));
        o[i] = (temperature == 0.0) ? __dmul_rn(sharpness, u) : __ddiv_rn(__dmul_rn(sharpness, u), temperature);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (temperature == 0.0) {
            // first-max one-hot (_kernels.pyx:63-74)
            int best = 0;
            double bv = o[0];
            for (int i = 1; i < vocab; ++i)
                if (o[i] > bv) { bv = o[i]; best = i; }
            red_m = (double)best;
        } else {
            double m = -__longlong_as_double(0x7ff0000000000000LL);
            for (int i = 0; i < vocab; ++i) m = o[i] > m ? o[i] : m;
            red_m = m;
        }
    }
    __syncthreads();
    if (temperature == 0.0) {
        int best = (int)red_m;
        for (int i = threadIdx.x; i < vocab; i += blockDim.x) o[i] = (i == best) ? 1.0 : 0.0;
        return;
    }
    const double m = red_m;
    for (int i = threadIdx.x; i < vocab; i += blockDim.x) o[i] = exp_cr(__dsub_rn(o[i], m));
    __syncthreads();
    __shared__ double z_sh;
    if (threadIdx.x == 0) {
        double z = 0.0;
        for (int i = 0; i < vocab; ++i) z = __dadd_rn(z, o[i]);   // sequential, token order
        z_sh = z;
    }
    __syncthreads();
    const double z = z_sh;
    for (int i = threadIdx.x; i < vocab; i += blockDim.x) o[i] = __ddiv_rn(o[i], z);
}

// ---------------------------------------------------------------- rows_topk
constexpr int kTopkMax = 32;

// (p desc, token asc): true if (pa, ta) ranks before (pb, tb)
__device__ __forceinline__ bool before(double pa, int ta, double pb, int tb) {
    return pa > pb || (pa == pb && ta < tb);
}

// One warp per row.  Each lane keeps a sorted local top-k of its strided
// tokens; k rounds of warp arg-best merge them.  Optional validation of the
// row (cache.py:204-208) is folded into the same pass.
__global__ void rows_topk_kernel(const double* __restrict__ dists, int n_rows, int vocab, int k,
                                 int32_t* __restrict__ out_tok, double* __restrict__ out_p,
                                 int32_t* __restrict__ out_cnt, int32_t* status) {
    const int row = blockIdx.x * (blockDim.x >> 5) + warp_id();
    if (row >= n_rows) return;
    const int lane = lane_id();
    const double* d = dists + (int64_t)row * vocab;
    double lp[kTopkMax];
    int lt[kTopkMax];
    int m = 0;
    bool bad = false;
    double sum = 0.0;
    for (int t = lane; t < vocab; t += 32) {
        double p = d[t];
        bad |= (p != p) || (p < 0.0);
        sum = __dadd_rn(sum, p);
        if (!(p > 0.0)) continue;
        // insertion into the local sorted list (tokens arrive ascending)
        int pos = m;
        while (pos > 0 && before(p, t, lp[pos - 1], lt[pos - 1])) --pos;
        if (pos >= k) continue;
        int end = m < k ? m : k - 1;
        for (int j = end; j > pos; --j) { lp[j] = lp[j - 1]; lt[j] = lt[j - 1]; }
        lp[pos] = p;
        lt[pos] = t;
        if (m < k) ++m;
    }
    if (status != nullptr) {
        for (int o = 16; o > 0; o >>= 1) sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
        unsigned any_bad = __ballot_sync(0xffffffffu, bad);
        if (lane == 0 && (any_bad || fabs(__dsub_rn(sum, 1.0)) > 1e-9)) atomicExch(status, CARD_E_INPUT);
    }
    int head = 0, cnt = 0;
    for (int r = 0; r < k; ++r) {
        double bp = head < m ? lp[head] : -1.0;
        int bt = head < m ? lt[head] : 0x7fffffff;
        int bl = lane;
        for (int o = 16; o > 0; o >>= 1) {
            double op = __shfl_xor_sync(0xffffffffu, bp, o);
            int ot = __shfl_xor_sync(0xffffffffu, bt, o);
            int ol = __shfl_xor_sync(0xffffffffu, bl, o);
            if (before(op, ot, bp, bt)) { bp = op; bt = ot; bl = ol; }
        }
        if (bp <= 0.0) break;   // every lane exhausted
        if (lane == 0) {
            out_tok[(int64_t)row * k + r] = bt;
            out_p[(int64_t)row * k + r] = bp;
        }
        if (lane == bl) ++head;
        ++cnt;
    }
    if (lane == 0) out_cnt[row] = cnt;
}

__global__ void log_cr_kernel(const double* x, double* y, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = log_cr(x[i]);
}
__global__ void exp_cr_kernel(const double* x, double* y, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = exp_cr(x[i]);
}

int launch_rows_topk(const double* dists, int n_rows, int vocab, int k, int32_t* tok, double* p,
                     int32_t* cnt, int32_t* status, cudaStream_t s) {
    if (n_rows <= 0) return CARD_OK;
    const int warps = 8;
    rows_topk_kernel<<<(n_rows + warps - 1) / warps, warps * 32, 0, s>>>(dists, n_rows, vocab, k, tok, p,
                                                                         cnt, status);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

}  // namespace card

using namespace card;

extern "C" {

int card_abi_version(void) { return CARD_ABI_VERSION; }

const char* card_strerror(int code) {
    switch (code) {
        case CARD_OK: return "ok";
        case CARD_E_INPUT: return "input error";
        case CARD_E_CONFIG: return "config error";
        case CARD_E_PROTOCOL: return "protocol error";
        case CARD_FRONTIER_FULL: return "frontier full";
        case CARD_E_CAPACITY: return "arena capacity exhausted";
        case CARD_E_CUDA: return "cuda error";
        case CARD_E_MASK: return "mask error";
        default: return "unknown status";
    }
}

const char* card_last_cuda_error(void) { return g_cuda_err; }

int card_kgram_dist(uint64_t seed, uint64_t seed2, double mix_weight, const int32_t* tails, int tail_len,
                    int tail_stride, int n_rows, int vocab, double sharpness, double temperature, double* out,
                    void* stream) {
    if (vocab < 1 || n_rows < 0 || tail_len < 0 || tail_stride < tail_len) return CARD_E_INPUT;
    if (n_rows == 0) return CARD_OK;
    kgram_dist_kernel<<<n_rows, 128, 0, (cudaStream_t)stream>>>(seed, seed2, mix_weight, tails, tail_len,
                                                               tail_stride, vocab, sharpness, temperature, out);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_rows_topk(const double* dists, int n_rows, int vocab, int k, int32_t* out_tok, double* out_p,
                   int32_t* out_cnt, int32_t* status, void* stream) {
    if (k < 1 || k > kTopkMax || vocab < 1 || n_rows < 0) return CARD_E_CONFIG;
    return launch_rows_topk(dists, n_rows, vocab, k, out_tok, out_p, out_cnt, status, (cudaStream_t)stream);
}

int card_log_cr(const double* x, double* y, int n, void* stream) {
    if (n <= 0) return CARD_OK;
    log_cr_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(x, y, n);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_exp_cr(const double* x, double* y, int n, void* stream) {
    if (n <= 0) return CARD_OK;
    exp_cr_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(x, y, n);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

}  // extern "C"
