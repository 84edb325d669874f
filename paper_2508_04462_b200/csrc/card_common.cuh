// card_common.cuh — shared device helpers for the CARD B200 library.
//
// Numerics note: the parity-path translation units (card_ops.cu,
// card_cache.cu) are compiled with --fmad=false so every a*b+c below is
// two IEEE operations, like the reference's -ffp-contract=off build
// (/root/reference/pkg/setup.py:23).  Explicit __fma_rn is used only where
// an exact product error term is wanted (two_prod).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/card_b200.h"

namespace card {

// ---------------------------------------------------------------- errors
void set_cuda_error(cudaError_t e);

#define CARD_CUDA_TRY(expr)                                   \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) {                              \
            card::set_cuda_error(_e);                         \
            return CARD_E_CUDA;                               \
        }                                                     \
    } while (0)

#define CARD_LAUNCH_CHECK()                                   \
    do {                                                      \
        cudaError_t _e = cudaGetLastError();                  \
        if (_e != cudaSuccess) {                              \
            card::set_cuda_error(_e);                         \
            return CARD_E_CUDA;                               \
        }                                                     \
    } while (0)

// ---------------------------------------------------------------- splitmix64
// _kernels.pyx:17-41 — pure integer arithmetic, bit-exact on any device.
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMixC1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t kMixC2 = 0x94D049BB133111EBULL;
constexpr uint64_t kSeedSalt = 0xD1B54A32D192ED03ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * kMixC1;
    z = (z ^ (z >> 27)) * kMixC2;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double to_unit(uint64_t v) {
    return (double)(v >> 11) * (1.0 / 9007199254740992.0);
}
// (float)to_unit(v) without the fp64 pipe: v >> 11 < 2^53 is exact in double,
// the scale is a power of two and the result is a normal float, so rounding
// the integer to float first and scaling after gives the same bits.
__device__ __forceinline__ float to_unit_f(uint64_t v) { return __ull2float_rn(v >> 11) * 0x1p-53f; }

// k-gram logit bias (agreement knob): logits[r][i] + sharp * (u1_i + mixw *
// u2_i), the splitmix64 k-gram stream of (seed, context tail of row r),
// _kernels.pyx:26-41.  Same fp32 arithmetic wherever it is applied (top-k /
// argmax readers, logit_bias_kernel, the fused lm_head epilogue).
struct KgBias {
    const int32_t* tail;
    int order, stride;
    uint64_t seed, seed2;
    float mixw, sharp;
};
__device__ __forceinline__ void kg_row_state(const KgBias& b, int r, uint64_t& s1, uint64_t& s2) {
    s1 = mix64(b.seed + kSeedSalt);
    s2 = mix64(b.seed2 + kSeedSalt);
    for (int j = 0; j < b.order; ++j) {
        const int t = b.tail[(int64_t)r * b.stride + j];
        if (t < 0) continue;
        s1 = mix64(s1 ^ mix64((uint64_t)t + 1));
        s2 = mix64(s2 ^ mix64((uint64_t)t + 1));
    }
}
// bias of token i given its splitmix64 stream offset step = (i + 1) * kGamma
__device__ __forceinline__ float kg_apply_step(const KgBias& b, float logit, uint64_t step, uint64_t s1, uint64_t s2) {
    float u = to_unit_f(mix64(s1 + step));
    if (b.mixw != 0.f) u += b.mixw * to_unit_f(mix64(s2 + step));
    return logit + b.sharp * u;
}
__device__ __forceinline__ float kg_apply(const KgBias& b, float logit, int i, uint64_t s1, uint64_t s2) {
    return kg_apply_step(b, logit, (uint64_t)(i + 1) * kGamma, s1, s2);
}


// ---------------------------------------------------------------- double-double
struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = __dadd_rn(p.lo, __dmul_rn(a.lo, b));
    return quick_two_sum(p.hi, p.lo);
}

// exp(x) - 1 in double-double for |x| small-ish via reduction x = k ln2 + r,
// r/1024 Taylor to degree 13, then 10 squarings in expm1 form.  Relative
// error ~2^-100, enough that rounding hi+lo is the correctly rounded exp
// except when the true value sits within ~2^-47 ulp of a midpoint.
__device__ __forceinline__ dd dd_exp_reduced(dd r, int* k_out, double x) {
    const dd kLn2 = {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
    double k = rint(x / 0x1.62e42fefa39efp-1);
    dd red = dd_add({x, 0.0}, dd_mul_d({-kLn2.hi, -kLn2.lo}, k));
    red = dd_add(red, r);
    *k_out = (int)k;
    // scale by 2^-10 (exact)
    red.hi = ldexp(red.hi, -10);
    red.lo = ldexp(red.lo, -10);
    const double inv_hi[14] = {0, 0x1.0p+0, 0x1.0p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
                               0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
                               0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
                               0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};
    const double inv_lo[14] = {0, 0, 0, 0x1.5555555555555p-57, 0x1.5555555555555p-59,
                               0x1.1111111111111p-63, -0x1.f49f49f49f49fp-65, 0x1.a01a01a01a01ap-73,
                               0x1.a01a01a01a01ap-76, -0x1.c154f8ddc6c00p-73, 0x1.cbbc05b4fa99ap-76,
                               -0x1.c062e06d1f209p-80, -0x1.2aec959e14c06p-83, 0x1.f28e0cc748ebep-87};
    // Horner: p = r*(1 + r*(1/2 + r*(1/6 + ...)))  == expm1(r)
    dd p = {inv_hi[13], inv_lo[13]};
    for (int i = 12; i >= 1; --i) {
        p = dd_mul(p, red);
        p = dd_add(p, {inv_hi[i], inv_lo[i]});
    }
    p = dd_mul(p, red);  // expm1(red)
    for (int i = 0; i < 10; ++i) {
        // (1+p)^2 - 1 = p*(2+p)
        p = dd_mul(p, dd_add({2.0, 0.0}, p));
    }
    return p;  // expm1 of (x + r) - k ln2
}

// Correctly rounded exp(x) (see dd_exp_reduced), x finite.
__device__ __forceinline__ double exp_cr(double x) {
    if (x != x) return x;
    if (x < -745.2) return 0.0;
    if (x > 709.79) return __longlong_as_double(0x7ff0000000000000LL);
    if (x == 0.0) return 1.0;
    int k;
    dd m1 = dd_exp_reduced({0.0, 0.0}, &k, x);
    dd e = dd_add({1.0, 0.0}, m1);
    if (k >= -1021) {   // e*2^k is normal (e >= 0.7)
        double r = __dadd_rn(e.hi, e.lo);
        return ldexp(r, k);
    }
    // subnormal result: round once on the 2^-1074 grid.  q = e * 2^(k+1074)
    // is exact (a power-of-two scaling into the normal range).
    const double qh = ldexp(e.hi, k + 1074), ql = ldexp(e.lo, k + 1074);
    double n = floor(qh);
    double r = __dadd_rn(__dsub_rn(qh, n), ql);
    while (r >= 1.0) { n += 1.0; r -= 1.0; }
    while (r < 0.0) { n -= 1.0; r += 1.0; }
    if (r > 0.5 || (r == 0.5 && fmod(n, 2.0) != 0.0)) n += 1.0;
    return ldexp(n, -1074);
}

// exp of a double-double argument as a double-double (for the log refinement).
__device__ __forceinline__ dd exp_dd(double x_hi) {
    int k;
    dd m1 = dd_exp_reduced({0.0, 0.0}, &k, x_hi);
    dd e = dd_add({1.0, 0.0}, m1);
    return {ldexp(e.hi, k), ldexp(e.lo, k)};
}

// Correctly rounded log(x) for normal positive x: one Newton step from the
// CUDA log (<= 1 ulp) against a double-double exp.
__device__ __forceinline__ double log_cr(double x) {
    if (!(x > 0.0)) return x == 0.0 ? __longlong_as_double(0xfff0000000000000LL)
                                     : __longlong_as_double(0x7ff8000000000000LL);
    if (x == 1.0) return 0.0;
    if (x < 2.2250738585072014e-308 || x > 1.7976931348623157e308) return log(x);
    double y0 = log(x);
    dd e = exp_dd(y0);
    // t = (x - e) / e   (x and e.hi agree to ~1 ulp: Sterbenz-exact subtraction)
    dd d = dd_add({x, 0.0}, {-e.hi, -e.lo});
    double t = __ddiv_rn(d.hi, e.hi);
    return __dadd_rn(y0, t);
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: kernels launched with launch_pdl may start
// (prologue, weight prefetch) while their predecessor drains; they must call
// pdl_wait() before reading anything the predecessor wrote.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#define CARD_PDL(kern, grid, block, smem, stream, ...)                        \
    do {                                                                      \
        cudaError_t _e = card::launch_pdl(kern, grid, block, smem, stream, __VA_ARGS__); \
        if (_e != cudaSuccess) {                                              \
            card::set_cuda_error(_e);                                         \
            return CARD_E_CUDA;                                               \
        }                                                                     \
    } while (0)

// ---------------------------------------------------------------- misc
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace card
