// Per-SM HBM -> shared-memory streaming rate: TMA bulk copies vs LDG.128 +
// STS vs both at once (tuning aid for the weight stream of the GEMMs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smbench tools/sm_stream_bench.cu
//   /tmp/smbench <ctas> <mode 0=tma 1=ldg 2=both> [MB per CTA]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kStage = 16384;
constexpr int kStages = 8;

__global__ void __launch_bounds__(384, 1) stream_kernel(const uint8_t* __restrict__ src, size_t per_cta, int mode,
                                                      unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[kStages];
    const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
    const int nblk = (int)(per_cta / kStage);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0)
        for (int i = 0; i < kStages; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    __syncthreads();
    unsigned long long acc = 0;
    // TMA part: warp 0 lane 0 streams blocks b with (mode 0: all) (mode 2: even b)
    if (warp == 0 && mode != 1) {
        if (threadIdx.x == 0) {
            uint32_t phase[kStages] = {0};
            int issued = 0, done = 0;
            const int step = mode == 2 ? 2 : 1;
            for (int b = 0; b < nblk; b += step) {
                const int s = issued % kStages;
                if (issued >= kStages) {   // wait for the block issued kStages ago
                    const uint32_t a = su32(&full[s]);
                    asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(a), "r"(phase[s]) : "memory");
                    phase[s] ^= 1;
                    acc += smem[s * kStage];
                    ++done;
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kStage) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(smem + s * kStage)),
                             "l"(base + (size_t)b * kStage), "r"(kStage), "r"(su32(&full[s])) : "memory");
                ++issued;
            }
            while (done < issued) {
                const int s = done % kStages;
                const uint32_t a = su32(&full[s]);
                asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(a), "r"(phase[s]) : "memory");
                phase[s] ^= 1;
                acc += smem[s * kStage];
                ++done;
            }
        }
    } else if (warp >= 4 && mode != 0) {
        // LDG part: warps 4..11 (256 threads) copy blocks b (mode 1: all, mode 2: odd b)
        // into a separate smem ring with 16-byte loads, 4 loads in flight per thread
        const int t = threadIdx.x - 128;
        uint8_t* ring = smem + kStages * kStage;
        const int step = mode == 2 ? 2 : 1;
        const int first = mode == 2 ? 1 : 0;
        int slot = 0;
        for (int b = first; b < nblk; b += step) {
            const uint4* s4 = reinterpret_cast<const uint4*>(base + (size_t)b * kStage);
            uint4 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w)
                             : "l"(s4 + t + 256 * j));
#pragma unroll
            for (int j = 0; j < 4; ++j) reinterpret_cast<uint4*>(ring + slot * kStage)[t + 256 * j] = v[j];
            slot = (slot + 1) % 4;
        }
        acc += ring[t];
    }
    if (acc == 0x123456789ull) *sink = acc;
}

int main(int argc, char** argv) {
    const int ctas = argc > 1 ? atoi(argv[1]) : 64;
    const int mode = argc > 2 ? atoi(argv[2]) : 0;
    const size_t mb = argc > 3 ? atoi(argv[3]) : 4;
    const size_t per_cta = mb << 20;
    uint8_t* src;
    unsigned long long* sink;
    cudaMalloc(&src, per_cta * ctas);
    cudaMemset(src, 1, per_cta * ctas);
    cudaMalloc(&sink, 8);
    uint8_t* flush;
    cudaMalloc(&flush, 256 << 20);
    const int smem = kStages * kStage + 4 * kStage;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        cudaEventRecord(a);
        stream_kernel<<<ctas, 384, smem>>>(src, per_cta, mode, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const cudaError_t e = cudaGetLastError();
    const double gbs = (double)per_cta * ctas / (best * 1e-3) / 1e9;
    printf("ctas %4d mode %d (%s): %.3f ms  total %.0f GB/s  per CTA %.1f GB/s  %s\n", ctas, mode,
           mode == 0 ? "tma " : mode == 1 ? "ldg " : "both", best, gbs, gbs / ctas, cudaGetErrorString(e));
    return 0;
}
