// Latency of the primitives the persistent forward's step boundaries are
// made of, on one SM of an otherwise idle B200: dependent L2 loads (pointer
// chase, near and whole-buffer), ld.acquire.gpu, atom.acq_rel.gpu, a store
// followed by fence + atomic, __nanosleep(32) and a 128-byte TMA-free
// load of a line another SM just wrote.  nvcc -arch=sm_100a -O3 lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long clk() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}

__global__ void chase(const int* __restrict__ next, int n, int steps, long long* out) {
    int i = 0;
    // warm
    for (int s = 0; s < steps; ++s) i = __ldcg(next + i);
    unsigned long long t0 = clk();
    for (int s = 0; s < steps; ++s) i = __ldcg(next + i);
    unsigned long long t1 = clk();
    out[0] = (long long)(t1 - t0) / steps;
    out[1] = i;
}

__global__ void prim(int* flag, int* data, long long* out) {
    const int n = 64;
    unsigned long long t0, t1;
    int v = 0;
    t0 = clk();
    for (int s = 0; s < n; ++s) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag + (v & 1)) : "memory");
    }
    t1 = clk();
    out[0] = (long long)(t1 - t0) / n;
    t0 = clk();
    for (int s = 0; s < n; ++s) {
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(flag + 2), "r"(1 + (v & 1)) : "memory");
        v += old;
    }
    t1 = clk();
    out[1] = (long long)(t1 - t0) / n;
    t0 = clk();
    for (int s = 0; s < n; ++s) {
        data[s * 32] = v;
        __threadfence();
        atomicAdd(flag + 3, 1);
    }
    t1 = clk();
    out[2] = (long long)(t1 - t0) / n;
    t0 = clk();
    for (int s = 0; s < n; ++s) __nanosleep(32);
    t1 = clk();
    out[3] = (long long)(t1 - t0) / n;
    t0 = clk();
    for (int s = 0; s < n; ++s) {
        int old;
        asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(flag + 4), "r"(1 + (v & 1)) : "memory");
        v += old;
    }
    t1 = clk();
    out[4] = (long long)(t1 - t0) / n;
    out[5] = v;
}

int main() {
    const int MB = 1 << 20;
    for (int size_mb : {1, 16, 64}) {
        int n = size_mb * MB / 4;
        int* h = new int[n];
        // random cyclic permutation at 128-byte granularity
        int lines = n / 32;
        int* perm = new int[lines];
        for (int i = 0; i < lines; ++i) perm[i] = i;
        unsigned s = 12345;
        for (int i = lines - 1; i > 0; --i) {
            s = s * 1103515245u + 12345u;
            int j = s % (i + 1);
            int t = perm[i];
            perm[i] = perm[j];
            perm[j] = t;
        }
        for (int i = 0; i < lines; ++i) h[perm[i] * 32] = perm[(i + 1) % lines] * 32;
        int* d;
        long long* o;
        cudaMalloc(&d, (size_t)n * 4);
        cudaMalloc(&o, 64);
        cudaMemcpy(d, h, (size_t)n * 4, cudaMemcpyHostToDevice);
        chase<<<1, 1>>>(d, n, 2000, o);
        long long r[2];
        cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
        printf("dependent __ldcg chase over %3d MB: %lld cycles/load\n", size_mb, r[0]);
        cudaFree(d);
        cudaFree(o);
        delete[] h;
        delete[] perm;
    }
    int* flag;
    int* data;
    long long* o;
    cudaMalloc(&flag, 64);
    cudaMalloc(&data, 64 * 32 * 4);
    cudaMalloc(&o, 64);
    cudaMemset(flag, 0, 64);
    prim<<<1, 1>>>(flag, data, o);
    long long r[6];
    cudaMemcpy(r, o, 48, cudaMemcpyDeviceToHost);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("ld.acquire.gpu: %lld cycles\natom.acq_rel.gpu: %lld\nstore + __threadfence + atomicAdd: %lld\n"
           "__nanosleep(32): %lld\natom.relaxed.gpu: %lld\n(SM clock attribute %d MHz)\n",
           r[0], r[1], r[2], r[3], r[4], clk_khz / 1000);
    return 0;
}
