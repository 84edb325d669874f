// Probe: green-context SM partitions on B200 — do plain launches, cooperative
// launches and CUDA-graph replays on a green-context stream stay on its SMs?
// nvcc -gencode arch=compute_100a,code=sm_100a -o green_probe green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <set>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s failed: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

__global__ void smid_kernel(int* out) {
    if (threadIdx.x == 0) {
        int s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        out[blockIdx.x] = s;
    }
    // keep the block alive a little so blocks spread
    long long t0 = clock64();
    while (clock64() - t0 < 20000) {}
}

__global__ void coop_kernel(int* out, int* ctr) {
    if (threadIdx.x == 0) {
        int s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        out[blockIdx.x] = s;
        atomicAdd(ctr, 1);
        while (atomicAdd(ctr, 0) < (int)gridDim.x) {}   // grid-wide: all blocks co-resident
    }
}

__global__ void busy_kernel(unsigned long long* t, int slot) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(t + slot, 0ULL, t0);
    long long c0 = clock64();
    while (clock64() - c0 < 4000000) {}   // ~2 ms
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMax(t + slot + 1, t1);
    }
}

static std::set<int> sms(const std::vector<int>& v) { return std::set<int>(v.begin(), v.end()); }

int main() {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    RK(cudaSetDevice(0));
    RK(cudaFree(0));   // primary context
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    unsigned int want = 56;
    CUdevResource grp[1], rest;
    unsigned int n = 1;
    CK(cuDevSmResourceSplitByCount(grp, &n, &all, &rest, 0, want));
    printf("group: %u SMs, remaining: %u SMs\n", grp[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc da, db;
    CK(cuDevResourceGenerateDesc(&da, &grp[0], 1));
    CK(cuDevResourceGenerateDesc(&db, &rest, 1));
    CUgreenCtx ga, gb;
    CK(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sa, sb;
    CK(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
    int *d_out, *d_ctr;
    RK(cudaMalloc(&d_out, 4096 * 4));   // primary-context memory
    RK(cudaMalloc(&d_ctr, 4));
    std::vector<int> h(4096);
    // 1. plain launches
    for (int k = 0; k < 2; ++k) {
        cudaStream_t s = (cudaStream_t)(k == 0 ? sa : sb);
        smid_kernel<<<1184, 64, 0, s>>>(d_out);
        RK(cudaStreamSynchronize(s));
        RK(cudaMemcpy(h.data(), d_out, 1184 * 4, cudaMemcpyDeviceToHost));
        auto S = sms(std::vector<int>(h.begin(), h.begin() + 1184));
        printf("plain launch on %s stream: %zu distinct SMs (min %d max %d)\n", k == 0 ? "group" : "rest", S.size(),
               *S.begin(), *S.rbegin());
    }
    // 2. cooperative launch with grid = group SM count
    {
        RK(cudaMemset(d_ctr, 0, 4));
        int G = grp[0].sm.smCount;
        void* args[] = {&d_out, &d_ctr};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)coop_kernel, dim3(G), dim3(32), args, 0, (cudaStream_t)sa);
        printf("cooperative launch grid %d on group stream: %s\n", G, cudaGetErrorString(e));
        if (e == cudaSuccess) {
            RK(cudaStreamSynchronize((cudaStream_t)sa));
            RK(cudaMemcpy(h.data(), d_out, G * 4, cudaMemcpyDeviceToHost));
            auto S = sms(std::vector<int>(h.begin(), h.begin() + G));
            printf("  -> %zu distinct SMs\n", S.size());
        }
        RK(cudaMemset(d_ctr, 0, 4));
        e = cudaLaunchCooperativeKernel((void*)coop_kernel, dim3(G + 8), dim3(32), args, 0, (cudaStream_t)sa);
        printf("cooperative launch grid %d (> group) on group stream: %s\n", G + 8, cudaGetErrorString(e));
        cudaGetLastError();
        cudaStreamSynchronize((cudaStream_t)sa);
    }
    // 3. graph captured on the group stream, replayed on it and on a primary stream
    {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        RK(cudaStreamBeginCapture((cudaStream_t)sa, cudaStreamCaptureModeGlobal));
        smid_kernel<<<1184, 64, 0, (cudaStream_t)sa>>>(d_out);
        RK(cudaStreamEndCapture((cudaStream_t)sa, &g));
        RK(cudaGraphInstantiate(&ge, g, 0));
        RK(cudaGraphLaunch(ge, (cudaStream_t)sa));
        RK(cudaStreamSynchronize((cudaStream_t)sa));
        RK(cudaMemcpy(h.data(), d_out, 1184 * 4, cudaMemcpyDeviceToHost));
        auto S = sms(std::vector<int>(h.begin(), h.begin() + 1184));
        printf("graph replay on group stream: %zu distinct SMs\n", S.size());
        cudaStream_t ps;
        RK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
        RK(cudaGraphLaunch(ge, ps));
        RK(cudaStreamSynchronize(ps));
        RK(cudaMemcpy(h.data(), d_out, 1184 * 4, cudaMemcpyDeviceToHost));
        S = sms(std::vector<int>(h.begin(), h.begin() + 1184));
        printf("graph (captured on group) replayed on a primary stream: %zu distinct SMs\n", S.size());
        // captured on a primary stream, replayed on the group stream
        cudaGraph_t g2;
        cudaGraphExec_t ge2;
        RK(cudaStreamBeginCapture(ps, cudaStreamCaptureModeGlobal));
        smid_kernel<<<1184, 64, 0, ps>>>(d_out);
        RK(cudaStreamEndCapture(ps, &g2));
        RK(cudaGraphInstantiate(&ge2, g2, 0));
        RK(cudaGraphLaunch(ge2, (cudaStream_t)sa));
        RK(cudaStreamSynchronize((cudaStream_t)sa));
        RK(cudaMemcpy(h.data(), d_out, 1184 * 4, cudaMemcpyDeviceToHost));
        S = sms(std::vector<int>(h.begin(), h.begin() + 1184));
        printf("graph (captured on primary) replayed on the group stream: %zu distinct SMs\n", S.size());
    }
    // 3b. concurrency: a ~2 ms kernel on each partition at once; globaltimer start/end per launch
    {
        unsigned long long* d_t;
        RK(cudaMalloc(&d_t, 64));
        RK(cudaMemset(d_t, 0, 64));
        busy_kernel<<<grp[0].sm.smCount, 64, 0, (cudaStream_t)sa>>>(d_t, 0);
        busy_kernel<<<rest.sm.smCount, 64, 0, (cudaStream_t)sb>>>(d_t, 2);
        RK(cudaDeviceSynchronize());
        unsigned long long t[4];
        RK(cudaMemcpy(t, d_t, 32, cudaMemcpyDeviceToHost));
        printf("concurrent partitions: A [%.1f, %.1f] us, B [%.1f, %.1f] us (relative to A start)\n", 0.0,
               (t[1] - t[0]) / 1e3, ((long long)t[2] - (long long)t[0]) / 1e3, ((long long)t[3] - (long long)t[0]) / 1e3);
        // the same two kernels on two primary-context streams
        cudaStream_t p1, p2;
        cudaStreamCreateWithFlags(&p1, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&p2, cudaStreamNonBlocking);
        RK(cudaMemset(d_t, 0, 64));
        busy_kernel<<<56, 64, 0, p1>>>(d_t, 0);
        busy_kernel<<<92, 64, 0, p2>>>(d_t, 2);
        RK(cudaDeviceSynchronize());
        RK(cudaMemcpy(t, d_t, 32, cudaMemcpyDeviceToHost));
        printf("two primary streams:    A [%.1f, %.1f] us, B [%.1f, %.1f] us\n", 0.0, (t[1] - t[0]) / 1e3,
               ((long long)t[2] - (long long)t[0]) / 1e3, ((long long)t[3] - (long long)t[0]) / 1e3);
    }
    // 4. cluster launches of sizes 2, 4, 8 on both partitions, with and without the max-cluster split flag
    for (int flag = 0; flag < 2; ++flag) {
        CUdevResource g2[1], r2;
        unsigned int n2 = 1;
        CUresult rr = cuDevSmResourceSplitByCount(g2, &n2, &all, &r2,
                                                  flag ? CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE : 0, want);
        if (rr != CUDA_SUCCESS) { printf("split flag %d failed\n", flag); continue; }
        CUdevResource* parts[2] = {&g2[0], &r2};
        for (int k = 0; k < 2; ++k) {
            CUdevResourceDesc dd;
            CUgreenCtx gc;
            CUstream st;
            CK(cuDevResourceGenerateDesc(&dd, parts[k], 1));
            CK(cuGreenCtxCreate(&gc, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM));
            CK(cuGreenCtxStreamCreate(&st, gc, CU_STREAM_NON_BLOCKING, 0));
            for (int cs = 2; cs <= 16; cs *= 2) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs * 4);
                cfg.blockDim = dim3(64);
                cfg.stream = (cudaStream_t)st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                if (cs == 16) cudaFuncSetAttribute(smid_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaError_t e = cudaLaunchKernelEx(&cfg, smid_kernel, d_out);
                cudaError_t e2 = cudaStreamSynchronize((cudaStream_t)st);
                printf("flag %d %s (%u SMs) cluster %d: launch %s, sync %s\n", flag, k ? "rest " : "group",
                       parts[k]->sm.smCount, cs, cudaGetErrorString(e), cudaGetErrorString(e2));
                cudaGetLastError();
            }
        }
    }
    printf("done\n");
    return 0;
}
