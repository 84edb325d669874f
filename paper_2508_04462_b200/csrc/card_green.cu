// card_green.cu — SM partitions for running the draft and the target side by
// side on ONE GPU (mode="concurrent", the reference's two threads of
// engine.py:320-389).
//
// The draft step is latency-bound (dependent phases, ~30 % of HBM
// bandwidth) and the verify step is bandwidth-bound; in the concurrent
// schedule they overlap.  Sharing SMs kernel by kernel does not overlap them
// (the draft's persistent forward is a cooperative grid over every SM), so
// the GPU is split into two green contexts — disjoint SM partitions with a
// stream each.  Kernels (and CUDA graphs captured) on a partition's stream
// run only on its SMs; memory is the device's, shared with every context.
#include <cuda.h>
#include <stdlib.h>

#include "card_common.cuh"

namespace {

struct DriverApi {
    CUresult (*deviceGet)(CUdevice*, int);
    CUresult (*getDevResource)(CUdevice, CUdevResource*, CUdevResourceType);
    CUresult (*smSplit)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                        unsigned int);
    CUresult (*genDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int);
    CUresult (*greenCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
    CUresult (*greenDestroy)(CUgreenCtx);
    CUresult (*greenStream)(CUstream*, CUgreenCtx, unsigned int, int);
    CUresult (*streamDestroy)(CUstream);
    bool ok;
};

DriverApi& api() {
    static DriverApi d = {};
    static bool init = false;
    if (init) return d;
    init = true;
    auto get = [](const char* name, void** fn) {
        cudaDriverEntryPointQueryResult q;
        return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
               q == cudaDriverEntryPointSuccess;
    };
    d.ok = get("cuDeviceGet", (void**)&d.deviceGet) && get("cuDeviceGetDevResource", (void**)&d.getDevResource) &&
           get("cuDevSmResourceSplitByCount", (void**)&d.smSplit) &&
           get("cuDevResourceGenerateDesc", (void**)&d.genDesc) && get("cuGreenCtxCreate", (void**)&d.greenCreate) &&
           get("cuGreenCtxDestroy", (void**)&d.greenDestroy) &&
           get("cuGreenCtxStreamCreate", (void**)&d.greenStream) && get("cuStreamDestroy", (void**)&d.streamDestroy);
    return d;
}

}  // namespace

struct card_green {
    CUgreenCtx ctx[2];
    CUstream stream[2];
    int sms[2];
};

extern "C" {

int card_green_destroy(card_green* g) {
    if (!g) return CARD_OK;
    DriverApi& d = api();
    for (int i = 0; i < 2; ++i) {
        if (g->stream[i]) d.streamDestroy(g->stream[i]);
        if (g->ctx[i]) d.greenDestroy(g->ctx[i]);
    }
    free(g);
    return CARD_OK;
}

int card_green_create(int device, int draft_sms, card_green** out) {
    if (!out || draft_sms <= 0) return CARD_E_INPUT;
    *out = nullptr;
    DriverApi& d = api();
    if (!d.ok) return CARD_E_CONFIG;
    cudaSetDevice(device);
    cudaFree(0);   // the primary context exists (memory is shared with it)
    CUdevice dev;
    if (d.deviceGet(&dev, device) != CUDA_SUCCESS) return CARD_E_CUDA;
    CUdevResource all, grp, rest;
    if (d.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return CARD_E_CUDA;
    if ((unsigned)draft_sms >= all.sm.smCount) return CARD_E_CONFIG;
    // the target's partition is the split-off group, built for the largest
    // clusters (its split-K GEMMs run 8-CTA clusters at one CTA per SM); the
    // draft takes the remaining SMs (its attention clusters are 4 wide)
    unsigned int n = 1;
    const unsigned tgt = all.sm.smCount - (unsigned)draft_sms;
    if (d.smSplit(&grp, &n, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, tgt) != CUDA_SUCCESS ||
        n != 1)
        return CARD_E_CONFIG;
    card_green* g = (card_green*)calloc(1, sizeof(card_green));
    CUdevResource* res[2] = {&rest, &grp};   // [draft, target]
    for (int i = 0; i < 2; ++i) {
        CUdevResourceDesc desc;
        if (d.genDesc(&desc, res[i], 1) != CUDA_SUCCESS ||
            d.greenCreate(&g->ctx[i], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
            d.greenStream(&g->stream[i], g->ctx[i], CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
            card_green_destroy(g);
            return CARD_E_CUDA;
        }
        g->sms[i] = (int)res[i]->sm.smCount;
    }
    *out = g;
    return CARD_OK;
}

// partition 0 = draft, 1 = target: its stream (cudaStream_t) and SM count
int card_green_stream(card_green* g, int part, void** stream, int* sms) {
    if (!g || part < 0 || part > 1) return CARD_E_INPUT;
    if (stream) *stream = (void*)g->stream[part];
    if (sms) *sms = g->sms[part];
    return CARD_OK;
}

}  // extern "C"
