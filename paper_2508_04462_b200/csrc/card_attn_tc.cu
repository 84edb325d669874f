// card_attn_tc.cu — tree / chain attention on the 5th-generation tensor cores.
//
// Row r of a forward attends to the prefix KV positions [0, plen[r]) plus the
// n_extra[r] KV slots listed in extra[r][..] (its tree ancestors and itself):
// the tree mask of mask.py:173-217 without materialising it.  Causal chains
// (target verify, draft catch-up, prefill) have plen = pos + 1 and no extras.
// Prefix positions map to KV slots through an optional page table (pages of
// 64 slots: slot = table[p / 64] * 64 + p % 64); extras are slots already.
//
// Grid (S, n_qt, nkv), thread-block cluster (S, 1, 1).  A CTA owns 128
// query-heads (row r, head h of kv head g's GQA group, ordered (r, h)) and
// the key list of its tile: [0, Kp) prefix positions (Kp = the tile's
// largest plen), then the tile rows' extra slots row after row.  The list is
// cut into rounds of 128 keys dealt to the S cluster ranks.  Per round:
//
//   loader warps   gather the round's K and V rows (cp.async, 16-byte
//                  chunks written in the SWIZZLE_128B layout the UMMA
//                  descriptors expect) into a double-buffered ring;
//   MMA thread     S = Q K^T   tcgen05.mma M=128 N=128 K=hd  -> TMEM (two
//                  S buffers: S of round i+1 is issued while round i is in
//                  softmax), then O_i = P V  M=128 N=hd K=128 -> TMEM, with P
//                  from shared memory (K-major) and V as an MN-major operand;
//   softmax warps  one thread per query-head = TMEM lane: row max over the
//                  valid keys (prefix range / own extras), p = exp(s - m) as
//                  bf16 into P, running (m, l), and O_acc = O_acc * alpha + O_i
//                  from TMEM (tcgen05.ld) into registers.
//
// The S ranks' partials (m, l, O) are pushed into the owner rank's shared
// memory (st.shared::cluster) and merged in rank order (deterministic); the
// owner writes o (bf16) for the o-projection GEMM.
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>

#include "card_common.cuh"
#include "card_llm.h"

namespace card {
namespace {

constexpr int kQT = 128;        // query-heads per tile = MMA M = TMEM lanes
constexpr int kKB = 128;        // keys per round = S MMA N = PV MMA K
constexpr int kMaxX = 1024;     // gathered extra keys per tile
constexpr int kMaxRows = 136;   // token rows per tile (GQA group >= 1)
constexpr int kMaxSeg = 64;     // request segments per tile (batched forwards)
constexpr int kSoftWarps = 8, kMmaWarp = 8, kLoadWarp0 = 9, kLoadWarps = 3;   // 12 warps: up to 168 registers
constexpr int kThreads = (kLoadWarp0 + kLoadWarps) * 32;   // 384
constexpr int kSub = 128 * 64 * 2;   // one [128 rows x 64 bf16] SW128 sub-block (16 KB)
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
#ifdef CARD_ATTN_WATCHDOG
#include <stdio.h>
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    for (long long it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred P;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P;\n\t}"
            : "=r"(ok)
            : "r"(su32(b)), "r"(parity)
            : "memory");
        if (ok) return;
        if (it == 20000000) {
            printf("attn_tc watchdog: block (%d,%d,%d) thread %d barrier smem 0x%x parity %u\n", blockIdx.x, blockIdx.y,
                   blockIdx.z, threadIdx.x, su32(b), parity);
            return;
        }
    }
}
#else
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra W_%=;\n\t}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
#endif
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
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
// K-major SWIZZLE_128B operand: 128-byte rows, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
// MN-major SWIZZLE_128B operand (V as the B of P.V): a 128-byte row holds 64
// consecutive N (head-dim) elements of one K (key) row; 8-key groups 1024 B
// apart (SBO); the next 64 N elements start one [128 x 64] sub-block later (LBO)
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(kSub >> 4) << 16) | ((uint64_t)64 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// byte offset of 16-byte chunk c (0..7) of row r in a [rows x 64 bf16] SW128 block
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// 3D TMA box (KV cache [slots, nkv, hd]: {64 dims, 1 head, 64 slots}) -> SW128 rows
__device__ __forceinline__ void tma3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void st16_zero(uint32_t dst) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0u) : "memory");
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_map(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cl_v4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void st_cl_v2(uint32_t addr, float a, float b) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
// remote shared-memory stores that complete_tx on the destination CTA's mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t addr, float a, float b, float c, float d, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     addr),
                 "f"(a), "f"(b), "f"(c), "f"(d), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, float a, float b, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "f"(a), "f"(b), "r"(bar)
                 : "memory");
}

__device__ unsigned long long* g_tc_trace = nullptr;   // tuning: [grid][8] %globaltimer stamps
__device__ __forceinline__ void tc_stamp(int k) {
    if (g_tc_trace && threadIdx.x == 0) {
        unsigned long long v;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
        g_tc_trace[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 8 + k] = v;
    }
}

struct TcAttnArgs {
    const float* q;   // [M, nh, hd] fp32, pre-scaled by 1/sqrt(hd)
    const int32_t* dM;
    const int32_t* plen;
    const int32_t* n_extra;
    const int32_t* extra;
    int extra_max;
    const __nv_bfloat16* kc;
    const __nv_bfloat16* vc;
    const int32_t* page_table;   // null: prefix position p is slot p
    int nh, nkv;
    __nv_bfloat16* o;   // [M, nh, hd]
    const uint8_t* qsw;   // non-null: Q tiles pre-swizzled bf16 (card_pfwd_set_qsw layout), q unused
    int qsw_tiles;
    // batched forwards: rows [i * seg_rows, (i + 1) * seg_rows) belong to
    // request i, whose prefix positions resolve through page_table + i *
    // pt_stride (seg_rows == 0: one request, page_table as is)
    int seg_rows, pt_stride;
};

template <int HD>
struct Smem {
    static constexpr int kNB = HD == 64 ? 2 : 1;       // K/V ring depth (hd 128: one round in flight)
    static constexpr int kQ = HD / 64 * kSub;          // Q tile [128 x HD]
    static constexpr int kKV = HD / 64 * kSub;         // one K (or V) round [128 keys x HD]
    static constexpr int kP = 2 * kSub;                // P [128 x 128 keys]
    // hd 64: P and O double-buffered, so the O accumulation of a round is
    // deferred behind the next round's softmax (TMEM: S 128 + 2 x O 64)
    static constexpr bool kDefer = HD == 64;
    static constexpr int kPB = kDefer ? 2 : 1;
    static constexpr int kRecvLd = HD + 4;             // merge record [m, l, pad, pad, O[HD]]
    static constexpr int oQ = 0, oK = kQ, oV = oK + kNB * kKV, oP = oV + kNB * kKV, oR = oP + kPB * kP;
    static constexpr int oMeta = oR + kQT * kRecvLd * 4;   // recv: one record per query-head row
    // meta: ext_slot[kMaxX], rplen/rnx/rxo[kMaxRows], xch[2][128], bars, tmem slot,
    // segment table seg_vb[kMaxSeg + 1] / seg_kp[kMaxSeg]
    static constexpr int kMeta = kMaxX * 4 + 3 * kMaxRows * 4 + 16 + 2 * kQT * 4 + 16 * 8 + 16 + (2 * kMaxSeg + 4) * 4;
    static constexpr int kTotal = oMeta + kMeta + 1024;   // + alignment slack
};

}  // namespace

template <int HD>
__global__ void __launch_bounds__(kThreads, 1) attn_tc_kernel(const __grid_constant__ TcAttnArgs a,
                                                              const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV) {
    using L = Smem<HD>;
    constexpr int HH = HD / 2;   // O columns per softmax half
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sQ = sm + L::oQ;
    uint8_t* sK = sm + L::oK;
    uint8_t* sV = sm + L::oV;
    uint8_t* sP = sm + L::oP;
    float* recv = reinterpret_cast<float*>(sm + L::oR);   // [S][RO][kRecvLd] partials of my rows
    int32_t* ext_slot = (int32_t*)(sm + L::oMeta);
    int32_t* rplen = ext_slot + kMaxX;
    int32_t* rnx = rplen + kMaxRows;
    int32_t* rxo = rnx + kMaxRows;
    int32_t* s_old = rxo + kMaxRows;          // prefix keys [0, s_old) predate this forward
    float* xch = (float*)(rxo + kMaxRows + 4);   // [2][128] half-row max / sum exchange
    uint64_t* bars = (uint64_t*)(xch + 2 * kQT);
    uint64_t* kv_full = bars;        // [2] loaders -> MMA
    uint64_t* kv_empty = bars + 2;   // [2] MMA commit -> loaders
    uint64_t* s_full = bars + 4;     // MMA commit -> softmax
    uint64_t* s_empty = bars + 6;    // softmax -> MMA
    uint64_t* p_full = bars + 8;     // softmax -> MMA
    // MMA commit -> softmax / softmax -> MMA, per O buffer (bars 9, 10 and 14, 15)
    auto o_full_b = [&](int ob) { return bars + (ob ? 14 : 9); };
    auto o_empty_b = [&](int ob) { return bars + (ob ? 15 : 10); };
    uint64_t* recv_bar = bars + 11;  // every rank's partials of my rows landed (st.async complete_tx)
    uint32_t* tmem_slot = (uint32_t*)(bars + 12);
    uint64_t* q_full = bars + 13;    // pre-swizzled Q tile landed (bulk copy)
    int32_t* seg_vb = (int32_t*)(bars + 16);   // [n_seg + 1] first virtual key of each segment's prefix rounds
    int32_t* seg_kp = seg_vb + kMaxSeg + 1;    // [n_seg] prefix keys of the segment (max plen of its rows)

    const int S = gridDim.x;
    const int rank = (int)cl_rank();
    const int qt = blockIdx.y, g = blockIdx.z;
    const int M = *a.dM;
    const int G = a.nh / a.nkv;
    const int nq = M * G;
    const int q0 = qt * kQT;
    if (q0 >= nq) return;   // every rank of the cluster shares qt: consistent exit
    tc_stamp(0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r_lo = q0 / G;
    const int r_hi = min(M, (q0 + kQT - 1) / G + 1);
    const int n_rows = r_hi - r_lo;

    // ---- row metadata (written before the previous kernel started: safe before the PDL wait)
    for (int i = threadIdx.x; i < n_rows; i += kThreads) {
        rplen[i] = a.plen[r_lo + i];
        rnx[i] = a.n_extra ? a.n_extra[r_lo + i] : 0;
    }
    if (threadIdx.x == 0) *s_old = 0x7fffffff;
    if (threadIdx.x == kMmaWarp * 32) {
        for (int i = 0; i < 2; ++i) {
            bar_init(&kv_full[i], kLoadWarps * 32);
            bar_init(&kv_empty[i], 1);
        }
        bar_init(s_full, 1);
        bar_init(s_empty, kSoftWarps * 32);
        bar_init(p_full, kSoftWarps * 32);
        for (int i = 0; i < 2; ++i) {
            bar_init(o_full_b(i), 1);
            bar_init(o_empty_b(i), kSoftWarps * 32);
        }
        bar_init(recv_bar, 1);
        bar_init(q_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (S > 1) {   // bytes the S ranks will push for my live rows
            const int RO = kQT / S;
            const int live = max(0, min(RO, nq - q0 - rank * RO));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(recv_bar)),
                         "r"((uint32_t)(live * S * (8 + 4 * HD)))
                         : "memory");
        }
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    // cluster-wide: every rank's recv barrier is initialised before anyone pushes
    if (S > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    tc_stamp(1);
    {   // the forward's own KV rows (chain rows write position plen - 1) are the
        // only prefix keys the previous kernels are still producing
        int mn = 0x7fffffff;
        for (int r = threadIdx.x; r < M; r += kThreads)
            if (!a.n_extra || a.n_extra[r] == 0) mn = min(mn, a.plen[r] - 1);
        if (mn != 0x7fffffff) atomicMin(s_old, mn);
    }
    int Kp = 0, Kx = 0;
    for (int i = 0; i < n_rows; ++i) {
        Kp = max(Kp, rplen[i]);
        Kx += rnx[i];
    }
    if (Kx > kMaxX) Kx = kMaxX;   // host guarantees rows * extra_max <= kMaxX
    // request segments of the tile's rows (one unless batched)
    const bool segm = a.seg_rows > 0;
    const int s_lo = segm ? r_lo / a.seg_rows : 0;
    const int n_seg = segm ? (r_hi - 1) / a.seg_rows - s_lo + 1 : 1;
    if (threadIdx.x == 0) {
        int x = 0;
        for (int i = 0; i < n_rows; ++i) {
            rxo[i] = x;
            x += rnx[i];
        }
        int vb = 0;
        for (int k = 0; k < n_seg; ++k) {
            int kp = 0;
            for (int i = 0; i < n_rows; ++i)
                if (!segm || (r_lo + i) / a.seg_rows == s_lo + k) kp = max(kp, rplen[i]);
            seg_vb[k] = vb;
            seg_kp[k] = kp;
            vb += (kp + kKB - 1) / kKB * kKB;
        }
        seg_vb[n_seg] = vb;
    }
    __syncthreads();
    for (int i = warp; i < n_rows; i += kThreads / 32) {
        const int n = rnx[i], xo = rxo[i];
        for (int j = lane; j < n && xo + j < kMaxX; j += 32)
            ext_slot[xo + j] = a.extra[(int64_t)(r_lo + i) * a.extra_max + j];
    }
    // Key rounds of 128: prefix positions [128 R, 128 R + 128) for R < n_pr,
    // then the gathered extras from virtual key XB = 128 n_pr on.  Rank s
    // takes rounds s, s + S, ...  The prefix rounds are anchored at position
    // 0 whatever the tile's rows, so a row's keys meet the same rounds, ranks
    // and summation order in an M = 1 decode step and in an M = r + 1 verify
    // (greedy CARD emits exactly the AR tokens).
    const int XB = seg_vb[n_seg];   // = 128 ceil(Kp / 128) for one segment
    const int n_pr = XB / kKB;
    const int n_tot = n_pr + (Kx + kKB - 1) / kKB;
    const int nr = rank < n_tot ? (n_tot - rank + S - 1) / S : 0;

    __syncthreads();   // ext_slot / s_old complete
    // Prefix rounds load by TMA: the round's two 64-key pages of K and V of
    // this kv head, one box per (page, 64-dim sub-block), straight into the
    // SW128 layout the UMMA descriptors read.  A page past the segment's
    // keys reloads its last page (finite values the softmax masks).  The
    // issuing loader thread's arrival is the expect_tx.
    auto tma_round = [&](int li) {
        const int b = li % L::kNB;
        const int j0 = (rank + li * S) * kKB;
        int sg = 0;
        while (j0 >= seg_vb[sg + 1]) ++sg;
        const int pp0 = j0 - seg_vb[sg];
        const int last_pg = seg_kp[sg] > 0 ? (seg_kp[sg] - 1) >> 6 : 0;
        const int32_t* pt = a.page_table ? a.page_table + (int64_t)(s_lo + sg) * a.pt_stride : nullptr;
        const uint32_t bar = su32(&kv_full[b]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)(2 * 2 * (HD / 64) * 8192))
                     : "memory");
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int pg = min((pp0 >> 6) + half, last_pg);
            const int slot0 = (pt ? pt[pg] : pg) * 64;
#pragma unroll
            for (int sb = 0; sb < HD / 64; ++sb) {
                const uint32_t off = (uint32_t)(sb * kSub + half * 8192);
                tma3d(su32(sK + b * L::kKV) + off, &tmK, bar, sb * 64, g, slot0);
                tma3d(su32(sV + b * L::kKV) + off, &tmV, bar, sb * 64, g, slot0);
            }
        }
    };
    int early = 0;   // prefix rounds whose pages all predate this forward, issued before the PDL wait
    if (warp >= kLoadWarp0 && threadIdx.x == kLoadWarp0 * 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
        const int old = segm ? 0 : min(*s_old, Kp);
        for (int li = 0; li < min(nr, L::kNB); ++li) {
            const int j0 = (rank + li * S) * kKB;
            if (j0 < XB && j0 + kKB <= old) {
                tma_round(li);
                early |= 1 << li;
            }
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");             // q and this forward's K/V rows are ready
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    tc_stamp(2);

    // ---- Q tile (softmax + MMA warps; the loaders go straight to this
    // forward's new K/V rows): fp32 -> bf16, SW128 K-major; or one bulk copy
    // of the tile the qkv epilogue already wrote in that layout
    if (a.qsw) {
        if (threadIdx.x == kMmaWarp * 32) {
            constexpr uint32_t qbytes = HD / 64 * kSub;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(q_full)), "r"(qbytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(sQ)),
                "l"(a.qsw + (size_t)(g * a.qsw_tiles + qt) * qbytes), "r"(qbytes), "r"(su32(q_full))
                : "memory");
        }
    } else if (warp < kLoadWarp0) {
#pragma unroll 4
        for (int idx = threadIdx.x; idx < kQT * (HD / 8); idx += kLoadWarp0 * 32) {
            const int t = idx / (HD / 8), c = idx % (HD / 8);
            const int qh = q0 + t;
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            if (qh < nq) {
                const int r = qh / G, head = g * G + qh % G;
                const float4* src = (const float4*)(a.q + ((int64_t)r * a.nh + head) * HD + c * 8);
                const float4 x0 = src[0], x1 = src[1];
                w[0] = pack_bf2(x0.x, x0.y);
                w[1] = pack_bf2(x0.z, x0.w);
                w[2] = pack_bf2(x1.x, x1.y);
                w[3] = pack_bf2(x1.z, x1.w);
            }
            const uint32_t dst = su32(sQ + (c >> 3) * kSub) + sw_off(t, c & 7);
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                         "r"(w[3])
                         : "memory");
        }
        fence_async_smem();
        named_bar_sync(5, kLoadWarp0 * 32);   // Q visible to the MMA issuer
    }
    tc_after();
    tc_stamp(3);
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem;          // S of the current round (128 columns)
    const uint32_t tO = tmem + 128;    // O of the current round (hd columns; hd 64: two buffers)

    // softmax state: warp w owns TMEM lanes 32 (w % 4) .. and S columns / O
    // columns of half h = w / 4; (m, l) of a row are shared by its two halves
    float m_run = -INFINITY, l_run = 0.f;
    float oacc[HH];
#pragma unroll
    for (int d = 0; d < HH; ++d) oacc[d] = 0.f;
    const int t = threadIdx.x & (kQT - 1);   // query-head row (softmax warps)
    const int h = warp >> 2;

    if (warp >= kLoadWarp0) {
        // ------------------------------------------------ loaders
        const int lt = threadIdx.x - kLoadWarp0 * 32;
        // virtual keys [jlo, jhi) of round li: cp.async into the ring slot, zeros for padding
        auto gather = [&](int li, int jlo, int jhi) {
            const int j0 = (rank + li * S) * kKB;
            const int b = li % L::kNB;
            const uint32_t kb = su32(sK + b * L::kKV), vb = su32(sV + b * L::kKV);
            const int k_lo = max(0, jlo - j0), k_hi = min(kKB, jhi - j0);
            for (int idx = k_lo * (HD / 8) + lt; idx < k_hi * (HD / 8); idx += kLoadWarps * 32) {
                const int kk = idx / (HD / 8), c = idx % (HD / 8);
                const int j = j0 + kk;
                const uint32_t off = (uint32_t)((c >> 3) * kSub) + sw_off(kk, c & 7);
                int sg = 0;   // the key's segment (prefix part)
                if (j < XB)
                    while (j >= seg_vb[sg + 1]) ++sg;
                const int pp = j - seg_vb[sg];
                if (j < XB ? pp < seg_kp[sg] : j - XB < Kx) {
                    int slot;
                    if (j < XB) {
                        const int32_t* pt = a.page_table ? a.page_table + (int64_t)(s_lo + sg) * a.pt_stride : nullptr;
                        slot = pt ? pt[pp >> 6] * 64 + (pp & 63) : pp;
                    } else {
                        slot = ext_slot[j - XB];
                    }
                    const int64_t e = ((int64_t)slot * a.nkv + g) * HD + c * 8;
                    cp16(kb + off, a.kc + e);
                    cp16(vb + off, a.vc + e);
                } else {
                    st16_zero(kb + off);
                    st16_zero(vb + off);
                }
            }
        };
        for (int li = 0; li < nr; ++li) {
            const int b = li % L::kNB;
            const int j0 = (rank + li * S) * kKB;
            if (li >= L::kNB) bar_wait(&kv_empty[b], ((li / L::kNB) - 1) & 1);
            if (j0 < XB) {   // prefix round: TMA (thread 0's arrival is its expect_tx)
                if (lt == 0) {
                    if (!((early >> li) & 1)) tma_round(li);
                } else {
                    bar_arrive(&kv_full[b]);
                }
            } else {         // tree extras: gathered slot by slot
                gather(li, j0, j0 + kKB);
                asm volatile("cp.async.wait_all;" ::: "memory");
                fence_async_smem();
                bar_arrive(&kv_full[b]);
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0 && nr > 0) {
            const uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kKB >> 3) << 17) |
                                 ((uint32_t)(kQT >> 4) << 24);
            const uint32_t idO = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) |
                                 ((uint32_t)(kQT >> 4) << 24);
            const uint32_t q_s = su32(sQ), p_s = su32(sP);
            if (a.qsw) bar_wait(q_full, 0);
            for (int li = 0; li < nr; ++li) {
                const int b = li % L::kNB;
                bar_wait(&kv_full[b], (li / L::kNB) & 1);
                if (li >= 1) bar_wait(s_empty, (li - 1) & 1);   // softmax has read S of the last round
                tc_after();
                const uint32_t k_s = su32(sK + b * L::kKV);
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const uint32_t o = (uint32_t)((k >> 2) * kSub + (k & 3) * 32);
                    tc_mma(tS, desc_kmajor(q_s + o), desc_kmajor(k_s + o), idS, k > 0 ? 1u : 0u);
                }
                tc_commit(s_full);
                bar_wait(p_full, li & 1);
                const int ob = L::kDefer ? (li & 1) : 0;
                if (L::kDefer) {
                    if (li >= 2) bar_wait(o_empty_b(ob), ((li - 2) >> 1) & 1);   // O of round li-2 accumulated
                } else if (li >= 1) {
                    bar_wait(o_empty_b(0), (li - 1) & 1);
                }
                tc_after();
                const uint32_t v_s = su32(sV + b * L::kKV);
                const uint32_t p_b = p_s + (uint32_t)(ob * L::kP);
                const uint32_t t_o = tO + (uint32_t)(ob * HD);
#pragma unroll
                for (int k = 0; k < kKB / 16; ++k) {
                    const uint32_t pa = p_b + (uint32_t)((k >> 2) * kSub + (k & 3) * 32);
                    tc_mma(t_o, desc_kmajor(pa), desc_mnmajor(v_s + (uint32_t)(k * 2048)), idO, k > 0 ? 1u : 0u);
                }
                tc_commit(o_full_b(ob));
                tc_commit(&kv_empty[b]);
            }
        }
    } else {
        // ------------------------------------------------ softmax (8 warps: 2 per TMEM lane quarter)
        const int qh = q0 + t;
        const bool live = qh < nq;
        const int ri = live ? qh / G - r_lo : 0;
        // valid keys of this row: [p0, plim) prefix (its segment's rounds), [e0, e1) its own extras
        const int sg = segm && live ? (r_lo + ri) / a.seg_rows - s_lo : 0;
        const int p0 = seg_vb[sg];
        const int plim = live ? p0 + min(rplen[ri], seg_kp[sg]) : 0;
        const int e0 = live ? XB + rxo[ri] : 0, e1 = live ? XB + rxo[ri] + rnx[ri] : 0;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const int pair_bar = 1 + (warp & 3);   // named barrier of warps w and w + 4
        float alpha_prev = 0.f;
        // O_acc = O_acc * alpha + O of round r (TMEM buffer r & 1 when double-buffered)
        auto accumulate_o = [&](int r, float alpha) {
            const int ob = L::kDefer ? (r & 1) : 0;
            bar_wait(o_full_b(ob), L::kDefer ? ((r >> 1) & 1) : (r & 1));
            tc_after();
            uint32_t orr[HH / 16][16];
#pragma unroll
            for (int c = 0; c < HH / 16; ++c)
                tmem_ld16_issue(tO + (uint32_t)(ob * HD) + lane_off + (uint32_t)(h * HH + c * 16), orr[c]);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < HH / 16; ++c)
#pragma unroll
                for (int u = 0; u < 16; ++u) oacc[c * 16 + u] = fmaf(oacc[c * 16 + u], alpha, __uint_as_float(orr[c][u]));
            tc_before();
            bar_arrive(o_empty_b(ob));
        };
        for (int li = 0; li < nr; ++li) {
            const int b = li & 1;
            const int j0 = (rank + li * S) * kKB;
            bar_wait(s_full, li & 1);
            if (li == 0) tc_stamp(5);   // (thread 0: the first S is in TMEM)
            tc_after();
            // 16-column validity masks of my half (c = 4h .. 4h+3)
            uint32_t msk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int jc = j0 + (4 * h + q) * 16;
                const int lim = plim - jc;
                uint32_t m = lim >= 16 ? 0xFFFFu : (lim > 0 ? (1u << lim) - 1u : 0u);
                const int lo = p0 - jc;   // 0 for a single segment
                if (lo > 0) m &= lo >= 16 ? 0u : ~((1u << lo) - 1u);
                const int x0 = max(0, e0 - jc), x1 = min(16, e1 - jc);
                if (x1 > x0) m |= ((1u << x1) - 1u) & ~((1u << x0) - 1u);
                msk[q] = m;
            }
            // my half of S in one batch of TMEM loads (one wait), kept in
            // registers for both passes; S's TMEM is free for the next round
            uint32_t sr[4][16];
            bool need[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                need[q] = __any_sync(0xffffffffu, msk[q] != 0u);
                if (need[q]) tmem_ld16_issue(tS + lane_off + (uint32_t)((4 * h + q) * 16), sr[q]);
            }
            tmem_wait_ld();
            tc_before();
            bar_arrive(s_empty);
            float mx = -INFINITY;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!need[q]) continue;
#pragma unroll
                for (int u = 0; u < 16; ++u) mx = ((msk[q] >> u) & 1u) ? fmaxf(mx, __uint_as_float(sr[q][u])) : mx;
            }
            xch[h * kQT + t] = mx;
            named_bar_sync(pair_bar, 64);
            const float m_new = fmaxf(m_run, fmaxf(mx, xch[(h ^ 1) * kQT + t]));
            const float mb = (m_new == -INFINITY) ? 0.f : m_new * kLog2e;
            float sum = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c = 4 * h + q;
                uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                if (need[q]) {
                    const uint32_t* v = sr[q];
#pragma unroll
                    for (int u = 0; u < 16; u += 2) {
                        const float p0 = ((msk[q] >> u) & 1u) ? exp2f(fmaf(__uint_as_float(v[u]), kLog2e, -mb)) : 0.f;
                        const float p1 =
                            ((msk[q] >> (u + 1)) & 1u) ? exp2f(fmaf(__uint_as_float(v[u + 1]), kLog2e, -mb)) : 0.f;
                        w[u >> 1] = pack_bf2(p0, p1);
                        const __nv_bfloat162 pr = *reinterpret_cast<__nv_bfloat162*>(&w[u >> 1]);
                        sum += __bfloat162float(pr.x) + __bfloat162float(pr.y);   // l sums what P.V uses
                    }
                }
                const uint32_t base = su32(sP + (L::kDefer ? (li & 1) * L::kP : 0) + (c >> 2) * kSub);
                const int ch = (c & 3) * 2;
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(base + sw_off(t, ch)), "r"(w[0]),
                             "r"(w[1]), "r"(w[2]), "r"(w[3])
                             : "memory");
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(base + sw_off(t, ch + 1)), "r"(w[4]),
                             "r"(w[5]), "r"(w[6]), "r"(w[7])
                             : "memory");
            }
            fence_async_smem();
            tc_before();
            bar_arrive(p_full);
            const float alpha = (m_run == -INFINITY) ? 0.f : exp2f((m_run - m_new) * kLog2e);
            l_run = l_run * alpha + sum;   // this half's share of l
            m_run = m_new;
            if (L::kDefer) {
                // O of the previous round, now that this round's P is out
                // (same accumulation order: O = O * alpha_r + O_r, r ascending)
                if (li >= 1) accumulate_o(li - 1, alpha_prev);
                alpha_prev = alpha;
            } else {
                accumulate_o(li, alpha);
            }
        }
        if (L::kDefer && nr >= 1) accumulate_o(nr - 1, alpha_prev);
        // the row's l = both halves' shares
        named_bar_sync(pair_bar, 64);
        xch[h * kQT + t] = l_run;
        named_bar_sync(pair_bar, 64);
        l_run += xch[(h ^ 1) * kQT + t];
    }
    tc_before();
    __syncthreads();
    tc_stamp(4);
    if (warp == kMmaWarp) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }

    // ---- combine the S ranks' partials (m, l, O) per query-head row
    if (S == 1) {
        if (warp < kSoftWarps) {
            const int qh = q0 + t;
            if (qh < nq) {
                const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
                const int r = qh / G, head = g * G + qh % G;
                __nv_bfloat16* dst = a.o + ((int64_t)r * a.nh + head) * HD + h * HH;
#pragma unroll
                for (int d = 0; d < HH; d += 8) {
                    uint4 w;
                    w.x = pack_bf2(oacc[d] * inv, oacc[d + 1] * inv);
                    w.y = pack_bf2(oacc[d + 2] * inv, oacc[d + 3] * inv);
                    w.z = pack_bf2(oacc[d + 4] * inv, oacc[d + 5] * inv);
                    w.w = pack_bf2(oacc[d + 6] * inv, oacc[d + 7] * inv);
                    *reinterpret_cast<uint4*>(dst + d) = w;
                }
            }
        }
        return;
    }
    // every rank pushes its partial (m, l, O) of each live row into the owner
    // rank's recv slot with st.async; the owner's recv_bar completes when all
    // bytes landed (no cluster barrier on this path)
    const int RO = kQT / S;   // rows owned per rank
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp < kSoftWarps && q0 + t < nq) {
        const int owner = t / RO, row = t % RO;
        const uint32_t base = cl_map(su32(recv + ((size_t)rank * RO + row) * L::kRecvLd), (uint32_t)owner);
        const uint32_t rbar = cl_map(su32(recv_bar), (uint32_t)owner);
        if (h == 0) st_async_v2(base, m_run, l_run, rbar);
#pragma unroll
        for (int d = 0; d < HH; d += 4)
            st_async_v4(base + (uint32_t)(4 + h * HH + d) * 4, oacc[d], oacc[d + 1], oacc[d + 2], oacc[d + 3], rbar);
    }
    bar_wait(recv_bar, 0);
    tc_stamp(6);
    for (int idx = threadIdx.x; idx < RO * (HD / 4); idx += kThreads) {
        const int row = idx / (HD / 4), d = (idx % (HD / 4)) * 4;
        const int tt = rank * RO + row, qh = q0 + tt;
        if (qh >= nq) continue;
        float mm = -INFINITY;
        for (int s = 0; s < S; ++s) mm = fmaxf(mm, recv[((size_t)s * RO + row) * L::kRecvLd]);
        float l = 0.f, o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
        for (int s = 0; s < S; ++s) {   // rank order: deterministic
            const float* rec = recv + ((size_t)s * RO + row) * L::kRecvLd;
            const float ms = rec[0];
            const float w = (ms == -INFINITY) ? 0.f : exp2f((ms - mm) * kLog2e);
            l = fmaf(rec[1], w, l);
            o0 = fmaf(rec[4 + d], w, o0);
            o1 = fmaf(rec[5 + d], w, o1);
            o2 = fmaf(rec[6 + d], w, o2);
            o3 = fmaf(rec[7 + d], w, o3);
        }
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const int r = qh / G, head = g * G + qh % G;
        __nv_bfloat16* dst = a.o + ((int64_t)r * a.nh + head) * HD + d;
        uint2 w;
        w.x = pack_bf2(o0 * inv, o1 * inv);
        w.y = pack_bf2(o2 * inv, o3 * inv);
        *reinterpret_cast<uint2*>(dst) = w;
    }
    tc_stamp(7);
}

// Host side --------------------------------------------------------------
int attn_tc_set_trace(unsigned long long* buf) {
    return cudaMemcpyToSymbol(g_tc_trace, &buf, sizeof(buf)) == cudaSuccess ? CARD_OK : CARD_E_CUDA;
}

bool attn_tc_fits(int m_max, int nh, int nkv, int hd, int extra_max) {
    if (hd != 64 && hd != 128) return false;
    const int G = nh / nkv;
    const int rows = kQT / G + 2;
    return rows <= kMaxRows && (int64_t)rows * extra_max <= kMaxX;
}
int attn_tc_max_segments() { return kMaxSeg; }

// ranks per tile: enough CTAs to cover the SMs once.  A function of the tile
// count alone (not of M or the context length), so a verify row and the same
// token decoded alone see the same key rounds on the same ranks.
static int attn_tc_ranks(int tiles) {
    return tiles <= 18 ? 8 : tiles <= 37 ? 4 : tiles <= 74 ? 2 : 1;   // portable clusters (<= 8)
}

typedef CUresult (*PFN_encodeTiled_attn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// KV cache [slots, nkv, hd] bf16 as a 3D tensor map, boxes of {64 dims, 1 head,
// 64 slots} with the 128-byte swizzle.  The slot extent is nominal (1 << 24):
// only slots of the caller's pages are ever addressed.
static int kv_map(CUtensorMap* m, const void* base, int nkv, int hd) {
    static PFN_encodeTiled_attn enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return CARD_E_CUDA;
        enc = (PFN_encodeTiled_attn)p;
    }
    cuuint64_t dims[3] = {(cuuint64_t)hd, (cuuint64_t)nkv, (cuuint64_t)1 << 24};
    cuuint64_t strides[2] = {(cuuint64_t)hd * 2, (cuuint64_t)nkv * hd * 2};
    cuuint32_t box[3] = {64, 1, 64};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? CARD_OK : CARD_E_CUDA;
}

template <int HD>
static cudaError_t launch_tc(const TcAttnArgs& a, dim3 grid, int S, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<HD>::kTotal);
        cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Smem<HD>::kTotal;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = S;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    CUtensorMap tmK, tmV;
    if (kv_map(&tmK, a.kc, a.nkv, HD) != CARD_OK || kv_map(&tmV, a.vc, a.nkv, HD) != CARD_OK)
        return cudaErrorInvalidValue;
    return cudaLaunchKernelEx(&cfg, attn_tc_kernel<HD>, a, tmK, tmV);
}

int launch_attn_tc(const float* q, const int32_t* dM, int m_max, const int32_t* plen, const int32_t* n_extra,
                   const int32_t* extra, int extra_max, const void* kc, const void* vc, const int32_t* page_table,
                   int nh, int nkv, int hd, int max_plen, void* o, cudaStream_t s, const void* qsw, int qsw_tiles,
                   int seg_rows, int pt_stride) {
    const int G = nh / nkv;
    const int n_qt = (m_max * G + kQT - 1) / kQT;
    if (qsw && qsw_tiles < n_qt) return CARD_E_CONFIG;
    const int S = attn_tc_ranks(n_qt * nkv);
    TcAttnArgs a{q, dM, plen, n_extra, extra, extra_max, (const __nv_bfloat16*)kc, (const __nv_bfloat16*)vc,
                 page_table, nh, nkv, (__nv_bfloat16*)o, (const uint8_t*)qsw, qsw_tiles, seg_rows, pt_stride};
    const dim3 grid(S, n_qt, nkv);
    const cudaError_t e = hd == 64 ? launch_tc<64>(a, grid, S, s) : launch_tc<128>(a, grid, S, s);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return CARD_E_CUDA;
    }
    return CARD_OK;
}

}  // namespace card
