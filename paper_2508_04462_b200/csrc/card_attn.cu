// card_attn.cu — one-launch attention for the draft tree forward and the
// target chain verify (bf16 KV, head_dim 64 / 128).
//
// Every query row r attends to the prefix KV slots [0, plen[r]) plus
// n_extra[r] listed slots (its tree ancestors and itself) — the tree mask of
// mask.py:173-217 without materialising it.  Causal chains (verify, draft
// catch-up, prefill) have plen = pos + 1 and no extras.
//
// Grid (S, n_qt, nkv), thread-block cluster (S, 1, 1):
//   * z = kv head g; y = tile of 64 query-heads (row r, head h in g's GQA
//     group, ordered (r, h)); x = cluster rank: rank s owns prefix chunks
//     s, s+S, ... (64 keys each).
//   * Each warp keeps 16 query-heads as bf16 mma.sync A fragments and runs a
//     flash-style online softmax over the rank's chunks (K and V staged
//     row-major by cp.async; V^T fragments via ldmatrix.trans).
//   * Tree extras are more chunks: the tile rows' extra slots are gathered
//     row after row into one key list; row i sees keys [xoff[i], xoff[i] +
//     n_extra) of it.  Extra chunks are dealt to the ranks after the prefix
//     chunks and use the same tensor-core path with a range mask.
//   * Combine without a global round trip: every rank pushes its partial
//     (m, l, o[HD]) into the owner rank's shared memory
//     (st.shared::cluster); after one cluster barrier each owner merges its
//     64/S query-heads in rank order and writes o (bf16) for the o-proj GEMM.
// This replaces the split-KV partial round trip through HBM (the old
// prefix + extra + combine kernels, kept for the fp32 parity path).
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include "card_common.cuh"
#include "card_llm.h"

namespace card {

namespace {

constexpr int kCh = 64;      // keys per chunk
constexpr int kMaxTileRows = 136;  // rows per tile of <= 128 query-heads (GQA group >= 1)
constexpr int kMaxExtra = 1024;    // gathered extra slots per tile (static smem: keep two CTAs per SM)

__device__ __forceinline__ uint32_t s_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
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
__device__ __forceinline__ void st_cl_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cl_v2(uint32_t addr, float a, float b) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}

__device__ unsigned long long* g_attn_trace = nullptr;   // tuning: [grid][8] %globaltimer stamps
__device__ __forceinline__ void at_stamp(int k) {
    if (g_attn_trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        g_attn_trace[cta * 8 + k] = t;
    }
}

}  // namespace

// smem: 2 x (K[kCh][HD+8] bf16 | V[kCh][HD+8] bf16) | recv[S][kQT/S][HD+2] f32
// QT query-heads per CTA: 64 (4 warps) for the verify, 128 (8 warps) for the
// wide draft tree (more queries per staged K/V chunk, half the tiles)
template <int HD, int QT>
__global__ void __launch_bounds__(QT * 2) attn_fused_kernel(const float* __restrict__ q, const int32_t* dM,
                                                             const int32_t* __restrict__ plen,
                                                             const int32_t* __restrict__ slot,
                                                             const int32_t* __restrict__ page_table,
                                                             const int32_t* __restrict__ n_extra,
                                                             const int32_t* __restrict__ extra, int extra_max,
                                                             const __nv_bfloat16* __restrict__ kc,
                                                             const __nv_bfloat16* __restrict__ vc, int nh, int nkv,
                                                             __nv_bfloat16* __restrict__ o_out) {
    constexpr int kThr = QT * 2;
    constexpr int LD = HD + 8;   // padded bf16 row: 16-byte aligned, conflict-free 32-bit fragment loads
    constexpr int PW = HD + 2;   // partial record: m, l, o[HD]
    extern __shared__ __align__(16) uint8_t smem[];
    __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem);   // [2][kCh][LD] (double buffer)
    __nv_bfloat16* Vs = Ks + 2 * kCh * LD;                         // [2][kCh][LD]
    float* recv = reinterpret_cast<float*>(Vs + 2 * kCh * LD);

    at_stamp(0);
    // Everything up to the first K/V chunk reads only the row block and old KV
    // slots, written before the previous kernel (the QKV GEMM) started; it runs
    // before griddepcontrol.wait and overlaps the GEMM's tail.
    const int S = gridDim.x;
    const int rank = (int)cl_rank();
    const int qt = blockIdx.y, g = blockIdx.z;
    const int M = *dM;
    const int G = nh / nkv;
    const int nq = M * G;
    const int q0 = qt * QT;
    if (q0 >= nq) return;   // the whole cluster shares qt: consistent early exit
    const int QO = QT / S;   // query-heads owned per rank in the combine
    const int warp = warp_id(), lane = lane_id();
    const int gq = lane >> 2, tq = lane & 3;

    const uint32_t ks_base = s_u32(Ks), vs_base = s_u32(Vs);
    auto stage_rows = [&](int c, int b, auto slot_of) {
        const int ks0 = c * kCh;
        const uint32_t kb = ks_base + (uint32_t)(b * kCh * LD * 2), vb = vs_base + (uint32_t)(b * kCh * LD * 2);
        for (int idx = threadIdx.x; idx < kCh * HD / 8; idx += kThr) {
            const int j = idx / (HD / 8), d8 = (idx % (HD / 8)) * 8;
            const int64_t src = (slot_of(ks0 + j) * nkv + g) * HD + d8;
            cp_async16(kb + (uint32_t)((j * LD + d8) * 2), kc + src);
            cp_async16(vb + (uint32_t)((j * LD + d8) * 2), vc + src);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // keys needed by this tile: max plen over its rows (prefix chunks), and
    // the tile rows' extra slots concatenated row by row (extra chunks: row
    // i's keys are [xoff[i], xoff[i] + xne[i]) of the gathered list)
    __shared__ int s_kmax, s_nx;
    __shared__ int xoff[kMaxTileRows], xne[kMaxTileRows];
    __shared__ int xs[kMaxExtra];
    const int r0 = q0 / G, r1 = min(M - 1, (q0 + QT - 1) / G);
    const int nrows = r1 - r0 + 1;   // <= kMaxTileRows
    // one thread per tile row loads (plen, n_extra); warp 0 scans the extra
    // counts (a serial single-thread loop of dependent loads cost ~10 us)
    if (threadIdx.x == 0) s_kmax = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < nrows; i += kThr) {   // both loads in flight together
        const int ne = n_extra[r0 + i], pl = plen[r0 + i];
        xne[i] = max(0, min(ne, extra_max));
        atomicMax(&s_kmax, pl);
    }
    __syncthreads();
    if (warp_id() == 0) {
        int carry = 0;
        for (int b0 = 0; b0 < nrows; b0 += 32) {
            const int i = b0 + lane_id();
            const int v = i < nrows ? xne[i] : 0;
            int x = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane_id() >= o) x += y;
            }
            if (i < nrows) {
                const int off = carry + x - v;
                xoff[i] = off;
                xne[i] = max(0, min(v, kMaxExtra - off));   // clip to the gathered-list capacity
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane_id() == 0) s_nx = min(carry, kMaxExtra);
    }
    __syncthreads();
    // gather over the flat (row, j) space: a few independent loads per thread
    // instead of one dependent load-store pair per tile row
    for (int e = threadIdx.x; e < nrows * extra_max; e += kThr) {
        const int i = e / extra_max, j = e - i * extra_max;
        if (j < xne[i]) xs[xoff[i] + j] = extra[(int64_t)r0 * extra_max + e];
    }
    const int n_ch = (s_kmax + kCh - 1) / kCh;
    const int n_xch = (s_nx + kCh - 1) / kCh;
    const int n_all = n_ch + n_xch;
    // prefix position k -> KV slot (pages of 64 slots when page_table is set)
    auto pslot = [&](int k) { return (int64_t)(page_table ? page_table[k >> 6] * 64 + (k & 63) : k); };
    // this rank's first chunk can be staged before the wait when it is a
    // prefix chunk below every position this forward writes (row 0 is the
    // lowest: catch-up / chain rows come first at position plen - 1; a tree
    // row 0 means the whole prefix is old)
    const int old_lim = (n_extra && n_extra[0] > 0) ? 0x7fffffff : plen[0] - 1;
    (void)slot;
    const bool prestaged = rank < n_ch && (rank + 1) * kCh <= old_lim;
    if (prestaged) stage_rows(rank, 0, pslot);
    pdl_wait();
    pdl_trigger();
    at_stamp(1);

    // this warp's 16 query-heads: rows a = gq, b = gq + 8
    const int qa = q0 + warp * 16 + gq, qb = qa + 8;
    const bool va = qa < nq, vb = qb < nq;
    const int ra = va ? qa / G : 0, rb = vb ? qb / G : 0;
    const int ha = g * G + (va ? qa % G : 0), hb = g * G + (vb ? qb % G : 0);
    const int pla = va ? plen[ra] : 0, plb = vb ? plen[rb] : 0;
    const int ia = ra - r0, ib = rb - r0;
    const bool warp_live = (q0 + warp * 16) < nq;

    uint32_t qf[HD / 16][4];
    {
        const float* qpa = q + ((int64_t)ra * nh + ha) * HD;
        const float* qpb = q + ((int64_t)rb * nh + hb) * HD;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
            const int d0 = ks * 16 + 2 * tq;
            const float2 a0 = va ? *reinterpret_cast<const float2*>(qpa + d0) : make_float2(0.f, 0.f);
            const float2 b0 = vb ? *reinterpret_cast<const float2*>(qpb + d0) : make_float2(0.f, 0.f);
            const float2 a1 = va ? *reinterpret_cast<const float2*>(qpa + d0 + 8) : make_float2(0.f, 0.f);
            const float2 b1 = vb ? *reinterpret_cast<const float2*>(qpb + d0 + 8) : make_float2(0.f, 0.f);
            qf[ks][0] = pack2(a0.x, a0.y);
            qf[ks][1] = pack2(b0.x, b0.y);
            qf[ks][2] = pack2(a1.x, a1.y);
            qf[ks][3] = pack2(b1.x, b1.y);
        }
    }
    float oacc[HD / 8][4];
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
    float ma = -INFINITY, mb = -INFINITY, la = 0.f, lb = 0.f;

    __syncthreads();   // xs complete
    at_stamp(2);
    // stage chunk c into buffer b (cp.async, one commit group per chunk)
    // gathered padding rows read slot xs[0] (finite data: 0 * V must stay 0)
    const int nx = s_nx;
    auto stage = [&](int c, int b) {
        if (c >= n_ch)
            stage_rows(c - n_ch, b, [&](int k) { return (int64_t)xs[k < nx ? k : 0]; });
        else
            stage_rows(c, b, pslot);
    };
    if (rank < n_all && !prestaged) stage(rank, 0);
    int buf = 0;
    for (int c = rank; c < n_all; c += S, buf ^= 1) {
        const bool xc = c >= n_ch;   // extra (gathered) chunk
        const int k0 = (xc ? c - n_ch : c) * kCh;
        __syncthreads();   // the other buffer (chunk c - S) is fully consumed
        // prefetch the next chunk into the other buffer while this one is used
        if (c + S < n_all) {
            stage(c + S, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();   // chunk c visible to every warp
        if (c == rank) at_stamp(3);
        const uint32_t kcur = ks_base + (uint32_t)(buf * kCh * LD * 2);
        const uint32_t vcur = vs_base + (uint32_t)(buf * kCh * LD * 2);
        const __nv_bfloat16* Kc = Ks + buf * kCh * LD;
        if (!warp_live) continue;
        // visible chunk keys of rows a / b: [loa, hia) / [lob, hib)
        int loa = 0, hia = pla - k0, lob = 0, hib = plb - k0;
        if (xc) {
            loa = va ? xoff[ia] - k0 : 0;
            hia = va ? loa + xne[ia] : 0;
            lob = vb ? xoff[ib] - k0 : 0;
            hib = vb ? lob + xne[ib] : 0;
        }
        if (__all_sync(0xffffffffu, max(0, loa) >= min(kCh, hia) && max(0, lob) >= min(kCh, hib))) continue;
        float s[kCh / 8][4];
#pragma unroll
        for (int n = 0; n < kCh / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks)
#pragma unroll
            for (int n = 0; n < kCh / 8; ++n) {
                const __nv_bfloat16* kr = Kc + (n * 8 + gq) * LD + ks * 16 + 2 * tq;
                uint32_t b[2];
                b[0] = *reinterpret_cast<const uint32_t*>(kr);
                b[1] = *reinterpret_cast<const uint32_t*>(kr + 8);
                mma16816(s[n], qf[ks], b);
            }
        float cma = -INFINITY, cmb = -INFINITY;
#pragma unroll
        for (int n = 0; n < kCh / 8; ++n) {
            const int j0 = n * 8 + 2 * tq;
            if (j0 < loa || j0 >= hia) s[n][0] = -INFINITY;
            if (j0 + 1 < loa || j0 + 1 >= hia) s[n][1] = -INFINITY;
            if (j0 < lob || j0 >= hib) s[n][2] = -INFINITY;
            if (j0 + 1 < lob || j0 + 1 >= hib) s[n][3] = -INFINITY;
            cma = fmaxf(cma, fmaxf(s[n][0], s[n][1]));
            cmb = fmaxf(cmb, fmaxf(s[n][2], s[n][3]));
        }
        cma = fmaxf(cma, __shfl_xor_sync(0xffffffffu, cma, 1));
        cma = fmaxf(cma, __shfl_xor_sync(0xffffffffu, cma, 2));
        cmb = fmaxf(cmb, __shfl_xor_sync(0xffffffffu, cmb, 1));
        cmb = fmaxf(cmb, __shfl_xor_sync(0xffffffffu, cmb, 2));
        const float na = fmaxf(ma, cma), nb = fmaxf(mb, cmb);
        const float sa = na == -INFINITY ? 0.f : na, sb = nb == -INFINITY ? 0.f : nb;
        const float fa = __expf(ma - sa), fb = __expf(mb - sb);   // 0 when the old max is -inf
        ma = na;
        mb = nb;
        float suma = 0.f, sumb = 0.f;
        uint32_t p[kCh / 16][4];
#pragma unroll
        for (int n = 0; n < kCh / 8; ++n) {
            const float e0 = __expf(s[n][0] - sa), e1 = __expf(s[n][1] - sa);
            const float e2 = __expf(s[n][2] - sb), e3 = __expf(s[n][3] - sb);
            suma += e0 + e1;
            sumb += e2 + e3;
            if ((n & 1) == 0) {
                p[n >> 1][0] = pack2(e0, e1);
                p[n >> 1][1] = pack2(e2, e3);
            } else {
                p[n >> 1][2] = pack2(e0, e1);
                p[n >> 1][3] = pack2(e2, e3);
            }
        }
        suma += __shfl_xor_sync(0xffffffffu, suma, 1);
        suma += __shfl_xor_sync(0xffffffffu, suma, 2);
        sumb += __shfl_xor_sync(0xffffffffu, sumb, 1);
        sumb += __shfl_xor_sync(0xffffffffu, sumb, 2);
        la = la * fa + suma;
        lb = lb * fb + sumb;
#pragma unroll
        for (int n = 0; n < HD / 8; ++n) {
            oacc[n][0] *= fa;
            oacc[n][1] *= fa;
            oacc[n][2] *= fb;
            oacc[n][3] *= fb;
        }
        // O += P V: B fragments of V (keys x dims) via ldmatrix.trans, two dim tiles per x4
        const int mat = lane >> 3, mrow = lane & 7;
#pragma unroll
        for (int kk = 0; kk < kCh / 16; ++kk)
#pragma unroll
            for (int nd = 0; nd < HD / 8; nd += 2) {
                // matrices: 0 keys kk*16+0..7 dims nd*8, 1 keys +8..15 dims nd*8, 2/3 the same for nd+1
                const int key = kk * 16 + (mat & 1) * 8 + mrow;
                const int dim = (nd + (mat >> 1)) * 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_trans(vcur + (uint32_t)((key * LD + dim) * 2), b0, b1, b2, b3);
                const uint32_t bA[2] = {b0, b1}, bB[2] = {b2, b3};
                mma16816(oacc[nd], p[kk], bA);
                mma16816(oacc[nd + 1], p[kk], bB);
            }
    }

    at_stamp(4);
    // push this rank's partial (m, l, o) for its 64 query-heads to the owners
    const uint32_t recv_base = s_u32(recv);
    if (warp_live) {
        const int la_loc = warp * 16 + gq, lb_loc = la_loc + 8;
        const int oa = la_loc / QO, ob = lb_loc / QO;
        const uint32_t da = cl_map(recv_base, (uint32_t)oa) + (uint32_t)(((rank * QO + la_loc - oa * QO) * PW) * 4);
        const uint32_t db = cl_map(recv_base, (uint32_t)ob) + (uint32_t)(((rank * QO + lb_loc - ob * QO) * PW) * 4);
        if (tq == 0) {
            st_cl_v2(da, ma, la);
            st_cl_v2(db, mb, lb);
        }
#pragma unroll
        for (int nd = 0; nd < HD / 8; ++nd) {
            const int d = nd * 8 + 2 * tq;
            st_cl_v2(da + (uint32_t)((2 + d) * 4), oacc[nd][0], oacc[nd][1]);
            st_cl_v2(db + (uint32_t)((2 + d) * 4), oacc[nd][2], oacc[nd][3]);
        }
    }
    at_stamp(5);
    cl_sync();   // every partial has landed in its owner's smem
    at_stamp(6);
    // owner merge: query-heads [rank*QO, rank*QO + QO), S partials.  The
    // weights w_s / L take one thread per (query-head, partial): QO * S = QT
    // threads, the S lanes of a query-head reduce by shuffles (S divides 32;
    // a fixed tree, the same for every M).  Then every output element is S
    // independent loads.
    __shared__ float s_w[QT][16];
    if (threadIdx.x < QT) {
        const int ql = threadIdx.x / S, s = threadIdx.x - ql * S;
        const float* rec = recv + (s * QO + ql) * PW;
        const float m_s = rec[0], l_s = rec[1];
        float Mx = m_s;
        for (int o = 1; o < S; o <<= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
        const float Ms = Mx == -INFINITY ? 0.f : Mx;
        const float w = m_s == -INFINITY ? 0.f : __expf(m_s - Ms);
        float L = w * l_s;
        for (int o = 1; o < S; o <<= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        s_w[ql][s] = L > 0.f ? w * (1.0f / L) : 0.f;
    }
    __syncthreads();
    // two adjacent dims per thread (8-byte smem loads, bf16x2 stores); the
    // rank loop is unrolled to the cluster-size bound so its loads overlap
    for (int e = threadIdx.x; e < QO * HD / 2; e += kThr) {
        const int ql = e / (HD / 2), d = 2 * (e - ql * (HD / 2));
        const int qi = q0 + rank * QO + ql;
        if (qi >= nq) break;
        float ax = 0.f, ay = 0.f;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            if (s < S) {
                const float w = s_w[ql][s];
                const float2 v = *reinterpret_cast<const float2*>(recv + (s * QO + ql) * PW + 2 + d);
                ax += w * v.x;
                ay += w * v.y;
            }
        }
        const int r = qi / G, h = g * G + (qi - r * G);
        *reinterpret_cast<__nv_bfloat162*>(o_out + ((int64_t)r * nh + h) * HD + d) = __floats2bfloat162_rn(ax, ay);
    }
    at_stamp(7);
}

int attn_set_trace(unsigned long long* buf) {
    return cudaMemcpyToSymbol(g_attn_trace, &buf, sizeof(buf)) == cudaSuccess ? CARD_OK : CARD_E_CUDA;
}

int attn_fused_smem(int hd, int S, int qt) { return 4 * kCh * (hd + 8) * 2 + S * (qt / S) * (hd + 2) * 4; }

template <int HD, int QT>
static cudaError_t launch_qt(cudaLaunchConfig_t& cfg, const float* q, const int32_t* dM, const int32_t* plen,
                             const int32_t* slot, const int32_t* page_table, const int32_t* n_extra,
                             const int32_t* extra, int extra_max, const void* kc, const void* vc, int nh, int nkv,
                             void* o) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_fused_kernel<HD, QT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(attn_fused_kernel<HD, QT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr = true;
    }
    return cudaLaunchKernelEx(&cfg, attn_fused_kernel<HD, QT>, q, dM, plen, slot, page_table, n_extra, extra, extra_max,
                              (const __nv_bfloat16*)kc, (const __nv_bfloat16*)vc, nh, nkv, (__nv_bfloat16*)o);
}

static int attn_qt(int m_max, int G) {
    return (m_max * G >= 512) ? 128 : 64;
}

// The fused kernel gathers every tile row's extra slots into one list of at
// most kMaxExtra keys; callers fall back to the split-KV kernels when a tile
// could need more (rows per tile x extra slots per row).
bool attn_fused_fits(int m_max, int nh, int nkv, int extra_max) {
    const int G = nh / nkv;
    const int QT = attn_qt(m_max, G);
    const int rows = QT / G + 2;
    return rows <= kMaxTileRows && rows * extra_max <= kMaxExtra;
}

int launch_attn_fused(const float* q, const int32_t* dM, int m_max, const int32_t* plen, const int32_t* slot,
                      const int32_t* page_table,
                      const int32_t* n_extra, const int32_t* extra, int extra_max, const void* kc, const void* vc,
                      int nh, int nkv, int hd, int max_plen, void* o, cudaStream_t s) {
    const int G = nh / nkv;
    const int n_ch = (max_plen + kCh - 1) / kCh;
    // wide (draft tree) forwards: 128 query-heads per CTA; narrow: 64
    const int QT = attn_qt(m_max, G);
    const int n_qt = (m_max * G + QT - 1) / QT;
    // narrow forwards (verify / AR: one query tile per kv head) spread the
    // context over 16 ranks (non-portable cluster; 2% faster verify forward
    // than 8); the wide draft tree forward is fastest with 4 (measured 4 <
    // 8 < 2 < 16 on the 1B draft at 116 rows)
    int S = QT == 128 ? 4 : n_qt * nkv <= 18 ? 16 : n_qt * nkv <= 37 ? 8 : 4;
    while (S > 1 && S > n_ch) S >>= 1;
    const int smem = attn_fused_smem(hd, S, QT);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S, n_qt, nkv);
    cfg.blockDim = dim3(QT * 2);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = S;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e;
    if (hd == 64)
        e = QT == 128 ? launch_qt<64, 128>(cfg, q, dM, plen, slot, page_table, n_extra, extra, extra_max, kc, vc, nh, nkv, o)
                      : launch_qt<64, 64>(cfg, q, dM, plen, slot, page_table, n_extra, extra, extra_max, kc, vc, nh, nkv, o);
    else
        e = QT == 128 ? launch_qt<128, 128>(cfg, q, dM, plen, slot, page_table, n_extra, extra, extra_max, kc, vc, nh, nkv, o)
                      : launch_qt<128, 64>(cfg, q, dM, plen, slot, page_table, n_extra, extra, extra_max, kc, vc, nh, nkv, o);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return CARD_E_CUDA;
    }
    return CARD_OK;
}

}  // namespace card
