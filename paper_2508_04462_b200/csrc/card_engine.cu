// card_engine.cu — the query-and-correct cycle as device kernels
// (engine.py:198-272, verify.py:38-132).  All per-cycle decisions stay on
// the GPU; the host replays a CUDA graph per draft step and one per target
// step and reads back a ~1 KB record once per cycle.
//
//   card_draft_rows    frontier (or flat) rows of the next draft forward:
//                      catch-up rows for committed tokens without draft KV
//                      (causal), then one row per frontier node listing its
//                      tree-KV ancestors (engine.py:198-221, mask.py:173-217)
//   card_target_rows   [root] + queried candidate path, causal (engine.py:228-245)
//   card_kgram_tails   context tails of output rows (toy k-gram models)
//   card_record_width  per-draft-step width log + empty-pool stop flag
//   card_verify_argmax greedy accept: longest argmax prefix + correction (verify.py:65-80)
//   card_verify_probs  greedy or lossless stochastic accept on fp64 rows
//                      (verify.py:43-51, 83-132), uniforms pre-drawn on the host
//   card_commit        max_new_tokens / EOS clipping, committed append (engine.py:247-262)
//   card_draft_promote accepted-chain tree KV -> draft prefix KV (KV rollforward)
//   card_kv_compact    move surviving tree KV rows after an arena compaction
//   card_cycle_end     snapshot the cycle record for the host
#include <cuda_bf16.h>
#include <stdio.h>

#include "card_common.cuh"
#include "card_llm.h"

extern "C" {
typedef struct card_engine_state {
    int32_t C, Pd, out_len, done;
    int32_t max_new, eos, stop, n_widths;
    int32_t hit, L, n_acc, corr;
    int32_t rec_acc, rec_lnew, cursor, n_uni;
    int32_t base_len, C_prev, order, sampling;
    int32_t rec_n_widths, rec_hit, rec_L, rec_n_acc;
    int32_t rec_corr, rec_done, n_commit, anchor_origin;
    int32_t widths[64];
    int32_t rec_widths[64];
    int32_t acc[64];
    int32_t committed_now[72];
    int32_t rec_depth, rec_alive;
    // target KV rollback of the last verify: KV rows [0, kv_keep)
    // stay valid, the kv_drop rows written above them are dead; uniforms
    // the verify consumed (verify.py:104-132 draw order)
    int32_t kv_keep, kv_drop, consumed, cursor_prev, spare[2];
} card_engine_state;
}

namespace card {

// prefix position -> KV slot: pages of 64 slots through the run's page table
// (NULL: identity); tree slots are tree_base + node id
__device__ __forceinline__ int pslot(const int32_t* pt, int p) { return pt ? pt[p >> 6] * 64 + (p & 63) : p; }

// ---------------------------------------------------------------- row builders
// A request's region of a batched row block: its rows start
// at row_base of the combined block (R points there), at most rows_cap of
// them, outputs at most out_cap; the rest of the region is padding rows
// (plen 0, no extras, KV written to dead_slot) so the combined forward can
// run over every region.  rows_cap == 0: a single request owning the block
// header (M, n_out).
struct RowSlot {
    int row_base, rows_cap, out_cap, dead_slot;
};

__device__ void pad_rows(CardRows R, const RowSlot& B, int m0, int o0, int tid, int nt) {
    for (int m = m0 + tid; m < B.rows_cap; m += nt) {
        R.tok[m] = 0;
        R.pos[m] = 0;
        R.slot[m] = B.dead_slot;
        R.plen[m] = 0;
        R.n_extra[m] = 0;
    }
    // padded outputs read the region's own rows in order (a target region's
    // outputs are then the identity map of its rows)
    for (int o = o0 + tid; o < B.out_cap; o += nt) R.out_rows[o] = B.row_base + (o < B.rows_cap ? o : B.rows_cap - 1);
}

__global__ void draft_rows_kernel(card_engine_state* E, const card_cache_state* S, const int32_t* __restrict__ ntoken,
                                  const int32_t* __restrict__ nparent, const int32_t* __restrict__ nlayer,
                                  const int32_t* __restrict__ frontier, const int32_t* __restrict__ committed,
                                  CardRows R, int tree_base, int32_t* ctx_tail, int order, const int32_t* pt,
                                  RowSlot B) {
    // one thread per catch-up row and per frontier row (the ancestor walks of
    // the frontier nodes run in parallel)
    const int tid = threadIdx.x;
    const bool batch = B.rows_cap > 0;
    // batched: spare[0] = expansions left in this cycle (set by the host,
    // min(ratio, max_depth - depth) as engine.py:303-310); spent -> stop
    const bool spent = batch && !E->stop && !E->done && E->spare[0] <= 0;
    __syncthreads();
    if (E->stop || E->done || spent) {
        if (batch) pad_rows(R, B, 0, 0, tid, blockDim.x);
        else if (tid == 0) {
            *R.M = 0;
            *R.n_out = 0;
        }
        // a spent budget stops this cycle's expansions; a finished request's
        // too (its padded outputs must not reach card_cache_expand_topk)
        if ((spent || (batch && E->done)) && tid == 0) E->stop = 1;
        return;
    }
    if (batch && tid == 0) E->spare[0] -= 1;
    const int C = E->C;
    const int nf = S->n_frontier;
    const int anchor = E->anchor_origin ? 0 : S->root;
    const int base = E->anchor_origin ? E->base_len : C;
    const int Pd = E->Pd;
    if (nf == 0) {
        // flat forward of the committed context (engine.py:210-213)
        const int start = Pd < C - 1 ? Pd : C - 1;
        if (batch && C - start > B.rows_cap) {   // region too small: fail loudly
            if (tid == 0) E->done = -1;
            pad_rows(R, B, 0, 0, tid, blockDim.x);
            return;
        }
        for (int p = start + tid; p < C; p += blockDim.x) {
            const int m = p - start;
            R.tok[m] = committed[p];
            R.pos[m] = p;
            R.slot[m] = pslot(pt, p);
            R.plen[m] = p + 1;
            R.n_extra[m] = 0;
        }
        if (ctx_tail)
            for (int j = tid; j < order; j += blockDim.x) {
                const int p = C - order + j;
                ctx_tail[j] = p >= 0 ? committed[p] : -1;
            }
        if (batch) pad_rows(R, B, C - start, 1, tid, blockDim.x);
        __syncthreads();
        if (tid == 0) {
            R.out_rows[0] = B.row_base + C - start - 1;
            if (!batch) {
                *R.n_out = 1;
                *R.M = C - start;
            }
            E->Pd = C;
        }
        return;
    }
    const int n_catch = Pd < base ? base - Pd : 0;
    if (batch && (n_catch + nf > B.rows_cap || nf > B.out_cap)) {
        if (tid == 0) E->done = -1;
        pad_rows(R, B, 0, 0, tid, blockDim.x);
        return;
    }
    for (int i = tid; i < n_catch; i += blockDim.x) {   // catch-up rows (no outputs)
        const int p = Pd + i;
        R.tok[i] = committed[p];
        R.pos[i] = p;
        R.slot[i] = pslot(pt, p);
        R.plen[i] = p + 1;
        R.n_extra[i] = 0;
    }
    const int anchor_layer = nlayer[anchor];
    for (int i = tid; i < nf; i += blockDim.x) {
        const int m = n_catch + i;
        const int f = frontier[i];
        const int d = nlayer[f] - anchor_layer;
        int32_t* ex = R.extra + (int64_t)m * R.extra_max;
        int cur = f;
        for (int j = d - 1; j >= 0; --j) {   // ancestors, root side first
            ex[j] = tree_base + cur;
            cur = nparent[cur];
        }
        R.tok[m] = ntoken[f];
        R.pos[m] = base - 1 + d;
        R.slot[m] = tree_base + f;
        R.plen[m] = base;
        R.n_extra[m] = d;
        R.out_rows[i] = B.row_base + m;
        if (ctx_tail) {
            // tail of base + path: last `order` tokens (path node = ex[q] - tree_base)
            for (int j = 0; j < order; ++j) {
                const int q = d - order + j;   // index into path (0..d-1), negative -> base
                int t;
                if (q >= 0) t = ntoken[ex[q] - tree_base];
                else {
                    const int p = base + q;
                    t = p >= 0 ? committed[p] : -1;
                }
                ctx_tail[(int64_t)i * order + j] = t;
            }
        }
    }
    if (batch) pad_rows(R, B, n_catch + nf, nf, tid, blockDim.x);
    __syncthreads();
    if (tid == 0) {
        if (!batch) {
            *R.n_out = nf;
            *R.M = n_catch + nf;
        }
        if (Pd < base) E->Pd = base;
    }
}

__global__ void target_rows_kernel(card_engine_state* E, const card_cache_state* S, const int32_t* __restrict__ q_tok,
                                   const int32_t* __restrict__ committed, CardRows R, int32_t* ctx_tail, int order,
                                   const int32_t* pt, RowSlot B) {
    if (threadIdx.x != 0) return;
    const bool batch = B.rows_cap > 0;
    if (E->done) {
        if (batch) pad_rows(R, B, 0, 0, 0, 1);
        else {
            *R.M = 0;
            *R.n_out = 0;
        }
        return;
    }
    const int C = E->C;
    const int L = S->q_hit ? S->q_len : 0;
    E->hit = S->q_hit;
    E->L = L;
    for (int i = 0; i <= L; ++i) {
        const int p = C - 1 + i;
        R.tok[i] = i == 0 ? committed[C - 1] : q_tok[i - 1];
        R.pos[i] = p;
        R.slot[i] = pslot(pt, p);
        R.plen[i] = p + 1;
        R.n_extra[i] = 0;
        R.out_rows[i] = B.row_base + i;
        if (ctx_tail)
            for (int j = 0; j < order; ++j) {
                const int q = i - order + j;   // index into candidate prefix
                int t;
                if (q >= 0) t = q_tok[q];
                else {
                    const int pp = C + q;
                    t = pp >= 0 ? committed[pp] : -1;
                }
                ctx_tail[(int64_t)i * order + j] = t;
            }
    }
    if (batch) pad_rows(R, B, L + 1, L + 1, 0, 1);
    else {
        *R.M = L + 1;
        *R.n_out = L + 1;
    }
}

// EOS is absorbing (lm.py:148-150): rows whose context ends in EOS become a one-hot.
__global__ void eos_fix_kernel(const int32_t* n_rows, const int32_t* ctx_tail, int order, int eos, int V,
                               double* probs) {
    const int r = blockIdx.x;
    if (r >= *n_rows || eos < 0) return;
    if (ctx_tail[(int64_t)r * order + order - 1] != eos) return;
    for (int i = threadIdx.x; i < V; i += blockDim.x) probs[(int64_t)r * V + i] = (i == eos) ? 1.0 : 0.0;
}

__global__ void record_width_kernel(card_engine_state* E, const card_cache_state* S, const int32_t* n_out) {
    if (E->done) return;
    const bool ran = !E->stop;
    const int w = (ran && S->status == CARD_OK) ? S->last_width : 0;
    if (ran) {
        if (E->n_widths < 64) E->widths[E->n_widths] = w;
        E->n_widths += 1;
    }
    if (w == 0) E->stop = 1;
}

// ---------------------------------------------------------------- verification
__device__ void finish_verify(card_engine_state* E, const int32_t* q_tok, int n, int corr) {
    E->cursor_prev = E->cursor;
    E->n_acc = n;
    E->corr = corr;
    for (int i = 0; i < n; ++i) E->acc[i] = q_tok[i];
}

__global__ void verify_argmax_kernel(card_engine_state* E, const int32_t* __restrict__ amax,
                                     const int32_t* __restrict__ q_tok) {
    if (threadIdx.x != 0 || E->done) return;
    const int L = E->L;
    int n = 0;
    while (n < L && amax[n] == q_tok[n]) ++n;   // verify.py:76-79
    finish_verify(E, q_tok, n, amax[n]);
}

// sample_index (verify.py:43-51): sequential cumsum, u*total, searchsorted right.
// `zero_tok` >= 0 zeroes that entry (the q=1 residual of verify.py:118-121).
__device__ __forceinline__ double resid(const double* p, int i, int tok, double q) {
    return i == tok ? fmax(p[i] - q, 0.0) : p[i];
}

__device__ int sample_row(const double* p, int V, int zero_tok, double q, double u, double* sh, int* shi) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (V <= 8192) {
        if (tid == 0) {
            double c = 0.0;
            for (int i = 0; i < V; ++i) c = c + resid(p, i, zero_tok, q);
            const double x = u * c;
            double run = 0.0;
            int idx = V;
            for (int i = 0; i < V; ++i) {
                run = run + resid(p, i, zero_tok, q);
                if (run > x) {
                    idx = i;
                    break;
                }
            }
            *shi = idx < V - 1 ? idx : V - 1;
        }
        __syncthreads();
        return *shi;
    }
    // large V: contiguous chunks per thread, ordered chunk scan
    const int chunk = (V + nt - 1) / nt;
    const int lo = tid * chunk, hi = min(V, lo + chunk);
    double s = 0.0;
    for (int i = lo; i < hi; ++i) s = s + resid(p, i, zero_tok, q);
    sh[tid] = s;
    __syncthreads();
    if (tid == 0) {
        double c = 0.0;
        for (int t = 0; t < nt; ++t) {
            const double v = sh[t];
            sh[t] = c;
            c = c + v;
        }
        sh[nt] = c;
        *shi = V - 1;
    }
    __syncthreads();
    const double x = u * sh[nt];
    double run = sh[tid];
    if (lo < hi && run + s > x && run <= x) {
        for (int i = lo; i < hi; ++i) {
            run = run + resid(p, i, zero_tok, q);
            if (run > x) {
                *shi = i < V - 1 ? i : V - 1;
                break;
            }
        }
    }
    __syncthreads();
    return *shi;
}

__global__ void __launch_bounds__(1024) verify_probs_kernel(card_engine_state* E, const double* __restrict__ probs,
                                                           int V, const int32_t* __restrict__ q_tok,
                                                           const double* __restrict__ qcond,
                                                           const double* __restrict__ uni) {
    extern __shared__ double sh[];
    __shared__ int shi, s_n, s_corr, s_done;
    if (E->done) return;
    const int L = E->L;
    const int tid = threadIdx.x;
    if (!E->sampling) {
        // greedy on probabilities: first maximum per row (np.argmax)
        __shared__ double bv[32];
        __shared__ int bi[32];
        int n = 0;
        for (int row = 0; row <= L; ++row) {
            const double* p = probs + (int64_t)row * V;
            double v = -1.0;
            int ix = 0x7fffffff;
            for (int i = tid; i < V; i += blockDim.x)
                if (p[i] > v) {
                    v = p[i];
                    ix = i;
                }
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
                if (ov > v || (ov == v && oi < ix)) {
                    v = ov;
                    ix = oi;
                }
            }
            if (lane_id() == 0) {
                bv[warp_id()] = v;
                bi[warp_id()] = ix;
            }
            __syncthreads();
            if (tid == 0) {
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                    if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) {
                        bv[0] = bv[w];
                        bi[0] = bi[w];
                    }
                shi = bi[0];
            }
            __syncthreads();
            const int am = shi;
            __syncthreads();
            if (row == L || am != q_tok[row]) {
                if (tid == 0) finish_verify(E, q_tok, n, am);
                return;
            }
            ++n;
        }
        return;
    }
    // lossless accept/reject with q = 1 (engine.py:241-242, verify.py:108-132)
    if (tid == 0) {
        s_n = 0;
        s_corr = -1;
        s_done = 0;
    }
    __syncthreads();
    int cur = E->cursor;
    for (int i = 0; i < L; ++i) {
        const double* p = probs + (int64_t)i * V;
        const int tok = q_tok[i];
        const double u = uni[cur++];
        const double pt = p[tok];
        const double qi = qcond ? qcond[i] : 1.0;
        const double ratio = pt / qi;
        const double accept = ratio < 1.0 ? ratio : 1.0;
        if (u < accept) {
            if (tid == 0) s_n = i + 1;
            continue;
        }
        // residual max(p - onehot(tok), 0); falls back to p when it has no mass
        __shared__ int any_mass;
        if (tid == 0) any_mass = 0;
        __syncthreads();
        for (int j = tid; j < V; j += blockDim.x)
            if (j != tok && p[j] > 0.0) any_mass = 1;
        if (tid == 0 && pt - qi > 0.0) any_mass = 1;
        __syncthreads();
        const double u2 = uni[cur++];
        const int c = sample_row(p, V, any_mass ? tok : -1, qi, u2, sh, &shi);
        if (tid == 0) {
            s_corr = c;
            s_done = 1;
        }
        __syncthreads();
        break;
    }
    __syncthreads();
    if (!s_done) {
        const double u3 = uni[cur++];
        const int c = sample_row(probs + (int64_t)L * V, V, -1, 0.0, u3, sh, &shi);
        if (tid == 0) s_corr = c;
        __syncthreads();
    }
    if (tid == 0) {
        finish_verify(E, q_tok, s_n, s_corr);
        E->cursor = cur;
    }
}

// ---------------------------------------------------------------- commit
__global__ void commit_kernel(card_engine_state* E, int32_t* committed) {
    if (threadIdx.x != 0 || E->done) return;
    const int n = E->n_acc;
    const int lnew = n + 1;
    int room = E->max_new - E->out_len;
    int cnt = lnew < room ? lnew : (room > 0 ? room : 0);
    int toks[72];
    for (int i = 0; i < cnt; ++i) toks[i] = i < n ? E->acc[i] : E->corr;
    if (E->eos >= 0)
        for (int i = 0; i < cnt; ++i)
            if (toks[i] == E->eos) {
                cnt = i + 1;
                break;
            }
    E->C_prev = E->C;
    for (int i = 0; i < cnt; ++i) {
        committed[E->C + i] = toks[i];
        E->committed_now[i] = toks[i];
    }
    E->n_commit = cnt;
    E->C += cnt;
    E->out_len += cnt;
    int done = (cnt < lnew) || (E->out_len >= E->max_new);
    if (cnt > 0 && E->eos >= 0 && toks[cnt - 1] == E->eos) done = 1;
    E->done = done;
    E->rec_acc = cnt > 0 ? cnt - 1 : 0;
    E->rec_lnew = cnt;
    // the verify wrote KV for positions C_prev-1 .. C_prev-1+L (root + L
    // candidates); the committed root and accepted tokens keep theirs, the
    // last committed token (the correction) has none yet
    E->kv_keep = E->C_prev + cnt - 1;
    E->kv_drop = E->L + 1 - cnt;
    E->consumed = E->cursor - E->cursor_prev;
    if (!E->anchor_origin) E->base_len = E->C;
}

// ---------------------------------------------------------------- draft KV maintenance
struct KVPtrs {
    void** k;
    void** v;
    int n_layers;
    int row_elems;   // nkv * hd
    int esize;       // bytes per element
};

__device__ __forceinline__ void copy_row(const KVPtrs& P, int layer, int64_t src, int64_t dst) {
    const int bytes = P.row_elems * P.esize;
    const char* ks = (const char*)P.k[layer] + src * bytes;
    char* kd = (char*)P.k[layer] + dst * bytes;
    const char* vs = (const char*)P.v[layer] + src * bytes;
    char* vd = (char*)P.v[layer] + dst * bytes;
    for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16) {
        *(uint4*)(kd + i) = *(const uint4*)(ks + i);
        *(uint4*)(vd + i) = *(const uint4*)(vs + i);
    }
}

// grid (n_layers, max_chain): run length of KV-bearing chain nodes starting
// at the current draft prefix end is promoted into the prefix region.
__global__ void draft_promote_kernel(card_engine_state* E, const card_cache_state* S, const int32_t* chain,
                                     const int32_t* chain_kv, KVPtrs P, int tree_base, const int32_t* pt) {
    if (E->done) return;
    const int j = blockIdx.y;
    const int clen = S->chain_len;
    if (E->Pd != E->C_prev || j >= clen) return;
    for (int i = 0; i <= j; ++i)
        if (!chain_kv[i]) return;
    copy_row(P, blockIdx.x, (int64_t)tree_base + chain[j], (int64_t)pslot(pt, E->C_prev + j));
}

__global__ void draft_promote_finish_kernel(card_engine_state* E, const card_cache_state* S, const int32_t* chain_kv) {
    if (E->done || E->Pd != E->C_prev) return;
    int r = 0;
    while (r < S->chain_len && chain_kv[r]) ++r;
    E->Pd = E->C_prev + r;
}

// compaction: gather kept tree rows into scratch (new ids), then scatter back
__global__ void kv_compact_gather_kernel(const card_engine_state* E, const card_cache_state* S,
                                         const int32_t* remap, KVPtrs P, KVPtrs scratch, int tree_base) {
    if (E->done || !S->compacted) return;
    const int bytes = P.row_elems * P.esize;
    const int l = blockIdx.x;
    for (int x = blockIdx.y; x < S->n_precompact; x += gridDim.y) {
    const int nx = remap[x];
    if (nx < 0) continue;
    const char* ks = (const char*)P.k[l] + ((int64_t)tree_base + x) * bytes;
    const char* vs = (const char*)P.v[l] + ((int64_t)tree_base + x) * bytes;
    char* kd = (char*)scratch.k[0] + ((int64_t)nx * P.n_layers + l) * bytes;
    char* vd = (char*)scratch.v[0] + ((int64_t)nx * P.n_layers + l) * bytes;
    for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16) {
        *(uint4*)(kd + i) = *(const uint4*)(ks + i);
        *(uint4*)(vd + i) = *(const uint4*)(vs + i);
    }
    }
}

__global__ void kv_compact_scatter_kernel(const card_engine_state* E, const card_cache_state* S, KVPtrs P,
                                          KVPtrs scratch, int tree_base) {
    if (E->done || !S->compacted) return;
    const int bytes = P.row_elems * P.esize;
    const int l = blockIdx.x;
    for (int nx = blockIdx.y; nx < S->n_nodes; nx += gridDim.y) {
    const char* ks = (const char*)scratch.k[0] + ((int64_t)nx * P.n_layers + l) * bytes;
    const char* vs = (const char*)scratch.v[0] + ((int64_t)nx * P.n_layers + l) * bytes;
    char* kd = (char*)P.k[l] + ((int64_t)tree_base + nx) * bytes;
    char* vd = (char*)P.v[l] + ((int64_t)tree_base + nx) * bytes;
    for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16) {
        *(uint4*)(kd + i) = *(const uint4*)(ks + i);
        *(uint4*)(vd + i) = *(const uint4*)(vs + i);
    }
    }
}

// concurrent mode: the target's commit outcome -> the draft-side state (the
// correction signal of engine.py:264-272; the draft keeps its own Pd)
__global__ void handoff_kernel(const card_engine_state* T, card_engine_state* D) {
    if (threadIdx.x != 0) return;
    D->C = T->C;
    D->C_prev = T->C_prev;
    D->base_len = T->base_len;
    D->done = T->done;
    D->out_len = T->out_len;
    D->n_acc = T->n_acc;
    D->corr = T->corr;
    for (int i = 0; i < 64; ++i) D->acc[i] = T->acc[i];
    D->stop = 0;
    D->n_widths = 0;
}

__global__ void cycle_end_kernel(card_engine_state* E, const card_cache_state* S, const int32_t* layer,
                                 const int32_t* frontier) {
    if (threadIdx.x != 0) return;
    if (S) E->rec_depth = S->n_frontier > 0 ? layer[frontier[0]] - layer[S->root] : 0;
    E->rec_n_widths = E->n_widths;
    for (int i = 0; i < 64; ++i) E->rec_widths[i] = E->widths[i];
    E->rec_hit = E->hit;
    E->rec_L = E->L;
    E->rec_n_acc = E->n_acc;
    E->rec_corr = E->corr;
    E->rec_done = E->done;
    E->n_widths = 0;
    E->stop = 0;
}

}  // namespace card

using namespace card;

static CardRows make_rows(int32_t* M, int32_t* n_out, int32_t* tok, int32_t* pos, int32_t* slot, int32_t* plen,
                          int32_t* n_extra, int32_t* extra, int32_t* out_rows, int rows_max, int extra_max) {
    CardRows r;
    r.M = M;
    r.n_out = n_out;
    r.tok = tok;
    r.pos = pos;
    r.slot = slot;
    r.plen = plen;
    r.n_extra = n_extra;
    r.extra = extra;
    r.out_rows = out_rows;
    r.rows_max = rows_max;
    r.extra_max = extra_max;
    return r;
}

extern "C" {

int card_engine_state_bytes(void) { return (int)sizeof(card_engine_state); }

// rows: int32 block [M, n_out, tok[rm], pos[rm], slot[rm], plen[rm], n_extra[rm], out_rows[rm], extra[rm*em]]
int card_draft_rows(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows, int rows_max,
                    int extra_max, int tree_base, int32_t* ctx_tail, int order, const int32_t* page_table,
                    void* stream) {
    card_cache_state* S;
    int32_t *tok, *par, *lay, *fr;
    int rc = card_cache_device_ptrs(h, &S, &tok, &par, &lay, &fr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    const int rm = rows_max;
    CardRows R = make_rows(rows, rows + 1, rows + 2, rows + 2 + rm, rows + 2 + 2 * rm, rows + 2 + 3 * rm,
                           rows + 2 + 4 * rm, rows + 2 + 6 * rm, rows + 2 + 5 * rm, rm, extra_max);
    draft_rows_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(E, S, tok, par, lay, fr, committed, R, tree_base, ctx_tail,
                                                         order, page_table, RowSlot{0, 0, 0, 0});
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_target_rows(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows, int rows_max,
                     int extra_max, int32_t* ctx_tail, int order, const int32_t* page_table, void* stream) {
    card_cache_state* S;
    int rc = card_cache_device_ptrs(h, &S, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    int32_t *qp, *qt;
    double* qe;
    card_cache_query_buffers(h, &qp, &qt, &qe);
    const int rm = rows_max;
    CardRows R = make_rows(rows, rows + 1, rows + 2, rows + 2 + rm, rows + 2 + 2 * rm, rows + 2 + 3 * rm,
                           rows + 2 + 4 * rm, rows + 2 + 6 * rm, rows + 2 + 5 * rm, rm, extra_max);
    target_rows_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(E, S, qt, committed, R, ctx_tail, order, page_table,
                                                         RowSlot{0, 0, 0, 0});
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

// target rows from an explicit query view (the mailbox driver: the query
// arrived in the target GPU's memory, card_mailbox_query_view)
int card_target_rows_view(card_engine_state* E, const card_cache_state* view, const int32_t* q_tok,
                          const int32_t* committed, int32_t* rows, int rows_max, int extra_max, int32_t* ctx_tail,
                          int order, const int32_t* page_table, void* stream) {
    if (!E || !view || !q_tok || !rows) return CARD_E_INPUT;
    const int rm = rows_max;
    CardRows R = make_rows(rows, rows + 1, rows + 2, rows + 2 + rm, rows + 2 + 2 * rm, rows + 2 + 3 * rm,
                           rows + 2 + 4 * rm, rows + 2 + 6 * rm, rows + 2 + 5 * rm, rm, extra_max);
    target_rows_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(E, view, q_tok, committed, R, ctx_tail, order, page_table,
                                                         RowSlot{0, 0, 0, 0});
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

// Batched row builders: the request writes its region
// [row_base, row_base + rows_cap) of a combined block of rows_max rows (and
// outputs [out_base, out_base + out_cap)); padding fills the rest of the
// region.  The block header (M, n_out) is the caller's (the region sizes).
// A request whose rows do not fit its region ends with done = -1.
int card_draft_rows_at(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows, int rows_max,
                       int extra_max, int row_base, int rows_cap, int out_base, int out_cap, int dead_slot,
                       int tree_base, int32_t* ctx_tail, int order, const int32_t* page_table, void* stream) {
    if (!E || !h || !rows || rows_cap <= 0 || out_cap <= 0 || row_base < 0 || row_base + rows_cap > rows_max ||
        out_base < 0 || out_base + out_cap > rows_max)
        return CARD_E_INPUT;
    card_cache_state* S;
    int32_t *tok, *par, *lay, *fr;
    int rc = card_cache_device_ptrs(h, &S, &tok, &par, &lay, &fr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    const int rm = rows_max, b = row_base;
    CardRows R = make_rows(rows, rows + 1, rows + 2 + b, rows + 2 + rm + b, rows + 2 + 2 * rm + b,
                           rows + 2 + 3 * rm + b, rows + 2 + 4 * rm + b, rows + 2 + 6 * rm + (int64_t)b * extra_max,
                           rows + 2 + 5 * rm + out_base, rows_cap, extra_max);
    draft_rows_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(E, S, tok, par, lay, fr, committed, R, tree_base,
                                                         ctx_tail ? ctx_tail + (int64_t)out_base * order : nullptr,
                                                         order, page_table, RowSlot{row_base, rows_cap, out_cap, dead_slot});
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_target_rows_at(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows, int rows_max,
                        int extra_max, int row_base, int rows_cap, int dead_slot, int32_t* ctx_tail, int order,
                        const int32_t* page_table, void* stream) {
    if (!E || !h || !rows || rows_cap <= 0 || row_base < 0 || row_base + rows_cap > rows_max) return CARD_E_INPUT;
    card_cache_state* S;
    int rc = card_cache_device_ptrs(h, &S, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    int32_t *qp, *qt;
    double* qe;
    card_cache_query_buffers(h, &qp, &qt, &qe);
    const int rm = rows_max, b = row_base;
    CardRows R = make_rows(rows, rows + 1, rows + 2 + b, rows + 2 + rm + b, rows + 2 + 2 * rm + b,
                           rows + 2 + 3 * rm + b, rows + 2 + 4 * rm + b, rows + 2 + 6 * rm + (int64_t)b * extra_max,
                           rows + 2 + 5 * rm + b, rows_cap, extra_max);
    target_rows_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(E, S, qt, committed, R,
                                                         ctx_tail ? ctx_tail + (int64_t)row_base * order : nullptr,
                                                         order, page_table, RowSlot{row_base, rows_cap, rows_cap, dead_slot});
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_eos_fix(const int32_t* n_rows, int m_max, const int32_t* ctx_tail, int order, int eos, int V, double* probs,
                 void* stream) {
    if (eos < 0 || m_max <= 0) return CARD_OK;
    eos_fix_kernel<<<m_max, 128, 0, (cudaStream_t)stream>>>(n_rows, ctx_tail, order, eos, V, probs);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_record_width(card_engine_state* E, card_cache* h, const int32_t* n_out, void* stream) {
    card_cache_state* S;
    card_cache_device_ptrs(h, &S, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    record_width_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(E, S, n_out);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_verify_argmax(card_engine_state* E, const int32_t* cand, const int32_t* amax, void* stream) {
    verify_argmax_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(E, amax, cand);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_verify_probs(card_engine_state* E, const int32_t* cand, const double* probs, int V, const double* qcond,
                      const double* uniforms, void* stream) {
    verify_probs_kernel<<<1, 1024, (1024 + 1) * sizeof(double), (cudaStream_t)stream>>>(E, probs, V, cand, qcond,
                                                                                      uniforms);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_commit(card_engine_state* E, int32_t* committed, void* stream) {
    commit_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(E, committed);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

// the last verify's outcome in the reference's terms: out[0] accepted
// prefix n, out[1] correction, out[2] uniforms consumed, out[3] kv_keep,
// out[4] KV rows rolled back, out[5] tokens committed (device int32[6])
__global__ void verify_result_kernel(const card_engine_state* E, int32_t* out) {
    if (threadIdx.x != 0) return;
    out[0] = E->n_acc;
    out[1] = E->corr;
    out[2] = E->consumed;
    out[3] = E->kv_keep;
    out[4] = E->kv_drop;
    out[5] = E->n_commit;
}

int card_verify_result(const card_engine_state* E, int32_t* out, void* stream) {
    if (!E || !out) return CARD_E_INPUT;
    verify_result_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(E, out);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_draft_promote(card_engine_state* E, card_cache* h, void** k_layers, void** v_layers, int n_layers,
                       int row_elems, int esize, int tree_base, int max_chain, const int32_t* page_table,
                       void* stream) {
    card_cache_state* S;
    int32_t *chain, *chain_kv;
    card_cache_device_ptrs(h, &S, nullptr, nullptr, nullptr, nullptr, nullptr, &chain, &chain_kv);
    KVPtrs P{k_layers, v_layers, n_layers, row_elems, esize};
    dim3 g(n_layers, max_chain);
    draft_promote_kernel<<<g, 128, 0, (cudaStream_t)stream>>>(E, S, chain, chain_kv, P, tree_base, page_table);
    draft_promote_finish_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(E, S, chain_kv);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_kv_compact(card_engine_state* E, card_cache* h, void** k_layers, void** v_layers, int n_layers, int row_elems,
                    int esize, int tree_base, void** scratch_kv, int capacity, void* stream) {
    card_cache_state* S;
    int32_t* remap;
    card_cache_device_ptrs(h, &S, nullptr, nullptr, nullptr, nullptr, &remap, nullptr, nullptr);
    KVPtrs P{k_layers, v_layers, n_layers, row_elems, esize};
    KVPtrs X{scratch_kv, scratch_kv + 1, n_layers, row_elems, esize};
    dim3 g(n_layers, capacity < 128 ? capacity : 128);
    kv_compact_gather_kernel<<<g, 128, 0, (cudaStream_t)stream>>>(E, S, remap, P, X, tree_base);
    kv_compact_scatter_kernel<<<g, 128, 0, (cudaStream_t)stream>>>(E, S, P, X, tree_base);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_enable_peer_access(int dev_a, int dev_b) {
    if (dev_a == dev_b) return CARD_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    int ok_ab = 0, ok_ba = 0;
    cudaDeviceCanAccessPeer(&ok_ab, dev_a, dev_b);
    cudaDeviceCanAccessPeer(&ok_ba, dev_b, dev_a);
    if (!ok_ab || !ok_ba) return CARD_E_CONFIG;
    for (int k = 0; k < 2; ++k) {
        cudaSetDevice(k == 0 ? dev_a : dev_b);
        cudaError_t e = cudaDeviceEnablePeerAccess(k == 0 ? dev_b : dev_a, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
            set_cuda_error(e);
            cudaSetDevice(prev);
            return CARD_E_CUDA;
        }
        cudaGetLastError();
    }
    cudaSetDevice(prev);
    return CARD_OK;
}

int card_engine_handoff(const card_engine_state* target_state, card_engine_state* draft_state, void* stream) {
    handoff_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(target_state, draft_state);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cycle_end(card_engine_state* E, card_cache* h, void* stream) {
    card_cache_state* S = nullptr;
    int32_t *lay = nullptr, *fr = nullptr;
    if (h) card_cache_device_ptrs(h, &S, nullptr, nullptr, &lay, &fr, nullptr, nullptr, nullptr);
    cycle_end_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(E, S, lay, fr);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

}  // extern "C"
