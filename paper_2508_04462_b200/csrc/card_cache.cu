// card_cache.cu — device-resident candidate tree (replaces cache.py:92-523).
//
// Layout in HBM (one allocation per request, struct of arrays):
//   state block (card_cache_state, 24 x int32)
//   token/parent/layer/nkids/mark/mark2/aux/remap int32[cap], alive/has_kv u8[cap],
//   log_score/edge_logp f64[cap], frontier/frontier_old int32[K],
//   open-addressing hash (parent<<32|token) -> child id, 2*cap rounded to a
//   power of two, probed 32 slots at a time by one warp,
//   per-row candidate scratch (token, value, count) [K x k],
//   query outputs [max_depth+1], correction chain [max_depth+2],
//   compaction scratch.
//
// Every operation is one single-CTA kernel (the tree is <= K*max_depth alive
// nodes, a few thousand): ordering work is a parallel rank sort with the
// reference's exact comparators, subtree work is a parallel parent-pointer
// climb, and compaction is a block-wide scan.  All decisions are integer
// compares or IEEE fp64 compares/adds, so results are bit-identical to the
// Python reference given identical inputs (edge log-probs use the correctly
// rounded log of card_common.cuh).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "card_common.cuh"

namespace card {

int launch_rows_topk(const double* dists, int n_rows, int vocab, int k, int32_t* tok, double* p,
                     int32_t* cnt, int32_t* status, cudaStream_t s);

constexpr unsigned long long kEmpty = ~0ULL;
constexpr int kThreads = 1024;
constexpr int kMaxK = 2048;        // frontier width bound (static smem)
constexpr int kMaxPool = 4096;     // K*k bound (dynamic smem)
constexpr int kCompactMinArena = 64;   // cache.py:30

struct Bufs {
    card_cache_state* st;
    int32_t *token, *parent, *layer, *nkids, *mark, *mark2, *aux, *remap;
    uint8_t *alive, *has_kv;
    double *score, *edge;
    int32_t *frontier, *frontier_old;
    unsigned long long* hkeys;
    int32_t* hvals;
    int32_t *c_tok, *c_cnt;
    double* c_val;
    int32_t *q_path, *q_tok;
    double* q_edge;
    int32_t* chain;
    int32_t* chain_kv;
    // compaction scratch
    int32_t *s_token, *s_parent, *s_layer;
    uint8_t* s_haskv;
    double *s_score, *s_edge;
};

}  // namespace card

struct card_cache {
    card::Bufs b;
    void* block;
    size_t bytes;
    int K, k, max_depth, eos, capacity, hcap;
};

namespace card {

// ---------------------------------------------------------------- hash
__device__ __forceinline__ unsigned long long hkey(int parent, int tok) {
    return ((unsigned long long)(uint32_t)parent << 32) | (uint32_t)tok;
}

__device__ void hash_insert(const Bufs& b, int parent, int tok, int id) {
    const unsigned long long key = hkey(parent, tok);
    const int mask = b.st->hash_mask;
    int i = (int)(mix64(key) & (unsigned long long)mask);
    while (true) {
        unsigned long long prev = atomicCAS(&b.hkeys[i], kEmpty, key);
        if (prev == kEmpty || prev == key) {
            b.hvals[i] = id;   // newest node for this (parent, token) wins
            return;
        }
        i = (i + 1) & mask;
    }
}

// Warp-cooperative lookup: 32 consecutive probe slots per step; returns the
// child id or -1.  Must be called by a full warp.
__device__ int hash_find_warp(const Bufs& b, int parent, int tok) {
    const unsigned long long key = hkey(parent, tok);
    const int mask = b.st->hash_mask;
    const int lane = lane_id();
    int base = (int)(mix64(key) & (unsigned long long)mask);
    for (int step = 0; step <= mask; step += 32) {
        int slot = (base + step + lane) & mask;
        unsigned long long k = b.hkeys[slot];
        unsigned hit = __ballot_sync(0xffffffffu, k == key);
        unsigned emp = __ballot_sync(0xffffffffu, k == kEmpty);
        if (hit) {
            // keys are unique and never deleted, so the first match is the entry
            const int src = __ffs(hit) - 1;
            return b.hvals[(base + step + src) & mask];
        }
        if (emp) return -1;
    }
    return -1;
}

// _alive_child (cache.py:337-342): the cached child must also be alive.
__device__ int alive_child_warp(const Bufs& b, int parent, int tok) {
    int c = hash_find_warp(b, parent, tok);
    if (c >= 0 && !b.alive[c]) c = -1;
    return c;
}

__device__ __forceinline__ bool descends(const Bufs& b, int h, int anc) {
    const int al = b.layer[anc];
    while (h >= 0 && b.layer[h] > al) h = b.parent[h];
    return h == anc;
}

// block-wide exclusive scan of 0/1 flags over [0, n); returns total.
__device__ int block_scan_flags(const uint8_t* flag_src, int32_t* out_idx, int n, int* sh_warp, int* sh_carry) {
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    if (tid == 0) *sh_carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += kThreads) {
        int i = base + tid;
        int f = (i < n) ? flag_src[i] : 0;
        unsigned bal = __ballot_sync(0xffffffffu, f);
        int pre = __popc(bal & ((1u << lane) - 1));
        if (lane == 31) sh_warp[w] = pre + f;
        __syncthreads();
        if (w == 0) {
            int v = sh_warp[lane];
            int x = v;
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            sh_warp[lane] = x - v;   // exclusive
        }
        __syncthreads();
        if (i < n) out_idx[i] = f ? (*sh_carry + sh_warp[w] + pre) : -1;
        __syncthreads();
        if (tid == kThreads - 1) *sh_carry += sh_warp[w] + pre + f;
        __syncthreads();
    }
    return *sh_carry;
}

// ---------------------------------------------------------------- init / reset
__global__ void clear_hash_kernel(Bufs b, int hcap) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < hcap; i += gridDim.x * blockDim.x) b.hkeys[i] = kEmpty;
}

__global__ void init_root_kernel(Bufs b, const int32_t* d_tok, int tok, int bump_epoch) {
    card_cache_state& S = *b.st;
    const int t = d_tok ? *d_tok : tok;
    b.token[0] = t;
    b.parent[0] = -1;
    b.layer[0] = 0;
    b.alive[0] = 1;
    b.has_kv[0] = 0;
    b.nkids[0] = 0;
    b.score[0] = 0.0;
    b.edge[0] = 0.0;
    b.mark[0] = 0;
    b.mark2[0] = 0;
    S.n_nodes = 1;
    S.root = 0;
    S.n_frontier = 0;
    S.dead = 0;
    S.top_layer = 0;
    S.status = (t < 0) ? CARD_E_INPUT : CARD_OK;
    S.vstatus = 0;
    S.last_width = 0;
    S.compacted = 0;
    if (bump_epoch) S.epoch += 1;
}

// ---------------------------------------------------------------- expansion
struct PoolSmem {
    double* w;
    double* e;
    ulonglong2* key;   // (-w, token, parent) as two u64 compared lexicographically
    uint32_t* k32;     // key.x >> 32, padded to a multiple of 4 (first-pass compare)
    int32_t* tok;
    int32_t* pid;
    int32_t* rank;
};

__device__ __forceinline__ PoolSmem carve_pool(char* smem, int P) {
    PoolSmem p;
    p.w = (double*)smem;
    p.e = p.w + P;
    p.key = (ulonglong2*)(p.e + P);
    p.k32 = (uint32_t*)(p.key + P);
    p.tok = (int32_t*)(p.k32 + ((P + 3) & ~3));
    p.pid = p.tok + P;
    p.rank = p.pid + P;
    return p;
}

// order key (-weight, token, parent node id) of cache.py:237-239 for pool
// slot s, compared as (hi, lo) pairs: weight descending by its bit pattern
// (-0.0 folds into +0.0 as the double compare does), then token, then parent
// ascending; invalid slots sort last
__device__ __forceinline__ ulonglong2 pool_key(const PoolSmem& p, int s) {
    if (p.tok[s] < 0) return make_ulonglong2(~0ull, ~0ull);
    const unsigned long long b = (unsigned long long)__double_as_longlong(p.w[s] + 0.0);
    const unsigned long long asc = (b >> 63) ? ~b : (b | (1ull << 63));   // ascending in w
    return make_ulonglong2(~asc, ((unsigned long long)(uint32_t)p.tok[s] << 32) | (uint32_t)p.pid[s]);
}

// Builds the extension pool (cache.py:190-222) into smem; returns P.
__device__ int build_pool(const Bufs& b, const int32_t* c_tok, const double* c_val, const int32_t* c_cnt,
                          int vals_are_logp, PoolSmem p, int npar, int k) {
    const card_cache_state& S = *b.st;
    const int P = npar * k;
    for (int s = threadIdx.x; s < P; s += blockDim.x) {
        const int row = s / k, j = s % k;
        const int par = S.n_frontier > 0 ? b.frontier[row] : S.root;
        bool ok = j < c_cnt[row] && !(S.eos >= 0 && b.token[par] == S.eos);
        p.pid[s] = par;
        if (ok) {
            double v = c_val[(int64_t)row * k + j];
            double e = vals_are_logp ? v : log_cr(v);
            p.e[s] = e;
            p.w[s] = __dadd_rn(b.score[par], e);
            p.tok[s] = c_tok[(int64_t)row * k + j];
        } else {
            p.tok[s] = -1;
        }
    }
    return P;
}


__global__ void __launch_bounds__(kThreads) expand_kernel(Bufs b, const int32_t* c_tok, const double* c_val,
                                                          const int32_t* c_cnt, int n_rows_host, int vals_are_logp,
                                                          const int32_t* skip) {
    extern __shared__ __align__(16) char smem[];
    __shared__ int sh_flag, sh_npar, sh_valid, sh_m, sh_cnt[3], sh_dead;
    __shared__ int lvl[2][kMaxK];
    card_cache_state& S = *b.st;
    const int tid = threadIdx.x;
    if (skip && *skip) {
        if (tid == 0) S.last_width = 0;
        return;
    }
    if (tid == 0) {
        const int npar = S.n_frontier > 0 ? S.n_frontier : 1;
        const int depth = S.n_frontier > 0 ? b.layer[b.frontier[0]] - b.layer[S.root] : 0;
        int st = CARD_OK;
        if (depth >= S.max_depth) st = CARD_FRONTIER_FULL;                 // cache.py:233-234
        else if (n_rows_host >= 0 && n_rows_host != npar) st = CARD_E_INPUT;  // cache.py:200-203
        else if (S.vstatus != 0) st = S.vstatus;                            // cache.py:204-208
        else if (S.n_nodes + S.K > S.capacity) st = CARD_E_CAPACITY;
        S.status = st;
        S.vstatus = 0;
        S.last_width = 0;
        S.compacted = 0;
        sh_flag = st;
        sh_npar = npar;
        sh_valid = 0;
        sh_dead = 0;
        sh_cnt[0] = 0;
        sh_m = S.n_frontier;
    }
    __syncthreads();
    if (sh_flag != CARD_OK) return;
    const int npar = sh_npar, K = S.K, k = S.k;
    const int n0 = S.n_nodes;
    for (int i = tid; i < sh_m; i += blockDim.x) {
        b.frontier_old[i] = b.frontier[i];
        lvl[0][i] = b.frontier[i];
    }
    PoolSmem p = carve_pool(smem, npar * k);
    const int P = build_pool(b, c_tok, c_val, c_cnt, vals_are_logp, p, npar, k);
    __syncthreads();
    // parallel rank sort; (token, parent) pairs are unique so ranks are
    // distinct.  Keys packed once; each slot's count is split over `parts`
    // threads (all warps busy instead of P / 32)
    const int P4 = (P + 3) & ~3;
    for (int s = tid; s < P4; s += blockDim.x) {
        const ulonglong2 ks = s < P ? pool_key(p, s) : make_ulonglong2(~0ull, ~0ull);
        if (s < P) {
            p.key[s] = ks;
            p.rank[s] = 0;
        }
        p.k32[s] = (uint32_t)(ks.x >> 32);
        // valid slots, one shared atomic per warp (same-address atomics serialise)
        const unsigned am = __activemask();
        const unsigned v = __ballot_sync(am, s < P && p.tok[s] >= 0);
        if ((tid & 31) == __ffs(am) - 1) atomicAdd(&sh_valid, __popc(v));
    }
    __syncthreads();
    {   // count the slots before s: the top 32 key bits decide all but near-ties
        const int parts = P <= (int)blockDim.x ? min(8, (int)blockDim.x / P) : 1;
        for (int i = tid; i < P * parts; i += blockDim.x) {
            const int s = i % P, part = i / P;
            if (p.tok[s] < 0) continue;
            const ulonglong2 ks = p.key[s];
            const uint32_t h = (uint32_t)(ks.x >> 32);
            int r = 0;
            const int t0 = (P4 / 4 * part / parts) * 4, t1 = (P4 / 4 * (part + 1) / parts) * 4;
            for (int t = t0; t < t1; t += 4) {
                const uint4 q = *reinterpret_cast<const uint4*>(p.k32 + t);
                r += (q.x < h) + (q.y < h) + (q.z < h) + (q.w < h);
                if (q.x == h || q.y == h || q.z == h || q.w == h) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const ulonglong2 kt = p.key[t + j];
                        if (t + j < P && (uint32_t)(kt.x >> 32) == h && (kt.x < ks.x || (kt.x == ks.x && kt.y < ks.y)))
                            ++r;
                    }
                }
            }
            if (parts == 1) p.rank[s] = r;
            else atomicAdd(&p.rank[s], r);
        }
    }
    __syncthreads();
    const int nnew = sh_valid < K ? sh_valid : K;
    // winners allocate arena nodes in rank order (cache.py:240-249)
    for (int s = tid; s < P; s += blockDim.x) {
        if (p.tok[s] < 0 || p.rank[s] >= K) continue;
        const int r = p.rank[s], id = n0 + r, par = p.pid[s];
        b.token[id] = p.tok[s];
        b.parent[id] = par;
        b.layer[id] = b.layer[par] + 1;
        b.score[id] = p.w[s];
        b.edge[id] = p.e[s];
        b.alive[id] = 1;
        b.has_kv[id] = 0;
        b.nkids[id] = 0;
        b.mark[id] = 0;
        b.mark2[id] = 0;
        b.frontier[r] = id;
        atomicAdd(&b.nkids[par], 1);
        hash_insert(b, par, p.tok[s], id);
    }
    // the parents of this layer were just forwarded: their tree KV exists
    if (S.n_frontier > 0)
        for (int i = tid; i < npar; i += blockDim.x) b.has_kv[b.frontier_old[i]] = 1;
    __syncthreads();
    const int stamp = S.stamp + 1;
    // Level-synchronous dead-end pruning from the old frontier
    // (cache.py:261-271).  The reference's `keep` set (ancestors of the new
    // frontier, cache.py:255-260) needs no pass of its own here: nkids counts
    // a node's alive children, and every ancestor of a new frontier node has
    // one (its child on that path), so `nkids != 0` already stops the climb
    // wherever `keep` would.
    // A parent joins the next level when this pass takes its last alive
    // child (the thread whose decrement reaches 0 pushes it, once): the
    // nodes the reference's per-branch climb would reach next.  Next-level
    // counts rotate over three slots so each level needs one barrier (slot
    // (i + 1) % 3 was last read before the previous barrier).
    int m = sh_m, cur_l = 0;
    const int root = S.root;
    for (int lv = 0; m > 0; ++lv) {
        if (tid == 0) sh_cnt[(lv + 1) % 3] = 0;
        for (int i = tid; i < m; i += blockDim.x) {
            const int x = lvl[cur_l][i];
            const int par = b.parent[x];
            if (x == root || (lv == 0 && (!b.alive[x] || b.nkids[x] != 0))) continue;
            b.alive[x] = 0;
            const unsigned am = __activemask();   // the lanes killing a node here
            if ((tid & 31) == __ffs(am) - 1) atomicAdd(&sh_dead, __popc(am));
            if (par >= 0 && atomicSub(&b.nkids[par], 1) == 1) lvl[cur_l ^ 1][atomicAdd(&sh_cnt[lv % 3], 1)] = par;
        }
        __syncthreads();
        m = sh_cnt[lv % 3];
        cur_l ^= 1;
    }
    if (tid == 0) {
        S.stamp = stamp;
        S.n_nodes = n0 + nnew;
        S.n_frontier = nnew;
        S.last_width = nnew;
        S.dead += sh_dead;
    }
}

// extension_pool() for the drop-in API: unsorted pool, P slots.
__global__ void pool_kernel(Bufs b, int32_t* o_tok, double* o_w, int32_t* o_pidx, double* o_e) {
    extern __shared__ __align__(16) char smem[];
    const card_cache_state& S = *b.st;
    const int npar = S.n_frontier > 0 ? S.n_frontier : 1;
    PoolSmem p = carve_pool(smem, npar * S.k);
    const int P = build_pool(b, b.c_tok, b.c_val, b.c_cnt, 0, p, npar, S.k);
    __syncthreads();
    for (int s = threadIdx.x; s < P; s += blockDim.x) {
        o_tok[s] = p.tok[s];
        o_w[s] = p.w[s];
        o_pidx[s] = s / S.k;
        o_e[s] = p.e[s];
    }
}

// ---------------------------------------------------------------- query
__global__ void __launch_bounds__(kThreads) query_kernel(Bufs b, int depth, const int32_t* skip) {
    if (skip && *skip) return;   // (mailbox driver: no correction arrived, nothing to query)
    card_cache_state& S = *b.st;
    __shared__ double bs[32];
    __shared__ int bt[32], bi[32];
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int root = S.root;
    if (b.nkids[root] == 0) {   // miss iff the root has no alive child (cache.py:287-288)
        if (tid == 0) {
            S.q_hit = 0;
            S.q_len = 0;
            S.status = CARD_OK;
        }
        return;
    }
    const int dbr = S.n_frontier > 0 ? b.layer[b.frontier[0]] - b.layer[root] : 0;
    const int d = depth < dbr ? depth : dbr;
    const int target = b.layer[root] + d;
    // best = min over frontier ancestors-at-depth-d of (-score, token, id)
    double ms = 0.0;
    int mt = 0x7fffffff, mi = -1;
    for (int i = tid; i < S.n_frontier; i += blockDim.x) {
        int cur = b.frontier[i];
        while (b.layer[cur] > target) cur = b.parent[cur];
        if (cur == root || !descends(b, cur, root)) continue;
        const double s = b.score[cur];
        const int t = b.token[cur];
        if (mi < 0 || s > ms || (s == ms && (t < mt || (t == mt && cur < mi)))) {
            ms = s;
            mt = t;
            mi = cur;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        double os = __shfl_xor_sync(0xffffffffu, ms, o);
        int ot = __shfl_xor_sync(0xffffffffu, mt, o);
        int oi = __shfl_xor_sync(0xffffffffu, mi, o);
        if (oi >= 0 && (mi < 0 || os > ms || (os == ms && (ot < mt || (ot == mt && oi < mi))))) {
            ms = os;
            mt = ot;
            mi = oi;
        }
    }
    if (lane == 0) {
        bs[w] = ms;
        bt[w] = mt;
        bi[w] = mi;
    }
    __syncthreads();
    if (tid == 0) {
        for (int j = 1; j < (int)(blockDim.x >> 5); ++j) {
            const double os = bs[j];
            const int ot = bt[j], oi = bi[j];
            if (oi >= 0 && (mi < 0 || os > ms || (os == ms && (ot < mt || (ot == mt && oi < mi))))) {
                ms = os;
                mt = ot;
                mi = oi;
            }
        }
        if (mi < 0) {   // the reference asserts here (cache.py:311)
            S.status = CARD_E_PROTOCOL;
            S.q_hit = 0;
            S.q_len = 0;
            return;
        }
        int len = b.layer[mi] - b.layer[root];
        int cur = mi;
        for (int j = len - 1; j >= 0; --j) {   // path_from_root (cache.py:151-162)
            b.q_path[j] = cur;
            b.q_tok[j] = b.token[cur];
            b.q_edge[j] = b.edge[cur];
            cur = b.parent[cur];
        }
        S.q_hit = 1;
        S.q_len = len;
        S.status = CARD_OK;
    }
}

// ---------------------------------------------------------------- correction
// Shared prologue of correct()/advance_root(): walk the accepted tokens
// (cache.py:324-335) and resolve the correction child.  Warp 0 only.
// Returns 0 ok, else a status.  chain[0..n) = chain ids.
__device__ int walk_chain(const Bufs& b, const int32_t* acc, int n_acc, int* anchor_out) {
    int cur = b.st->root;
    for (int i = 0; i < n_acc; ++i) {
        int nxt = alive_child_warp(b, cur, acc[i]);
        if (nxt < 0) return CARD_E_PROTOCOL;
        if (lane_id() == 0) b.chain[i] = nxt;
        cur = nxt;
    }
    *anchor_out = cur;
    return CARD_OK;
}

__global__ void __launch_bounds__(kThreads) correct_kernel(Bufs b, const int32_t* acc, const int32_t* n_acc_p,
                                                           const int32_t* corr_p, const int32_t* skip) {
    card_cache_state& S = *b.st;
    if (skip && *skip) {
        if (threadIdx.x == 0) S.compacted = 0;
        return;
    }
    __shared__ int sh_flag, sh_new_root, sh_fresh, sh_plen, sh_dead, sh_ns, sh_total;
    __shared__ int path[72];   // max_depth <= 64
    __shared__ int surv[kMaxK];
    __shared__ int sh_warp[32], sh_carry;
    const int tid = threadIdx.x;
    const int n_acc = *n_acc_p, corr = *corr_p;
    const int root = S.root;
    if (tid < 32) {
        int st = CARD_OK, anchor = root, new_root = -1, fresh = 0;
        if (n_acc < 0) st = CARD_E_INPUT;
        else if (n_acc > S.max_depth + 1) st = CARD_E_PROTOCOL;   // cannot be a cached chain
        if (st == CARD_OK) st = walk_chain(b, acc, n_acc, &anchor);
        if (st == CARD_OK) {
            if (corr < 0) {
                if (n_acc == 0) st = CARD_E_INPUT;   // cache.py:369-370
                new_root = anchor;
            } else {
                new_root = alive_child_warp(b, anchor, corr);
                if (new_root < 0) {
                    if (S.n_nodes >= S.capacity) st = CARD_E_CAPACITY;
                    fresh = 1;
                }
            }
        }
        if (tid == 0) {
            S.status = st;
            S.compacted = 0;
            sh_flag = st;
            if (st == CARD_OK) {
                if (fresh) {   // fresh node: parent's score, edge 0 (cache.py:374-379)
                    const int id = S.n_nodes;
                    b.token[id] = corr;
                    b.parent[id] = anchor;
                    b.layer[id] = b.layer[anchor] + 1;
                    b.score[id] = b.score[anchor];
                    b.edge[id] = 0.0;
                    b.alive[id] = 1;
                    b.has_kv[id] = 0;
                    b.nkids[id] = 0;
                    b.mark[id] = 0;
                    b.mark2[id] = 0;
                    b.nkids[anchor] += 1;
                    S.n_nodes = id + 1;
                    new_root = id;
                }
                // path = [root] + chain + [new_root if != anchor]
                int pl = 0;
                path[pl++] = root;
                for (int i = 0; i < n_acc; ++i) path[pl++] = b.chain[i];
                if (new_root != anchor) path[pl++] = new_root;
                if (new_root != anchor) b.chain[n_acc] = new_root;
                for (int i = 1; i < pl; ++i) b.chain_kv[i - 1] = b.has_kv[path[i]];
                sh_plen = pl;
                sh_new_root = new_root;
                sh_fresh = fresh;
                S.fresh = fresh;
                S.new_root = new_root;
                S.chain_len = n_acc + (new_root != anchor ? 1 : 0);
                S.stamp += 1;
                sh_dead = 0;
                sh_ns = 0;
            }
        }
    }
    __syncthreads();
    if (sh_flag != CARD_OK) return;
    const int stamp = S.stamp, new_root = sh_new_root, plen = sh_plen;
    if (tid == 0 && sh_fresh) hash_insert(b, b.parent[new_root], corr, new_root);
    for (int i = tid; i < plen; i += blockDim.x) {
        b.mark[path[i]] = stamp;
        b.aux[path[i]] = i;
    }
    __syncthreads();
    const int n = S.n_nodes;
    // kill every alive node whose nearest path ancestor is not the new root
    // (cache.py:383-388: each off-path sibling subtree is killed whole)
    for (int x = tid; x < n; x += blockDim.x) {
        if (!b.alive[x] || b.mark[x] == stamp) continue;
        int cur = b.parent[x];
        while (cur >= 0 && b.mark[cur] != stamp) cur = b.parent[cur];
        if (cur >= 0 && b.aux[cur] != plen - 1) {
            b.alive[x] = 0;
            atomicAdd(&sh_dead, 1);
            atomicSub(&b.nkids[b.parent[x]], 1);
        }
    }
    __syncthreads();
    // survivors: old frontier nodes strictly under the new root, re-sorted by
    // (-score, token, id) on pre-rebase scores and truncated to K (cache.py:392-408)
    const int nf = S.n_frontier;
    if (!sh_fresh) {
        for (int i = tid; i < nf; i += blockDim.x) {
            const int h = b.frontier[i];
            if (b.alive[h] && h != new_root && descends(b, h, new_root)) surv[atomicAdd(&sh_ns, 1)] = h;
        }
    }
    __syncthreads();
    const int ns = sh_ns;
    for (int i = tid; i < ns; i += blockDim.x) {
        const int h = surv[i];
        const double s = b.score[h];
        const int t = b.token[h];
        int r = 0;
        for (int j = 0; j < ns; ++j) {
            const int g = surv[j];
            const double sg = b.score[g];
            const int tg = b.token[g];
            if (sg > s || (sg == s && (tg < t || (tg == t && g < h)))) ++r;
        }
        b.aux[h] = r;   // reuse aux: not a path node any more
    }
    __syncthreads();
    for (int i = tid; i < ns; i += blockDim.x) {
        const int h = surv[i];
        const int r = b.aux[h];
        if (r < S.K) b.frontier[r] = h;
    }
    // rebase the alive subtree of the new root (cache.py:454-469)
    const double base = b.score[new_root];
    __syncthreads();
    if (base != 0.0) {
        for (int x = tid; x < n; x += blockDim.x)
            if (b.alive[x] && descends(b, x, new_root)) b.score[x] = __dsub_rn(b.score[x], base);
        __syncthreads();
        if (tid == 0) b.score[new_root] = 0.0;
    }
    if (tid == 0) {
        S.n_frontier = ns < S.K ? ns : S.K;
        S.root = new_root;
        S.epoch += 1;
        S.dead += sh_dead;
        // cache.py:471-474; and, unlike the reference's unbounded arena, when
        // the next cycle's expansions (<= max_depth layers of <= K nodes) could
        // overflow the fixed device arena.  At small K the reference's
        // condition can stay false for a whole decode (the committed chain
        // stays alive as ancestors).  Compaction is order-preserving, so every
        // decision (sort / query tie-breaks on node ids) is unchanged; only
        // absolute ids differ from the reference's arena from then on.
        const bool ref_rule = n >= kCompactMinArena && (double)S.dead > 0.75 * (double)n;
        const bool pressure = n + S.K * (S.max_depth + 1) + 2 > S.capacity;
        sh_flag = (ref_rule || pressure) ? 1 : 0;
        S.n_precompact = n;
    }
    __syncthreads();
    if (!sh_flag) return;
    // ---- order-preserving compaction (cache.py:475-504)
    // keep flag = alive and in the root's subtree; reuse s_haskv as the flag buffer
    for (int x = tid; x < n; x += blockDim.x) b.s_haskv[x] = (b.alive[x] && descends(b, x, new_root)) ? 1 : 0;
    __syncthreads();
    const int total = block_scan_flags(b.s_haskv, b.remap, n, sh_warp, &sh_carry);
    for (int x = tid; x < n; x += blockDim.x) {
        const int nx = b.remap[x];
        if (nx < 0) continue;
        const int par = b.parent[x];
        b.s_token[nx] = b.token[x];
        b.s_parent[nx] = (x == new_root || par < 0 || b.remap[par] < 0) ? -1 : b.remap[par];
        b.s_layer[nx] = b.layer[x];
        b.s_score[nx] = b.score[x];
        b.s_edge[nx] = b.edge[x];
        b.aux[nx] = b.has_kv[x];   // staged (aux is free now)
    }
    __syncthreads();
    for (int i = tid; i < S.n_frontier; i += blockDim.x) b.frontier[i] = b.remap[b.frontier[i]];
    for (int x = tid; x < total; x += blockDim.x) {
        b.token[x] = b.s_token[x];
        b.parent[x] = b.s_parent[x];
        b.layer[x] = b.s_layer[x];
        b.score[x] = b.s_score[x];
        b.edge[x] = b.s_edge[x];
        b.has_kv[x] = (uint8_t)b.aux[x];
        b.alive[x] = 1;
        b.nkids[x] = 0;
        b.mark[x] = 0;
        b.mark2[x] = 0;
    }
    const int hcap = S.hash_mask + 1;
    for (int i = tid; i < hcap; i += blockDim.x) b.hkeys[i] = kEmpty;
    __syncthreads();
    for (int x = tid; x < total; x += blockDim.x) {
        const int par = b.parent[x];
        if (par >= 0) {
            atomicAdd(&b.nkids[par], 1);
            hash_insert(b, par, b.token[x], x);
        }
    }
    if (tid == 0) {
        const int nr = b.remap[new_root];
        S.root = nr;
        S.new_root = nr;
        S.n_nodes = total;
        S.dead = 0;
        S.top_layer = b.s_layer[nr];
        S.compacted = 1;
        sh_total = total;
    }
}

__global__ void advance_root_kernel(Bufs b, const int32_t* acc, const int32_t* n_acc_p, const int32_t* corr_p) {
    card_cache_state& S = *b.st;
    if (threadIdx.x >= 32) return;
    const int n_acc = *n_acc_p, corr = *corr_p;
    int anchor = S.root, st = CARD_OK;
    if (n_acc < 0) st = CARD_E_INPUT;
    else if (n_acc > S.max_depth + 1) st = CARD_E_PROTOCOL;
    if (st == CARD_OK) st = walk_chain(b, acc, n_acc, &anchor);
    int new_root = anchor;
    if (st == CARD_OK) {
        if (corr < 0) {
            if (n_acc == 0) st = CARD_E_INPUT;
        } else {
            new_root = alive_child_warp(b, anchor, corr);
        }
    }
    if (lane_id() != 0) return;
    S.status = st;
    S.compacted = 0;
    if (st != CARD_OK) return;
    if (new_root < 0) {   // not cached: caller resets (cache.py:430-432)
        S.moved = 0;
        return;
    }
    S.root = new_root;
    S.new_root = new_root;
    S.chain_len = n_acc + (corr >= 0 ? 1 : 0);
    if (corr >= 0) b.chain[n_acc] = new_root;
    int m = 0;
    for (int i = 0; i < S.n_frontier; ++i)
        if (b.alive[b.frontier[i]]) b.frontier[m++] = b.frontier[i];
    S.n_frontier = m;
    S.epoch += 1;
    S.moved = 1;
}

__global__ void count_alive_kernel(Bufs b) {
    card_cache_state& S = *b.st;
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int root = S.root;
    int c = 0;
    for (int x = threadIdx.x; x < S.n_nodes; x += blockDim.x)
        if (x != root && b.alive[x] && descends(b, x, root)) ++c;
    atomicAdd(&cnt, c);
    __syncthreads();
    if (threadIdx.x == 0) S.alive_below = cnt;
}

__global__ void clear_status_kernel(Bufs b) {
    b.st->status = 0;
    b.st->vstatus = 0;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// w, e, key, k32 (padded to 4), tok, pid, rank
static int pool_smem_bytes(int P) { return P * (8 + 8 + 16 + 4 + 4 + 4 + 4) + 16; }

}  // namespace card

using namespace card;

extern "C" {

int card_cache_create(int root_token, int K, int k, int max_depth, int eos_token, int capacity, card_cache** out) {
    if (!out) return CARD_E_INPUT;
    *out = nullptr;
    if (root_token < 0) return CARD_E_INPUT;
    if (K < 1 || k < 1 || max_depth < 1 || K > kMaxK || (long)K * k > kMaxPool || k > 32 || max_depth > 64)
        return CARD_E_CONFIG;
    if (capacity <= 0) capacity = 6 * K * (max_depth + 1) + 256;
    int hcap = 1;
    while (hcap < 2 * capacity) hcap <<= 1;
    const int md2 = max_depth + 2;
    // carve one allocation
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = align_up(off, 256);
        off = o + bytes;
        return o;
    };
    const size_t o_st = take(sizeof(card_cache_state));
    const size_t cap = (size_t)capacity;
    size_t o_i32[8];
    for (int i = 0; i < 8; ++i) o_i32[i] = take(cap * 4);
    const size_t o_alive = take(cap), o_haskv = take(cap);
    const size_t o_score = take(cap * 8), o_edge = take(cap * 8);
    const size_t o_fr = take((size_t)K * 4), o_fro = take((size_t)K * 4);
    const size_t o_hk = take((size_t)hcap * 8), o_hv = take((size_t)hcap * 4);
    const size_t o_ctok = take((size_t)K * k * 4), o_ccnt = take((size_t)K * 4), o_cval = take((size_t)K * k * 8);
    const size_t o_qp = take(md2 * 4), o_qt = take(md2 * 4), o_qe = take(md2 * 8), o_ch = take(md2 * 4);
    const size_t o_chkv = take(md2 * 4);
    const size_t o_st_tok = take(cap * 4), o_st_par = take(cap * 4), o_st_lay = take(cap * 4);
    const size_t o_st_hk = take(cap), o_st_sc = take(cap * 8), o_st_ed = take(cap * 8);
    void* block = nullptr;
    CARD_CUDA_TRY(cudaMalloc(&block, off));
    CARD_CUDA_TRY(cudaMemset(block, 0, off));
    char* base = (char*)block;
    card_cache* h = (card_cache*)calloc(1, sizeof(card_cache));
    h->block = block;
    h->bytes = off;
    h->K = K;
    h->k = k;
    h->max_depth = max_depth;
    h->eos = eos_token < 0 ? -1 : eos_token;
    h->capacity = capacity;
    h->hcap = hcap;
    Bufs& b = h->b;
    b.st = (card_cache_state*)(base + o_st);
    int32_t** i32s[8] = {&b.token, &b.parent, &b.layer, &b.nkids, &b.mark, &b.mark2, &b.aux, &b.remap};
    for (int i = 0; i < 8; ++i) *i32s[i] = (int32_t*)(base + o_i32[i]);
    b.alive = (uint8_t*)(base + o_alive);
    b.has_kv = (uint8_t*)(base + o_haskv);
    b.score = (double*)(base + o_score);
    b.edge = (double*)(base + o_edge);
    b.frontier = (int32_t*)(base + o_fr);
    b.frontier_old = (int32_t*)(base + o_fro);
    b.hkeys = (unsigned long long*)(base + o_hk);
    b.hvals = (int32_t*)(base + o_hv);
    b.c_tok = (int32_t*)(base + o_ctok);
    b.c_cnt = (int32_t*)(base + o_ccnt);
    b.c_val = (double*)(base + o_cval);
    b.q_path = (int32_t*)(base + o_qp);
    b.q_tok = (int32_t*)(base + o_qt);
    b.q_edge = (double*)(base + o_qe);
    b.chain = (int32_t*)(base + o_ch);
    b.chain_kv = (int32_t*)(base + o_chkv);
    b.s_token = (int32_t*)(base + o_st_tok);
    b.s_parent = (int32_t*)(base + o_st_par);
    b.s_layer = (int32_t*)(base + o_st_lay);
    b.s_haskv = (uint8_t*)(base + o_st_hk);
    b.s_score = (double*)(base + o_st_sc);
    b.s_edge = (double*)(base + o_st_ed);
    card_cache_state st;
    memset(&st, 0, sizeof(st));
    st.K = K;
    st.k = k;
    st.max_depth = max_depth;
    st.eos = h->eos;
    st.capacity = capacity;
    st.hash_mask = hcap - 1;
    CARD_CUDA_TRY(cudaMemcpy(b.st, &st, sizeof(st), cudaMemcpyHostToDevice));
    static bool attr_done = false;
    if (!attr_done) {
        CARD_CUDA_TRY(cudaFuncSetAttribute(expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           pool_smem_bytes(kMaxPool)));
        CARD_CUDA_TRY(cudaFuncSetAttribute(pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           pool_smem_bytes(kMaxPool)));
        attr_done = true;
    }
    clear_hash_kernel<<<64, 256>>>(b, hcap);
    CARD_LAUNCH_CHECK();
    init_root_kernel<<<1, 1>>>(b, nullptr, root_token, 0);
    CARD_LAUNCH_CHECK();
    CARD_CUDA_TRY(cudaDeviceSynchronize());
    *out = h;
    return CARD_OK;
}

int card_cache_destroy(card_cache* h) {
    if (!h) return CARD_OK;
    cudaFree(h->block);
    free(h);
    return CARD_OK;
}

namespace card {
__global__ void state_init_kernel(card_cache_state* st, int K, int k, int max_depth, int eos, int capacity,
                                  int hash_mask) {
    st->K = K;
    st->k = k;
    st->max_depth = max_depth;
    st->eos = eos;
    st->capacity = capacity;
    st->hash_mask = hash_mask;
}
}  // namespace card

int card_cache_clear(card_cache* h, int root_token, void* stream) {
    if (!h) return CARD_E_INPUT;
    if (root_token < 0) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    CARD_CUDA_TRY(cudaMemsetAsync(h->block, 0, h->bytes, s));
    state_init_kernel<<<1, 1, 0, s>>>(h->b.st, h->K, h->k, h->max_depth, h->eos, h->capacity, h->hcap - 1);
    clear_hash_kernel<<<64, 256, 0, s>>>(h->b, h->hcap);
    init_root_kernel<<<1, 1, 0, s>>>(h->b, nullptr, root_token, 0);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_reset(card_cache* h, const int32_t* d_root_token, int root_token, void* stream) {
    if (!h) return CARD_E_INPUT;
    if (!d_root_token && root_token < 0) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    clear_hash_kernel<<<64, 256, 0, s>>>(h->b, h->hcap);
    init_root_kernel<<<1, 1, 0, s>>>(h->b, d_root_token, root_token, 1);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_expand(card_cache* h, const double* dists, int n_rows, int vocab, void* stream) {
    if (!h) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    const int rows = n_rows >= 0 ? n_rows : h->K;
    if (rows > h->K || rows < 0) return CARD_E_INPUT;
    int rc = launch_rows_topk(dists, rows, vocab, h->k, h->b.c_tok, h->b.c_val, h->b.c_cnt, &h->b.st->vstatus, s);
    if (rc) return rc;
    const int P = (n_rows >= 0 ? (n_rows > 0 ? n_rows : 1) : h->K) * h->k;
    expand_kernel<<<1, kThreads, pool_smem_bytes(P), s>>>(h->b, h->b.c_tok, h->b.c_val, h->b.c_cnt, n_rows, 0,
                                                          nullptr);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_expand_topk(card_cache* h, const int32_t* tok, const double* val, const int32_t* cnt, int n_rows,
                           int values_are_probs, const int32_t* skip, void* stream) {
    if (!h) return CARD_E_INPUT;
    const int P = (n_rows > 0 ? n_rows : h->K) * h->k;
    expand_kernel<<<1, kThreads, pool_smem_bytes(P), (cudaStream_t)stream>>>(h->b, tok, val, cnt, n_rows,
                                                                             values_are_probs ? 0 : 1, skip);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_pool(card_cache* h, const double* dists, int n_rows, int vocab, int32_t* out_tok, double* out_w,
                    int32_t* out_pidx, double* out_edge, void* stream) {
    if (!h || n_rows < 1 || n_rows > h->K) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    int rc = launch_rows_topk(dists, n_rows, vocab, h->k, h->b.c_tok, h->b.c_val, h->b.c_cnt, &h->b.st->vstatus, s);
    if (rc) return rc;
    pool_kernel<<<1, 256, pool_smem_bytes(n_rows * h->k), s>>>(h->b, out_tok, out_w, out_pidx, out_edge);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_query(card_cache* h, int depth, void* stream) {
    if (!h) return CARD_E_INPUT;
    if (depth < 1) return CARD_E_INPUT;
    query_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(h->b, depth, nullptr);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

// card_cache_query unless *skip (device flag)
int card_cache_query_if(card_cache* h, int depth, const int32_t* skip, void* stream) {
    if (!h || depth < 1) return CARD_E_INPUT;
    query_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(h->b, depth, skip);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_query_buffers(card_cache* h, int32_t** path, int32_t** tok, double** edge) {
    if (!h) return CARD_E_INPUT;
    if (path) *path = h->b.q_path;
    if (tok) *tok = h->b.q_tok;
    if (edge) *edge = h->b.q_edge;
    return CARD_OK;
}

int card_cache_correct(card_cache* h, const int32_t* accepted, const int32_t* n_accepted, const int32_t* correction,
                       const int32_t* skip, void* stream) {
    if (!h) return CARD_E_INPUT;
    correct_kernel<<<1, kThreads, 0, (cudaStream_t)stream>>>(h->b, accepted, n_accepted, correction, skip);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_advance_root(card_cache* h, const int32_t* accepted, const int32_t* n_accepted,
                            const int32_t* correction, void* stream) {
    if (!h) return CARD_E_INPUT;
    advance_root_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(h->b, accepted, n_accepted, correction);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_count_alive(card_cache* h, void* stream) {
    if (!h) return CARD_E_INPUT;
    count_alive_kernel<<<1, kThreads, 0, (cudaStream_t)stream>>>(h->b);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_clear_status(card_cache* h, void* stream) {
    if (!h) return CARD_E_INPUT;
    clear_status_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(h->b);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_cache_read_state(card_cache* h, card_cache_state* st, void* stream) {
    if (!h || !st) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    CARD_CUDA_TRY(cudaMemcpyAsync(st, h->b.st, sizeof(*st), cudaMemcpyDeviceToHost, s));
    CARD_CUDA_TRY(cudaStreamSynchronize(s));
    return CARD_OK;
}

int card_cache_snapshot(card_cache* h, int32_t* token, int32_t* parent, int32_t* layer, uint8_t* alive, double* score,
                        double* edge, int32_t* frontier, void* stream) {
    if (!h) return CARD_E_INPUT;
    cudaStream_t s = (cudaStream_t)stream;
    card_cache_state st;
    CARD_CUDA_TRY(cudaMemcpyAsync(&st, h->b.st, sizeof(st), cudaMemcpyDeviceToHost, s));
    CARD_CUDA_TRY(cudaStreamSynchronize(s));
    const size_t n = (size_t)st.n_nodes;
    if (token) CARD_CUDA_TRY(cudaMemcpyAsync(token, h->b.token, n * 4, cudaMemcpyDeviceToHost, s));
    if (parent) CARD_CUDA_TRY(cudaMemcpyAsync(parent, h->b.parent, n * 4, cudaMemcpyDeviceToHost, s));
    if (layer) CARD_CUDA_TRY(cudaMemcpyAsync(layer, h->b.layer, n * 4, cudaMemcpyDeviceToHost, s));
    if (alive) CARD_CUDA_TRY(cudaMemcpyAsync(alive, h->b.alive, n, cudaMemcpyDeviceToHost, s));
    if (score) CARD_CUDA_TRY(cudaMemcpyAsync(score, h->b.score, n * 8, cudaMemcpyDeviceToHost, s));
    if (edge) CARD_CUDA_TRY(cudaMemcpyAsync(edge, h->b.edge, n * 8, cudaMemcpyDeviceToHost, s));
    if (frontier) CARD_CUDA_TRY(cudaMemcpyAsync(frontier, h->b.frontier, (size_t)st.n_frontier * 4,
                                                cudaMemcpyDeviceToHost, s));
    CARD_CUDA_TRY(cudaStreamSynchronize(s));
    return CARD_OK;
}

int card_cache_device_ptrs(card_cache* h, card_cache_state** st, int32_t** token, int32_t** parent, int32_t** layer,
                           int32_t** frontier, int32_t** remap, int32_t** chain, int32_t** chain_kv) {
    if (!h) return CARD_E_INPUT;
    if (st) *st = h->b.st;
    if (token) *token = h->b.token;
    if (parent) *parent = h->b.parent;
    if (layer) *layer = h->b.layer;
    if (frontier) *frontier = h->b.frontier;
    if (remap) *remap = h->b.remap;
    if (chain) *chain = h->b.chain;
    if (chain_kv) *chain_kv = h->b.chain_kv;
    return CARD_OK;
}

}  // extern "C"
