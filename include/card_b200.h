/*
 * card_b200.h — C-ABI of the B200-native CARD query-and-correct path.
 *
 * Plain pointers and sizes only.  Unless stated otherwise every pointer
 * argument is a DEVICE pointer owned by the caller, every call is
 * asynchronous on the caller's cudaStream_t (passed as void*), and every
 * call returns an int status (CARD_OK or a negative CARD_E_* code).  No
 * C++ exception crosses this boundary.  Device-side protocol errors (a
 * rejected walk, a full frontier, a bad distribution) are written to the
 * cache's status word and read back with card_cache_status().
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/specache):
 *   operator plug-in  backend.py:42-47 get_kernels() module protocol
 *                     {kgram_dist (_kernels.pyx:44-93), rows_topk (_kernels.pyx:96-145)}
 *   candidate cache   cache.py:92-523 TreeCache
 *   verification      verify.py:43-132
 *   model plug-in     lm.py:109-196 ToyModel.next_distribution / batch_tree_forward
 * One cache handle per request, never shared by two writers.
 */
#ifndef CARD_B200_H
#define CARD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CARD_ABI_VERSION 1

/* status codes; the Python mirror maps them onto errors.py:6-45 */
#define CARD_OK              0
#define CARD_E_INPUT        -1   /* InputError      */
#define CARD_E_CONFIG       -2   /* ConfigError     */
#define CARD_E_PROTOCOL     -3   /* ProtocolError   */
#define CARD_FRONTIER_FULL  -4   /* FrontierFull    */
#define CARD_E_CAPACITY     -5   /* arena capacity exhausted (sizing bug) */
#define CARD_E_CUDA         -6   /* CUDA runtime error */
#define CARD_E_MASK         -7   /* MaskError       */

int         card_abi_version(void);
const char* card_strerror(int code);
/* last CUDA error string recorded by a failing call (host memory, static) */
const char* card_last_cuda_error(void);

/* ------------------------------------------------------------------ *
 * operator plug-in (backend.py:42-47)
 * ------------------------------------------------------------------ */

/* Hashed k-gram next-token distributions for n_rows contexts.
 * tails: [n_rows, tail_len] int32 (the last `order` tokens of each context,
 * -1 marking "context shorter than the order");
 * out: [n_rows, vocab] float64.  Replaces _kernels.pyx:44-93 (bit-exact
 * integer stream; fp64 softmax with a correctly rounded exp). */
int card_kgram_dist(uint64_t seed, uint64_t seed2, double mix_weight,
                    const int32_t* tails, int tail_len, int tail_stride, int n_rows, int vocab,
                    double sharpness, double temperature, double* out, void* stream);

/* Per-row top-k by (p desc, token asc), p <= 0 excluded.  dists:
 * [n_rows, vocab] float64; out_tok/out_p: [n_rows, k]; out_cnt: [n_rows].
 * If status != NULL, rows are also validated as in cache.py:204-208
 * (no NaN / negative, sum within 1e-9 of 1) and *status gets CARD_E_INPUT
 * on failure.  Replaces _kernels.pyx:96-145. */
int card_rows_topk(const double* dists, int n_rows, int vocab, int k,
                   int32_t* out_tok, double* out_p, int32_t* out_cnt,
                   int32_t* status, void* stream);

/* Correctly rounded natural log / exp over n doubles (parity helpers). */
int card_log_cr(const double* x, double* y, int n, void* stream);
int card_exp_cr(const double* x, double* y, int n, void* stream);

/* ------------------------------------------------------------------ *
 * device candidate tree (cache.py:92-523)
 * ------------------------------------------------------------------ */

typedef struct card_cache card_cache;

/* Host-visible copy of the device state word block (card_cache_state). */
typedef struct card_cache_state {
    int32_t n_nodes, root, n_frontier, epoch;
    int32_t dead, status, vstatus, stamp;
    int32_t top_layer, last_width, compacted, moved;
    int32_t K, k, max_depth, eos;
    int32_t capacity, hash_mask, fresh, new_root;
    int32_t q_hit, q_len, chain_len, alive_below;
    int32_t n_precompact, reserved[7];
} card_cache_state;

/* Create a cache rooted at root_token (cache.py:95-105).  eos_token < 0
 * means None.  capacity <= 0 picks a bound that covers the corrected
 * protocol (compaction keeps the arena below ~5*K*max_depth).  This call
 * allocates device memory and synchronises. */
int card_cache_create(int root_token, int K, int k, int max_depth, int eos_token,
                      int capacity, card_cache** out);
int card_cache_destroy(card_cache* h);

/* Return the handle to the state card_cache_create(root_token, ...) leaves
 * it in (arena, hash, frontier, epoch and counters), asynchronously on
 * `stream`.  No reference counterpart: it lets a serving session reuse one
 * arena (and the CUDA graphs that point into it) across requests. */
int card_cache_clear(card_cache* h, int root_token, void* stream);

/* reset(root_token) (cache.py:439-444).  If d_root_token != NULL the token
 * is read on the device (engine path), else root_token is used. */
int card_cache_reset(card_cache* h, const int32_t* d_root_token, int root_token, void* stream);

/* expand_layer(distributions) (cache.py:224-251): validate, row top-k,
 * edge = log(p), global top-K by (-weight, token, parent id), allocate,
 * prune dead ends.  n_rows must equal len(expansion_parents()); pass -1 to
 * take it from the device (engine path). */
int card_cache_expand(card_cache* h, const double* dists, int n_rows, int vocab, void* stream);

/* Same, from precomputed per-row candidates — the fused lm_head top-k output
 * (log-probs) or a row top-k over fp64 distributions (probabilities, the
 * log is taken on the device).  tok/val: [n_rows, k]; cnt: [n_rows].  If
 * skip is non-NULL and *skip != 0 on the device, the call is a no-op. */
int card_cache_expand_topk(card_cache* h, const int32_t* tok, const double* val,
                           const int32_t* cnt, int n_rows, int values_are_probs,
                           const int32_t* skip, void* stream);

/* Candidate pool of extension_pool() (cache.py:190-222) for the drop-in:
 * writes P = n_rows*k slots of (token or -1, weight, parent index, edge). */
int card_cache_pool(card_cache* h, const double* dists, int n_rows, int vocab,
                    int32_t* out_tok, double* out_w, int32_t* out_pidx, double* out_edge,
                    void* stream);

/* query(depth) (cache.py:277-318).  Result in the state block (q_hit, q_len)
 * and in the cache's query buffers (card_cache_query_buffers). */
int card_cache_query(card_cache* h, int depth, void* stream);
/* card_cache_query unless *skip != 0 (device flag; the mailbox driver's
 * "no correction arrived" flag) */
int card_cache_query_if(card_cache* h, int depth, const int32_t* skip, void* stream);
int card_cache_query_buffers(card_cache* h, int32_t** path, int32_t** tok, double** edge);

/* correct(accepted, correction) (cache.py:355-413).  All inputs on the
 * device: accepted[0..*n_accepted), *correction < 0 means None; skip as above.
 * Before compaction the kernel records the walked chain (+ new root) in the
 * chain buffer and whether each had tree KV (chain_kv), and sets
 * state.n_precompact / state.compacted / remap[] for the draft KV mover. */
int card_cache_correct(card_cache* h, const int32_t* accepted, const int32_t* n_accepted,
                       const int32_t* correction, const int32_t* skip, void* stream);

/* advance_root (cache.py:415-437); state.moved = 1 on success, 0 if the
 * correction token is not cached (caller then resets). */
int card_cache_advance_root(card_cache* h, const int32_t* accepted, const int32_t* n_accepted,
                            const int32_t* correction, void* stream);

/* alive_below_root() (cache.py:174-184) into state.alive_below. */
int card_cache_count_alive(card_cache* h, void* stream);

/* Clear the status word (stream-ordered). */
int card_cache_clear_status(card_cache* h, void* stream);

/* Synchronous host reads (parity / drop-in API).  Arrays are host buffers of
 * at least state.n_nodes (arena) / K (frontier) entries; NULL skips one. */
int card_cache_read_state(card_cache* h, card_cache_state* st, void* stream);
int card_cache_snapshot(card_cache* h, int32_t* token, int32_t* parent, int32_t* layer,
                        uint8_t* alive, double* score, double* edge, int32_t* frontier,
                        void* stream);
/* Device pointers of the state block and arrays (engine kernels chain on them). */
int card_cache_device_ptrs(card_cache* h, card_cache_state** st, int32_t** token,
                           int32_t** parent, int32_t** layer, int32_t** frontier,
                           int32_t** remap, int32_t** chain, int32_t** chain_kv);


/* ------------------------------------------------------------------ *
 * model plug-in: KV-cached transformer forward (lm.py:109-196)
 * ------------------------------------------------------------------ *
 * dtype codes: 0 = bf16, 1 = fp32.  `dM` / `n_out` are device row counts so
 * one captured CUDA graph serves every step of a decode. */

typedef struct card_linear card_linear;

/* Y[M,N] = X[M,K] . W[N,K]^T with a fused epilogue (0 store f32, 1 residual
 * add f32, 2 store bf16, 3 SwiGLU -> bf16 with gate/up rows interleaved per
 * 128-row tile, 4 QKV RoPE + KV-cache write, see card_linear_fuse_rope).  wdtype: 0 bf16 row-major (tcgen05 + tensor-map TMA for
 * m_max >= 2, 128-bit-load GEMV for m_max == 1), 1 fp32 (parity kernel),
 * 2 bf16 pre-tiled [N/128][K/64][128x64] blocks in SWIZZLE_128B order
 * (card_tile_weights; one contiguous 16 KB bulk copy per pipeline stage).
 * X must hold round_up(m_max, 16) rows.  bias: optional fp32 [N]. */
int card_linear_create(const void* W, int N, int K, int wdtype, const void* X, int m_max, int epi,
                       void* out, int ldo, const float* bias, card_linear** out_h);
int card_linear_run(card_linear* h, const int32_t* dM, void* stream);
int card_linear_info(card_linear* h, int32_t* info8);
/* Fused epilogues (bf16 tcgen05 path only):
 * fuse_norm: the linear consumes the bf16 residual and applies RMSNorm as a
 *   per-token output scale rsqrt(sum_p ssq[p*ld + off + m] / H + eps) (the norm
 *   weight is folded into W at pack time); x_row_off (device, may be NULL) is
 *   the first X row — the lm_head runs over a contiguous output-row range.
 * fuse_resid: an EPI_RESID_F32 linear also writes bf16(x_new) to xb_out and
 *   the per-16-column sum of squares of x_new to ssq_out[(col/16)*ld + m].
 * fuse_rope: an EPI_QKV_ROPE (4) linear writes RoPE(q)/sqrt(hd) to q_out
 *   [m, nh*hd] fp32 and RoPE(k), v to the KV cache rows slot[m] (bf16).
 * These replace the rmsnorm and rope kernels between the GEMMs of a layer. */
int card_linear_fuse_norm(card_linear* h, const float* ssq, int parts, int ld, float eps, int H,
                          const int32_t* x_row_off);
int card_linear_fuse_resid(card_linear* h, float* ssq_out, int ld, void* xb_out);
int card_linear_fuse_rope(card_linear* h, const int32_t* pos, const int32_t* slot, const float* cos_t,
                          const float* sin_t, int nh, int nkv, int hd, float* q_out, void* k_cache, void* v_cache);
/* fuse_kgram: an EPI_STORE_F32 lm_head adds the k-gram logit bias of
 * card_logit_bias (_kernels.pyx:44-93 uniforms, output row m's context tail
 * ctx_tail[m*stride ..]) to every logit it stores, so the top-k / argmax
 * readers run without it.  Same fp32 arithmetic as the readers' on-the-fly
 * bias (bit-identical logits).  ctx_tail == NULL turns it off. */
int card_linear_fuse_kgram(card_linear* h, const int32_t* ctx_tail, int order, int stride, uint64_t seed,
                           uint64_t seed2, float mix_weight, float sharpness);
/* fuse_topk: an EPI_TOPK (5) lm_head (pre-tiled bf16 weights) stores no
 * logits.  For every output row m and 128-token vocab tile t it writes the
 * record out[(m * (N/128) + t) * 10] = [max, sum exp(x - max), (x, token) x 4]
 * over x = logit * inv_temp (k-gram bias first, if fused; tokens >= V are
 * padding and skipped).  card_lmhead_topk_merge combines the records into the
 * rows_topk result (fused lm_head + softmax + top-k). */
int card_linear_fuse_topk(card_linear* h, int V, float inv_temp);
/* Merge the EPI_TOPK records of rows [0, *dM): fp64 log-sum-exp over the
 * n_tiles tiles and the top-k (k <= 4) by (value desc, token asc); out_logp =
 * value - lse (same output contract as card_topk_logits). */
int card_lmhead_topk_merge(const float* work, const int32_t* dM, int m_max, int n_tiles, int k, int V,
                           int32_t* out_tok, double* out_logp, int32_t* out_cnt, void* stream);
/* tuning: per-CTA %globaltimer stamps [grid][16] (NULL disables) */
int card_linear_trace(card_linear* h, unsigned long long* trace);
int card_linear_destroy(card_linear* h);

/* Persistent wide forward (draft tree steps, 16 < m_max <= 128 rows; bf16,
 * folded norms).  One CTA per SM walks steps = (layer, phase), phase 0 qkv,
 * 1 attention, 2 o, 3 gate/up, 4 down: weight blocks stream into a ring across
 * step boundaries, split-K partials meet in an L2 workspace and are reduced
 * in fixed split order with the qkv (RoPE, KV write) / residual / SwiGLU
 * epilogues of card_linear_fuse_*.  Replaces the per-GEMM launches of the
 * draft forward behind lm.py:155-196 batch_tree_forward (engine.py:198-221).
 * layer_w: host array [n_layers*4] of pre-tiled wqkv, wo, wgu (interleaved),
 * wd; bqkv: host array [n_layers] (NULL: no bias); kv: [n_layers*2] k, v
 * caches [slots, nkv, hd] bf16.  Buffers as the fused forward's (x fp32
 * [rows,H], xb bf16 [rows,H], ssq [H/16][ssq_ld], q fp32 [rows, nh*hd],
 * o bf16 [rows, nh*hd], g bf16 [rows, F]); act_rows = their row count.
 * card_pfwd_run executes steps [step_begin, step_end) on the stream (a
 * cooperative launch); attention steps are run by card_attention_paged between
 * runs, so a range must not contain one (CARD_E_CONFIG). */
typedef struct card_pfwd card_pfwd;
int card_pfwd_create(int n_layers, int H, int F, int nh, int nkv, int hd, int m_max, const void* const* layer_w,
                     const float* const* bqkv, void* const* kv, float* x, void* xb, float* ssq, int ssq_ld, float* q,
                     void* o, void* g, int act_rows, const int32_t* pos, const int32_t* slot, const float* cos_t,
                     const float* sin_t, float eps, card_pfwd** out);
int card_pfwd_run(card_pfwd* h, const int32_t* dM, int step_begin, int step_end, void* stream);
/* grid (CTAs, one per SM) of the next launches, with the split-K ways
 * re-derived for it: the SM count of the partition the forward runs on
 * (card_green); 0 = the whole device */
int card_pfwd_set_grid(card_pfwd* h, int grid);
/* qkv epilogue writes Q as pre-swizzled bf16 tiles for card_attention_tree
 * ([nkv][tiles][hd/64][128 x 64] SWIZZLE_128B; tiles >= ceil(Mpad*nh/nkv/128))
 * instead of fp32 q; NULL restores fp32 q */
int card_pfwd_set_qsw(card_pfwd* h, void* qsw, int tiles);
/* bind the row block's positions and KV slots (qkv epilogue) */
int card_pfwd_bind(card_pfwd* h, const int32_t* pos, const int32_t* slot);
/* info16: grid, smem, weight stages, activation stages, Mpad, then (splits,
 * units) per phase, [15] epilogue worker groups */
int card_pfwd_info(card_pfwd* h, int32_t* info16);
/* tuning: per-CTA %globaltimer stamps [grid][2 + 8 * steps] of the next runs (NULL disables) */
int card_pfwd_trace(card_pfwd* h, unsigned long long* trace);
/* tuning: split-K ways (1..10) of one GEMM phase (0 qkv, 2 o, 4 down) */
int card_pfwd_tune(card_pfwd* h, int phase, int splits);
int card_pfwd_destroy(card_pfwd* h);

/* The lm_head reads its n_out input rows as one contiguous block; for a
 * batched draft step (whose output rows are spread over the requests'
 * regions) copy row out_rows[o] of the bf16 residual and of its
 * per-16-column sums of squares to row o of xb_out / ssq_out first. */
int card_gather_rows(const int32_t* out_rows, const int32_t* n_out, int m_max, int H, const void* xb, const float* ssq,
                     int ssq_ld, void* xb_out, float* ssq_out, int ssq_out_ld, void* stream);
/* x[r] = E[tok[r]] (fp32 residual); if xb != NULL also its bf16 copy and the
 * per-16-column sums of squares ssq[(col/16)*ssq_ld + r] (fused-norm input) */
/* Tensor-parallel target: after the NCCL all-reduce of a
 * row-parallel o / down projection partial, x += part and refresh the bf16
 * residual copy + per-16-column sums of squares (ssq[H/16][ssq_ld]). */
int card_resid_add(const int32_t* dM, int m_max, int H, float* x, const float* part, void* xb, float* ssq, int ssq_ld,
                   void* stream);
int card_embed(const int32_t* tok, const int32_t* dM, int m_max, const void* E, int wdtype, int H,
               float* x, void* xb, float* ssq, int ssq_ld, void* stream);
int card_rmsnorm(const float* x, const float* w, int H, float eps, const int32_t* dM, int m_max,
                 const int32_t* gather, void* y, int ydtype, void* stream);
int card_rope_kv(const float* qkv, const int32_t* dM, int m_max, const int32_t* pos, const int32_t* slot,
                 const float* cos_t, const float* sin_t, int nh, int nkv, int hd, float* q,
                 void* k_cache, void* v_cache, int kvdtype, void* stream);
int card_attention_work_floats(int m_max, int nh, int hd, int max_plen);
/* tuning: per-CTA %globaltimer stamps [grid][8] of the fused attention (NULL disables) */
int card_attention_trace(unsigned long long* buf);
/* slot: the rows' KV slots (row block), lets the fused bf16 kernel start on old
 * KV before the QKV GEMM that writes the new rows has finished */
int card_attention(const float* q, const int32_t* dM, int m_max, const int32_t* plen, const int32_t* slot,
                   const int32_t* n_extra, const int32_t* extra, int extra_max, const void* k_cache,
                   const void* v_cache, int kvdtype, int nh, int nkv, int hd, int max_plen, float* work,
                   void* o, int odtype, void* stream);
/* Tree / chain attention over a paged KV cache (bf16 K/V and output, head_dim
 * 64 or 128): prefix position p of every row lives in KV slot
 * page_table[p / 64] * 64 + p % 64 (page_table NULL: slot p); extra slots are
 * physical.  Wide forwards (>= 256 query-heads per KV head: draft tree rows,
 * prefill) run the tcgen05 kernel (S = QK^T and O = PV in TMEM); verify / AR
 * rows the register-resident mma.sync kernel.  The bf16 model forward's
 * attention.  Replaces the tree-mask forward of mask.py:173-217 /
 * lm.py:155-196. */
int card_attention_paged(const float* q, const int32_t* dM, int m_max, const int32_t* plen,
                         const int32_t* n_extra, const int32_t* extra, int extra_max, const void* k_cache,
                         const void* v_cache, const int32_t* page_table, int nh, int nkv, int hd, int max_plen,
                         void* o, void* stream);
/* card_attention_paged's tcgen05 kernel with the Q operand read as
 * pre-swizzled bf16 tiles (the persistent forward's qkv epilogue output,
 * card_pfwd_set_qsw) instead of converted from fp32 q: one bulk copy per
 * tile.  Same arithmetic and results as card_attention_paged. */
int card_attention_tree(const void* qsw, int qsw_tiles, const int32_t* dM, int m_max, const int32_t* plen,
                        const int32_t* n_extra, const int32_t* extra, int extra_max, const void* k_cache,
                        const void* v_cache, const int32_t* page_table, int nh, int nkv, int hd, int max_plen,
                        void* o, void* stream);
/* Batched forward of several requests: rows [i*seg_rows,
 * (i+1)*seg_rows) belong to request i, whose prefix position p lives in KV
 * slot page_tables[i*pt_stride + p/64]*64 + p%64; extras are physical slots.
 * Rows with plen = 0 and no extras are padding (output zero).  Always the
 * tcgen05 kernel; Q from fp32 q, or from pre-swizzled tiles when qsw != NULL
 * (card_pfwd_set_qsw).  A tile's rows may span requests: each request's
 * prefix is its own run of key rounds, masked per row. */
int card_attention_batch(const float* q, const void* qsw, int qsw_tiles, const int32_t* dM, int m_max,
                         const int32_t* plen, const int32_t* n_extra, const int32_t* extra, int extra_max,
                         const void* k_cache, const void* v_cache, const int32_t* page_tables, int pt_stride,
                         int seg_rows, int nh, int nkv, int hd, int max_plen, void* o, void* stream);
/* draft lm_head epilogue: per-row top-k by (logit desc, token asc) with
 * log-probs logit/T - logsumexp (replaces extension_pool's rows_topk+log).
 * If ctx_tail != NULL the k-gram logit bias of card_logit_bias is applied on
 * the fly (same arithmetic); likewise for card_argmax_logits. */
int card_lmhead_work_floats(int m_max, int k);
int card_topk_logits(const float* logits, const int32_t* dM, int m_max, int V, int k, double inv_temp,
                     int32_t* out_tok, double* out_logp, int32_t* out_cnt, float* work, const int32_t* ctx_tail,
                     int order, int stride, uint64_t seed, uint64_t seed2, float mix_weight, float sharpness,
                     void* stream);
/* target greedy: first maximum per row (verify.py:38-40); vocab split over
 * CTAs, merged in a second launch.  work: card_lmhead_work_floats floats. */
int card_argmax_logits(const float* logits, const int32_t* dM, int m_max, int V, int32_t* out, float* work,
                       const int32_t* ctx_tail, int order, int stride, uint64_t seed, uint64_t seed2,
                       float mix_weight, float sharpness, void* stream);
int card_softmax64(const float* logits, const int32_t* dM, int m_max, int V, double inv_temp, double* out,
                   void* stream);
/* agreement knob: logits[r] += sharpness * (u1 + mix_weight * u2), u the
 * splitmix64 k-gram stream of (seed, ctx_tail[r]) (_kernels.pyx:26-41). */
int card_logit_bias(float* logits, const int32_t* dM, int m_max, int V, const int32_t* ctx_tail, int order,
                    int stride, uint64_t seed, uint64_t seed2, float mix_weight, float sharpness, void* stream);

/* ------------------------------------------------------------------ *
 * engine: the query-and-correct cycle (engine.py:198-317) on the device
 * ------------------------------------------------------------------ *
 * card_engine_state is a device struct of int32 fields (layout in
 * paper_2508_04462_b200/_lib.py: EngineState); `rows` is an int32 block
 * [M, n_out, tok[R], pos[R], slot[R], plen[R], n_extra[R], out_rows[R],
 * extra[R*E]] with R = rows_max, E = extra_max. */
typedef struct card_engine_state card_engine_state;
int card_engine_state_bytes(void);
/* page_table (NULL: identity): the run's prefix pages, 64 KV slots each —
 * chain rows write their K/V to slot page_table[p / 64] * 64 + p % 64. */
int card_draft_rows(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows,
                    int rows_max, int extra_max, int tree_base, int32_t* ctx_tail, int order,
                    const int32_t* page_table, void* stream);
int card_target_rows(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows,
                     int rows_max, int extra_max, int32_t* ctx_tail, int order, const int32_t* page_table,
                     void* stream);
/* SM partitions of one GPU for mode="concurrent" (engine.py:320-389): two
 * green contexts, draft_sms SMs (rounded up to the partition granularity)
 * for the draft and the rest for the target, each with a stream.  Kernels
 * and CUDA graphs captured on a partition's stream run on its SMs only;
 * memory is shared with the primary context. */
typedef struct card_green card_green;
int card_green_create(int device, int draft_sms, card_green** out);
int card_green_stream(card_green* g, int part, void** stream, int* sms);
int card_green_destroy(card_green* g);

/* Draft <-> target mailboxes of mode="concurrent" across two GPUs
 * (engine.py:320-389 lock + epoch).  Each direction is
 * a box in the receiver's memory written by the sender's kernel with P2P
 * stores and published by a system-scope release of a sequence number:
 * the query box (target GPU) carries the path queried after a correction
 * and the tree epoch; the commit box (draft GPU) the verify outcome.
 *   draft stream, every draft step: poll_commit (a new commit -> the draft
 *     state, skip flag 0; else 1), card_cache_correct / card_cache_query_if
 *     gated by the skip flag, publish_query (force = 0: only after a
 *     correction), then the expansion;
 *   target stream, every verify: wait_query (blocks on an acquire poll),
 *     card_target_rows_view on the delivered query, forward, verify,
 *     commit, publish_commit.
 * Devices may be equal (then the boxes are local). */
typedef struct card_mailbox card_mailbox;
int card_mailbox_create(int draft_dev, int target_dev, card_mailbox** out);
int card_mailbox_destroy(card_mailbox* m);
/* boxes and sequence numbers to zero between requests (both devices idle) */
int card_mailbox_reset(card_mailbox* m);
int card_mailbox_skip_flag(card_mailbox* m, int32_t** skip);
int card_mailbox_query_view(card_mailbox* m, card_cache_state** view, int32_t** q_tok);
int card_mailbox_poll_commit(card_mailbox* m, card_engine_state* draft_state, void* stream);
int card_mailbox_publish_query(card_mailbox* m, card_cache* h, int force, void* stream);
int card_mailbox_wait_query(card_mailbox* m, void* stream);
int card_mailbox_publish_commit(card_mailbox* m, const card_engine_state* target_state, void* stream);

/* Batched decode (the reference runs one request at a time,
 * engine.py:275-287): each request builds its rows into its own region
 * [row_base, row_base + rows_cap) of one combined row block of rows_max rows
 * (outputs [out_base, out_base + out_cap)) and pads the rest of the region
 * (plen 0, KV to dead_slot), so one forward serves every request.  The
 * caller owns the block header (M = all regions, n_out = all output
 * regions).  A request whose rows overflow its region ends with done = -1
 * (raised as ProtocolError by the host). */
int card_draft_rows_at(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows, int rows_max,
                       int extra_max, int row_base, int rows_cap, int out_base, int out_cap, int dead_slot,
                       int tree_base, int32_t* ctx_tail, int order, const int32_t* page_table, void* stream);
int card_target_rows_at(card_engine_state* E, card_cache* h, const int32_t* committed, int32_t* rows, int rows_max,
                        int extra_max, int row_base, int rows_cap, int dead_slot, int32_t* ctx_tail, int order,
                        const int32_t* page_table, void* stream);
/* card_target_rows with the queried path taken from an explicit view (the
 * q_hit / q_len fields of a card_cache_state and the path tokens), e.g. the
 * copy a card_mailbox delivered into the target GPU's memory. */
int card_target_rows_view(card_engine_state* E, const card_cache_state* view, const int32_t* q_tok,
                          const int32_t* committed, int32_t* rows, int rows_max, int extra_max, int32_t* ctx_tail,
                          int order, const int32_t* page_table, void* stream);
int card_eos_fix(const int32_t* n_rows, int m_max, const int32_t* ctx_tail, int order, int eos, int V,
                 double* probs, void* stream);
int card_record_width(card_engine_state* E, card_cache* h, const int32_t* n_out, void* stream);
/* accept-and-correct over L = state.L candidate tokens cand[0..L): greedy
 * from per-row argmax, or greedy / lossless stochastic from fp64 rows
 * [L+1, V] with draft conditionals qcond (NULL = the point mass q = 1 of
 * engine.py:242) and host-drawn uniforms consumed from state.cursor.
 * Writes accepted tokens, n, correction into the state. */
int card_verify_argmax(card_engine_state* E, const int32_t* cand, const int32_t* amax, void* stream);
int card_verify_probs(card_engine_state* E, const int32_t* cand, const double* probs, int V,
                      const double* qcond, const double* uniforms, void* stream);
int card_commit(card_engine_state* E, int32_t* committed, void* stream);
/* Outcome of the last verify + commit (replaces the return of
 * verify.py:65-132 and the rollback the reference leaves implicit in
 * engine.py:247-262): out = device int32[6] {accepted prefix
 * n, correction token, uniforms consumed (the host advances its PCG64 by
 * this), kv_keep (target KV rows [0, kv_keep) stay valid = C_prev + n for an
 * unclipped commit), KV rows rolled back (L - n unclipped), tokens
 * committed}. */
int card_verify_result(const card_engine_state* E, int32_t* out, void* stream);
/* KV rollback / roll-forward of the draft: promote accepted-chain tree KV
 * rows into the prefix; move surviving tree rows after an arena compaction. */
int card_draft_promote(card_engine_state* E, card_cache* h, void** k_layers, void** v_layers,
                       int n_layers, int row_elems, int esize, int tree_base, int max_chain,
                       const int32_t* page_table, void* stream);
int card_kv_compact(card_engine_state* E, card_cache* h, void** k_layers, void** v_layers, int n_layers,
                    int row_elems, int esize, int tree_base, void** scratch_kv, int capacity, void* stream);
int card_cycle_end(card_engine_state* E, card_cache* h, void* stream);
/* mode="concurrent": copy the target state's commit outcome (C, accepted
 * tokens, correction, done) into the draft-side state before the correction
 * is applied on the draft stream (engine.py:320-389 lock + epoch protocol). */
int card_engine_handoff(const card_engine_state* target_state, card_engine_state* draft_state, void* stream);
/* Two-GPU draft||target placement: enable P2P access both ways between the
 * draft and the target device (the kernels of each side read the other's
 * query result / commit outcome / committed tokens over NVLink).  Returns
 * CARD_E_CONFIG when the devices cannot access each other. */
int card_enable_peer_access(int dev_a, int dev_b);

#ifdef __cplusplus
}
#endif
#endif /* CARD_B200_H */
