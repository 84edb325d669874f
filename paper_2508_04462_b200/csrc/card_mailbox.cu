// card_mailbox.cu — the draft <-> target exchange of mode="concurrent" as
// device mailboxes (engine.py:320-389).
//
// The reference's two threads share one TreeCache under a lock and an epoch:
// the target queries the best path, verifies, commits and corrects; the
// draft keeps expanding and drops an expansion whose epoch went stale.  With
// the draft and the target on two GPUs (NVLink peers), each direction is a
// mailbox in the RECEIVER's memory, written by the sender's kernel with P2P
// stores and published by a system-scope release of its sequence number:
//
//   query box  (target GPU)  <- draft GPU after a correction: the queried path
//                               (hit, length, tokens) and the tree epoch
//   commit box (draft GPU)   <- target GPU after each commit: the verify
//                               outcome (accepted tokens, correction, done)
//
// Receivers poll with acquire loads.  The draft polls without blocking at
// the start of every draft step: a new commit is handed to its engine state
// and the step corrects the tree, queries it and publishes the query before
// expanding (so expansions always follow the latest correction on the one
// stream that mutates the tree — nothing can go stale).  The target blocks
// at the start of every verify until a query newer than the last one it
// verified arrives.  No host round trip sits between the two sides.
#include <stdio.h>

#include "card_common.cuh"

extern "C" {
typedef struct card_engine_state card_engine_state;
}

namespace card {
namespace {

constexpr int kMaxPath = 64;

struct QueryBox {
    uint32_t seq;
    int32_t epoch, hit, len;
    int32_t tok[kMaxPath];
};

struct CommitBox {
    uint32_t seq;
    int32_t C, C_prev, base_len, done, out_len, n_acc, corr;
    int32_t acc[kMaxPath];
};

// the fields of card_engine_state the exchange touches (card_engine.cu layout)
struct EngineView {
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
    int32_t kv_keep, kv_drop, consumed, cursor_prev, spare[2];
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// draft GPU: publish the query of the last correction (pending != 0) or a forced one
__global__ void publish_query_kernel(QueryBox* box, const card_cache_state* S, const int32_t* q_tok,
                                     const int32_t* skip, uint32_t* sent) {
    if (threadIdx.x != 0) return;
    if (skip && *skip) return;
    const int len = S->q_hit ? S->q_len : 0;
    for (int i = 0; i < len && i < kMaxPath; ++i) box->tok[i] = q_tok[i];
    box->epoch = S->epoch;
    box->hit = S->q_hit;
    box->len = len;
    const uint32_t s = *sent + 1;
    *sent = s;
    st_release_sys(&box->seq, s);   // payload (P2P stores) before the sequence number
}

// target GPU: wait for a query newer than the last verified one; expose it
// as the cache-state view card_target_rows reads (q_hit, q_len, epoch) + tokens
__global__ void wait_query_kernel(const QueryBox* box, uint32_t* seen, card_cache_state* view, int32_t* q_tok) {
    if (threadIdx.x != 0) return;
    const uint32_t want = *seen + 1;
    uint32_t s;
    while ((s = ld_acquire_sys(&box->seq)) < want) __nanosleep(64);
    *seen = s;
    const int len = box->len;
    for (int i = 0; i < len; ++i) q_tok[i] = box->tok[i];
    view->q_hit = box->hit;
    view->q_len = len;
    view->epoch = box->epoch;
}

// target GPU: publish the commit outcome into the draft GPU's box
__global__ void publish_commit_kernel(CommitBox* box, const EngineView* E, uint32_t* sent) {
    if (threadIdx.x != 0) return;
    box->C = E->C;
    box->C_prev = E->C_prev;
    box->base_len = E->base_len;
    box->done = E->done;
    box->out_len = E->out_len;
    box->n_acc = E->n_acc;
    box->corr = E->corr;
    for (int i = 0; i < E->n_acc && i < kMaxPath; ++i) box->acc[i] = E->acc[i];
    const uint32_t s = *sent + 1;
    *sent = s;
    st_release_sys(&box->seq, s);
}

// draft GPU, every draft step: a new commit -> the draft state (the hand-off
// of card_engine_handoff), skip flag 0 (correct and query run); else skip 1
__global__ void poll_commit_kernel(const CommitBox* box, uint32_t* seen, EngineView* D, int32_t* skip) {
    if (threadIdx.x != 0) return;
    const uint32_t s = ld_acquire_sys(&box->seq);
    if (s <= *seen) {
        *skip = 1;
        return;
    }
    *seen = s;
    D->C = box->C;
    D->C_prev = box->C_prev;
    D->base_len = box->base_len;
    D->done = box->done;
    D->out_len = box->out_len;
    D->n_acc = box->n_acc;
    D->corr = box->corr;
    for (int i = 0; i < box->n_acc && i < 64; ++i) D->acc[i] = box->acc[i];
    D->stop = 0;
    D->n_widths = 0;
    *skip = 0;
}

}  // namespace
}  // namespace card

using namespace card;

struct card_mailbox {
    QueryBox* qbox;      // on the target device
    CommitBox* cbox;     // on the draft device
    uint32_t* q_sent;    // draft device: queries published
    uint32_t* q_seen;    // target device: queries consumed
    uint32_t* c_sent;    // target device: commits published
    uint32_t* c_seen;    // draft device: commits consumed
    int32_t* skip;       // draft device: 1 = no new commit this draft step
    card_cache_state* view;   // target device: the consumed query as card_target_rows reads it
    int32_t* q_tok;           // target device [kMaxPath]
    int dev_d, dev_t;
};

static cudaError_t alloc_on(int dev, void** p, size_t bytes) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) e = cudaMemset(*p, 0, bytes);
    cudaSetDevice(prev);
    return e;
}

extern "C" {

int card_mailbox_create(int draft_dev, int target_dev, card_mailbox** out) {
    if (!out) return CARD_E_INPUT;
    card_mailbox* m = (card_mailbox*)calloc(1, sizeof(card_mailbox));
    m->dev_d = draft_dev;
    m->dev_t = target_dev;
    cudaError_t e = alloc_on(target_dev, (void**)&m->qbox, sizeof(QueryBox));
    if (e == cudaSuccess) e = alloc_on(draft_dev, (void**)&m->cbox, sizeof(CommitBox));
    if (e == cudaSuccess) e = alloc_on(draft_dev, (void**)&m->q_sent, 64);
    if (e == cudaSuccess) e = alloc_on(target_dev, (void**)&m->q_seen, 64);
    if (e == cudaSuccess) e = alloc_on(target_dev, (void**)&m->c_sent, 64);
    if (e == cudaSuccess) e = alloc_on(draft_dev, (void**)&m->c_seen, 64);
    if (e == cudaSuccess) e = alloc_on(draft_dev, (void**)&m->skip, 64);
    if (e == cudaSuccess) e = alloc_on(target_dev, (void**)&m->view, sizeof(card_cache_state));
    if (e == cudaSuccess) e = alloc_on(target_dev, (void**)&m->q_tok, kMaxPath * sizeof(int32_t));
    if (e != cudaSuccess) {
        set_cuda_error(e);
        *out = m;
        card_mailbox_destroy(m);
        *out = nullptr;
        return CARD_E_CUDA;
    }
    *out = m;
    return CARD_OK;
}

int card_mailbox_destroy(card_mailbox* m) {
    if (!m) return CARD_OK;
    void* ps[] = {m->qbox, m->cbox, m->q_sent, m->q_seen, m->c_sent, m->c_seen, m->skip, m->view, m->q_tok};
    for (void* p : ps)
        if (p) cudaFree(p);
    free(m);
    return CARD_OK;
}

// both boxes and sequence counters back to zero (between requests; the
// caller has synchronised both devices)
int card_mailbox_reset(card_mailbox* m) {
    if (!m) return CARD_E_INPUT;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(m->dev_t);
    if (e == cudaSuccess) e = cudaMemset(m->qbox, 0, sizeof(QueryBox));
    if (e == cudaSuccess) e = cudaMemset(m->q_seen, 0, 64);
    if (e == cudaSuccess) e = cudaMemset(m->c_sent, 0, 64);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaSetDevice(m->dev_d);
    if (e == cudaSuccess) e = cudaMemset(m->cbox, 0, sizeof(CommitBox));
    if (e == cudaSuccess) e = cudaMemset(m->q_sent, 0, 64);
    if (e == cudaSuccess) e = cudaMemset(m->c_seen, 0, 64);
    if (e == cudaSuccess) e = cudaMemset(m->skip, 0, 64);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return CARD_E_CUDA;
    }
    return CARD_OK;
}

// (draft side) the per-step skip flag: 1 when no commit arrived since the last step
int card_mailbox_skip_flag(card_mailbox* m, int32_t** skip) {
    if (!m || !skip) return CARD_E_INPUT;
    *skip = m->skip;
    return CARD_OK;
}

// (target side) the consumed query as card_target_rows_view reads it
int card_mailbox_query_view(card_mailbox* m, card_cache_state** view, int32_t** q_tok) {
    if (!m) return CARD_E_INPUT;
    if (view) *view = m->view;
    if (q_tok) *q_tok = m->q_tok;
    return CARD_OK;
}

int card_mailbox_poll_commit(card_mailbox* m, card_engine_state* draft_state, void* stream) {
    if (!m || !draft_state) return CARD_E_INPUT;
    poll_commit_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(m->cbox, m->c_seen, (EngineView*)draft_state, m->skip);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_mailbox_publish_query(card_mailbox* m, card_cache* h, int force, void* stream) {
    if (!m || !h) return CARD_E_INPUT;
    card_cache_state* S;
    int rc = card_cache_device_ptrs(h, &S, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (rc) return rc;
    int32_t *qp, *qt;
    double* qe;
    card_cache_query_buffers(h, &qp, &qt, &qe);
    publish_query_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(m->qbox, S, qt, force ? nullptr : m->skip, m->q_sent);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_mailbox_wait_query(card_mailbox* m, void* stream) {
    if (!m) return CARD_E_INPUT;
    wait_query_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(m->qbox, m->q_seen, m->view, m->q_tok);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

int card_mailbox_publish_commit(card_mailbox* m, const card_engine_state* target_state, void* stream) {
    if (!m || !target_state) return CARD_E_INPUT;
    publish_commit_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(m->cbox, (const EngineView*)target_state, m->c_sent);
    CARD_LAUNCH_CHECK();
    return CARD_OK;
}

}  // extern "C"
