// card_llm.h — internal declarations shared by the model / engine kernels.
#pragma once
#include <stdint.h>

#include "../../include/card_b200.h"

#include <cuda_runtime.h>

namespace card {
// fused attention (card_attn.cu): prefix chunks + tree extras + cluster combine
int launch_attn_fused(const float* q, const int32_t* dM, int m_max, const int32_t* plen, const int32_t* slot,
                      const int32_t* page_table,
                      const int32_t* n_extra,
                      const int32_t* extra, int extra_max, const void* kc, const void* vc, int nh, int nkv, int hd,
                      int max_plen, void* o, cudaStream_t s);
int attn_set_trace(unsigned long long* buf);
bool attn_fused_fits(int m_max, int nh, int nkv, int extra_max);
// tcgen05 attention over a paged KV cache (card_attn_tc.cu)
bool attn_tc_fits(int m_max, int nh, int nkv, int hd, int extra_max);
int attn_tc_set_trace(unsigned long long* buf);
int launch_attn_tc(const float* q, const int32_t* dM, int m_max, const int32_t* plen, const int32_t* n_extra,
                   const int32_t* extra, int extra_max, const void* kc, const void* vc, const int32_t* page_table,
                   int nh, int nkv, int hd, int max_plen, void* o, cudaStream_t s, const void* qsw = nullptr,
                   int qsw_tiles = 0, int seg_rows = 0, int pt_stride = 0);
int attn_tc_max_segments();
}  // namespace card

// GEMM epilogues (card_gemm.cu)
enum {
    EPI_STORE_F32 = 0,
    EPI_RESID_F32 = 1,
    EPI_STORE_BF16 = 2,
    EPI_SWIGLU_BF16 = 3,
    EPI_QKV_ROPE = 4,   // RoPE + q scale + KV-cache write (card_linear_fuse_rope)
    EPI_TOPK = 5,       // lm_head: per (row, 128-token vocab tile) top-4 + max / sum-exp records
};
constexpr int kTopkKT = 4;                  // candidates per (row, vocab tile) record
constexpr int kTopkRec = 2 + 2 * kTopkKT;   // [max, sum, (value, token) x KT] floats

// Per-forward row descriptors written by the row builders (card_engine.cu)
// and consumed by the model kernels (card_llm.cu).  Device memory.
//   tok[r]     input token of row r
//   pos[r]     RoPE position
//   slot[r]    KV slot the row's K/V are written to
//   plen[r]    number of prefix KV slots [0, plen) the row attends to
//   n_extra[r] number of extra slots (tree ancestors + self) in extra[r][..]
//   out_rows   rows whose hidden state reaches the lm_head, in output order
struct CardRows {
    int32_t* M;         // [1] number of rows this forward
    int32_t* n_out;     // [1] number of output rows
    int32_t* tok;
    int32_t* pos;
    int32_t* slot;
    int32_t* plen;
    int32_t* n_extra;
    int32_t* extra;     // [rows_max * extra_max]
    int32_t* out_rows;  // [rows_max]
    int rows_max;
    int extra_max;
};
