// kernels.h -- host launchers of the device stages (internal to libpbs_b200.so).
// Every launcher is stream-ordered, allocation-free and returns a PBS_* status.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace pbs_b200 {

// ---- stage 1 (importance.cu) ------------------------------------------------
// Workspace for the exact importance estimate: E [Hq, N, take] f32 (logits,
// then exps, key-major), rowmax [Hq, take] u32, w [Hq, take] f32.
size_t importance_workspace_bytes(int hq, int64_t n, int64_t block);
// q_rows: rows per head in q (0 = n; `take` = only the last take rows were passed)
int launch_importance(const void* q, const void* k, int dtype, int hq, int hkv, int64_t n, int d,
                      int64_t block, float scale, float* scores, void* ws, size_t ws_bytes,
                      cudaStream_t st, int64_t q_rows = 0);
// the same in two parts: logits (+ row maxima) of heads [h0, h0 + nh) (q / k still
// point at head 0 / KV head 0), then the exps, denominators and scores of all heads
int launch_importance_logits(const void* q, const void* k, int dtype, int hq, int hkv, int h0, int nh, int64_t n,
                             int d, int64_t block, float scale, void* ws, size_t ws_bytes, cudaStream_t st,
                             int64_t q_rows = 0);
// exps, denominators and scores of heads [h0, h0 + nh) of an hq-head workspace
int launch_importance_finish(int hq, int h0, int nh, int64_t n, int64_t block, float* scores, void* ws,
                             size_t ws_bytes, cudaStream_t st);
// per segment stable sort; primary_keys: 0 = descending f32 scores, 1 = ascending u32 groups
int launch_segmented_sort(const void* keys, int key_kind, int heads, int64_t n, int64_t segment,
                          int32_t* perm, int32_t* inv, cudaStream_t st);
size_t query_perm_workspace_bytes(int hq, int64_t n, int d, int64_t block);
int launch_query_groups(const void* q, const void* k, int dtype, int hq, int k_heads, int64_t n,
                        int d, int64_t block, uint32_t* groups, void* ws, size_t ws_bytes,
                        cudaStream_t st);
int launch_identity(int32_t* perm, int heads, int64_t n, cudaStream_t st);
// TMA map (a CUtensorMap, 64 bytes) over fp32 [d2][d1][d0] with a [1][box1][box0] box (attn_sm100.cu)
int make_f32_map_3d(void* map, const float* base, int64_t d0, int64_t d1, int64_t d2, int box0, int box1);
// bf16 [d2][d1][d0] with rows of `row_elems` (>= d0, 16-byte multiple) and a
// [1, box1, box0] SW128 box: the tcgen05 K-major operand tiles
int make_bf16_sw128_map_3d(void* map, const void* base, int64_t d0, int64_t d1, int64_t d2, int64_t row_elems,
                           int box0, int box1);

// ---- stage 2 (gather.cu) ------------------------------------------------------
// the un-permute: dst[h][perm[h][i]] = src[h][i] (pipeline.hpp:178-180)
int launch_scatter_rows(const int32_t* perm, const void* src, int heads, int64_t rows, int cols, int esize,
                        void* dst, cudaStream_t st);
int launch_apply_rows(const int32_t* perm, const void* src, int src_heads, int dst_heads,
                      int64_t rows, int cols, int esize, void* dst, cudaStream_t st);

// ---- stage 3 (select.cu) ------------------------------------------------------
size_t select_workspace_bytes(int hq, int64_t n, int d, int64_t block);
// pooled block means of Q' (per q head) and K' (gathered through pi from raw
// K or read directly from a per-q-head K'); k_perm == nullptr means identity.
int launch_pool(const void* x, int dtype, int src_heads, int dst_heads, const int32_t* perm,
                int64_t n, int d, int64_t block, float* pooled, cudaStream_t st);
// block logits GEMM into logits_ws [hq, t, t] + softmax (+ optional dense
// score output) + (select != 0) selection and CSR
int launch_score_select(const float* qbar, const float* kbar, float* logits_ws, int hq, int64_t t, int d,
                        int64_t block, int64_t segment, float scale, double tau, int forced_first, int forced_band,
                        int select, float* scores_out, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt,
                        double* row_cov, cudaStream_t st, int top_k = 0);
// mask -> per-row ascending key-block lists (the attention's CSR)
int launch_mask_to_lists(const uint8_t* mask, int hq, int64_t t, int32_t* kv_idx, int32_t* kv_cnt, cudaStream_t st);
// coverage[h] = mean over rows of exp(lse_sparse - lse_dense) (attention_coverage)
int launch_coverage_reduce(const float* lse_sparse, const float* lse_dense, int hq, int64_t n, double* coverage,
                           cudaStream_t st);
// selection from precomputed scores (pbs_select_blocks)
int launch_select_from_scores(const float* scores, int hq, int64_t t, int64_t block,
                              int64_t segment, double tau, int forced_first, int forced_band,
                              uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt, cudaStream_t st, int top_k = 0);

// ---- stage 4 (attn_simt.cu / attn_sm100.cu) -----------------------------------
struct AttnParams {
  const void* q;  // [Hq, N, d] (permuted Q')
  const void* k;  // [kv_heads, N, d]
  const void* v;  // [kv_heads, N, d]
  void* out;      // [Hq, N, d]
  int dtype;
  int hq, kv_heads, d;
  int64_t n, block;
  float scale;
  const int32_t* kv_idx;  // [Hq, T, T] or nullptr (dense causal)
  const int32_t* kv_cnt;  // [Hq, T]
  const int32_t* q_orig;  // sigma [Hq, N] or nullptr
  const int32_t* k_orig;  // pi [Hq, N] or nullptr
  const int32_t* out_rows;  // sigma for the fused un-permute, or nullptr
  int32_t* status;          // device int32[2] or nullptr
  // per-row log-sum-exp of the scaled, admissible scores (natural log; -inf for
  // a row with no admissible key), f32 [Hq, N] in output-row order, or nullptr
  float* lse;
  int causal;               // dense causal comparator mode
  // query blocks [qb_begin, qb_end) only (qb_end == 0: all; qb_begin even on the
  // tensor-core path): a head-parallel shard that cuts inside a head
  int64_t qb_begin;
  int64_t qb_end;
};
int launch_attention_simt(const AttnParams& p, cudaStream_t st);
bool attention_sm100_supported(const AttnParams& p);
int launch_attention_sm100(const AttnParams& p, void* sched_ws, cudaStream_t st);
size_t attention_sm100_workspace_bytes(int hq, int64_t n, int64_t block);

// debug: device expf port
int launch_debug_expf(const float* x, float* y, int64_t n, cudaStream_t st);

}  // namespace pbs_b200
