// pbs_b200.hpp -- header-only C++ face of libpbs_b200.so for C++ callers of the
// reference's operator API (namespace pbs in /root/reference/proj/include/pbs/).
//
// The reference is header-only C++20 over host Matrix<T> values; this header
// keeps its names and argument meaning but works on device buffers (plus one
// host-buffer entry, pbs_attention_host, for drop-in use with host matrices),
// and maps the C ABI status codes back onto exceptions carrying the
// reference's exit codes (errors.hpp:11-89).  Only <pbs_cabi.h> is required;
// link with -lpbs_b200.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "pbs_cabi.h"

namespace pbs_b200 {

/// pbs::Error (errors.hpp:18-30): what() is the "E_*: message" line,
/// exit_code() the reference CLI exit code (2 config, 3 io, 4 resource,
/// 5 degenerate; 1 = CUDA).
class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  int exit_code() const { return code_; }

 private:
  int code_;
};

inline void check(int rc) {
  if (rc != PBS_OK) throw Error(rc, pbs_last_error());
}

enum class PermutationStrategy : int32_t {  // pipeline.hpp:19
  none = PBS_STRATEGY_NONE,
  key_permute = PBS_STRATEGY_KEY_PERMUTE,
  query_permute = PBS_STRATEGY_QUERY_PERMUTE,
  both = PBS_STRATEGY_BOTH
};

/// PipelineConfig (pipeline.hpp:30-49) with the reference defaults.
struct PipelineConfig {
  std::size_t block_size = 128;
  std::size_t segment_size = 256;
  double tau = 0.9;
  PermutationStrategy strategy = PermutationStrategy::key_permute;
  bool forced_first_block = true;
  bool forced_diagonal_band = true;
  double scale = 0.0;
  int top_k = 0;  // extension: > 0 keeps the top_k blocks per row instead of the tau prefix

  pbs_pipeline_config c() const {
    pbs_pipeline_config r{};
    r.block_size = (int64_t)block_size;
    r.segment_size = (int64_t)segment_size;
    r.tau = tau;
    r.strategy = (int32_t)strategy;
    r.forced_first_block = forced_first_block ? 1 : 0;
    r.forced_diagonal_band = forced_diagonal_band ? 1 : 0;
    r.scale = scale;
    r.top_k = top_k;
    return r;
  }
};

/// [Hq, N, d] query / [Hkv, N, d] key-value problem shape.
inline pbs_shape make_shape(int dtype, int q_heads, int kv_heads, std::size_t n, int d) {
  pbs_shape s{};
  s.dtype = dtype;
  s.num_q_heads = q_heads;
  s.num_kv_heads = kv_heads;
  s.head_dim = d;
  s.seq_len = (int64_t)n;
  return s;
}

/// PipelineReport (pipeline.hpp:63-74) + StageTimings (51-61).
using PipelineReport = pbs_report;

// ---- operators on device buffers (stream-ordered) ----------------------------

/// estimate_key_importance (permutation.hpp:143-178); scores f32 [Hq, N].
inline void estimate_key_importance(const void* q, const void* k, const pbs_shape& s, std::size_t block,
                                    double scale, float* scores, void* ws, std::size_t ws_bytes,
                                    void* stream = nullptr) {
  check(pbs_estimate_key_importance(q, k, &s, (int64_t)block, scale, scores, ws, ws_bytes, stream));
}

/// build_key_permutation + flatten + inverse (permutation.hpp:182-201, 118-126, 51-55).
inline void build_key_permutation(const float* scores, int heads, std::size_t n, std::size_t segment,
                                  int32_t* perm, int32_t* inv = nullptr, void* stream = nullptr) {
  check(pbs_build_key_permutation(scores, heads, (int64_t)n, (int64_t)segment, perm, inv, stream));
}

/// apply_rows (permutation.hpp:79-89) with the GQA broadcast.
inline void apply_rows(const int32_t* perm, const void* src, int src_heads, int dst_heads, std::size_t rows,
                       int cols, int dtype, void* dst, void* stream = nullptr) {
  check(pbs_apply_rows(perm, src, src_heads, dst_heads, (int64_t)rows, cols, dtype, dst, stream));
}

/// Workspace bytes build_query_permutation needs.
inline std::size_t query_permutation_workspace_size(const pbs_shape& s, std::size_t block) {
  return pbs_query_permutation_workspace_size(&s, (int64_t)block);
}

/// build_query_permutation (permutation.hpp:206-275); k may be K' (strategy both).
inline void build_query_permutation(const void* q, const void* k, int k_heads, const pbs_shape& s,
                                    std::size_t block, std::size_t segment, int32_t* perm, int32_t* inv, void* ws,
                                    std::size_t ws_bytes, void* stream = nullptr) {
  check(pbs_build_query_permutation(q, k, k_heads, &s, (int64_t)block, (int64_t)segment, perm, inv, ws, ws_bytes,
                                    stream));
}

/// meanpool_block_scores (block_selection.hpp:120-161) under the segment-band mask.
inline void meanpool_block_scores(const void* qp, const void* kp, const pbs_shape& s, std::size_t block,
                                  std::size_t segment, double scale, float* scores, void* ws, std::size_t ws_bytes,
                                  void* stream = nullptr) {
  check(pbs_meanpool_block_scores(qp, kp, &s, (int64_t)block, (int64_t)segment, scale, scores, ws, ws_bytes,
                                  stream));
}

/// select_blocks (block_selection.hpp:171-206); top_k > 0 selects by rank instead (extension).
inline void select_blocks(const float* scores, int heads, std::size_t t, std::size_t block, std::size_t segment,
                          double tau, uint8_t* mask, int32_t* kv_idx = nullptr, int32_t* kv_cnt = nullptr,
                          bool forced_first = true, bool forced_band = true, int top_k = 0,
                          void* stream = nullptr) {
  if (top_k > 0)
    check(pbs_select_blocks_top_k(scores, heads, (int64_t)t, (int64_t)block, (int64_t)segment, top_k,
                                  forced_first ? 1 : 0, forced_band ? 1 : 0, mask, kv_idx, kv_cnt, stream));
  else
    check(pbs_select_blocks(scores, heads, (int64_t)t, (int64_t)block, (int64_t)segment, tau, forced_first ? 1 : 0,
                            forced_band ? 1 : 0, mask, kv_idx, kv_cnt, stream));
}

/// attention_block_sparse (attention.hpp:259-310) over the selected blocks, with the
/// original-position element mask (q_orig = sigma, k_orig = pi) and the fused un-permute.
inline void attention_block_sparse(const void* qp, const void* kp, const void* vp, int kv_heads,
                                   const pbs_shape& s, std::size_t block, const int32_t* kv_idx,
                                   const int32_t* kv_cnt, void* out, const int32_t* q_orig = nullptr,
                                   const int32_t* k_orig = nullptr, const int32_t* out_rows = nullptr,
                                   int32_t* status = nullptr, double scale = 0.0, void* stream = nullptr) {
  check(pbs_block_sparse_attention_fwd(qp, kp, vp, kv_heads, &s, (int64_t)block, scale, kv_idx, kv_cnt, q_orig,
                                       k_orig, out_rows, out, status, stream));
}

/// The dense causal comparator (attention_tiled, causal, attention.hpp:314-321).
inline void dense_causal_attention(const void* q, const void* k, const void* v, const pbs_shape& s, void* out,
                                   double scale = 0.0, void* stream = nullptr) {
  check(pbs_dense_causal_attention_fwd(q, k, v, &s, scale, out, stream));
}

/// PBST files (tensor_io.hpp) to and from device memory.
inline pbs_tensor_info tensor_info(const char* path) {
  pbs_tensor_info i{};
  check(pbs_tensor_info_read(path, &i));
  return i;
}
inline void load_tensor(const char* path, void* dst, int dst_dtype, void* stream = nullptr) {
  check(pbs_tensor_load(path, dst, dst_dtype, stream));
}
inline void save_tensor(const char* path, const void* src, int src_dtype, std::size_t heads, std::size_t rows,
                        std::size_t cols, bool f64_file = false, bool as_stack = true, void* stream = nullptr) {
  check(pbs_tensor_save(path, src, src_dtype, (int64_t)heads, (int64_t)rows, (int64_t)cols, f64_file ? 1 : 0,
                        as_stack ? 1 : 0, stream));
}

/// The stage-5 un-permute (pipeline.hpp:178-180): dst[h][sigma[h][i]] = src[h][i].
inline void unpermute(const int32_t* sigma, const void* src, int heads, std::size_t rows, int cols, int dtype,
                      void* dst, void* stream = nullptr) {
  check(pbs_unpermute(sigma, src, heads, (int64_t)rows, cols, dtype, dst, stream));
}

/// The full Algorithm 1 (pbs_attention, pipeline.hpp:107-193) on device buffers.
inline std::size_t workspace_size(const pbs_shape& s, const PipelineConfig& cfg) {
  const pbs_pipeline_config c = cfg.c();
  const std::size_t n = pbs_workspace_size(&s, &c);
  if (n == 0) throw Error(PBS_ERR_CONFIG, pbs_last_error());
  return n;
}

inline PipelineReport pbs_attention(const void* q, const void* k, const void* v, const pbs_shape& s,
                                    const PipelineConfig& cfg, void* out, void* ws, std::size_t ws_bytes,
                                    int32_t* sigma = nullptr, int32_t* pi = nullptr, uint8_t* mask = nullptr,
                                    void* stream = nullptr) {
  const pbs_pipeline_config c = cfg.c();
  PipelineReport rep{};
  check(::pbs_attention(q, k, v, &s, &c, out, sigma, pi, mask, ws, ws_bytes, &rep, stream));
  return rep;
}

/// Drop-in for pbs::pbs_attention on host matrices of one head: q, k, v are
/// row-major [N, d] float (Matrix<float>::data()), out likewise.
inline PipelineReport pbs_attention_host(const float* q, const float* k, const float* v, std::size_t n, int d,
                                         const PipelineConfig& cfg, float* out, int32_t* sigma = nullptr,
                                         int32_t* pi = nullptr, uint8_t* mask = nullptr) {
  const pbs_shape s = make_shape(PBS_DTYPE_F32, 1, 1, n, d);
  const pbs_pipeline_config c = cfg.c();
  PipelineReport rep{};
  check(::pbs_attention_host(q, k, v, &s, &c, out, sigma, pi, mask, &rep));
  return rep;
}

/// attention_coverage (pipeline.hpp:198-243) on device buffers: per-head
/// coverage into the device array `coverage` (double [Hq]).
inline std::size_t coverage_workspace_size(const pbs_shape& s, std::size_t block) {
  const std::size_t n = pbs_coverage_workspace_size(&s, (int64_t)block);
  if (n == 0) throw Error(PBS_ERR_CONFIG, pbs_last_error());
  return n;
}
inline void attention_coverage(const void* q, const void* k, const pbs_shape& s, std::size_t block,
                               const uint8_t* mask, const int32_t* sigma, const int32_t* pi, double* coverage,
                               void* ws, std::size_t ws_bytes, double scale = 0.0, void* stream = nullptr) {
  check(pbs_attention_coverage(q, k, &s, (int64_t)block, mask, sigma, pi, scale, coverage, ws, ws_bytes, stream));
}

}  // namespace pbs_b200
