// pbs_dropin.hpp -- the reference's C++ operator API, on the B200 library.
//
// A header-swap drop-in for callers of the reference headers
// (proj/include/pbs/, namespace pbs): the same types (pbs::Matrix<T>,
// pbs::PipelineConfig, pbs::PipelineResult<T>, pbs::BlockMask,
// pbs::Permutation, pbs::SegmentedPermutation, pbs::ImportanceScores<T>,
// pbs::BlockScoreMatrix<T>, pbs::ElementMask), the same function names and
// argument meaning, the same exceptions (pbs::ConfigError, ShapeError,
// ResourceError, DegenerateRowError, errors.hpp), computed by libpbs_b200.so
// through the C ABI (pbs_cabi.h).  The functions live in namespace pbs::b200;
// a caller switches with one using-declaration per name, e.g. the reference
// CLI's per-head run (tools/pbs_main.cpp:212):
//
//     #include "pbs/pipeline.hpp"      // the reference's types (unchanged)
//     #include "pbs_dropin.hpp"        // this header
//     using pbs::b200::pbs_attention;  // instead of pbs::pbs_attention
//
// Build: -I <reference>/proj/include -I <this repo>/include, link -lpbs_b200.
//
// Precision: the device computes in f32 with the reference's f32 arithmetic
// (permutations and masks bit-exact; outputs within 1e-4 of the reference's
// f32 outputs).  The reference's f64 instantiation (its default Precision,
// pipeline.hpp:35) has no device counterpart: every entry here refuses
// T = double with pbs::ConfigError ("precision f64 is not supported ...").
// Shapes: self-attention only (N == M, like pbs_attention) and V's head dim
// equal to Q's (the C ABI carries one d).
#pragma once

#include <algorithm>
#include <concepts>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "pbs/attention.hpp"
#include "pbs/block_selection.hpp"
#include "pbs/errors.hpp"
#include "pbs/matrix.hpp"
#include "pbs/permutation.hpp"
#include "pbs/pipeline.hpp"
#include "pbs_cabi.h"

namespace pbs::b200 {
namespace detail {

// C-ABI status -> the reference's exception types (errors.hpp:32-89), with the
// library's message (the "E_*: " prefix stripped: pbs::Error adds its own)
[[noreturn]] inline void rethrow(int rc) {
  std::string msg = pbs_last_error();
  const auto colon = msg.find(": ");
  const std::string prefix = colon == std::string::npos ? "" : msg.substr(0, colon);
  const std::string body = colon == std::string::npos ? msg : msg.substr(colon + 2);
  switch (rc) {
    case PBS_ERR_CONFIG:
      if (prefix == "E_SHAPE") throw ShapeError(body);
      throw ConfigError(body);
    case PBS_ERR_IO:
      throw IoError(body);
    case PBS_ERR_RESOURCE:
      throw Error(ErrorCode::resource, "E_RESOURCE", body);
    case PBS_ERR_DEGENERATE: {
      std::size_t qb = 0;
      const auto at = body.find("query block ");
      if (at != std::string::npos) qb = std::stoul(body.substr(at + 12));
      throw DegenerateRowError(qb);
    }
    default:
      throw std::runtime_error(msg);  // E_CUDA: not a pbs::Error (no device, launch failure)
  }
}
inline void check(int rc) {
  if (rc != PBS_OK) rethrow(rc);
}

template <typename T>
void require_f32() {
  if constexpr (!std::is_same_v<T, float>)
    throw ConfigError("precision f64 is not supported by the B200 device path (use f32)");
}

inline pbs_pipeline_config to_c(const PipelineConfig& c) {
  pbs_pipeline_config r{};
  r.block_size = (int64_t)c.block_size;
  r.segment_size = (int64_t)c.segment_size;
  r.tau = c.tau;
  r.strategy = (int32_t)c.strategy;
  r.forced_first_block = c.forced.first_block ? 1 : 0;
  r.forced_diagonal_band = c.forced.diagonal_band ? 1 : 0;
  r.top_k = 0;
  r.scale = c.scale;
  return r;
}

inline pbs_shape shape_f32(std::size_t n, std::size_t d) {
  pbs_shape s{};
  s.dtype = PBS_DTYPE_F32;
  s.num_q_heads = 1;
  s.num_kv_heads = 1;
  s.head_dim = (int32_t)d;
  s.seq_len = (int64_t)n;
  return s;
}

// device buffer through the C ABI (no CUDA runtime needed by the caller)
class Dev {
 public:
  Dev() = default;
  explicit Dev(std::size_t bytes) { check(pbs_malloc(bytes, &p_)); }
  Dev(const void* host, std::size_t bytes) : Dev(bytes) { put(host, bytes); }
  ~Dev() { pbs_free(p_); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  void put(const void* host, std::size_t bytes) { check(pbs_memcpy(p_, host, bytes, PBS_COPY_H2D, nullptr)); }
  void get(void* host, std::size_t bytes) const {
    check(pbs_memcpy(host, p_, bytes, PBS_COPY_D2H, nullptr));
    check(pbs_stream_synchronize(nullptr));
  }
  template <typename U = void>
  U* as() const {
    return static_cast<U*>(p_);
  }

 private:
  void* p_ = nullptr;
};

inline std::vector<int32_t> to_i32(const std::vector<std::size_t>& v) {
  return std::vector<int32_t>(v.begin(), v.end());
}
inline std::vector<std::size_t> to_size(const std::vector<int32_t>& v) {
  return std::vector<std::size_t>(v.begin(), v.end());
}
inline std::vector<int32_t> map_of(const Permutation& p) { return to_i32(p.map()); }

// per-row ascending block lists (kv_idx / kv_cnt) of a BlockMask, for the kernel
inline void csr_of(const BlockMask& m, std::vector<int32_t>& idx, std::vector<int32_t>& cnt) {
  const std::size_t t = m.rows();
  idx.assign(t * m.cols(), 0);
  cnt.assign(t, 0);
  for (std::size_t i = 0; i < t; ++i)
    for (std::size_t j = 0; j < m.cols(); ++j)
      if (m.at(i, j)) idx[i * m.cols() + (std::size_t)cnt[i]++] = (int32_t)j;
}

}  // namespace detail

/// pbs::pbs_attention (pipeline.hpp:107-193) on the device: one head, host
/// Matrix<float> in and out, the same PipelineResult.
template <std::floating_point T>
PipelineResult<T> pbs_attention(const Matrix<T>& q, const Matrix<T>& k, const Matrix<T>& v,
                                const PipelineConfig& cfg) {
  cfg.validate();
  if (q.rows() != k.rows())
    throw ConfigError("pipeline expects self-attention: N == M, got " + std::to_string(q.rows()) + " vs " +
                      std::to_string(k.rows()));
  if (q.cols() != k.cols() || k.rows() != v.rows()) throw ShapeError("pipeline inputs have inconsistent shapes");
  if (q.rows() == 0) throw ShapeError("pipeline inputs are empty");
  detail::require_f32<T>();
  if (v.cols() != q.cols()) throw ShapeError("pbs_b200: V head dim must equal Q/K head dim");
  const std::size_t n = q.rows(), d = q.cols(), b = cfg.block_size, s = cfg.segment_size;
  const std::size_t t = (n + b - 1) / b;
  const pbs_shape sh = detail::shape_f32(n, d);
  const pbs_pipeline_config c = detail::to_c(cfg);
  Matrix<T> out(n, d);
  std::vector<int32_t> sigma(n), pi(n);
  std::vector<uint8_t> mask(t * t);
  pbs_report rep{};
  detail::check(pbs_attention_host(q.data(), k.data(), v.data(), &sh, &c, out.data(), sigma.data(), pi.data(),
                                   mask.data(), &rep));
  PipelineResult<T> r{std::move(out), PipelineReport{}, Permutation(detail::to_size(sigma)),
                      Permutation(detail::to_size(pi)), BlockMask(t, t, b, s)};
  for (std::size_t i = 0; i < t; ++i)
    for (std::size_t j = 0; j < t; ++j) r.mask.set(i, j, mask[i * t + j] != 0);
  r.report.block_density = rep.block_density;
  r.report.causal_density_baseline = rep.causal_density_baseline;
  r.report.pooled_score_coverage = rep.pooled_score_coverage;
  r.report.selected_blocks = (std::size_t)rep.selected_blocks;
  r.report.total_admissible_blocks = (std::size_t)rep.total_admissible_blocks;
  r.report.timings.estimate_us = rep.estimate_us;
  r.report.timings.permute_us = rep.permute_us;
  r.report.timings.select_us = rep.select_us;
  r.report.timings.attention_us = rep.attention_us;
  r.report.timings.unpermute_us = rep.unpermute_us;
  return r;
}

/// pbs::attention_coverage (pipeline.hpp:198-243): no N^2 cap on the device.
template <std::floating_point T>
double attention_coverage(const Matrix<T>& q, const Matrix<T>& k, const BlockMask& mask, const Permutation& sigma,
                          const Permutation& pi, double scale = 0.0) {
  if (q.rows() != k.rows() || q.cols() != k.cols())
    throw ShapeError("attention_coverage expects square self-attention inputs");
  if (sigma.size() != q.rows() || pi.size() != k.rows())
    throw ShapeError("attention_coverage: permutation lengths do not match inputs");
  const std::size_t n = q.rows(), d = q.cols(), b = mask.block_size();
  if (mask.rows() != (n + b - 1) / b || mask.cols() != (n + b - 1) / b)
    throw ShapeError("attention_coverage: mask grid does not match inputs");
  detail::require_f32<T>();
  const std::size_t t = mask.rows();
  std::vector<uint8_t> m(t * t);
  for (std::size_t i = 0; i < t; ++i)
    for (std::size_t j = 0; j < t; ++j) m[i * t + j] = mask.at(i, j) ? 1 : 0;
  const auto sg = detail::map_of(sigma), pp = detail::map_of(pi);
  const pbs_shape sh = detail::shape_f32(n, d);
  detail::Dev dq(q.data(), n * d * 4), dk(k.data(), n * d * 4), dm(m.data(), m.size()), ds(sg.data(), n * 4),
      dp(pp.data(), n * 4), dc(sizeof(double));
  const std::size_t wsb = pbs_coverage_workspace_size(&sh, (int64_t)b);
  detail::Dev ws(wsb);
  detail::check(pbs_attention_coverage(dq.as(), dk.as(), &sh, (int64_t)b, dm.as<uint8_t>(), ds.as<int32_t>(),
                                       dp.as<int32_t>(), scale, dc.as<double>(), ws.as(), wsb, nullptr));
  double cov = 0.0;
  dc.get(&cov, sizeof cov);
  return cov;
}

/// pbs::estimate_key_importance (permutation.hpp:143-178), bit-exact.
template <std::floating_point T>
ImportanceScores<T> estimate_key_importance(const Matrix<T>& q, const Matrix<T>& k, const AttentionConfig& cfg) {
  if (k.rows() == 0) throw ShapeError("estimate_key_importance: empty key matrix");
  if (q.rows() == 0) throw ShapeError("estimate_key_importance: empty query matrix");
  if (q.cols() != k.cols()) throw ShapeError("estimate_key_importance: head dims differ");
  detail::require_f32<T>();
  if (q.rows() != k.rows()) throw ShapeError("pbs_b200: estimate_key_importance takes N == M");
  const std::size_t n = q.rows(), d = q.cols();
  const pbs_shape sh = detail::shape_f32(n, d);
  const std::size_t take = std::min(cfg.block_size, n);
  const std::size_t wsb = n * take * 4 + take * 8 + 4096;
  detail::Dev dq(q.data(), n * d * 4), dk(k.data(), n * d * 4), ds(n * 4), ws(wsb);
  detail::check(pbs_estimate_key_importance(dq.as(), dk.as(), &sh, (int64_t)cfg.block_size, cfg.scale,
                                            ds.as<float>(), ws.as(), wsb, nullptr));
  ImportanceScores<T> out;
  out.scores.resize(n);
  ds.get(out.scores.data(), n * 4);
  out.source_query_block = (n - 1) / cfg.block_size;
  return out;
}

/// pbs::build_key_permutation (permutation.hpp:182-201): stable descending
/// sort per segment (ties by index), same SegmentedPermutation.
template <std::floating_point T>
SegmentedPermutation build_key_permutation(const ImportanceScores<T>& imp, std::size_t segment_size) {
  if (segment_size == 0) throw ConfigError("build_key_permutation: segment size must be >= 1");
  detail::require_f32<T>();
  const std::size_t n = imp.scores.size();
  std::vector<int32_t> perm(n);
  if (n > 0) {
    detail::Dev ds(imp.scores.data(), n * 4), dp(n * 4);
    detail::check(pbs_build_key_permutation(ds.as<float>(), 1, (int64_t)n, (int64_t)segment_size, dp.as<int32_t>(),
                                            nullptr, nullptr));
    dp.get(perm.data(), n * 4);
  }
  std::vector<Permutation> locals;
  for (std::size_t g = 0; g < n / segment_size; ++g) {
    std::vector<std::size_t> m(segment_size);
    for (std::size_t i = 0; i < segment_size; ++i) m[i] = (std::size_t)perm[g * segment_size + i] - g * segment_size;
    locals.emplace_back(std::move(m));
  }
  return SegmentedPermutation(segment_size, n, std::move(locals));
}

/// pbs::meanpool_block_scores (block_selection.hpp:120-161), bit-exact.  The
/// device builds the segment-band causal mask itself; `causal` must be that
/// mask (build_block_causal_mask), as in the pipeline.
template <std::floating_point T>
BlockScoreMatrix<T> meanpool_block_scores(const Matrix<T>& qp, const Matrix<T>& kp, std::size_t block_size,
                                          std::size_t segment_size, const Matrix<T>& causal, double scale = 0.0) {
  detail::require_f32<T>();
  if (qp.rows() != kp.rows() || qp.cols() != kp.cols())
    throw ShapeError("pbs_b200: meanpool_block_scores takes square self-attention inputs");
  const std::size_t n = qp.rows(), d = qp.cols(), t = (n + block_size - 1) / block_size;
  if (causal.rows() != t || causal.cols() != t) throw ShapeError("meanpool_block_scores: causal grid mismatch");
  if (!(causal == build_block_causal_mask<T>(t, t, block_size, segment_size)))
    throw ConfigError("pbs_b200: meanpool_block_scores takes the segment-band causal mask");
  const pbs_shape sh = detail::shape_f32(n, d);
  const std::size_t wsb = 2 * (t * d * 4 + 256) + t * t * 4 + 8192;
  detail::Dev dq(qp.data(), n * d * 4), dk(kp.data(), n * d * 4), ds(t * t * 4), ws(wsb);
  detail::check(pbs_meanpool_block_scores(dq.as(), dk.as(), &sh, (int64_t)block_size, (int64_t)segment_size, scale,
                                          ds.as<float>(), ws.as(), wsb, nullptr));
  BlockScoreMatrix<T> out;
  out.scores = Matrix<T>(t, t);
  ds.get(out.scores.data(), t * t * 4);
  out.causal = causal;
  out.block_size = block_size;
  out.segment_size = segment_size;
  return out;
}

/// pbs::select_blocks (block_selection.hpp:171-206), bit-exact.
template <std::floating_point T>
BlockMask select_blocks(const BlockScoreMatrix<T>& bsm, double tau, ForcedPolicy forced = {}) {
  detail::require_f32<T>();
  if (!(tau >= 0.0 && tau <= 1.0)) throw ConfigError("tau must lie in [0, 1]");
  const std::size_t t = bsm.scores.rows();
  if (bsm.scores.cols() != t) throw ShapeError("pbs_b200: select_blocks takes a square block grid");
  detail::Dev ds(bsm.scores.data(), t * t * 4), dm(t * t), di(t * t * 4), dc(t * 4);
  detail::check(pbs_select_blocks(ds.as<float>(), 1, (int64_t)t, (int64_t)bsm.block_size,
                                  (int64_t)bsm.segment_size, tau, forced.first_block ? 1 : 0,
                                  forced.diagonal_band ? 1 : 0, dm.as<uint8_t>(), di.as<int32_t>(), dc.as<int32_t>(),
                                  nullptr));
  std::vector<uint8_t> m(t * t);
  dm.get(m.data(), m.size());
  BlockMask out(t, t, bsm.block_size, bsm.segment_size);
  for (std::size_t i = 0; i < t; ++i)
    for (std::size_t j = 0; j < t; ++j) out.set(i, j, m[i * t + j] != 0);
  return out;
}

/// pbs::attention_block_sparse (attention.hpp:259-310): the selected blocks of
/// `mask`, the ElementMask when given (else causal per cfg.causal, else none).
template <std::floating_point T>
Matrix<T> attention_block_sparse(const Matrix<T>& q, const Matrix<T>& k, const Matrix<T>& v,
                                 const AttentionConfig& cfg, const BlockMask& mask, const ElementMask* em = nullptr) {
  detail::require_f32<T>();
  if (q.rows() != k.rows() || q.cols() != k.cols() || v.rows() != k.rows() || v.cols() != q.cols())
    throw ShapeError("pbs_b200: attention_block_sparse takes square self-attention inputs with d_v == d");
  const std::size_t n = q.rows(), d = q.cols(), b = cfg.block_size, t = (n + b - 1) / b;
  if (mask.rows() != t || mask.cols() != t)
    throw ShapeError("attention: block mask grid is " + std::to_string(mask.rows()) + "x" +
                     std::to_string(mask.cols()) + ", expected " + std::to_string(t) + "x" + std::to_string(t));
  if (mask.block_size() != b) throw ShapeError("attention: block mask block size differs from config");
  std::vector<int32_t> idx, cnt;
  detail::csr_of(mask, idx, cnt);
  std::vector<int32_t> qo, ko;
  if (em) {
    if (em->query_len() != n || em->key_len() != n)
      throw ShapeError("attention: element mask lengths do not match inputs");
    qo.resize(n);
    ko.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
      qo[i] = (int32_t)em->q_orig(i);
      ko[i] = (int32_t)em->k_orig(i);
    }
  } else if (cfg.causal) {
    qo.resize(n);
    std::iota(qo.begin(), qo.end(), 0);
  }
  const pbs_shape sh = detail::shape_f32(n, d);
  detail::Dev dq(q.data(), n * d * 4), dk(k.data(), n * d * 4), dv(v.data(), n * d * 4), di(idx.data(), idx.size() * 4),
      dc(cnt.data(), t * 4), dout(n * d * 4), dst(8);
  detail::Dev dqo(qo.empty() ? nullptr : qo.data(), qo.size() * 4), dko(ko.empty() ? nullptr : ko.data(), ko.size() * 4);
  const int32_t st0[2] = {0, 0x7fffffff};
  dst.put(st0, sizeof st0);
  detail::check(pbs_block_sparse_attention_fwd(dq.as(), dk.as(), dv.as(), 1, &sh, (int64_t)b, cfg.scale,
                                               di.as<int32_t>(), dc.as<int32_t>(),
                                               qo.empty() ? nullptr : dqo.as<int32_t>(),
                                               ko.empty() ? nullptr : dko.as<int32_t>(), nullptr, dout.as(),
                                               dst.as<int32_t>(), nullptr));
  detail::check(pbs_check_status(dst.as<int32_t>(), (int64_t)t, nullptr));
  Matrix<T> out(n, d);
  dout.get(out.data(), n * d * 4);
  return out;
}

}  // namespace pbs::b200
