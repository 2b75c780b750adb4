// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference headers, compiled in place
// from /root/reference/proj/include (never copied) by oracle/Makefile into
// oracle/_ref/libpbsref.so with the reference's own flags (-O3 -std=gnu++20,
// no -march; proj/CMakeLists.txt:3-8).  It is used (a) to pin the C
// restatement in oracle/pbs_oracle.c bit-for-bit, and (b) as the CPU
// reference arm of bench.py (`--impl reference`, cpu_baseline kind
// "reference"), fanning heads over std::thread like pbs_main.cpp:99-122.
//
// Signatures match oracle/pbs_oracle.h with the prefix pbsref_.
#include <array>
#include <cstring>
#include <mutex>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "../include/pbs_cabi.h"
#include "pbs/attention.hpp"
#include "pbs/block_selection.hpp"
#include "pbs/errors.hpp"
#include "pbs/permutation.hpp"
#include "pbs/pipeline.hpp"
#include "pbs/tensor_io.hpp"
#include "pbs/workload.hpp"

namespace {

thread_local std::string g_err;

int fail(const pbs::Error& e) {
  g_err = std::string(e.prefix()) + ": " + e.what();
  return e.exit_code();
}
int fail_other(const std::exception& e) {
  g_err = std::string("E_INTERNAL: ") + e.what();
  return 1;
}

template <typename T>
pbs::Matrix<T> to_mat(const T* p, std::size_t rows, std::size_t cols) {
  pbs::Matrix<T> m(rows, cols);
  if (rows != 0 && cols != 0) std::memcpy(m.data(), p, sizeof(T) * rows * cols);
  return m;
}

template <typename T>
void from_mat(const pbs::Matrix<T>& m, T* p) {
  if (m.size()) std::memcpy(p, m.data(), sizeof(T) * m.size());
}

void perm_out(const pbs::Permutation& p, int32_t* out) {
  for (std::size_t i = 0; i < p.size(); ++i) out[i] = static_cast<int32_t>(p[i]);
}

std::vector<std::size_t> idx_in(const int32_t* p, std::size_t n) {
  std::vector<std::size_t> v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = p ? static_cast<std::size_t>(p[i]) : i;
  return v;
}

pbs::PipelineConfig to_cfg(const pbs_pipeline_config* c, pbs::Precision prec) {
  pbs::PipelineConfig cfg;
  cfg.block_size = static_cast<std::size_t>(c->block_size);
  cfg.segment_size = static_cast<std::size_t>(c->segment_size);
  cfg.tau = c->tau;
  cfg.strategy = static_cast<pbs::PermutationStrategy>(c->strategy);
  cfg.precision = prec;
  cfg.forced.first_block = c->forced_first_block != 0;
  cfg.forced.diagonal_band = c->forced_diagonal_band != 0;
  cfg.scale = c->scale;
  return cfg;
}

template <typename T>
int estimate(const T* q, std::size_t n, const T* k, std::size_t m, std::size_t d,
             std::size_t block, double scale, T* scores, std::size_t* src) {
  try {
    const auto imp = pbs::estimate_key_importance(to_mat(q, n, d), to_mat(k, m, d),
                                                  pbs::AttentionConfig::make(block, d, false, scale));
    std::memcpy(scores, imp.scores.data(), sizeof(T) * imp.scores.size());
    if (src) *src = imp.source_query_block;
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int key_perm(const T* scores, std::size_t n, std::size_t segment, int32_t* perm) {
  try {
    pbs::ImportanceScores<T> imp;
    imp.scores.assign(scores, scores + n);
    perm_out(pbs::build_key_permutation(imp, segment).flatten(), perm);
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int query_perm(const T* q, std::size_t n, const T* k, std::size_t m, std::size_t d,
               std::size_t block, std::size_t segment, int32_t* perm) {
  try {
    perm_out(pbs::build_query_permutation(to_mat(q, n, d), to_mat(k, m, d),
                                          pbs::AttentionConfig::make(block, d), segment)
                 .flatten(),
             perm);
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int causal_mask(std::size_t t_r, std::size_t t_c, std::size_t block, std::size_t segment, T* out) {
  try {
    from_mat(pbs::build_block_causal_mask<T>(t_r, t_c, block, segment), out);
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int meanpool(const T* qp, std::size_t n, const T* kp, std::size_t m, std::size_t d,
             std::size_t block, const T* causal, double scale, T* scores) {
  try {
    const std::size_t t_r = (n + block - 1) / block, t_c = (m + block - 1) / block;
    const auto bsm = pbs::meanpool_block_scores(to_mat(qp, n, d), to_mat(kp, m, d), block, 0,
                                                to_mat(causal, t_r, t_c), scale);
    from_mat(bsm.scores, scores);
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int select(const T* scores, const T* causal, std::size_t t_r, std::size_t t_c, std::size_t block,
           std::size_t segment, double tau, int first, int band, uint8_t* mask) {
  try {
    pbs::BlockScoreMatrix<T> bsm;
    bsm.scores = to_mat(scores, t_r, t_c);
    bsm.causal = to_mat(causal, t_r, t_c);
    bsm.block_size = block;
    bsm.segment_size = segment;
    pbs::ForcedPolicy fp;
    fp.first_block = first != 0;
    fp.diagonal_band = band != 0;
    const auto bm = pbs::select_blocks(bsm, tau, fp);
    for (std::size_t i = 0; i < t_r; ++i)
      for (std::size_t j = 0; j < t_c; ++j) mask[i * t_c + j] = bm.at(i, j) ? 1 : 0;
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int sparse_attn(const T* q, std::size_t n, const T* k, const T* v, std::size_t m, std::size_t d,
                std::size_t dv, std::size_t block, double scale, int causal, const uint8_t* mask,
                const int32_t* q_orig, const int32_t* k_orig, T* out, std::size_t* degenerate) {
  try {
    const auto cfg = pbs::AttentionConfig::make(block, d, causal != 0, scale);
    const std::size_t t_r = (n + block - 1) / block, t_c = (m + block - 1) / block;
    pbs::BlockMask bm = pbs::BlockMask::full(t_r, t_c, block);
    if (mask)
      for (std::size_t i = 0; i < t_r; ++i)
        for (std::size_t j = 0; j < t_c; ++j) bm.set(i, j, mask[i * t_c + j] != 0);
    const bool em_on = q_orig || k_orig;
    std::unique_ptr<pbs::ElementMask> em;
    if (em_on) em = std::make_unique<pbs::ElementMask>(idx_in(q_orig, n), idx_in(k_orig, m));
    from_mat(pbs::attention_block_sparse(to_mat(q, n, d), to_mat(k, m, d), to_mat(v, m, dv), cfg, bm,
                                         em.get()),
             out);
    return 0;
  } catch (const pbs::DegenerateRowError& e) {
    if (degenerate) *degenerate = e.query_block();
    return fail(e);
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int oracle_attn(const T* q, std::size_t n, const T* k, const T* v, std::size_t m, std::size_t d,
                std::size_t dv, std::size_t block, double scale, int causal, const int32_t* q_orig,
                const int32_t* k_orig, T* out) {
  try {
    const auto cfg = pbs::AttentionConfig::make(block, d, causal != 0, scale);
    std::unique_ptr<pbs::ElementMask> em;
    if (q_orig || k_orig) em = std::make_unique<pbs::ElementMask>(idx_in(q_orig, n), idx_in(k_orig, m));
    from_mat(pbs::attention_oracle(to_mat(q, n, d), to_mat(k, m, d), to_mat(v, m, dv), cfg, em.get()), out);
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
int coverage(const T* q, const T* k, std::size_t n, std::size_t d, const uint8_t* mask, std::size_t block,
             const int32_t* sigma, const int32_t* pi, double scale, double* out) {
  try {
    const std::size_t t = (n + block - 1) / block;
    pbs::BlockMask bm(t, t, block, 0);
    for (std::size_t r = 0; r < t; ++r)
      for (std::size_t c = 0; c < t; ++c) bm.set(r, c, mask[r * t + c] != 0);
    *out = pbs::attention_coverage(to_mat(q, n, d), to_mat(k, n, d), bm, pbs::Permutation(idx_in(sigma, n)),
                                   pbs::Permutation(idx_in(pi, n)), scale);
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

template <typename T>
void fill_report(const pbs::PipelineResult<T>& res, pbs_report* rep) {
  if (!rep) return;
  rep->block_density = res.report.block_density;
  rep->causal_density_baseline = res.report.causal_density_baseline;
  rep->pooled_score_coverage = res.report.pooled_score_coverage;
  rep->selected_blocks = static_cast<int64_t>(res.report.selected_blocks);
  rep->total_admissible_blocks = static_cast<int64_t>(res.report.total_admissible_blocks);
  rep->estimate_us = res.report.timings.estimate_us;
  rep->permute_us = res.report.timings.permute_us;
  rep->select_us = res.report.timings.select_us;
  rep->attention_us = res.report.timings.attention_us;
  rep->unpermute_us = res.report.timings.unpermute_us;
}

template <typename T>
int pipeline(const T* q, const T* k, const T* v, std::size_t n, std::size_t d,
             const pbs_pipeline_config* c, T* out, int32_t* sigma, int32_t* pi, uint8_t* mask,
             pbs_report* rep) {
  try {
    const auto cfg = to_cfg(c, sizeof(T) == 4 ? pbs::Precision::f32 : pbs::Precision::f64);
    const auto res = pbs::pbs_attention(to_mat(q, n, d), to_mat(k, n, d), to_mat(v, n, d), cfg);
    from_mat(res.output, out);
    if (sigma) perm_out(res.sigma, sigma);
    if (pi) perm_out(res.pi, pi);
    if (mask)
      for (std::size_t i = 0; i < res.mask.rows(); ++i)
        for (std::size_t j = 0; j < res.mask.cols(); ++j)
          mask[i * res.mask.cols() + j] = res.mask.at(i, j) ? 1 : 0;
    fill_report(res, rep);
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) { return fail_other(e); }
}

}  // namespace

extern "C" {

const char* pbsref_last_error(void) { return g_err.c_str(); }

#define PBSREF_DEFS(T, SFX)                                                                        \
  int pbsref_estimate_key_importance_##SFX(const T* q, size_t n, const T* k, size_t m, size_t d,   \
                                           size_t block, double scale, T* scores, size_t* src) {   \
    return estimate<T>(q, n, k, m, d, block, scale, scores, src);                                  \
  }                                                                                                \
  int pbsref_build_key_permutation_##SFX(const T* scores, size_t n, size_t segment,                \
                                         int32_t* perm) {                                          \
    return key_perm<T>(scores, n, segment, perm);                                                  \
  }                                                                                                \
  int pbsref_build_query_permutation_##SFX(const T* q, size_t n, const T* k, size_t m, size_t d,   \
                                           size_t block, size_t segment, int32_t* perm) {          \
    return query_perm<T>(q, n, k, m, d, block, segment, perm);                                     \
  }                                                                                                \
  int pbsref_block_causal_mask_##SFX(size_t t_r, size_t t_c, size_t block, size_t segment,         \
                                     T* causal) {                                                  \
    return causal_mask<T>(t_r, t_c, block, segment, causal);                                       \
  }                                                                                                \
  int pbsref_meanpool_block_scores_##SFX(const T* qp, size_t n, const T* kp, size_t m, size_t d,   \
                                         size_t block, const T* causal, double scale,              \
                                         T* scores) {                                              \
    return meanpool<T>(qp, n, kp, m, d, block, causal, scale, scores);                             \
  }                                                                                                \
  int pbsref_select_blocks_##SFX(const T* scores, const T* causal, size_t t_r, size_t t_c,         \
                                 size_t block, size_t segment, double tau, int first, int band,    \
                                 uint8_t* mask) {                                                  \
    return select<T>(scores, causal, t_r, t_c, block, segment, tau, first, band, mask);            \
  }                                                                                                \
  int pbsref_attention_block_sparse_##SFX(const T* q, size_t n, const T* k, const T* v, size_t m,  \
                                          size_t d, size_t dv, size_t block, double scale,         \
                                          int causal, const uint8_t* mask, const int32_t* qo,      \
                                          const int32_t* ko, T* out, size_t* degenerate) {         \
    return sparse_attn<T>(q, n, k, v, m, d, dv, block, scale, causal, mask, qo, ko, out,           \
                          degenerate);                                                             \
  }                                                                                                \
  int pbsref_attention_oracle_##SFX(const T* q, size_t n, const T* k, const T* v, size_t m,        \
                                    size_t d, size_t dv, size_t block, double scale, int causal,   \
                                    const int32_t* qo, const int32_t* ko, T* out) {                \
    return oracle_attn<T>(q, n, k, v, m, d, dv, block, scale, causal, qo, ko, out);                \
  }                                                                                                \
  int pbsref_pbs_attention_##SFX(const T* q, const T* k, const T* v, size_t n, size_t d,           \
                                 const pbs_pipeline_config* cfg, T* out, int32_t* sigma,           \
                                 int32_t* pi, uint8_t* mask, pbs_report* rep) {                    \
    return pipeline<T>(q, k, v, n, d, cfg, out, sigma, pi, mask, rep);                             \
  }                                                                                                \
  int pbsref_attention_coverage_##SFX(const T* q, const T* k, size_t n, size_t d,                  \
                                      const uint8_t* mask, size_t block, const int32_t* sigma,     \
                                      const int32_t* pi, double scale, double* cov) {              \
    return coverage<T>(q, k, n, d, mask, block, sigma, pi, scale, cov);                            \
  }

PBSREF_DEFS(float, f32)
PBSREF_DEFS(double, f64)

// Multi-head CPU run (the reference CLI's for_each_head, pbs_main.cpp:99-122):
// heads [H, N, d] f32 each, K/V head = h / (Hq / Hkv) (GQA repeated per q head
// since the reference has no GQA), `threads` workers, reports summed.
int pbsref_pbs_attention_heads_f32(const float* q, const float* k, const float* v, int hq, int hkv,
                                   size_t n, size_t d, const pbs_pipeline_config* cfg, float* out,
                                   int threads, pbs_report* rep_sum) {
  if (hkv <= 0 || hq <= 0 || hq % hkv != 0) {
    g_err = "E_SHAPE: query heads must be a whole number of GQA groups";
    return PBS_ERR_CONFIG;
  }
  const int g = hq / hkv;
  std::vector<pbs_report> reps(hq);
  std::vector<int> rcs(hq, 0);
  std::vector<std::string> errs(hq);
  int next = 0;
  std::mutex mu;
  auto worker = [&]() {
    for (;;) {
      int h;
      {
        std::lock_guard<std::mutex> lk(mu);
        if (next >= hq) return;
        h = next++;
      }
      const std::size_t off_q = static_cast<std::size_t>(h) * n * d;
      const std::size_t off_kv = static_cast<std::size_t>(h / g) * n * d;
      std::memset(&reps[h], 0, sizeof(pbs_report));
      rcs[h] = pipeline<float>(q + off_q, k + off_kv, v + off_kv, n, d, cfg, out + off_q, nullptr,
                               nullptr, nullptr, &reps[h]);
      if (rcs[h]) errs[h] = g_err;
    }
  };
  std::vector<std::thread> pool;
  const int nt = threads < 1 ? 1 : threads;
  for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  if (rep_sum) std::memset(rep_sum, 0, sizeof(pbs_report));
  for (int h = 0; h < hq; ++h) {  // deterministic merge by head index
    if (rcs[h]) {
      g_err = errs[h];
      return rcs[h];
    }
    if (rep_sum) {
      rep_sum->block_density += reps[h].block_density / hq;
      rep_sum->causal_density_baseline += reps[h].causal_density_baseline / hq;
      rep_sum->pooled_score_coverage += reps[h].pooled_score_coverage / hq;
      rep_sum->selected_blocks += reps[h].selected_blocks;
      rep_sum->total_admissible_blocks += reps[h].total_admissible_blocks;
      rep_sum->estimate_us += reps[h].estimate_us;
      rep_sum->permute_us += reps[h].permute_us;
      rep_sum->select_us += reps[h].select_us;
      rep_sum->attention_us += reps[h].attention_us;
      rep_sum->unpermute_us += reps[h].unpermute_us;
    }
  }
  return 0;
}

// Stages 1-3 of pbs_attention (pipeline.hpp:129-171) under key_permute, per
// head over `threads` workers, each stage timed like StageClock (pipeline.hpp:
// 86-99): estimate_key_importance + build_key_permutation (estimate),
// apply_rows of K and V (permute), meanpool_block_scores + select_blocks
// (select).  The CPU baseline times these at full length and extrapolates only
// the attention.  stage_us[3] and the selected-block count are
// summed over heads.
int pbsref_pbs_stages_heads_f32(const float* q, const float* k, const float* v, int hq, int hkv, size_t n,
                                size_t d, const pbs_pipeline_config* c, int threads, double* stage_us,
                                int64_t* selected) {
  if (hkv <= 0 || hq <= 0 || hq % hkv != 0 || c->strategy != PBS_STRATEGY_KEY_PERMUTE) {
    g_err = "E_CONFIG: stage timing covers key_permute over whole GQA groups";
    return PBS_ERR_CONFIG;
  }
  const int g = hq / hkv;
  std::vector<std::array<double, 3>> us(hq);
  std::vector<int64_t> sel(hq, 0);
  std::vector<int> rcs(hq, 0);
  std::vector<std::string> errs(hq);
  int next = 0;
  std::mutex mu;
  const pbs::PipelineConfig cfg = to_cfg(c, pbs::Precision::f32);
  auto worker = [&]() {
    for (;;) {
      int h;
      {
        std::lock_guard<std::mutex> lk(mu);
        if (next >= hq) return;
        h = next++;
      }
      try {
        const auto qm = to_mat(q + (size_t)h * n * d, n, d);
        const auto km = to_mat(k + (size_t)(h / g) * n * d, n, d);
        const auto vm = to_mat(v + (size_t)(h / g) * n * d, n, d);
        const auto acfg = pbs::AttentionConfig::make(cfg.block_size, d, false, cfg.scale);
        pbs::detail::StageClock clock;
        const auto imp = pbs::estimate_key_importance(qm, km, acfg);
        const pbs::Permutation pi = pbs::build_key_permutation(imp, cfg.segment_size).flatten();
        us[h][0] = clock.lap_us();
        const auto qp = pbs::apply_rows(pbs::Permutation::identity(n), qm);  // sigma = identity
        const auto kp = pbs::apply_rows(pi, km);
        const auto vp = pbs::apply_rows(pi, vm);
        us[h][1] = clock.lap_us();
        const std::size_t t = (n + cfg.block_size - 1) / cfg.block_size;
        const auto causal = pbs::build_block_causal_mask<float>(t, t, cfg.block_size, cfg.segment_size);
        const auto bsm = pbs::meanpool_block_scores(qp, kp, cfg.block_size, cfg.segment_size, causal, cfg.scale);
        const auto mask = pbs::select_blocks(bsm, cfg.tau, cfg.forced);
        us[h][2] = clock.lap_us();
        sel[h] = (int64_t)mask.selected_count();
        (void)vp;
      } catch (const pbs::Error& e) {
        rcs[h] = fail(e);
        errs[h] = g_err;
      } catch (const std::exception& e) {
        rcs[h] = fail_other(e);
        errs[h] = g_err;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < (threads < 1 ? 1 : threads); ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  for (int i = 0; i < 3; ++i) stage_us[i] = 0.0;
  *selected = 0;
  for (int h = 0; h < hq; ++h) {
    if (rcs[h]) {
      g_err = errs[h];
      return rcs[h];
    }
    for (int i = 0; i < 3; ++i) stage_us[i] += us[h][i];
    *selected += sel[h];
  }
  return 0;
}

// Synthetic workload (workload.hpp:145-198), one head, for golden fixtures:
// kind 0 gaussian, 1 vertical_lines, 2 block_diag, 3 mixed; scatter 0
// clustered, 1 scattered.  Writes q, k, v [n, d] and returns the planted
// line count (positions into `planted` when non-null).
#define PBSREF_GEN(T, SFX)                                                                         \
  int pbsref_generate_head_##SFX(int kind, size_t n, size_t d, uint64_t seed, size_t line_count,   \
                                 double line_strength, int scatter, size_t head,                   \
                                 size_t block, size_t segment, T* q, T* k, T* v,                   \
                                 int64_t* planted) {                                               \
    try {                                                                                          \
      pbs::WorkloadSpec spec;                                                                      \
      spec.kind = static_cast<pbs::WorkloadKind>(kind);                                            \
      spec.n = n;                                                                                  \
      spec.d = d;                                                                                  \
      spec.heads = head + 1;                                                                       \
      spec.seed = seed;                                                                            \
      spec.line_count = line_count;                                                                \
      spec.line_strength = line_strength;                                                          \
      spec.scatter = scatter ? pbs::LineScatter::scattered : pbs::LineScatter::clustered;          \
      spec.validate();                                                                             \
      pbs::Matrix<T> mq, mk, mv;                                                                   \
      std::vector<std::size_t> pl;                                                                 \
      pbs::generate_head<T>(spec, head, block, segment, mq, mk, mv, pl);                           \
      from_mat(mq, q);                                                                             \
      from_mat(mk, k);                                                                             \
      from_mat(mv, v);                                                                             \
      if (planted)                                                                                 \
        for (std::size_t i = 0; i < pl.size(); ++i) planted[i] = static_cast<int64_t>(pl[i]);      \
      return static_cast<int>(pl.size());                                                          \
    } catch (const pbs::Error& e) { return -fail(e); }                                             \
  }
PBSREF_GEN(float, f32)
PBSREF_GEN(double, f64)

// PBST files through the reference's own tensor_io.hpp: write_tensor(_stack)
// of `heads` row-major [rows, cols] matrices, and read_tensor into a caller
// buffer (dims[3] = heads, rows, cols; *file_dtype 0 f32 / 1 f64; values
// widened to double).  Errors return the reference's code and E_* text.
#define PBSREF_TIO(T, SFX)                                                                         \
  int pbsref_write_tensor_##SFX(const char* path, const T* data, size_t heads, size_t rows,        \
                                size_t cols, int as_stack) {                                       \
    try {                                                                                          \
      std::vector<pbs::Matrix<T>> hs;                                                              \
      for (size_t h = 0; h < heads; ++h) hs.push_back(to_mat(data + h * rows * cols, rows, cols)); \
      pbs::write_tensor<T>(path, std::span<const pbs::Matrix<T>>(hs.data(), hs.size()),           \
                           as_stack != 0);                                                         \
      return 0;                                                                                    \
    } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) {            \
      return fail_other(e);                                                                        \
    }                                                                                              \
  }
PBSREF_TIO(float, f32)
PBSREF_TIO(double, f64)

int pbsref_read_tensor(const char* path, double* out, size_t capacity, int64_t* dims, int* file_dtype,
                       int* ndim) {
  try {
    const pbs::LoadedTensor t = pbs::read_tensor(path);
    *file_dtype = static_cast<int>(t.dtype);
    *ndim = t.is_stack ? 3 : 2;
    auto emit = [&](const auto& heads) {
      dims[0] = static_cast<int64_t>(heads.size());
      dims[1] = heads.empty() ? 0 : static_cast<int64_t>(heads[0].rows());
      dims[2] = heads.empty() ? 0 : static_cast<int64_t>(heads[0].cols());
      size_t o = 0;
      for (const auto& m : heads)
        for (size_t i = 0; i < m.size() && o < capacity; ++i) out[o++] = static_cast<double>(m.data()[i]);
    };
    if (t.dtype == pbs::Dtype::f32) emit(t.as<float>());
    else emit(t.as<double>());
    return 0;
  } catch (const pbs::Error& e) { return fail(e); } catch (const std::exception& e) {
    return fail_other(e);
  }
}

}  // extern "C"
