// workload.cu -- the reference's synthetic workload generator (workload.hpp:145-198,
// rng.hpp), host code, so that run manifests naming a `workload` instead of
// input files (manifest.hpp:26-39, pbs_main.cpp:70-80) run on the device path
// with the same tensors, bit for bit, as the reference CLI generates.
//
// The reference pins the bytes by construction: mt19937_64 seeded through
// std::seed_seq {seed lo, seed hi, stream lo, stream hi} (fully specified by
// the C++ standard), uniforms from the top 53 bits, Box-Muller normals with a
// cached spare (std::sqrt / std::log / std::sin / std::cos of glibc, as in the
// reference build), values converted to the precision T only when stored.  The
// same operations in the same order are restated here; tests/test_workload.py
// compares every element with the compiled reference.
#include <cmath>
#include <cstdint>

#include <random>
#include <string>
#include <vector>

#include "common.cuh"
#include "pbs_cabi.h"

namespace pbs_b200 {
namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;  // std::numbers::pi (the same double)

class Rng {  // rng.hpp:15-49
 public:
  Rng(uint64_t seed, uint64_t stream) {
    std::seed_seq seq{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), static_cast<uint32_t>(stream),
                      static_cast<uint32_t>(stream >> 32)};
    engine_.seed(seq);
  }
  double uniform() { return double(engine_() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 == 0.0) u1 = uniform();
    const double u2 = uniform();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * kPi * u2;
    spare_ = mag * std::sin(ang);
    has_spare_ = true;
    return mag * std::cos(ang);
  }

 private:
  std::mt19937_64 engine_;
  double spare_ = 0;
  bool has_spare_ = false;
};

// plan_line_positions (workload.hpp:68-107)
std::vector<int64_t> line_positions(int64_t n, int64_t line_count, int scatter, int64_t block, int64_t segment) {
  std::vector<int64_t> pos;
  if (line_count == 0) return pos;
  const uint64_t un = (uint64_t)n, lc = (uint64_t)line_count, b = (uint64_t)block, s = (uint64_t)segment;
  if (scatter == PBS_SCATTER_CLUSTERED) {
    const uint64_t start = std::min(un / 2, un - lc);
    for (uint64_t t = 0; t < lc; ++t) pos.push_back((int64_t)(start + t));
    return pos;
  }
  const uint64_t groups = s > 0 ? un / s : 0;
  if (groups == 0 || s < b) {
    for (uint64_t t = 0; t < lc; ++t) pos.push_back((int64_t)((2 * t + 1) * un / (2 * lc)));
    return pos;
  }
  uint64_t per_seg = std::max<uint64_t>(1, s / b);
  uint64_t used = (lc + per_seg - 1) / per_seg;
  if (used > groups) {
    used = groups;
    per_seg = (lc + groups - 1) / groups;
  }
  const uint64_t stride = std::max<uint64_t>(1, s / per_seg);
  for (uint64_t t = 0; t < lc; ++t) {
    const uint64_t u = t / per_seg;
    const uint64_t g = (2 * u + 1) * groups / (2 * used);
    const uint64_t p = g * s + (t % per_seg) * stride + stride / 2;
    pos.push_back((int64_t)std::min(p, un - 1));
  }
  return pos;
}

std::vector<double> random_unit(int64_t d, Rng& rng) {  // detail::random_unit (workload.hpp:125-139)
  std::vector<double> u((size_t)d);
  double norm = 0;
  do {
    norm = 0;
    for (auto& x : u) {
      x = rng.normal();
      norm += x * x;
    }
  } while (norm == 0);
  norm = std::sqrt(norm);
  for (auto& x : u) x /= norm;
  return u;
}

// generate_head (workload.hpp:145-198) into row-major [n, d] buffers of T
template <typename T>
int generate(const pbs_workload_spec& w, int64_t head, int64_t block, int64_t segment, T* q, T* k, T* v,
             int64_t* planted, int64_t* planted_count) {
  const int64_t n = w.n, d = w.d;
  Rng rng(w.seed, (uint64_t)head);
  for (T* m : {q, k, v})  // detail::fill_normal, row by row
    for (int64_t i = 0; i < n * d; ++i) m[i] = T(rng.normal());
  const bool lines = w.kind == PBS_WORKLOAD_VERTICAL_LINES || w.kind == PBS_WORKLOAD_MIXED;
  const bool blockish = w.kind == PBS_WORKLOAD_BLOCK_DIAG || w.kind == PBS_WORKLOAD_MIXED;
  if (blockish) {
    const int64_t blocks = (n + block - 1) / block;
    const double kappa = std::sqrt(10.0 * std::sqrt(double(d)));
    std::vector<std::vector<double>> dirs((size_t)blocks);
    for (auto& dir : dirs) dir = random_unit(d, rng);
    for (int64_t r = 0; r < n; ++r) {
      const auto& dir = dirs[(size_t)(r / block)];
      for (int64_t c = 0; c < d; ++c) {
        q[r * d + c] += T(kappa * dir[(size_t)c]);
        k[r * d + c] += T(kappa * dir[(size_t)c]);
      }
    }
  }
  int64_t np = 0;
  if (lines) {
    const auto u = random_unit(d, rng);
    const double query_bias = std::sqrt(double(d));
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < d; ++c) q[r * d + c] += T(query_bias * u[(size_t)c]);
    const auto pos = line_positions(n, w.line_count, w.scatter, block, segment);
    for (int64_t p : pos) {
      for (int64_t c = 0; c < d; ++c) k[p * d + c] += T(w.line_strength * u[(size_t)c]);
      if (planted) planted[np] = p;
      ++np;
    }
  }
  if (planted_count) *planted_count = np;
  for (T* m : {q, k, v})
    for (int64_t i = 0; i < n * d; ++i)
      if (!std::isfinite((double)m[i])) return fail(PBS_ERR_CONFIG, "E_CONFIG", "workload generated non-finite values");
  return PBS_OK;
}

}  // namespace
}  // namespace pbs_b200

using namespace pbs_b200;

extern "C" {

int pbs_generate_workload_head(const pbs_workload_spec* w, int64_t head, int64_t block_size, int64_t segment_size,
                               int32_t host_dtype, void* q, void* k, void* v, int64_t* planted,
                               int64_t* planted_count) {
  if (!w || !q || !k || !v) return fail(PBS_ERR_CONFIG, "E_CONFIG", "generate_workload_head: null pointer");
  // WorkloadSpec::validate (workload.hpp:30-37)
  if (w->n <= 0 || w->d <= 0 || w->heads <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "workload dims must be >= 1");
  if (w->kind < PBS_WORKLOAD_GAUSSIAN || w->kind > PBS_WORKLOAD_MIXED)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "unknown workload kind");
  if (w->kind == PBS_WORKLOAD_VERTICAL_LINES || w->kind == PBS_WORKLOAD_MIXED) {
    if (w->line_count < 0 || w->line_count > w->n)
      return fail(PBS_ERR_CONFIG, "E_CONFIG", "line count exceeds sequence length");
    if (!(w->line_strength > 0)) return fail(PBS_ERR_CONFIG, "E_CONFIG", "line strength must be > 0");
  }
  if (head < 0 || head >= w->heads) return fail(PBS_ERR_CONFIG, "E_CONFIG", "head index out of range");
  if (block_size <= 0 || segment_size < 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (host_dtype == PBS_HOST_F64)
    return generate<double>(*w, head, block_size, segment_size, static_cast<double*>(q), static_cast<double*>(k),
                            static_cast<double*>(v), planted, planted_count);
  if (host_dtype == PBS_HOST_F32)
    return generate<float>(*w, head, block_size, segment_size, static_cast<float*>(q), static_cast<float*>(k),
                           static_cast<float*>(v), planted, planted_count);
  return fail(PBS_ERR_CONFIG, "E_CONFIG", "workload precision must be f32 or f64");
}

}  // extern "C"
