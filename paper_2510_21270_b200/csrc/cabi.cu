// cabi.cu -- the extern "C" boundary (include/pbs_cabi.h) and the fused
// Algorithm-1 orchestration (pbs_attention, pipeline.hpp:107-193).
//
// Host code here only validates, carves the caller's workspace and launches
// the device stages on the caller's stream; there is no CPU compute path.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "pipeline.h"

namespace pbs_b200 {

namespace {
thread_local std::string g_err;
std::atomic<long long> g_launches{0};
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) return 148;
  cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

void set_error(const char* prefix, const std::string& msg) { g_err = std::string(prefix) + ": " + msg; }

int fail(int code, const char* prefix, const std::string& msg) {
  set_error(prefix, msg);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  set_error("E_CUDA", std::string(where) + ": " + cudaGetErrorString(e));
  return PBS_ERR_CUDA;
}


int esize_of(int dtype) { return dtype == PBS_DTYPE_BF16 ? 2 : 4; }

float effective_scale(double scale, int d) {
  // AttentionConfig::effective_scale (attention.hpp:32-34), cast to float at use
  return (float)(scale > 0.0 ? scale : 1.0 / sqrt((double)d));
}

int check_shape(const pbs_shape* s) {
  if (!s) return fail(PBS_ERR_CONFIG, "E_SHAPE", "null shape");
  if (s->dtype != PBS_DTYPE_BF16 && s->dtype != PBS_DTYPE_F32)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "dtype must be bf16 or f32");
  if (s->num_q_heads <= 0 || s->num_kv_heads <= 0 || s->num_q_heads % s->num_kv_heads != 0)
    return fail(PBS_ERR_CONFIG, "E_SHAPE", "num_q_heads must be a positive multiple of num_kv_heads");
  if (s->head_dim <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "head dim must be >= 1");
  if (s->seq_len <= 0) return fail(PBS_ERR_CONFIG, "E_SHAPE", "pipeline inputs are empty");
  if (s->seq_len > (int64_t)1 << 30) return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "sequence longer than 2^30");
  return PBS_OK;
}

// PipelineConfig::validate (pipeline.hpp:39-48)
int check_cfg(const pbs_pipeline_config* c) {
  if (!c) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null config");
  if (c->block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (c->segment_size < 0 ||
      (c->segment_size != 0 && (c->segment_size < c->block_size || c->segment_size % c->block_size != 0)))
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "segment size must be 0 or a multiple of the block size");
  if (!(c->tau >= 0.0 && c->tau <= 1.0)) return fail(PBS_ERR_CONFIG, "E_CONFIG", "tau must lie in [0, 1]");
  if (c->strategy < PBS_STRATEGY_NONE || c->strategy > PBS_STRATEGY_BOTH)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "unknown permutation strategy");
  if (c->segment_size == 0 && c->strategy != PBS_STRATEGY_NONE)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "segment size 0 requires strategy none");
  if (c->scale < 0.0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "scale must be > 0");
  if (c->top_k < 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "top_k must be >= 0 (0 selects by tau)");
  return PBS_OK;
}

bool uses_pi(int s) { return s == PBS_STRATEGY_KEY_PERMUTE || s == PBS_STRATEGY_BOTH; }
bool uses_sigma(int s) { return s == PBS_STRATEGY_QUERY_PERMUTE || s == PBS_STRATEGY_BOTH; }


size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

Layout plan(const pbs_shape* s, const pbs_pipeline_config* c) {
  Layout L{};
  const int64_t n = s->seq_len, hq = s->num_q_heads, d = s->head_dim, b = c->block_size;
  const int64_t t = ceil_div(n, b);
  const size_t es = esize_of(s->dtype);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al(bytes);
    return o;
  };
  L.status = take(16);
  L.imp = take(uses_pi(c->strategy) ? importance_workspace_bytes((int)hq, n, b) : 0);
  L.scores = take(uses_pi(c->strategy) ? (size_t)hq * n * 4 : 0);
  L.pi = take((size_t)hq * n * 4);
  L.pi_inv = take(uses_pi(c->strategy) ? (size_t)hq * n * 4 : 0);
  L.sigma = take((size_t)hq * n * 4);
  L.sigma_inv = take(uses_sigma(c->strategy) ? (size_t)hq * n * 4 : 0);
  L.groups = take(uses_sigma(c->strategy) ? (size_t)hq * n * 4 : 0);
  L.qperm = take(uses_sigma(c->strategy) ? query_perm_workspace_bytes((int)hq, n, (int)d, b) : 0);
  L.kp = take(uses_pi(c->strategy) ? (size_t)hq * n * d * es : 0);
  L.vp = take(uses_pi(c->strategy) ? (size_t)hq * n * d * es : 0);
  L.qp = take(uses_sigma(c->strategy) ? (size_t)hq * n * d * es : 0);
  L.qbar = take((size_t)hq * t * d * 4);
  L.kbar = take((size_t)hq * t * d * 4);
  L.blog = take((size_t)hq * t * t * 4);
  L.mask = take((size_t)hq * t * t);
  L.kv_idx = take((size_t)hq * t * t * 4);
  L.kv_cnt = take((size_t)hq * t * 4);
  L.row_cov = take((size_t)hq * t * 8);
  L.sched = take(attention_sm100_workspace_bytes((int)hq, n, b));
  L.total = off + 256;
  return L;
}


int run_attention(const AttnParams& p, void* sched, cudaStream_t st) {
  if (attention_sm100_supported(p)) return launch_attention_sm100(p, sched, st);
  if (getenv("PBS_REQUIRE_TC"))  // tests: the shape must take the tensor-core kernel
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "PBS_REQUIRE_TC: this attention call would take the SIMT kernel");
  return launch_attention_simt(p, st);
}

}  // namespace pbs_b200

using namespace pbs_b200;

extern "C" {

const char* pbs_last_error(void) { return g_err.c_str(); }

const char* pbs_version(void) { return "pbs-b200 0.1 (sm_100a)"; }

int64_t pbs_kernel_launches(void) { return (int64_t)g_launches.load(); }

size_t pbs_workspace_size(const pbs_shape* shape, const pbs_pipeline_config* cfg) {
  if (check_shape(shape) || check_cfg(cfg)) return 0;
  return plan(shape, cfg).total;
}

int pbs_estimate_key_importance(const void* q, const void* k, const pbs_shape* shape, int64_t block_size,
                                double scale, float* scores, void* workspace, size_t workspace_bytes,
                                void* stream) {
  if (int rc = check_shape(shape)) return rc;
  if (block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (scale < 0.0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "scale must be > 0");
  return launch_importance(q, k, shape->dtype, shape->num_q_heads, shape->num_kv_heads, shape->seq_len,
                           shape->head_dim, block_size, effective_scale(scale, shape->head_dim), scores, workspace,
                           workspace_bytes, as_stream(stream));
}

int pbs_build_key_permutation(const float* scores, int32_t num_heads, int64_t seq_len, int64_t segment_size,
                              int32_t* perm, int32_t* inv, void* stream) {
  if (segment_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "build_key_permutation: segment size must be >= 1");
  if (num_heads <= 0 || seq_len < 0) return fail(PBS_ERR_CONFIG, "E_SHAPE", "bad head count or length");
  return launch_segmented_sort(scores, 0, num_heads, seq_len, segment_size, perm, inv, as_stream(stream));
}

int pbs_build_query_permutation(const void* q, const void* k, int32_t k_heads, const pbs_shape* shape,
                                int64_t block_size, int64_t segment_size, int32_t* perm, int32_t* inv,
                                void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_shape(shape)) return rc;
  if (segment_size <= 0)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "build_query_permutation: segment size must be >= 1");
  if (block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (k_heads <= 0 || shape->num_q_heads % k_heads != 0)
    return fail(PBS_ERR_CONFIG, "E_SHAPE", "k_heads must divide num_q_heads");
  const int64_t n = shape->seq_len;
  const size_t need = query_perm_workspace_bytes(shape->num_q_heads, n, shape->head_dim, block_size) +
                      al((size_t)shape->num_q_heads * n * 4);
  if (workspace_bytes < need) return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "query permutation workspace too small");
  uint32_t* groups = static_cast<uint32_t*>(workspace);
  void* rest = static_cast<char*>(workspace) + al((size_t)shape->num_q_heads * n * 4);
  cudaStream_t st = as_stream(stream);
  if (int rc = launch_query_groups(q, k, shape->dtype, shape->num_q_heads, k_heads, n, shape->head_dim,
                                   block_size, groups, rest, workspace_bytes - al((size_t)shape->num_q_heads * n * 4),
                                   st))
    return rc;
  return launch_segmented_sort(groups, 1, shape->num_q_heads, n, segment_size, perm, inv, st);
}

size_t pbs_query_permutation_workspace_size(const pbs_shape* shape, int64_t block_size) {
  if (!shape || check_shape(shape) || block_size <= 0) return 0;
  return query_perm_workspace_bytes(shape->num_q_heads, shape->seq_len, shape->head_dim, block_size) +
         al((size_t)shape->num_q_heads * shape->seq_len * 4);
}

int pbs_apply_rows(const int32_t* perm, const void* src, int32_t src_heads, int32_t dst_heads, int64_t rows,
                   int32_t cols, int32_t dtype, void* dst, void* stream) {
  if (dtype != PBS_DTYPE_BF16 && dtype != PBS_DTYPE_F32) return fail(PBS_ERR_CONFIG, "E_CONFIG", "bad dtype");
  return launch_apply_rows(perm, src, src_heads, dst_heads, rows, cols, esize_of(dtype), dst, as_stream(stream));
}

int pbs_unpermute(const int32_t* sigma, const void* src, int32_t num_heads, int64_t rows, int32_t cols,
                  int32_t dtype, void* dst, void* stream) {
  if (dtype != PBS_DTYPE_BF16 && dtype != PBS_DTYPE_F32) return fail(PBS_ERR_CONFIG, "E_CONFIG", "bad dtype");
  if (num_heads < 0 || rows < 0 || cols < 0) return fail(PBS_ERR_CONFIG, "E_SHAPE", "unpermute: negative shape");
  return launch_scatter_rows(sigma, src, num_heads, rows, cols, esize_of(dtype), dst, as_stream(stream));
}

int pbs_meanpool_block_scores(const void* qp, const void* kp, const pbs_shape* shape, int64_t block_size,
                              int64_t segment_size, double scale, float* scores, void* workspace,
                              size_t workspace_bytes, void* stream) {
  if (int rc = check_shape(shape)) return rc;
  if (block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (segment_size != 0 && (segment_size < block_size || segment_size % block_size != 0))
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "segment size must be 0 or a multiple of the block size");
  const int64_t n = shape->seq_len, t = ceil_div(n, block_size);
  const int hq = shape->num_q_heads, d = shape->head_dim;
  const size_t need = 2 * al((size_t)hq * t * d * 4) + al((size_t)hq * t * t * 4);
  if (workspace_bytes < need) return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "meanpool workspace too small");
  float* qbar = static_cast<float*>(workspace);
  float* kbar = reinterpret_cast<float*>(static_cast<char*>(workspace) + al((size_t)hq * t * d * 4));
  float* blog = reinterpret_cast<float*>(static_cast<char*>(workspace) + 2 * al((size_t)hq * t * d * 4));
  cudaStream_t st = as_stream(stream);
  if (int rc = launch_pool(qp, shape->dtype, hq, hq, nullptr, n, d, block_size, qbar, st)) return rc;
  if (int rc = launch_pool(kp, shape->dtype, shape->num_kv_heads, hq, nullptr, n, d, block_size, kbar, st)) return rc;
  // scores only (no selection)
  return launch_score_select(qbar, kbar, blog, hq, t, d, block_size, segment_size, effective_scale(scale, d), 1.0, 0,
                             0, 0, scores, nullptr, nullptr, nullptr, nullptr, st);
}

int pbs_select_blocks(const float* scores, int32_t num_heads, int64_t num_blocks, int64_t block_size,
                      int64_t segment_size, double tau, int32_t forced_first_block, int32_t forced_diagonal_band,
                      uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt, void* stream) {
  if (!(tau >= 0.0 && tau <= 1.0)) return fail(PBS_ERR_CONFIG, "E_CONFIG", "tau must lie in [0, 1]");
  if (block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (segment_size != 0 && (segment_size < block_size || segment_size % block_size != 0))
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "segment size must be 0 or a multiple of the block size");
  return launch_select_from_scores(scores, num_heads, num_blocks, block_size, segment_size, tau, forced_first_block,
                                   forced_diagonal_band, mask, kv_idx, kv_cnt, as_stream(stream));
}

int pbs_select_blocks_top_k(const float* scores, int32_t num_heads, int64_t num_blocks, int64_t block_size,
                            int64_t segment_size, int32_t top_k, int32_t forced_first_block,
                            int32_t forced_diagonal_band, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt,
                            void* stream) {
  if (top_k < 1) return fail(PBS_ERR_CONFIG, "E_CONFIG", "top_k must be >= 1");
  if (block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (segment_size != 0 && (segment_size < block_size || segment_size % block_size != 0))
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "segment size must be 0 or a multiple of the block size");
  return launch_select_from_scores(scores, num_heads, num_blocks, block_size, segment_size, 1.0, forced_first_block,
                                   forced_diagonal_band, mask, kv_idx, kv_cnt, as_stream(stream), top_k);
}

int pbs_block_sparse_attention_fwd(const void* qp, const void* kp, const void* vp, int32_t kv_heads,
                                   const pbs_shape* shape, int64_t block_size, double scale, const int32_t* kv_idx,
                                   const int32_t* kv_cnt, const int32_t* q_orig, const int32_t* k_orig,
                                   const int32_t* out_rows, void* out, int32_t* status, void* stream) {
  if (int rc = check_shape(shape)) return rc;
  if (block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "attention: block size must be >= 1");
  if (kv_heads <= 0 || shape->num_q_heads % kv_heads != 0)
    return fail(PBS_ERR_CONFIG, "E_SHAPE", "kv_heads must divide num_q_heads");
  if ((kv_idx == nullptr) != (kv_cnt == nullptr))
    return fail(PBS_ERR_CONFIG, "E_SHAPE", "kv_idx and kv_cnt must be given together");
  AttnParams p{};
  p.q = qp;
  p.k = kp;
  p.v = vp;
  p.out = out;
  p.dtype = shape->dtype;
  p.hq = shape->num_q_heads;
  p.kv_heads = kv_heads;
  p.d = shape->head_dim;
  p.n = shape->seq_len;
  p.block = block_size;
  p.scale = effective_scale(scale, shape->head_dim);
  p.kv_idx = kv_idx;
  p.kv_cnt = kv_cnt;
  p.q_orig = q_orig;
  p.k_orig = k_orig;
  p.out_rows = out_rows;
  p.status = status;
  p.causal = 0;
  return run_attention(p, nullptr, as_stream(stream));
}

int pbs_dense_causal_attention_fwd(const void* q, const void* k, const void* v, const pbs_shape* shape, double scale,
                                   void* out, void* stream) {
  if (int rc = check_shape(shape)) return rc;
  AttnParams p{};
  p.q = q;
  p.k = k;
  p.v = v;
  p.out = out;
  p.dtype = shape->dtype;
  p.hq = shape->num_q_heads;
  p.kv_heads = shape->num_kv_heads;
  p.d = shape->head_dim;
  p.n = shape->seq_len;
  p.block = 128;
  p.scale = effective_scale(scale, shape->head_dim);
  p.causal = 1;
  return run_attention(p, nullptr, as_stream(stream));
}

namespace {
struct CoverageLayout {
  size_t qp, kp, o, lse_s, lse_d, kv_idx, kv_cnt, total;
};
CoverageLayout coverage_plan(const pbs_shape* shape, int64_t block) {
  const int64_t n = shape->seq_len, d = shape->head_dim, hq = shape->num_q_heads, t = ceil_div(n, block);
  const size_t es = shape->dtype == PBS_DTYPE_BF16 ? 2 : 4;
  CoverageLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off += (bytes + 255) & ~(size_t)255;
    return at;
  };
  L.qp = take((size_t)hq * n * d * es);
  L.kp = take((size_t)hq * n * d * es);
  L.o = take((size_t)hq * n * d * es);
  L.lse_s = take((size_t)hq * n * 4);
  L.lse_d = take((size_t)hq * n * 4);
  L.kv_idx = take((size_t)hq * t * t * 4);
  L.kv_cnt = take((size_t)hq * t * 4);
  L.total = off + 256;
  return L;
}
}  // namespace

size_t pbs_coverage_workspace_size(const pbs_shape* shape, int64_t block_size) {
  if (check_shape(shape) || block_size <= 0) return 0;
  return coverage_plan(shape, block_size).total;
}

int pbs_attention_coverage(const void* q, const void* k, const pbs_shape* shape, int64_t block_size,
                           const uint8_t* mask, const int32_t* sigma, const int32_t* pi, double scale,
                           double* coverage, void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_shape(shape)) return rc;
  if (block_size <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "attention_coverage: block size must be >= 1");
  if (!mask || !coverage) return fail(PBS_ERR_CONFIG, "E_SHAPE", "attention_coverage: mask and coverage are required");
  const CoverageLayout L = coverage_plan(shape, block_size);
  if (workspace == nullptr || workspace_bytes < L.total)
    return fail(PBS_ERR_RESOURCE, "E_RESOURCE",
                "coverage workspace of " + std::to_string(workspace_bytes) + " bytes, need " + std::to_string(L.total));
  cudaStream_t st = as_stream(stream);
  char* ws = static_cast<char*>(workspace);
  const int hq = shape->num_q_heads, hkv = shape->num_kv_heads, d = shape->head_dim;
  const int64_t n = shape->seq_len, t = ceil_div(n, block_size);
  const int es = shape->dtype == PBS_DTYPE_BF16 ? 2 : 4;
  int32_t* kv_idx = reinterpret_cast<int32_t*>(ws + L.kv_idx);
  int32_t* kv_cnt = reinterpret_cast<int32_t*>(ws + L.kv_cnt);
  float* lse_s = reinterpret_cast<float*>(ws + L.lse_s);
  float* lse_d = reinterpret_cast<float*>(ws + L.lse_d);
  if (int rc = launch_mask_to_lists(mask, hq, t, kv_idx, kv_cnt, st)) return rc;
  // the permuted grid: Q' = sigma Q, K' = pi K (V is irrelevant to the mass: K' stands in)
  const void* qp = q;
  const void* kp = k;
  int kv_heads = hkv;
  if (sigma) {
    if (int rc = launch_apply_rows(sigma, q, hq, hq, n, d, es, ws + L.qp, st)) return rc;
    qp = ws + L.qp;
  }
  if (pi) {
    if (int rc = launch_apply_rows(pi, k, hkv, hq, n, d, es, ws + L.kp, st)) return rc;
    kp = ws + L.kp;
    kv_heads = hq;
  }
  AttnParams p{};
  p.q = qp;
  p.k = kp;
  p.v = kp;
  p.out = ws + L.o;
  p.dtype = shape->dtype;
  p.hq = hq;
  p.kv_heads = kv_heads;
  p.d = d;
  p.n = n;
  p.block = block_size;
  p.scale = effective_scale(scale, d);
  p.kv_idx = kv_idx;
  p.kv_cnt = kv_cnt;
  p.q_orig = sigma;
  p.k_orig = pi;
  p.out_rows = sigma;  // lse rows back in original order
  p.causal = (sigma == nullptr && pi == nullptr) ? 1 : 0;
  p.lse = lse_s;
  if (int rc = run_attention(p, nullptr, st)) return rc;
  // the true causal mass of every row (dense causal pass over the original order)
  AttnParams dp{};
  dp.q = q;
  dp.k = k;
  dp.v = k;
  dp.out = ws + L.o;
  dp.dtype = shape->dtype;
  dp.hq = hq;
  dp.kv_heads = hkv;
  dp.d = d;
  dp.n = n;
  dp.block = 128;
  dp.scale = effective_scale(scale, d);
  dp.causal = 1;
  dp.lse = lse_d;
  if (int rc = run_attention(dp, nullptr, st)) return rc;
  return launch_coverage_reduce(lse_s, lse_d, hq, n, coverage, st);
}

int pbs_check_status(const int32_t* status, int64_t num_blocks, void* stream) {
  int32_t h[2] = {0, 0};
  PBS_CUDA_CHECK(cudaMemcpyAsync(h, status, sizeof h, cudaMemcpyDeviceToHost, as_stream(stream)));
  PBS_CUDA_CHECK(cudaStreamSynchronize(as_stream(stream)));
  if (h[0]) {
    const int64_t qb = num_blocks > 0 ? h[1] % num_blocks : h[1];
    const int64_t head = num_blocks > 0 ? h[1] / num_blocks : 0;
    return fail(PBS_ERR_DEGENERATE, "E_DEGENERATE",
                "query block " + std::to_string(qb) + " (head " + std::to_string(head) +
                    ") has an empty softmax denominator (all keys masked)");
  }
  return PBS_OK;
}

}  // extern "C"

namespace pbs_b200 {
// Algorithm 1 enqueued on `stream` (no synchronisation); stage events go to tm.
// pi_given (key_permute only): pi of every head, computed beforehand (the host
// entry estimates all heads at once from the keys and the last query rows).
int pipeline_enqueue(const void* q, const void* k, const void* v, const pbs_shape* shape,
                     const pbs_pipeline_config* cfg, void* out, int32_t* sigma_out, int32_t* pi_out,
                     uint8_t* mask_out, void* workspace, size_t workspace_bytes, Timer& tm, void* stream,
                     const int32_t* pi_given, int64_t qb_begin, int64_t qb_end) {
  if (int rc = check_shape(shape)) return rc;
  if (int rc = check_cfg(cfg)) return rc;
  const Layout L = plan(shape, cfg);
  if (workspace_bytes < L.total || workspace == nullptr)
    return fail(PBS_ERR_RESOURCE, "E_RESOURCE",
                "workspace of " + std::to_string(workspace_bytes) + " bytes, need " + std::to_string(L.total));
  cudaStream_t st = as_stream(stream);
  char* ws = static_cast<char*>(workspace);
  auto at = [&](size_t off) { return static_cast<void*>(ws + off); };
  const int hq = shape->num_q_heads, hkv = shape->num_kv_heads, d = shape->head_dim, dt = shape->dtype;
  const int64_t n = shape->seq_len, b = cfg->block_size, s = cfg->segment_size, t = ceil_div(n, b);
  const int es = esize_of(dt);
  const float scale = effective_scale(cfg->scale, d);
  const int strategy = cfg->strategy;
  int32_t* status = static_cast<int32_t*>(at(L.status));
  int32_t* pi = pi_given ? const_cast<int32_t*>(pi_given) : pi_out ? pi_out : static_cast<int32_t*>(at(L.pi));
  int32_t* sigma = sigma_out ? sigma_out : static_cast<int32_t*>(at(L.sigma));
  uint8_t* mask = mask_out ? mask_out : static_cast<uint8_t*>(at(L.mask));
  int32_t* kv_idx = static_cast<int32_t*>(at(L.kv_idx));
  int32_t* kv_cnt = static_cast<int32_t*>(at(L.kv_cnt));
  double* row_cov = static_cast<double*>(at(L.row_cov));
  // status = {0, 0x7f7f7f7f}: memsets (not a host copy) keep the call capturable in a CUDA graph
  PBS_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  PBS_CUDA_CHECK(cudaMemsetAsync(status + 1, 0x7f, sizeof(int32_t), st));

  tm.mark();
  // ---- stage 1: estimate (pipeline.hpp:129-155)
  const void* kp = k;
  int kv_heads = hkv;
  if (pi_given && strategy != PBS_STRATEGY_KEY_PERMUTE)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "a precomputed pi is only taken under key_permute");
  if (pi_given) {
    // stage 1 already done by the caller
  } else if (uses_pi(strategy)) {
    float* scores = static_cast<float*>(at(L.scores));
    if (int rc = launch_importance(q, k, dt, hq, hkv, n, d, b, scale, scores, at(L.imp),
                                   importance_workspace_bytes(hq, n, b), st))
      return rc;
    if (int rc = launch_segmented_sort(scores, 0, hq, n, s, pi, static_cast<int32_t*>(at(L.pi_inv)), st)) return rc;
  } else if (pi_out) {
    if (int rc = launch_identity(pi_out, hq, n, st)) return rc;
  }
  if (strategy == PBS_STRATEGY_BOTH) {
    // keys first; sigma is computed against K' = pi K (pipeline.hpp:144-153)
    if (int rc = launch_apply_rows(pi, k, hkv, hq, n, d, es, at(L.kp), st)) return rc;
    kp = at(L.kp);
    kv_heads = hq;
  }
  if (uses_sigma(strategy)) {
    uint32_t* groups = static_cast<uint32_t*>(at(L.groups));
    if (int rc = launch_query_groups(q, kp, dt, hq, kv_heads, n, d, b, groups, at(L.qperm),
                                     query_perm_workspace_bytes(hq, n, d, b), st))
      return rc;
    if (int rc = launch_segmented_sort(groups, 1, hq, n, s, sigma, static_cast<int32_t*>(at(L.sigma_inv)), st))
      return rc;
  } else if (sigma_out) {
    if (int rc = launch_identity(sigma_out, hq, n, st)) return rc;
  }
  tm.mark();
  // ---- stage 2: permute (pipeline.hpp:157-165)
  const void* qp = q;
  const void* vp = v;
  if (uses_sigma(strategy)) {
    if (int rc = launch_apply_rows(sigma, q, hq, hq, n, d, es, at(L.qp), st)) return rc;
    qp = at(L.qp);
  }
  if (strategy == PBS_STRATEGY_KEY_PERMUTE) {
    if (int rc = launch_apply_rows(pi, k, hkv, hq, n, d, es, at(L.kp), st)) return rc;
    kp = at(L.kp);
    kv_heads = hq;
  }
  if (uses_pi(strategy)) {
    if (int rc = launch_apply_rows(pi, v, hkv, hq, n, d, es, at(L.vp), st)) return rc;
    vp = at(L.vp);
  }
  tm.mark();
  // ---- stage 3: select (pipeline.hpp:167-171)
  float* qbar = static_cast<float*>(at(L.qbar));
  float* kbar = static_cast<float*>(at(L.kbar));
  if (int rc = launch_pool(qp, dt, hq, hq, nullptr, n, d, b, qbar, st)) return rc;
  if (int rc = launch_pool(kp, dt, kv_heads, hq, nullptr, n, d, b, kbar, st)) return rc;
  if (int rc = launch_score_select(qbar, kbar, static_cast<float*>(at(L.blog)), hq, t, d, b, s, scale, cfg->tau,
                                   cfg->forced_first_block, cfg->forced_diagonal_band, 1, nullptr, mask, kv_idx,
                                   kv_cnt, row_cov, st, cfg->top_k))
    return rc;
  tm.mark();
  // ---- stage 4: attention with the original-position element mask (173-176)
  AttnParams p{};
  p.q = qp;
  p.k = kp;
  p.v = vp;
  p.out = out;
  p.dtype = dt;
  p.hq = hq;
  p.kv_heads = kv_heads;
  p.d = d;
  p.n = n;
  p.block = b;
  p.scale = scale;
  p.kv_idx = kv_idx;
  p.kv_cnt = kv_cnt;
  p.q_orig = uses_sigma(strategy) ? sigma : nullptr;
  p.k_orig = uses_pi(strategy) ? pi : nullptr;
  // ---- stage 5 fused: output row i of the permuted grid goes to row sigma[i]
  p.out_rows = uses_sigma(strategy) ? sigma : nullptr;
  p.status = status;
  // ElementMask(sigma, pi) with both identities is exactly the causal mask
  p.causal = (p.q_orig == nullptr && p.k_orig == nullptr) ? 1 : 0;
  p.qb_begin = qb_begin;
  p.qb_end = qb_end;
  if (int rc = run_attention(p, at(L.sched), st)) return rc;
  tm.mark();
  tm.mark();  // un-permute is fused into the attention epilogue
  return PBS_OK;
}

// The per-row counters the report needs, copied to host memory on `st`
// (asynchronous; complete once `st` reaches this point).
int report_fetch(const pbs_shape* shape, const pbs_pipeline_config* cfg, const void* workspace, int32_t* cnt,
                 double* cov, int32_t* hs, cudaStream_t st) {
  const Layout L = plan(shape, cfg);
  const char* ws = static_cast<const char*>(workspace);
  const int64_t t = ceil_div(shape->seq_len, cfg->block_size), hq = shape->num_q_heads;
  PBS_CUDA_CHECK(cudaMemcpyAsync(cnt, ws + L.kv_cnt, (size_t)hq * t * 4, cudaMemcpyDeviceToHost, st));
  PBS_CUDA_CHECK(cudaMemcpyAsync(cov, ws + L.row_cov, (size_t)hq * t * 8, cudaMemcpyDeviceToHost, st));
  PBS_CUDA_CHECK(cudaMemcpyAsync(hs, ws + L.status, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  return PBS_OK;
}

// ---- report (pipeline.hpp:182-191) from the fetched counters
int report_build(const pbs_shape* shape, const pbs_pipeline_config* cfg, const int32_t* cnt, const double* cov,
                 const int32_t* hs, const Timer& tm, pbs_report* report, int64_t qb_begin, int64_t qb_end) {
  const int hq = shape->num_q_heads;
  const int64_t b = cfg->block_size, s = cfg->segment_size, t = ceil_div(shape->seq_len, b);
  const int64_t lo = qb_begin, hi = qb_end > 0 ? std::min<int64_t>(qb_end, t) : t;
  if (hs[0]) {
    return fail(PBS_ERR_DEGENERATE, "E_DEGENERATE",
                "query block " + std::to_string(hs[1] % t) + " (head " + std::to_string(hs[1] / t) +
                    ") has an empty softmax denominator (all keys masked)");
  }
  memset(report, 0, sizeof *report);
  int64_t adm = 0;
  for (int64_t i = lo; i < hi; ++i) adm += admissible_prefix(i, t, b, s);
  double dens = 0.0, covsum = 0.0;
  for (int h = 0; h < hq; ++h) {
    int64_t sel = 0;
    double c = 0.0;
    for (int64_t i = lo; i < hi; ++i) {
      sel += cnt[(size_t)h * t + i];
      c += cov[(size_t)h * t + i];
    }
    report->selected_blocks += sel;
    dens += (double)sel / (double)(t * t);
    covsum += c / (double)t;
  }
  report->block_density = dens / hq;
  report->pooled_score_coverage = covsum / hq;
  report->causal_density_baseline = (double)(t + 1) / (double)(2 * t);
  report->total_admissible_blocks = adm * hq;
  report->estimate_us = tm.us(0);
  report->permute_us = tm.us(1);
  report->select_us = tm.us(2);
  report->attention_us = tm.us(3);
  report->unpermute_us = tm.us(4);
  return PBS_OK;
}
}  // namespace pbs_b200

extern "C" {

int pbs_attention(const void* q, const void* k, const void* v, const pbs_shape* shape, const pbs_pipeline_config* cfg,
                  void* out, int32_t* sigma_out, int32_t* pi_out, uint8_t* mask_out, void* workspace,
                  size_t workspace_bytes, pbs_report* report, void* stream) {
  cudaStream_t st = as_stream(stream);
  Timer tm(report != nullptr, st);
  if (int rc = pipeline_enqueue(q, k, v, shape, cfg, out, sigma_out, pi_out, mask_out, workspace, workspace_bytes,
                                tm, stream))
    return rc;
  if (!report) return PBS_OK;
  const int64_t t = ceil_div(shape->seq_len, cfg->block_size), hq = shape->num_q_heads;
  std::vector<int32_t> cnt((size_t)hq * t);
  std::vector<double> cov((size_t)hq * t);
  int32_t hs[2];
  if (int rc = report_fetch(shape, cfg, workspace, cnt.data(), cov.data(), hs, st)) return rc;
  PBS_CUDA_CHECK(cudaStreamSynchronize(st));
  return report_build(shape, cfg, cnt.data(), cov.data(), hs, tm, report);
}

// ---- host-buffer entry: library-owned device arena, pipelined by KV group ------
//
// The host call streams the problem through the GPU one KV group (a KV head
// and its Hq/Hkv query heads) at a time, double-buffered on three streams:
// H2D of group g+1 and D2H of group g-1 overlap the compute of group g.  Heads
// share nothing, so the result is identical to one whole call.
namespace {
// One arena = device memory for two group slots (+ the estimate-first
// buffers), three streams and their events, on one device.  Calls check an
// arena out of a per-process pool and return it when they finish, so
// concurrent host callers (one per thread, like pbs_main.cpp:99-122's head
// fan-out) each get their own arena and never serialise on each other; a
// sequential caller reuses the same arena call after call.
struct Arena {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = -1;
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  cudaEvent_t ev_rep[2] = {nullptr, nullptr};
  cudaEvent_t ev_comp[2] = {nullptr, nullptr};  // per slot: the group's compute is done (its inputs are free)
  cudaEvent_t ev_q0a = nullptr;  // group 0's V and the first half of its Q are on the device
  std::vector<cudaEvent_t> ev_k;  // per KV head: its keys are on the device (estimate-first path)
  // per slot: stage timers and pinned copies of the report counters, so a
  // group's report is built while the next group computes
  Timer* timer[2] = {nullptr, nullptr};
  char* pinned = nullptr;
  size_t pinned_bytes = 0;
};

struct ArenaPool {
  std::mutex mu;
  std::vector<Arena*> idle;
};
ArenaPool g_pool;

// an idle arena of the current device (streams and events are per device), or a new one
Arena* arena_acquire(int dev) {
  {
    std::lock_guard<std::mutex> lk(g_pool.mu);
    for (size_t i = 0; i < g_pool.idle.size(); ++i) {
      if (g_pool.idle[i]->device != dev) continue;
      Arena* a = g_pool.idle[i];
      g_pool.idle.erase(g_pool.idle.begin() + (long)i);
      return a;
    }
  }
  Arena* a = new Arena();
  a->device = dev;
  return a;
}

void arena_release(Arena* a) {
  std::lock_guard<std::mutex> lk(g_pool.mu);
  g_pool.idle.push_back(a);
}

struct ArenaLease {
  Arena* a;
  explicit ArenaLease(int dev) : a(arena_acquire(dev)) {}
  ~ArenaLease() {
    // an early error return may leave copies in flight on the arena's streams
    for (auto s : a->st)
      if (s) cudaStreamSynchronize(s);
    arena_release(a);
  }
};

int arena_streams(Arena& A) {
  if (A.st[0]) return PBS_OK;
  for (auto& x : A.st) PBS_CUDA_CHECK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    PBS_CUDA_CHECK(cudaEventCreateWithFlags(&A.ev_in[i], cudaEventDisableTiming));
    PBS_CUDA_CHECK(cudaEventCreateWithFlags(&A.ev_done[i], cudaEventDisableTiming));
    PBS_CUDA_CHECK(cudaEventCreateWithFlags(&A.ev_out[i], cudaEventDisableTiming));
    PBS_CUDA_CHECK(cudaEventCreateWithFlags(&A.ev_rep[i], cudaEventDisableTiming));
    PBS_CUDA_CHECK(cudaEventCreateWithFlags(&A.ev_comp[i], cudaEventDisableTiming));
    A.timer[i] = new Timer(true, A.st[1]);
  }
  PBS_CUDA_CHECK(cudaEventCreateWithFlags(&A.ev_q0a, cudaEventDisableTiming));
  return PBS_OK;
}
}  // namespace

namespace {
// debug (PBS_HOST_TRACE=1): the host entry's timeline, CUDA events on its three
// streams, printed to stderr as ms after the first event once the call is done
struct HostTrace {
  bool on = getenv("PBS_HOST_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void mark(const std::string& name, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, st);
    ev.emplace_back(name, e);
  }
  ~HostTrace() {
    if (!on || ev.empty()) return;
    cudaDeviceSynchronize();
    for (auto& x : ev) {
      float ms = 0.0f;
      const cudaError_t e = cudaEventElapsedTime(&ms, ev.front().second, x.second);
      fprintf(stderr, "pbs_host_trace %8.3f ms  %s%s\n", ms, x.first.c_str(),
              e == cudaSuccess ? "" : (std::string(" (") + cudaGetErrorString(e) + ")").c_str());
    }
    for (auto& x : ev) cudaEventDestroy(x.second);
  }
};
}  // namespace

int pbs_attention_host(const void* q, const void* k, const void* v, const pbs_shape* shape,
                       const pbs_pipeline_config* cfg, void* out, int32_t* sigma, int32_t* pi, uint8_t* mask,
                       pbs_report* report) {
  if (int rc = check_shape(shape)) return rc;
  if (int rc = check_cfg(cfg)) return rc;
  const int64_t n = shape->seq_len, hq = shape->num_q_heads, hkv = shape->num_kv_heads, d = shape->head_dim;
  const int64_t g = hq / hkv;  // query heads per chunk (one KV head)
  const int64_t t = ceil_div(n, cfg->block_size);
  const size_t es = esize_of(shape->dtype);
  pbs_shape cs = *shape;  // chunk shape
  cs.num_q_heads = (int32_t)g;
  cs.num_kv_heads = 1;
  const size_t qb = (size_t)g * n * d * es, kvb = (size_t)n * d * es;
  const size_t pb = (size_t)g * n * 4, mb = (size_t)g * t * t;
  const size_t ws = pbs_workspace_size(&cs, cfg);
  const size_t slot = al(qb) * 2 + al(kvb) * 2 + al(pb) * 2 + al(mb) + al(ws);
  const int nslots = hkv > 1 ? 2 : 1;
  // key_permute over several KV groups: estimate every head up front from K and
  // the last `take` query rows (stage 1 reads nothing else), so the per-group
  // pipelines skip it.  One all-heads estimate fills the GPU; per-group ones
  // (4 heads) leave its sequential denominator chains on a few SMs.
  const bool est_first = cfg->strategy == PBS_STRATEGY_KEY_PERMUTE && hkv > 1;
  const int64_t take = std::min<int64_t>(cfg->block_size, n);
  const size_t kall_b = (size_t)hkv * kvb, qtail_b = (size_t)hq * take * d * es;
  const size_t imp_b = importance_workspace_bytes((int)hq, n, cfg->block_size);
  const size_t est_bytes = est_first ? al(kall_b) + al(qtail_b) + al(imp_b) + 3 * al((size_t)hq * n * 4) : 0;
  int dev = 0;
  PBS_CUDA_CHECK(cudaGetDevice(&dev));
  ArenaLease lease(dev);
  Arena& A = *lease.a;
  if (int rc = arena_streams(A)) return rc;
  if (A.bytes < slot * nslots + est_bytes) {
    if (A.ptr) cudaFree(A.ptr);
    A.ptr = nullptr;
    A.bytes = 0;
    PBS_CUDA_CHECK(cudaMalloc(&A.ptr, slot * nslots + est_bytes));
    A.bytes = slot * nslots + est_bytes;
  }
  struct Slot {
    char *q, *k, *v, *out, *ws;
    int32_t *sig, *pi;
    uint8_t* mask;
  } sl[2];
  for (int i = 0; i < nslots; ++i) {
    char* p = static_cast<char*>(A.ptr) + (size_t)i * slot;
    auto take = [&](size_t bytes) {
      char* r = p;
      p += al(bytes);
      return r;
    };
    sl[i].q = take(qb);
    sl[i].k = take(kvb);
    sl[i].v = take(kvb);
    sl[i].out = take(qb);
    sl[i].sig = reinterpret_cast<int32_t*>(take(pb));
    sl[i].pi = reinterpret_cast<int32_t*>(take(pb));
    sl[i].mask = reinterpret_cast<uint8_t*>(take(mb));
    sl[i].ws = take(ws);
  }
  cudaStream_t s_in = A.st[0], s_run = A.st[1], s_out = A.st[2];
  HostTrace tr;
  tr.mark("start", s_in);
  const char* hq_ = static_cast<const char*>(q);
  const char* hk_ = static_cast<const char*>(k);
  const char* hv_ = static_cast<const char*>(v);
  char* k_all = nullptr;
  char* q_tail = nullptr;
  char* imp = nullptr;
  float* scores = nullptr;
  int32_t* pi_all = nullptr;
  int32_t* pi_inv = nullptr;
  Timer est_tm(report != nullptr, s_run);
  const float sc = effective_scale(cfg->scale, (int)d);
  if (est_first) {
    char* p = static_cast<char*>(A.ptr) + (size_t)nslots * slot;
    auto take_b = [&](size_t bytes) {
      char* r = p;
      p += al(bytes);
      return r;
    };
    k_all = take_b(kall_b);
    q_tail = take_b(qtail_b);
    imp = take_b(imp_b);
    scores = reinterpret_cast<float*>(take_b((size_t)hq * n * 4));
    pi_all = reinterpret_cast<int32_t*>(take_b((size_t)hq * n * 4));
    pi_inv = reinterpret_cast<int32_t*>(take_b((size_t)hq * n * 4));
    while (A.ev_k.size() < (size_t)hkv) {
      cudaEvent_t e;
      PBS_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      A.ev_k.push_back(e);
    }
  }
  // estimate of the query heads of KV groups [c0, c1) (stage 1 reads only K and
  // the last `take` query rows): logits per group as its keys land, then the
  // exps / denominators / scores and the segmented sort for those heads
  auto estimate_groups = [&](int64_t c0, int64_t c1) -> int {
    for (int64_t c = c0; c < c1; ++c) {
      PBS_CUDA_CHECK(cudaStreamWaitEvent(s_run, A.ev_k[c], 0));
      if (c == c0) est_tm.mark();
      if (int rc = launch_importance_logits(q_tail, k_all, shape->dtype, (int)hq, (int)hkv, (int)(c * g), (int)g, n,
                                            (int)d, cfg->block_size, sc, imp, imp_b, s_run, take))
        return rc;
    }
    const int h0 = (int)(c0 * g), nh = (int)((c1 - c0) * g);
    if (int rc = launch_importance_finish((int)hq, h0, nh, n, cfg->block_size, scores, imp, imp_b, s_run)) return rc;
    if (int rc = launch_segmented_sort(scores + (size_t)h0 * n, 0, nh, n, cfg->segment_size, pi_all + (size_t)h0 * n,
                                       pi_inv + (size_t)h0 * n, s_run))
      return rc;
    est_tm.mark();
    tr.mark("run: estimate groups " + std::to_string(c0) + ".." + std::to_string(c1 - 1) + " done", s_run);
    return PBS_OK;
  };
  char* ho_ = static_cast<char*>(out);
  pbs_report total{};
  double dens = 0.0, cov = 0.0;
  // pinned report counters per chunk parity: kv_cnt (int32), row_cov (double), status
  const size_t rep_bytes = al((size_t)g * t * 4) + al((size_t)g * t * 8) + 256;
  if (report && A.pinned_bytes < rep_bytes * 2) {
    if (A.pinned) cudaFreeHost(A.pinned);
    A.pinned = nullptr;
    A.pinned_bytes = 0;
    PBS_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&A.pinned), rep_bytes * 2, cudaHostAllocDefault));
    A.pinned_bytes = rep_bytes * 2;
  }
  auto rep_cnt = [&](int i) { return reinterpret_cast<int32_t*>(A.pinned + i * rep_bytes); };
  auto rep_cov = [&](int i) { return reinterpret_cast<double*>(A.pinned + i * rep_bytes + al((size_t)g * t * 4)); };
  auto rep_hs = [&](int i) {
    return reinterpret_cast<int32_t*>(A.pinned + i * rep_bytes + al((size_t)g * t * 4) + al((size_t)g * t * 8));
  };
  // Work chunks: one per KV group, except that the FIRST and the LAST group
  // (key_permute, pi precomputed) run in two head halves: the first half of
  // group 0 starts once its V and half of its Q are in (the fill before the
  // first kernel is half a group's queries), and the output of the last group's
  // first half goes back to the host while the second computes (the drain after
  // the last kernel is half a group).  Single-head slices cost more in
  // per-launch tails than they save: measured 1.85 ms per 1-head slice vs 1.26
  // per head.
  struct Chunk {
    int64_t c, a, b;  // KV group c, its query heads [a, b) (local to the group)
  };
  std::vector<Chunk> chunks;
  const bool split0 = est_first && g >= 2;
  for (int64_t c = 0; c < hkv; ++c) {
    const int64_t parts = (est_first && (c == hkv - 1 || c == 0)) ? std::min<int64_t>(g, 2) : 1;
    for (int64_t j = 0; j < parts; ++j) chunks.push_back(Chunk{c, j * g / parts, (j + 1) * g / parts});
  }
  // fold the report of chunk kk (its counters were fetched on s_run) into the total
  auto fold = [&](size_t kk) -> int {
    const int i = (int)(kk % 2);
    const Chunk& ch = chunks[kk];
    pbs_shape cs2 = cs;
    cs2.num_q_heads = (int32_t)(ch.b - ch.a);
    PBS_CUDA_CHECK(cudaEventSynchronize(A.ev_rep[i]));
    pbs_report r{};
    if (int rc = report_build(&cs2, cfg, rep_cnt(i), rep_cov(i), rep_hs(i), *A.timer[i], &r)) {
      if (rc == PBS_ERR_DEGENERATE) {  // name the head in the whole problem
        const int32_t hfull = (int32_t)(ch.c * g + ch.a + rep_hs(i)[1] / t);
        return fail(PBS_ERR_DEGENERATE, "E_DEGENERATE",
                    "query block " + std::to_string(rep_hs(i)[1] % t) + " (head " + std::to_string(hfull) +
                        ") has an empty softmax denominator (all keys masked)");
      }
      return rc;
    }
    total.selected_blocks += r.selected_blocks;
    total.total_admissible_blocks += r.total_admissible_blocks;
    dens += r.block_density * (double)(ch.b - ch.a);
    cov += r.pooled_score_coverage * (double)(ch.b - ch.a);
    total.causal_density_baseline = r.causal_density_baseline;
    total.estimate_us += r.estimate_us;
    total.permute_us += r.permute_us;
    total.select_us += r.select_us;
    total.attention_us += r.attention_us;
    total.unpermute_us += r.unpermute_us;
    return PBS_OK;
  };
  auto copy_in = [&](int64_t c) -> int {
    Slot& S = sl[c % nslots];
    // the slot's Q / K / V buffers are free once group c - nslots has been
    // COMPUTED (its output buffer, written again by group c, is guarded on
    // s_run by ev_out below), so the inputs of the next group stream in while
    // the previous output is still being copied out
    if (c >= nslots) PBS_CUDA_CHECK(cudaStreamWaitEvent(s_in, A.ev_comp[c % nslots], 0));
    if (c == 0 && split0) {  // V, then Q in the two head halves of the first chunks
      const size_t qh = (size_t)(g / 2) * n * d * es;
      PBS_CUDA_CHECK(cudaMemcpyAsync(S.v, hv_, kvb, cudaMemcpyHostToDevice, s_in));
      PBS_CUDA_CHECK(cudaMemcpyAsync(S.q, hq_, qh, cudaMemcpyHostToDevice, s_in));
      PBS_CUDA_CHECK(cudaEventRecord(A.ev_q0a, s_in));
      PBS_CUDA_CHECK(cudaMemcpyAsync(S.q + qh, hq_ + qh, qb - qh, cudaMemcpyHostToDevice, s_in));
      PBS_CUDA_CHECK(cudaEventRecord(A.ev_in[0], s_in));
      tr.mark("in: Q,V of group 0 landed", s_in);
      return PBS_OK;
    }
    PBS_CUDA_CHECK(cudaMemcpyAsync(S.q, hq_ + (size_t)c * qb, qb, cudaMemcpyHostToDevice, s_in));
    if (!est_first) PBS_CUDA_CHECK(cudaMemcpyAsync(S.k, hk_ + (size_t)c * kvb, kvb, cudaMemcpyHostToDevice, s_in));
    PBS_CUDA_CHECK(cudaMemcpyAsync(S.v, hv_ + (size_t)c * kvb, kvb, cudaMemcpyHostToDevice, s_in));
    PBS_CUDA_CHECK(cudaEventRecord(A.ev_in[c % nslots], s_in));
    tr.mark("in: Q,V of group " + std::to_string(c) + " landed", s_in);
    return PBS_OK;
  };
  if (est_first) {
    // Fill order: the last `take` rows of every query head, K of group 0, then
    // group 0's Q and V, then the other groups' K.  Group 0 is estimated alone
    // and starts as soon as its own inputs are in; the other groups' estimate
    // runs after it, while their K (and group 1's Q, V) stream in.
    PBS_CUDA_CHECK(cudaMemcpy2DAsync(q_tail, (size_t)take * d * es, hq_ + (size_t)(n - take) * d * es,
                                     (size_t)n * d * es, (size_t)take * d * es, (size_t)hq, cudaMemcpyHostToDevice,
                                     s_in));
    PBS_CUDA_CHECK(cudaMemcpyAsync(k_all, hk_, kvb, cudaMemcpyHostToDevice, s_in));
    PBS_CUDA_CHECK(cudaEventRecord(A.ev_k[0], s_in));
    if (int rc = copy_in(0)) return rc;
    for (int64_t c = 1; c < hkv; ++c) {
      PBS_CUDA_CHECK(cudaMemcpyAsync(k_all + (size_t)c * kvb, hk_ + (size_t)c * kvb, kvb, cudaMemcpyHostToDevice, s_in));
      PBS_CUDA_CHECK(cudaEventRecord(A.ev_k[c], s_in));
    }
    tr.mark("in: all K landed", s_in);
    if (int rc = estimate_groups(0, 1)) return rc;
  } else {
    if (int rc = copy_in(0)) return rc;
  }
  for (size_t kk = 0; kk < chunks.size(); ++kk) {
    const Chunk& ch = chunks[kk];
    const int64_t c = ch.c;
    const int i = (int)(c % nslots);
    const int ri = (int)(kk % 2);
    Slot& S = sl[i];
    const bool first_of_group = ch.a == 0;
    if (first_of_group) {
      if (c + 1 < hkv && nslots > 1)
        if (int rc = copy_in(c + 1)) return rc;
      if (est_first && c == 1)
        if (int rc = estimate_groups(1, hkv)) return rc;
      if (c >= nslots) PBS_CUDA_CHECK(cudaStreamWaitEvent(s_run, A.ev_out[i], 0));  // S.out copied out
    }
    // the chunk's inputs: all of the group's, or for group 0's first half its V and half of its Q
    PBS_CUDA_CHECK(cudaStreamWaitEvent(s_run, (c == 0 && split0 && ch.a == 0) ? A.ev_q0a : A.ev_in[i], 0));
    pbs_shape cs2 = cs;
    cs2.num_q_heads = (int32_t)(ch.b - ch.a);
    const size_t qoff = (size_t)ch.a * n * d * es, poff = (size_t)ch.a * n, moff = (size_t)ch.a * t * t;
    const size_t qbytes = (size_t)(ch.b - ch.a) * n * d * es, pbytes = (size_t)(ch.b - ch.a) * n * 4,
                 mbytes = (size_t)(ch.b - ch.a) * t * t;
    Timer& tm = *A.timer[ri];
    tm.restart(s_run);
    tm.on = report != nullptr;
    const int32_t* pi_c = est_first ? pi_all + (size_t)c * g * n + poff : nullptr;
    if (int rc = pipeline_enqueue(S.q + qoff, est_first ? k_all + (size_t)c * kvb : S.k, S.v, &cs2, cfg, S.out + qoff,
                                  sigma ? S.sig + poff : nullptr, (pi && !est_first) ? S.pi + poff : nullptr,
                                  mask ? S.mask + moff : nullptr, S.ws, ws, tm, s_run, pi_c))
      return rc;
    if (report) {
      if (int rc = report_fetch(&cs2, cfg, S.ws, rep_cnt(ri), rep_cov(ri), rep_hs(ri), s_run)) return rc;
      PBS_CUDA_CHECK(cudaEventRecord(A.ev_rep[ri], s_run));
    }
    PBS_CUDA_CHECK(cudaEventRecord(A.ev_done[ri], s_run));
    if (ch.b == g) PBS_CUDA_CHECK(cudaEventRecord(A.ev_comp[i], s_run));
    tr.mark("run: chunk " + std::to_string(kk) + " (group " + std::to_string(c) + " heads " + std::to_string(ch.a) +
                ".." + std::to_string(ch.b - 1) + ") computed",
            s_run);
    PBS_CUDA_CHECK(cudaStreamWaitEvent(s_out, A.ev_done[ri], 0));
    const size_t hoff = (size_t)c * g + ch.a;  // first query head of the chunk
    PBS_CUDA_CHECK(cudaMemcpyAsync(ho_ + hoff * n * d * es, S.out + qoff, qbytes, cudaMemcpyDeviceToHost, s_out));
    if (sigma)
      PBS_CUDA_CHECK(cudaMemcpyAsync(sigma + hoff * n, S.sig + poff, pbytes, cudaMemcpyDeviceToHost, s_out));
    if (pi)
      PBS_CUDA_CHECK(cudaMemcpyAsync(pi + hoff * n, est_first ? pi_c : S.pi + poff, pbytes, cudaMemcpyDeviceToHost,
                                     s_out));
    if (mask) PBS_CUDA_CHECK(cudaMemcpyAsync(mask + hoff * t * t, S.mask + moff, mbytes, cudaMemcpyDeviceToHost, s_out));
    PBS_CUDA_CHECK(cudaEventRecord(A.ev_out[i], s_out));
    tr.mark("out: chunk " + std::to_string(kk) + " copied out", s_out);
    // the previous chunk's report, while this one computes (its counters are
    // overwritten only two chunks later, after this fold)
    if (report && kk > 0)
      if (int rc = fold(kk - 1)) return rc;
    const bool last_of_group = ch.b == g;
    if (nslots == 1 && last_of_group && c + 1 < hkv) {
      PBS_CUDA_CHECK(cudaStreamSynchronize(s_out));
      if (int rc = copy_in(c + 1)) return rc;
    }
  }
  if (report && !chunks.empty())
    if (int rc = fold(chunks.size() - 1)) return rc;
  if (report && est_first) {  // events complete: every fold synchronised later work
    total.estimate_us += est_tm.us(0);
    if (hkv > 1) total.estimate_us += est_tm.us(2);
  }
  PBS_CUDA_CHECK(cudaStreamSynchronize(s_out));
  total.block_density = dens / (double)hq;
  total.pooled_score_coverage = cov / (double)hq;
  if (report) *report = total;
  return PBS_OK;
}

// ---- device memory for C-ABI callers without the CUDA runtime (FFI bindings,
// the pbs:: drop-in header); the hot calls themselves never allocate
int pbs_malloc(size_t bytes, void** ptr) {
  if (!ptr) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null pointer");
  *ptr = nullptr;
  if (bytes == 0) return PBS_OK;
  const cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaErrorMemoryAllocation)
    return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "device allocation of " + std::to_string(bytes) + " bytes failed");
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return PBS_OK;
}

int pbs_free(void* ptr) {
  if (ptr) PBS_CUDA_CHECK(cudaFree(ptr));
  return PBS_OK;
}

int pbs_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream) {
  if (bytes == 0) return PBS_OK;
  const cudaMemcpyKind k = kind == PBS_COPY_H2D ? cudaMemcpyHostToDevice
                           : kind == PBS_COPY_D2H ? cudaMemcpyDeviceToHost
                                                  : cudaMemcpyDeviceToDevice;
  PBS_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, k, as_stream(stream)));
  return PBS_OK;
}

int pbs_stream_synchronize(void* stream) {
  PBS_CUDA_CHECK(cudaStreamSynchronize(as_stream(stream)));
  return PBS_OK;
}

int pbs_debug_expf(const float* x, float* y, int64_t n, void* stream) {
  return launch_debug_expf(x, y, n, as_stream(stream));
}

}  // extern "C"
