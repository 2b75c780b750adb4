// dist.cu -- head-parallel multi-GPU PBS-Attn behind the C ABI.
//
// The reference's only parallelism is the per-head fan-out of its CLI
// (tools/pbs_main.cpp:99-122): heads share nothing.  Here one
// process per GPU owns a contiguous range of (query head, query-block pair)
// work units, cut so that every rank gets the same causal work; whole heads
// when the head count divides evenly (Llama: 32 q heads on 1/2/4/8 GPUs), a
// cut inside a head otherwise (Qwen: 28 q heads on 8 GPUs = 3.5 heads each),
// instead of the 4 + 3 head split that caps efficiency at 87.5%.  A rank
// needs only the K/V heads of its query heads.  Because heads and units are
// assigned in head-major order, each rank's output rows are one contiguous
// byte range of the [Hq, N, d] output, so the single exchange is an
// all-gather-v: one in-place ncclBroadcast per rank inside one NCCL group,
// straight into the full output buffer (no staging, no other collective).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): the library loads
// and runs single-GPU without it, and the multi-GPU entries fail loudly with
// E_RESOURCE when it is missing.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "pipeline.h"

namespace pbs_b200 {
namespace {

// ---- work model and shard plan -------------------------------------------------
// Unit = (head h, pair p): the query blocks of one pair of 128-row tiles (the
// attention kernel's item): blocks 2p, 2p + 1 at B = 128, 4p .. 4p + 3 at
// B = 64 (two blocks per tile), 2p, 2p + 1 for other block sizes.  Weight = the
// causal key blocks its query blocks visit, qb + 1 each: the PBS selection
// keeps a similar fraction of every row, so causal work is the balance proxy.
struct Units {
  int64_t t, per, pairs, head_w;
  explicit Units(int64_t n, int64_t b) {
    t = ceil_div(n, b);
    per = b == 64 ? 4 : 2;
    pairs = ceil_div(t, per);
    head_w = before(pairs);
  }
  // work of pairs [0, p) of one head: sum over query blocks qb < per p of (qb + 1)
  int64_t before(int64_t p) const {
    const int64_t m = std::min<int64_t>(per * p, t);
    return m * (m + 1) / 2;
  }
  // first unit whose preceding work (global, head-major) is >= target
  void boundary(int64_t target, int64_t hq, int64_t& h, int64_t& p) const {
    if (head_w == 0) {
      h = hq;
      p = 0;
      return;
    }
    h = target / head_w;
    int64_t rem = target - h * head_w;
    if (h >= hq) {
      h = hq;
      p = 0;
      return;
    }
    int64_t lo = 0, hi = pairs;  // smallest p with before(p) >= rem
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (before(mid) >= rem) hi = mid;
      else lo = mid + 1;
    }
    p = lo;
    if (p == pairs) {  // rem beyond this head's last pair start: next head
      ++h;
      p = 0;
    }
  }
};

int shard_plan(const pbs_shape* g, int64_t block, int32_t world, int32_t rank, pbs_shard* s) {
  if (int rc = check_shape(g)) return rc;
  if (block <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "block size must be >= 1");
  if (world <= 0 || rank < 0 || rank >= world) return fail(PBS_ERR_CONFIG, "E_CONFIG", "rank outside [0, world_size)");
  const Units u(g->seq_len, block);
  const int64_t hq = g->num_q_heads, grp = hq / g->num_kv_heads;
  const int64_t total = u.head_w * hq;
  int64_t h0, p0, h1, p1;
  u.boundary(total / world * rank + (total % world) * rank / world, hq, h0, p0);
  u.boundary(total / world * (rank + 1) + (total % world) * (rank + 1) / world, hq, h1, p1);
  memset(s, 0, sizeof *s);
  // [h0:p0, h1:p1) in head-major unit order -> heads [head_begin, head_end),
  // the first from block qb_begin, the last up to block qb_end
  s->head_begin = (int32_t)h0;
  s->qb_begin = u.per * p0;
  if (p1 == 0) {
    s->head_end = (int32_t)h1;
    s->qb_end = u.t;
  } else {
    s->head_end = (int32_t)(h1 + 1);
    s->qb_end = u.per * p1;
  }
  if (h0 >= hq || (h0 == h1 && p0 == p1)) {  // no work for this rank
    s->head_begin = s->head_end = (int32_t)std::min<int64_t>(h0, hq);
    s->qb_begin = s->qb_end = 0;
    s->kv_begin = s->kv_end = s->head_begin / (int32_t)grp;
    s->out_row_begin = s->out_rows = 0;
    return PBS_OK;
  }
  s->kv_begin = (int32_t)(s->head_begin / grp);
  s->kv_end = (int32_t)((s->head_end - 1) / grp + 1);
  const int64_t n = g->seq_len;
  s->out_row_begin = (int64_t)s->head_begin * n + s->qb_begin * block;
  const int64_t end = (int64_t)(s->head_end - 1) * n + std::min<int64_t>(s->qb_end * block, n);
  s->out_rows = end - s->out_row_begin;
  return PBS_OK;
}

// A run: consecutive query heads of the shard with one query-block range and
// whole-group K/V (one KV head, or several whole GQA groups), i.e. one
// pipeline_enqueue over a [hq_run, N, d] slice.
struct Run {
  int32_t h0, h1;        // global query heads [h0, h1)
  int32_t kv0, kv1;      // global KV heads [kv0, kv1)
  int64_t qb0, qb1;      // query blocks [qb0, qb1) (0, t: all)
};

std::vector<Run> runs_of(const pbs_shape* g, const pbs_shard& s, int64_t t) {
  const int32_t grp = g->num_q_heads / g->num_kv_heads;
  std::vector<Run> per_kv;  // maximal runs of one KV head and one query-block range
  for (int32_t h = s.head_begin; h < s.head_end; ++h) {
    const int64_t qb0 = (h == s.head_begin) ? s.qb_begin : 0;
    const int64_t qb1 = (h == s.head_end - 1) ? s.qb_end : t;
    const int32_t kv = h / grp;
    if (!per_kv.empty()) {
      Run& r = per_kv.back();
      if (r.qb0 == qb0 && r.qb1 == qb1 && r.kv0 == kv) {
        r.h1 = h + 1;
        continue;
      }
    }
    per_kv.push_back(Run{h, h + 1, kv, kv + 1, qb0, qb1});
  }
  // whole GQA groups with full ranges merge into one pipeline call
  auto whole = [&](const Run& r) { return r.h0 == r.kv0 * grp && r.h1 == r.kv1 * grp && r.qb0 == 0 && r.qb1 == t; };
  std::vector<Run> out;
  for (const Run& r : per_kv) {
    if (!out.empty() && whole(out.back()) && whole(r) && out.back().kv1 == r.kv0) {
      out.back().h1 = r.h1;
      out.back().kv1 = r.kv1;
    } else {
      out.push_back(r);
    }
  }
  return out;
}

pbs_shape run_shape(const pbs_shape* g, const Run& r) {
  pbs_shape s = *g;
  s.num_q_heads = r.h1 - r.h0;
  s.num_kv_heads = r.kv1 - r.kv0;
  return s;
}

size_t shard_workspace(const pbs_shape* g, const pbs_pipeline_config* cfg, const pbs_shard& s) {
  const int64_t t = ceil_div(g->seq_len, cfg->block_size);
  size_t need = 0;
  for (const Run& r : runs_of(g, s, t)) {
    const pbs_shape rs = run_shape(g, r);
    need = std::max(need, plan(&rs, cfg).total);
  }
  return need;
}

// local sums for the global report: selected, admissible, sum of per-head
// densities, sum of per-head pooled coverages (the report averages over Hq)
struct LocalReport {
  double v[4] = {0, 0, 0, 0};
  pbs_report timing{};
};

int shard_enqueue(const void* q_local, const void* k_local, const void* v_local, const pbs_shape* g,
                  const pbs_pipeline_config* cfg, const pbs_shard& s, void* out_full, void* ws, size_t ws_bytes,
                  LocalReport* rep, cudaStream_t st) {
  const int64_t n = g->seq_len, d = g->head_dim, t = ceil_div(n, cfg->block_size);
  const size_t es = esize_of(g->dtype);
  for (const Run& r : runs_of(g, s, t)) {
    const pbs_shape rs = run_shape(g, r);
    const char* q = static_cast<const char*>(q_local) + (size_t)(r.h0 - s.head_begin) * n * d * es;
    const char* k = static_cast<const char*>(k_local) + (size_t)(r.kv0 - s.kv_begin) * n * d * es;
    const char* v = static_cast<const char*>(v_local) + (size_t)(r.kv0 - s.kv_begin) * n * d * es;
    char* out = static_cast<char*>(out_full) + (size_t)r.h0 * n * d * es;
    Timer tm(rep != nullptr, st);
    const int64_t qb1 = r.qb1 == t ? 0 : r.qb1;
    if (int rc = pipeline_enqueue(q, k, v, &rs, cfg, out, nullptr, nullptr, nullptr, ws, ws_bytes, tm, st, nullptr,
                                  r.qb0, qb1))
      return rc;
    if (rep) {
      std::vector<int32_t> cnt((size_t)rs.num_q_heads * t);
      std::vector<double> cov((size_t)rs.num_q_heads * t);
      int32_t hs[2];
      if (int rc = report_fetch(&rs, cfg, ws, cnt.data(), cov.data(), hs, st)) return rc;
      PBS_CUDA_CHECK(cudaStreamSynchronize(st));
      pbs_report pr{};
      if (int rc = report_build(&rs, cfg, cnt.data(), cov.data(), hs, tm, &pr, r.qb0, qb1)) {
        if (rc == PBS_ERR_DEGENERATE)
          return fail(PBS_ERR_DEGENERATE, "E_DEGENERATE",
                      "query block " + std::to_string(hs[1] % t) + " (head " +
                          std::to_string(r.h0 + hs[1] / t) + ") has an empty softmax denominator (all keys masked)");
        return rc;
      }
      rep->v[0] += (double)pr.selected_blocks;
      rep->v[1] += (double)pr.total_admissible_blocks;
      rep->v[2] += pr.block_density * rs.num_q_heads;
      rep->v[3] += pr.pooled_score_coverage * rs.num_q_heads;
      rep->timing.estimate_us += pr.estimate_us;
      rep->timing.permute_us += pr.permute_us;
      rep->timing.select_us += pr.select_us;
      rep->timing.attention_us += pr.attention_us;
      rep->timing.unpermute_us += pr.unpermute_us;
      rep->timing.causal_density_baseline = pr.causal_density_baseline;
    }
  }
  return PBS_OK;
}

void finish_report(const pbs_shape* g, const double* v, const pbs_report& timing, pbs_report* out) {
  *out = timing;
  const int64_t hq = g->num_q_heads;
  out->selected_blocks = (int64_t)(v[0] + 0.5);
  out->total_admissible_blocks = (int64_t)(v[1] + 0.5);
  out->block_density = v[2] / (double)hq;
  out->pooled_score_coverage = v[3] / (double)hq;
}

// ---- NCCL, resolved at run time ------------------------------------------------
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl lib;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      lib.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    lib.GetUniqueId = reinterpret_cast<decltype(lib.GetUniqueId)>(sym("ncclGetUniqueId"));
    lib.CommInitRank = reinterpret_cast<decltype(lib.CommInitRank)>(sym("ncclCommInitRank"));
    lib.CommDestroy = reinterpret_cast<decltype(lib.CommDestroy)>(sym("ncclCommDestroy"));
    lib.Broadcast = reinterpret_cast<decltype(lib.Broadcast)>(sym("ncclBroadcast"));
    lib.AllReduce = reinterpret_cast<decltype(lib.AllReduce)>(sym("ncclAllReduce"));
    lib.GroupStart = reinterpret_cast<decltype(lib.GroupStart)>(sym("ncclGroupStart"));
    lib.GroupEnd = reinterpret_cast<decltype(lib.GroupEnd)>(sym("ncclGroupEnd"));
    lib.GetErrorString = reinterpret_cast<decltype(lib.GetErrorString)>(sym("ncclGetErrorString"));
    lib.ok = lib.GetUniqueId && lib.CommInitRank && lib.CommDestroy && lib.Broadcast && lib.AllReduce &&
             lib.GroupStart && lib.GroupEnd && lib.GetErrorString;
    if (!lib.ok) lib.why = "libnccl.so.2 lacks a required symbol";
  });
  return lib;
}

int nccl_fail(ncclResult_t r, const char* where) {
  return fail(PBS_ERR_CUDA, "E_NCCL", std::string(where) + ": " + nccl().GetErrorString(r));
}
#define PBS_NCCL_CHECK(expr)                                    \
  do {                                                          \
    ncclResult_t _r = (expr);                                   \
    if (_r != ncclSuccess) return nccl_fail(_r, #expr);         \
  } while (0)

int need_nccl() {
  if (!nccl().ok) return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "multi-GPU needs NCCL: " + nccl().why);
  return PBS_OK;
}

}  // namespace
}  // namespace pbs_b200

using namespace pbs_b200;

struct pbs_dist {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
  double* red = nullptr;  // device scratch for the report reduction
};

extern "C" {

int pbs_shard_plan(const pbs_shape* global_shape, int64_t block_size, int32_t world_size, int32_t rank,
                   pbs_shard* shard) {
  if (!shard) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null shard");
  return shard_plan(global_shape, block_size, world_size, rank, shard);
}

size_t pbs_shard_workspace_size(const pbs_shape* global_shape, const pbs_pipeline_config* cfg, int32_t world_size,
                                int32_t rank) {
  pbs_shard s;
  if (check_cfg(cfg) || shard_plan(global_shape, cfg->block_size, world_size, rank, &s)) return 0;
  return std::max<size_t>(shard_workspace(global_shape, cfg, s), 256);
}

int pbs_attention_shard(const void* q_local, const void* k_local, const void* v_local, const pbs_shape* global_shape,
                        const pbs_pipeline_config* cfg, int32_t world_size, int32_t rank, void* out_full,
                        void* workspace, size_t workspace_bytes, pbs_report* report, void* stream) {
  if (int rc = check_cfg(cfg)) return rc;
  pbs_shard s;
  if (int rc = shard_plan(global_shape, cfg->block_size, world_size, rank, &s)) return rc;
  LocalReport lr;
  if (int rc = shard_enqueue(q_local, k_local, v_local, global_shape, cfg, s, out_full, workspace, workspace_bytes,
                             report ? &lr : nullptr, as_stream(stream)))
    return rc;
  if (report) finish_report(global_shape, lr.v, lr.timing, report);
  return PBS_OK;
}

int pbs_dist_unique_id(uint8_t id[PBS_NCCL_UNIQUE_ID_BYTES]) {
  if (int rc = need_nccl()) return rc;
  static_assert(sizeof(ncclUniqueId) == PBS_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  PBS_NCCL_CHECK(nccl().GetUniqueId(&u));
  memcpy(id, &u, sizeof u);
  return PBS_OK;
}

int pbs_dist_create(const uint8_t id[PBS_NCCL_UNIQUE_ID_BYTES], int32_t world_size, int32_t rank,
                    pbs_dist** handle) {
  if (!handle) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null handle");
  *handle = nullptr;
  if (world_size <= 0 || rank < 0 || rank >= world_size)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "rank outside [0, world_size)");
  if (int rc = need_nccl()) return rc;
  pbs_dist* d = new pbs_dist();
  d->world = world_size;
  d->rank = rank;
  if (cudaGetDevice(&d->device) != cudaSuccess || cudaMalloc(&d->red, 4 * sizeof(double)) != cudaSuccess) {
    delete d;
    return fail(PBS_ERR_CUDA, "E_CUDA", "pbs_dist_create: no CUDA device");
  }
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  const ncclResult_t r = nccl().CommInitRank(&d->comm, world_size, u, rank);
  if (r != ncclSuccess) {
    cudaFree(d->red);
    delete d;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *handle = d;
  return PBS_OK;
}

int pbs_dist_destroy(pbs_dist* handle) {
  if (!handle) return PBS_OK;
  if (handle->comm) nccl().CommDestroy(handle->comm);
  if (handle->red) cudaFree(handle->red);
  delete handle;
  return PBS_OK;
}

size_t pbs_dist_workspace_size(const pbs_dist* handle, const pbs_shape* global_shape, const pbs_pipeline_config* cfg) {
  if (!handle) return 0;
  return pbs_shard_workspace_size(global_shape, cfg, handle->world, handle->rank);
}

int pbs_dist_attention(pbs_dist* h, const void* q_local, const void* k_local, const void* v_local,
                       const pbs_shape* global_shape, const pbs_pipeline_config* cfg, void* out_full,
                       void* workspace, size_t workspace_bytes, pbs_report* report, void* stream) {
  if (!h) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null pbs_dist handle");
  if (int rc = check_cfg(cfg)) return rc;
  pbs_shard s;
  if (int rc = shard_plan(global_shape, cfg->block_size, h->world, h->rank, &s)) return rc;
  cudaStream_t st = as_stream(stream);
  LocalReport lr;
  if (int rc = shard_enqueue(q_local, k_local, v_local, global_shape, cfg, s, out_full, workspace, workspace_bytes,
                             report ? &lr : nullptr, st))
    return rc;
  // the one exchange: every rank's contiguous output rows, broadcast in place
  const size_t row_bytes = (size_t)global_shape->head_dim * esize_of(global_shape->dtype);
  PBS_NCCL_CHECK(nccl().GroupStart());
  for (int32_t r = 0; r < h->world; ++r) {
    pbs_shard sr;
    if (int rc = shard_plan(global_shape, cfg->block_size, h->world, r, &sr)) {
      nccl().GroupEnd();
      return rc;
    }
    if (sr.out_rows == 0) continue;
    char* p = static_cast<char*>(out_full) + (size_t)sr.out_row_begin * row_bytes;
    const ncclResult_t br = nccl().Broadcast(p, p, (size_t)sr.out_rows * row_bytes, ncclUint8, r, h->comm, st);
    if (br != ncclSuccess) {
      nccl().GroupEnd();
      return nccl_fail(br, "ncclBroadcast");
    }
  }
  PBS_NCCL_CHECK(nccl().GroupEnd());
  if (report) {  // collective: every rank asks for the report or none does
    PBS_CUDA_CHECK(cudaMemcpyAsync(h->red, lr.v, sizeof lr.v, cudaMemcpyHostToDevice, st));
    PBS_NCCL_CHECK(nccl().AllReduce(h->red, h->red, 4, ncclFloat64, ncclSum, h->comm, st));
    double v[4];
    PBS_CUDA_CHECK(cudaMemcpyAsync(v, h->red, sizeof v, cudaMemcpyDeviceToHost, st));
    PBS_CUDA_CHECK(cudaStreamSynchronize(st));
    finish_report(global_shape, v, lr.timing, report);
  }
  return PBS_OK;
}

}  // extern "C"
