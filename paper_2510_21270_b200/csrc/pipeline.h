// pipeline.h -- internal: Algorithm 1 enqueued on a stream, shared by the
// single-call C-ABI entries (cabi.cu) and the head-parallel multi-GPU entry
// (dist.cu).  Not part of the public ABI (include/pbs_cabi.h).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace pbs_b200 {

int esize_of(int dtype);
float effective_scale(double scale, int d);
int check_shape(const pbs_shape* s);
int check_cfg(const pbs_pipeline_config* c);
bool uses_pi(int s);
bool uses_sigma(int s);
size_t al(size_t x);

// workspace carve-up for pbs_attention
struct Layout {
  size_t status, imp, scores, pi, pi_inv, sigma, sigma_inv, groups, qperm, kp, vp, qp, qbar, kbar, blog, mask,
      kv_idx, kv_cnt, row_cov, sched, total;
};

Layout plan(const pbs_shape* s, const pbs_pipeline_config* c);

// CUDA-event stage timer (StageTimings, pipeline.hpp:51-61)
struct Timer {
  bool on;
  cudaStream_t st;
  cudaEvent_t ev[6];
  int k = 0;
  Timer(bool enabled, cudaStream_t s) : on(enabled), st(s) {
    if (on)
      for (auto& e : ev) cudaEventCreate(&e);
  }
  ~Timer() {
    if (on)
      for (auto& e : ev) cudaEventDestroy(e);
  }
  Timer(const Timer&) = delete;
  Timer& operator=(const Timer&) = delete;
  void restart(cudaStream_t s) {
    st = s;
    k = 0;
  }
  void mark() {
    if (on && k < 6) cudaEventRecord(ev[k++], st);
  }
  double us(int a) const {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ev[a], ev[a + 1]);
    return ms * 1000.0;
  }
};

int run_attention(const AttnParams& p, void* sched, cudaStream_t st);

// Algorithm 1 (pipeline.hpp:107-193) enqueued on `stream`, no synchronisation;
// stage events go to tm.  pi_given (key_permute only): pi of every head,
// computed beforehand.  [qb_begin, qb_end): the query blocks whose output rows
// this call writes (0, 0: all) -- every other stage runs on whole heads.
int pipeline_enqueue(const void* q, const void* k, const void* v, const pbs_shape* shape,
                     const pbs_pipeline_config* cfg, void* out, int32_t* sigma_out, int32_t* pi_out,
                     uint8_t* mask_out, void* workspace, size_t workspace_bytes, Timer& tm, void* stream,
                     const int32_t* pi_given = nullptr, int64_t qb_begin = 0, int64_t qb_end = 0);

// The per-row counters the report needs, copied to host memory on `st`
// (asynchronous; complete once `st` reaches this point).
int report_fetch(const pbs_shape* shape, const pbs_pipeline_config* cfg, const void* workspace, int32_t* cnt,
                 double* cov, int32_t* hs, cudaStream_t st);

// PipelineReport (pipeline.hpp:182-191) from the fetched counters, over the
// query blocks [qb_begin, qb_end) of every head (0, 0: all)
int report_build(const pbs_shape* shape, const pbs_pipeline_config* cfg, const int32_t* cnt, const double* cov,
                 const int32_t* hs, const Timer& tm, pbs_report* report, int64_t qb_begin = 0, int64_t qb_end = 0);

}  // namespace pbs_b200
