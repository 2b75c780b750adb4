// common.cuh -- shared device/host helpers for the sm_100a PBS-Attn library.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include "../../include/pbs_cabi.h"

namespace pbs_b200 {

// ---- thread-local error text (pbs_last_error) -------------------------------
void set_error(const char* prefix, const std::string& msg);
int fail(int code, const char* prefix, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define PBS_CUDA_CHECK(expr)                                        \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) return ::pbs_b200::cuda_fail(_e, #expr); \
  } while (0)

// every kernel launch of the library is followed by exactly one of these;
// it also feeds the process-wide launch counter (pbs_kernel_launches)
void count_launch();
#define PBS_LAUNCH_CHECK(where)                                       \
  do {                                                                \
    ::pbs_b200::count_launch();                                       \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::pbs_b200::cuda_fail(_e, where);   \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Per-device one-time setup of a call site (function attributes such as the
// dynamic shared-memory size are per device).  The device's bit is set only
// after the setup succeeded, under a lock, so a second host thread never
// launches before the attribute is in place and a failed setup is retried.
struct DeviceOnce {
  std::atomic<uint64_t> done{0};
  std::mutex mu;
};
template <class F>
int once_per_device(DeviceOnce& o, F&& setup) {
  int dev = 0;
  PBS_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return setup();
  const uint64_t bit = 1ull << dev;
  if (o.done.load(std::memory_order_acquire) & bit) return PBS_OK;
  std::lock_guard<std::mutex> lk(o.mu);
  if (o.done.load(std::memory_order_relaxed) & bit) return PBS_OK;
  if (int rc = setup()) return rc;
  o.done.fetch_or(bit, std::memory_order_release);
  return PBS_OK;
}

// SM count of the current device (cached per device)
int num_sms();

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// ---- element access (inputs are bf16 or f32; the arithmetic is f32) ---------
template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// segment_of_block (block_selection.hpp:19-23)
__host__ __device__ __forceinline__ int64_t segment_of_block(int64_t b, int64_t block, int64_t segment) {
  return segment == 0 ? b : b * block / segment;
}

// number of admissible key blocks of block-row i under the segment-band causal
// mask (build_block_causal_mask, block_selection.hpp:86-97): seg(j) <= seg(i)
// holds exactly for j < (seg(i) + 1) * S / B, a prefix of the row.
__host__ __device__ __forceinline__ int64_t admissible_prefix(int64_t i, int64_t t, int64_t block,
                                                              int64_t segment) {
  if (segment == 0) return i + 1;
  const int64_t per = segment / block;
  const int64_t end = (i / per + 1) * per;
  return end < t ? end : t;
}

// order-preserving float -> uint32 (ascending), -0 folded onto +0 so that
// the reference's `>` comparison (which treats them equal) is reproduced.
__device__ __forceinline__ uint32_t float_order_key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// atomic max on floats through the order-preserving encoding
__device__ __forceinline__ void atomic_max_float(unsigned int* addr, float v) {
  atomicMax(addr, float_order_key(v));
}
__device__ __forceinline__ float decode_order_key(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

}  // namespace pbs_b200
