// gather.cu -- K4/K7: apply_rows (permutation.hpp:79-89) batched over heads with
// the GQA broadcast: dst[h][i][:] = src[h / G][perm[h][i]][:].
//
// HBM-bound row copy: algorithmic bytes = 2 * rows * cols * esize per head
// (read + write).  One warp moves one row with 16-byte vector accesses; a
// grid of 148 * 16 CTAs strides over all (head, row) pairs.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pbs_b200 {
namespace {

// kVecPerRow 16-byte vectors per row; a warp moves 32 / kVecPerRow rows per
// pass (all lanes busy for 256-byte rows) and kUnroll passes' loads are issued
// before any store, so each lane keeps kUnroll 16-byte loads in flight.
template <int kVecPerRow>
__global__ void __launch_bounds__(256) apply_rows_vec_kernel(const int32_t* __restrict__ perm,
                                                             const int4* __restrict__ src, int group,
                                                             int64_t rows, int64_t total_rows,
                                                             int4* __restrict__ dst) {
  constexpr int kRowsPerPass = kVecPerRow >= 32 ? 1 : 32 / kVecPerRow;
  constexpr int kVecPerLane = kVecPerRow >= 32 ? kVecPerRow / 32 : 1;
  constexpr int kUnroll = 4;
  const int lane = threadIdx.x & 31;
  const int sub = kVecPerRow >= 32 ? 0 : lane / kVecPerRow;  // row of the pass
  const int col = kVecPerRow >= 32 ? lane : lane % kVecPerRow;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t step = nwarps * kRowsPerPass;
  for (int64_t base = warp * kRowsPerPass * kUnroll; base < total_rows; base += step * kUnroll) {
    int4 v[kUnroll][kVecPerLane];
    int64_t rr[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t r = base + (int64_t)u * kRowsPerPass + sub;
      rr[u] = r;
      if (r < total_rows) {
        // 32-bit head / row split (total_rows < 2^31 is checked at launch):
        // a 64-bit division per row cost more issue slots than the copy
        const uint32_t r32 = (uint32_t)r, rows32 = (uint32_t)rows;
        const uint32_t h = r32 / rows32, i = r32 - h * rows32;
        const int64_t s = perm ? __ldg(perm + r) : (int64_t)i;
        const int4* sp = src + ((int64_t)(h / (uint32_t)group) * rows + s) * kVecPerRow;
#pragma unroll
        for (int w = 0; w < kVecPerLane; ++w) v[u][w] = __ldg(sp + col + w * 32);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (rr[u] < total_rows) {
        int4* dp = dst + rr[u] * kVecPerRow;
#pragma unroll
        for (int w = 0; w < kVecPerLane; ++w) dp[col + w * 32] = v[u][w];
      }
    }
  }
}

__global__ void apply_rows_generic_kernel(const int32_t* __restrict__ perm, const char* __restrict__ src,
                                          int group, int64_t rows, int64_t row_bytes, int64_t total_rows,
                                          char* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < total_rows; r += nwarps) {
    const int64_t h = r / rows, i = r % rows;
    const int64_t s = perm ? perm[r] : i;
    const char* sp = src + ((h / group) * rows + s) * row_bytes;
    char* dp = dst + r * row_bytes;
    for (int64_t b = lane; b < row_bytes; b += 32) dp[b] = sp[b];
  }
}

// the stage-5 un-permute as a scatter: dst[h][perm[h][i]] = src[h][i]
// (O = apply_rows(sigma^-1, O'), pipeline.hpp:178-180, without forming sigma^-1)
template <int kVecPerRow>
__global__ void __launch_bounds__(256) scatter_rows_vec_kernel(const int32_t* __restrict__ perm,
                                                               const int4* __restrict__ src, int64_t rows,
                                                               int64_t total_rows, int4* __restrict__ dst) {
  constexpr int kRowsPerPass = kVecPerRow >= 32 ? 1 : 32 / kVecPerRow;
  constexpr int kVecPerLane = kVecPerRow >= 32 ? kVecPerRow / 32 : 1;
  const int lane = threadIdx.x & 31;
  const int sub = kVecPerRow >= 32 ? 0 : lane / kVecPerRow;
  const int col = kVecPerRow >= 32 ? lane : lane % kVecPerRow;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp * kRowsPerPass + sub; r < total_rows; r += nwarps * kRowsPerPass) {
    const uint32_t r32 = (uint32_t)r, rows32 = (uint32_t)rows;
    const uint32_t h = r32 / rows32;
    const int64_t to = (int64_t)h * rows + __ldg(perm + r);
    const int4* sp = src + r * kVecPerRow;
    int4* dp = dst + to * kVecPerRow;
#pragma unroll
    for (int w = 0; w < kVecPerLane; ++w) dp[col + w * 32] = __ldg(sp + col + w * 32);
  }
}

__global__ void scatter_rows_generic_kernel(const int32_t* __restrict__ perm, const char* __restrict__ src,
                                            int64_t rows, int64_t row_bytes, int64_t total_rows,
                                            char* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < total_rows; r += nwarps) {
    const int64_t h = r / rows;
    char* dp = dst + (h * rows + perm[r]) * row_bytes;
    const char* sp = src + r * row_bytes;
    for (int64_t b = lane; b < row_bytes; b += 32) dp[b] = sp[b];
  }
}

}  // namespace

int launch_scatter_rows(const int32_t* perm, const void* src, int heads, int64_t rows, int cols, int esize,
                        void* dst, cudaStream_t st) {
  if (rows == 0 || cols == 0 || heads == 0) return PBS_OK;
  if (!perm) return fail(PBS_ERR_CONFIG, "E_CONFIG", "unpermute: sigma is required");
  const int64_t total = rows * heads;
  const int64_t row_bytes = (int64_t)cols * esize;
  const int blocks = (int)min64(ceil_div(total, 8 * 8), 148 * 16);
  const bool aligned = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0) &&
                       total < ((int64_t)1 << 31);
  if (aligned && row_bytes == 256) {
    scatter_rows_vec_kernel<16><<<blocks, 256, 0, st>>>(perm, static_cast<const int4*>(src), rows, total,
                                                       static_cast<int4*>(dst));
  } else if (aligned && row_bytes == 512) {
    scatter_rows_vec_kernel<32><<<blocks, 256, 0, st>>>(perm, static_cast<const int4*>(src), rows, total,
                                                       static_cast<int4*>(dst));
  } else {
    scatter_rows_generic_kernel<<<blocks, 256, 0, st>>>(perm, static_cast<const char*>(src), rows, row_bytes, total,
                                                        static_cast<char*>(dst));
  }
  PBS_LAUNCH_CHECK("scatter_rows_kernel");
  return PBS_OK;
}

int launch_apply_rows(const int32_t* perm, const void* src, int src_heads, int dst_heads, int64_t rows,
                      int cols, int esize, void* dst, cudaStream_t st) {
  if (rows == 0 || cols == 0 || dst_heads == 0) return PBS_OK;
  if (src_heads <= 0 || dst_heads % src_heads != 0)
    return fail(PBS_ERR_CONFIG, "E_SHAPE", "apply_rows: dst heads must be a multiple of src heads");
  const int group = dst_heads / src_heads;
  const int64_t total = rows * dst_heads;
  const int64_t row_bytes = (int64_t)cols * esize;
  const int blocks = (int)min64(ceil_div(total, 8 * 8), 148 * 16);
  const bool aligned = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0) &&
                       total < ((int64_t)1 << 31);  // the vector kernels split rows in 32 bits
  if (aligned && row_bytes == 256) {
    apply_rows_vec_kernel<16><<<blocks, 256, 0, st>>>(perm, static_cast<const int4*>(src), group, rows, total,
                                                     static_cast<int4*>(dst));
  } else if (aligned && row_bytes == 512) {
    apply_rows_vec_kernel<32><<<blocks, 256, 0, st>>>(perm, static_cast<const int4*>(src), group, rows, total,
                                                     static_cast<int4*>(dst));
  } else {
    apply_rows_generic_kernel<<<blocks, 256, 0, st>>>(perm, static_cast<const char*>(src), group, rows, row_bytes,
                                                      total, static_cast<char*>(dst));
  }
  PBS_LAUNCH_CHECK("apply_rows_kernel");
  return PBS_OK;
}

}  // namespace pbs_b200
