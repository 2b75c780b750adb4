// select.cu -- stage 3 of Algorithm 1: pooled block scores and block selection.
//
//  pool          meanpool (block_selection.hpp:134-147): sequential row sums in
//                permuted order, / rc (short final block uses its real length)
//  score_select  per (head, query block) CTA:
//                logits = qbar . kbar (sequential c, matrix.hpp:87-94), *= s (152-153)
//                softmax_rows under the segment-band mask (matrix.hpp:122-144):
//                  row max, e = expf(v - mx), sequential denominator, e / denom
//                select_blocks (block_selection.hpp:171-206): stable descending
//                  order (ties by index), double cumulative sum until >= tau,
//                  forced block 0 and forced diagonal band
//                compaction into the ascending kv list the attention kernel
//                  iterates (the reference's kb loop order, attention.hpp:283)
//
// All arithmetic feeding a comparison is restated exactly (non-fused mul/add,
// IEEE div, glibc expf port), so masks are bit-identical to the reference.
// Admissible blocks of row i are the prefix j < (seg(i)+1)*S/B (segment band,
// block_selection.hpp:86-97), so no causal matrix is materialised.
#include <algorithm>

#include "common.cuh"
#include "expf_glibc.cuh"
#include "kernels.h"

namespace pbs_b200 {
namespace {

// pooled[h][b][c] = (sum_{r in block b} x[h / G][perm[h][r]][c]) / rc
template <typename T>
__global__ void pool_kernel(const T* __restrict__ x, int group, const int32_t* __restrict__ perm, int64_t n,
                            int d, int64_t block, int64_t t, float* __restrict__ pooled) {
  const int64_t h = blockIdx.y;
  const int64_t b = blockIdx.x;
  const int64_t r0 = b * block;
  const int64_t rc = min(block, n - r0);
  const T* xs = x + (h / group) * n * d;
  const int32_t* ph = perm ? perm + h * n : nullptr;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.0f;
    for (int64_t r = r0; r < r0 + rc; ++r) {
      const int64_t src = ph ? ph[r] : r;
      acc = __fadd_rn(acc, to_f32(xs[src * d + c]));
    }
    pooled[(h * t + b) * d + c] = __fdiv_rn(acc, (float)rc);
  }
}

constexpr int kSelThreads = 256;

__device__ __forceinline__ float block_max(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? red[l] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

// One CTA per (query block i, head h).  mode 0: compute scores from pooled
// Q/K; mode 1: read precomputed scores (pbs_select_blocks).
__global__ void __launch_bounds__(kSelThreads) score_select_kernel(
    int mode, const float* __restrict__ qbar, const float* __restrict__ kbar,
    const float* __restrict__ scores_in, int64_t t, int d, int64_t block, int64_t segment, float scale,
    double tau, int forced_first, int forced_band, int pow2, float* __restrict__ scores_out,
    uint8_t* __restrict__ mask, int32_t* __restrict__ kv_idx, int32_t* __restrict__ kv_cnt,
    double* __restrict__ row_cov) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);  // [pow2]
  float* sv = reinterpret_cast<float*>(keys + pow2);                      // [t]
  float* qs = sv + t;                                                      // [d]
  uint8_t* mrow = reinterpret_cast<uint8_t*>(qs + d);                      // [t]
  __shared__ float red[32];
  __shared__ float s_denom;
  __shared__ int s_take;

  const int64_t h = blockIdx.y, i = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t a = admissible_prefix(i, t, block, segment);

  if (mode == 0) {
    for (int c = tid; c < d; c += blockDim.x) qs[c] = qbar[(h * t + i) * d + c];
    __syncthreads();
    const float* kb = kbar + h * t * d;
    float mx = -INFINITY;
    for (int64_t j = tid; j < a; j += blockDim.x) {
      const float* kr = kb + j * d;
      float acc = 0.0f;
      for (int c = 0; c < d; ++c) acc = __fadd_rn(acc, __fmul_rn(qs[c], kr[c]));
      const float v = __fmul_rn(acc, scale);
      sv[j] = v;
      mx = fmaxf(mx, v);
    }
    mx = block_max(mx, red);
    for (int64_t j = tid; j < a; j += blockDim.x) sv[j] = expf_glibc(__fsub_rn(sv[j], mx));
    __syncthreads();
    if (tid == 0) {
      float denom = 0.0f;
      for (int64_t j = 0; j < a; ++j) denom = __fadd_rn(denom, sv[j]);
      s_denom = denom;
    }
    __syncthreads();
    const float denom = s_denom;
    for (int64_t j = tid; j < a; j += blockDim.x) sv[j] = __fdiv_rn(sv[j], denom);
    __syncthreads();
    if (scores_out) {
      float* so = scores_out + (h * t + i) * t;
      for (int64_t j = tid; j < t; j += blockDim.x) so[j] = j < a ? sv[j] : 0.0f;
    }
  } else {
    const float* si = scores_in + (h * t + i) * t;
    for (int64_t j = tid; j < a; j += blockDim.x) sv[j] = si[j];
    __syncthreads();
  }

  // descending stable order of the admissible blocks
  for (int j = tid; j < pow2; j += blockDim.x)
    keys[j] = j < a ? (((unsigned long long)(~float_order_key(sv[j])) << 32) | (unsigned)j) : ~0ull;
  for (int64_t j = tid; j < t; j += blockDim.x) mrow[j] = 0;
  __syncthreads();
  for (int size = 2; size <= pow2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int x = tid; x < pow2 / 2; x += blockDim.x) {
        const int lo = 2 * x - (x & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long p = keys[lo], q = keys[hi];
        if ((p > q) == up) {
          keys[lo] = q;
          keys[hi] = p;
        }
      }
      __syncthreads();
    }
  if (tid == 0) {
    double cum = 0.0;
    int take = (int)a;  // fallback: every admissible block (line 188)
    for (int k = 0; k < a; ++k) {
      cum += (double)sv[keys[k] & 0xffffffffu];
      if (cum >= tau) {
        take = k + 1;
        break;
      }
    }
    s_take = take;
  }
  __syncthreads();
  const int take = s_take;
  for (int k = tid; k < take; k += blockDim.x) mrow[keys[k] & 0xffffffffu] = 1;
  __syncthreads();
  if (tid == 0) {
    if (forced_first && t > 0) mrow[0] = 1;
    if (forced_band) {
      int64_t lo, hi;
      if (segment == 0) {
        lo = i;
        hi = i + 1;
      } else {
        const int64_t per = segment / block;
        lo = (i / per) * per;
        hi = min(lo + per, t);
      }
      for (int64_t j = lo; j < hi; ++j) mrow[j] = 1;
    }
  }
  __syncthreads();
  if (mask) {
    uint8_t* mo = mask + (h * t + i) * t;
    for (int64_t j = tid; j < t; j += blockDim.x) mo[j] = mrow[j];
  }
  // warp 0: ascending compaction of the selected blocks + coverage partial
  if (tid < 32) {
    int cnt = 0;
    double cov = 0.0;
    int32_t* out = kv_idx ? kv_idx + (h * t + i) * t : nullptr;
    for (int64_t j0 = 0; j0 < t; j0 += 32) {
      const int64_t j = j0 + tid;
      const bool sel = j < t && mrow[j];
      const unsigned bal = __ballot_sync(0xffffffffu, sel);
      if (sel && out) out[cnt + __popc(bal & ((1u << tid) - 1))] = (int32_t)j;
      cnt += __popc(bal);
    }
    if (tid == 0) {
      // pooled_score_coverage partial (pipeline.hpp:186-191), j ascending
      if (mode == 0)
        for (int64_t j = 0; j < a; ++j)
          if (mrow[j]) cov += (double)sv[j];
      if (kv_cnt) kv_cnt[h * t + i] = cnt;
      if (row_cov) row_cov[h * t + i] = cov;
    }
  }
}

inline size_t select_smem(int64_t t, int d, int pow2) {
  return (size_t)pow2 * 8 + (size_t)t * 4 + (size_t)d * 4 + (size_t)t + 16;
}

}  // namespace

size_t select_workspace_bytes(int hq, int64_t n, int d, int64_t block) {
  const int64_t t = ceil_div(n, block);
  return 2 * (size_t)hq * t * d * 4 + (size_t)hq * t * 8 + 1024;
}

int launch_pool(const void* x, int dtype, int src_heads, int dst_heads, const int32_t* perm, int64_t n, int d,
                int64_t block, float* pooled, cudaStream_t st) {
  const int64_t t = ceil_div(n, block);
  if (t == 0) return PBS_OK;
  const int group = dst_heads / src_heads;
  const int threads = std::min(128, ((d + 31) / 32) * 32);
  dim3 grid((unsigned)t, (unsigned)dst_heads);
  if (dtype == PBS_DTYPE_BF16)
    pool_kernel<__nv_bfloat16><<<grid, threads, 0, st>>>(static_cast<const __nv_bfloat16*>(x), group, perm, n, d,
                                                         block, t, pooled);
  else
    pool_kernel<float><<<grid, threads, 0, st>>>(static_cast<const float*>(x), group, perm, n, d, block, t, pooled);
  PBS_LAUNCH_CHECK("pool_kernel");
  return PBS_OK;
}

static int launch_select_common(int mode, const float* qbar, const float* kbar, const float* scores_in, int hq,
                                int64_t t, int d, int64_t block, int64_t segment, float scale, double tau,
                                int forced_first, int forced_band, float* scores_out, uint8_t* mask,
                                int32_t* kv_idx, int32_t* kv_cnt, double* row_cov, cudaStream_t st) {
  if (t == 0 || hq == 0) return PBS_OK;
  if (t > 16384) return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "block grid wider than 16384 blocks");
  int pow2 = 1;
  while (pow2 < t) pow2 <<= 1;
  const size_t smem = select_smem(t, d, pow2);
  static bool attr_set = false;
  if (!attr_set) {
    PBS_CUDA_CHECK(cudaFuncSetAttribute(score_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set = true;
  }
  score_select_kernel<<<dim3((unsigned)t, (unsigned)hq), kSelThreads, smem, st>>>(
      mode, qbar, kbar, scores_in, t, d, block, segment, scale, tau, forced_first, forced_band, pow2, scores_out,
      mask, kv_idx, kv_cnt, row_cov);
  PBS_LAUNCH_CHECK("score_select_kernel");
  return PBS_OK;
}

int launch_score_select(const float* qbar, const float* kbar, int hq, int64_t t, int d, int64_t block,
                        int64_t segment, float scale, double tau, int forced_first, int forced_band,
                        float* scores_out, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt, double* row_cov,
                        cudaStream_t st) {
  return launch_select_common(0, qbar, kbar, nullptr, hq, t, d, block, segment, scale, tau, forced_first,
                              forced_band, scores_out, mask, kv_idx, kv_cnt, row_cov, st);
}

int launch_select_from_scores(const float* scores, int hq, int64_t t, int64_t block, int64_t segment, double tau,
                              int forced_first, int forced_band, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt,
                              cudaStream_t st) {
  return launch_select_common(1, nullptr, nullptr, scores, hq, t, 0, block, segment, 0.0f, tau, forced_first,
                              forced_band, nullptr, mask, kv_idx, kv_cnt, nullptr, st);
}

}  // namespace pbs_b200
