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
#include "exact_gemm.cuh"
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

// bf16, d % 8 == 0: a thread owns 8 columns (one 16-byte load per row) of one
// block and sums its rows in order; 128 threads cover 128 / (d / 8) blocks, and
// four rows' loads (row indices prefetched) are in flight ahead of the adds.
__global__ void __launch_bounds__(128) pool_bf16x8_kernel(const __nv_bfloat16* __restrict__ x, int group,
                                                          const int32_t* __restrict__ perm, int64_t n, int d,
                                                          int64_t block, int64_t t, float* __restrict__ pooled) {
  const int cg_per_row = d / 8;
  const int blocks_per_cta = blockDim.x / cg_per_row;
  const int64_t h = blockIdx.y;
  const int64_t b = (int64_t)blockIdx.x * blocks_per_cta + threadIdx.x / cg_per_row;
  const int c0 = (threadIdx.x % cg_per_row) * 8;
  if (b >= t || threadIdx.x >= blocks_per_cta * cg_per_row) return;
  const int64_t r0 = b * block;
  const int64_t rc = min(block, n - r0);
  const __nv_bfloat16* xs = x + (h / group) * n * d + c0;
  const int32_t* ph = perm ? perm + h * n : nullptr;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  constexpr int kU = 4;
  int64_t r = r0;
  for (; r + kU <= r0 + rc; r += kU) {
    uint4 raw[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t src = ph ? __ldg(ph + r + u) : r + u;
      raw[u] = __ldg(reinterpret_cast<const uint4*>(xs + src * d));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw[u]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(p2[q]);
        acc[2 * q] = __fadd_rn(acc[2 * q], f.x);
        acc[2 * q + 1] = __fadd_rn(acc[2 * q + 1], f.y);
      }
    }
  }
  for (; r < r0 + rc; ++r) {
    const int64_t src = ph ? ph[r] : r;
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(xs + src * d));
    const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(p2[q]);
      acc[2 * q] = __fadd_rn(acc[2 * q], f.x);
      acc[2 * q + 1] = __fadd_rn(acc[2 * q + 1], f.y);
    }
  }
  float* dst = pooled + (h * t + b) * d + c0;
#pragma unroll
  for (int q = 0; q < 8; ++q) dst[q] = __fdiv_rn(acc[q], (float)rc);
}

constexpr int kSelThreads = 128;

// block logits: Lb[h][i][j] = (qbar_i . kbar_j) * s for the admissible prefix
// j < A_i only (matrix.hpp:87-94 then block_selection.hpp:152-153).
__global__ void __launch_bounds__(xgemm::kThreads) block_logits_kernel(const float* __restrict__ qbar,
                                                                      const float* __restrict__ kbar, int64_t t, int d,
                                                                      int64_t block, int64_t segment, float scale,
                                                                      float* __restrict__ lb) {
  __shared__ __align__(16) xgemm::Smem sm;
  const int64_t h = blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.x * xgemm::kTile;
  const int64_t j0 = (int64_t)blockIdx.y * xgemm::kTile;
  const int a_rows = (int)min64(xgemm::kTile, t - i0);
  if (j0 >= admissible_prefix(i0 + a_rows - 1, t, block, segment)) return;  // tile above the band
  const int b_rows = (int)min64(xgemm::kTile, t - j0);
  float acc[8][8];
  if (d % 16 == 0)
    xgemm::tile<float, float, false, true>(qbar + (h * t + i0) * d, a_rows, kbar + (h * t + j0) * d, b_rows, d, acc,
                                            sm);
  else
    xgemm::tile<float, float, false, false>(qbar + (h * t + i0) * d, a_rows, kbar + (h * t + j0) * d, b_rows, d,
                                             acc, sm);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) {
    const int64_t i = i0 + xgemm::tile_row(ii, ty);
    if (i >= i0 + a_rows) continue;
    const int64_t a = admissible_prefix(i, t, block, segment);
    float* row = lb + (h * t + i) * t;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int64_t j = j0 + xgemm::tile_row(jj, tx);
      if (j < a) row[j] = __fmul_rn(acc[ii][jj], scale);
    }
  }
}

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

// One CTA per (query block i, head h).  mode 0: softmax of the block logits
// row; mode 1: precomputed scores (pbs_select_blocks).  Sequential chains
// (the softmax denominator, the double cumulative sum, the coverage sum) run
// in warp 0 as a broadcast chain: every lane pulls element k with a shuffle
// and performs the identical add, so the order is exactly the reference's.
__global__ void __launch_bounds__(kSelThreads) select_kernel(
    int mode, const float* __restrict__ rows_in, int64_t t, int64_t block, int64_t segment, double tau, int top_k,
    int forced_first, int forced_band, int select, float* __restrict__ scores_out, uint8_t* __restrict__ mask,
    int32_t* __restrict__ kv_idx, int32_t* __restrict__ kv_cnt, double* __restrict__ row_cov) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t h = blockIdx.y, i = blockIdx.x;
  const int64_t a = admissible_prefix(i, t, block, segment);
  int pow2 = 1;
  while (pow2 < a) pow2 <<= 1;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);  // [pow2]
  float* sv = reinterpret_cast<float*>(keys + pow2);                      // [a]
  uint8_t* mrow = reinterpret_cast<uint8_t*>(sv + ((a + 3) & ~3));        // [t]
  __shared__ float red[32];
  __shared__ float s_denom;
  __shared__ int s_take;
  __shared__ uint64_t tab[32];
  load_exp2f_table(tab);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* in = rows_in + (h * t + i) * t;
  for (int64_t j = tid; j < a; j += blockDim.x) sv[j] = in[j];
  __syncthreads();
  if (mode == 0) {
    float mx = -INFINITY;
    for (int64_t j = tid; j < a; j += blockDim.x) mx = fmaxf(mx, sv[j]);
    mx = block_max(mx, red);
    for (int64_t j = tid; j < a; j += blockDim.x) sv[j] = expf_glibc(__fsub_rn(sv[j], mx), tab);
    __syncthreads();
    if (tid == 0) {
      // one thread, values straight from smem (loads run ahead of the add chain)
      float denom = 0.0f;
      int64_t j = 0;
      for (; j + 8 <= a; j += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = sv[j + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) denom = __fadd_rn(denom, v[u]);
      }
      for (; j < a; ++j) denom = __fadd_rn(denom, sv[j]);
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
  }
  if (!select) return;

  // descending stable order of the admissible blocks (composite unique keys)
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
      // comparisons x in [32w, 32w + 32) (+ multiples of the block) touch only
      // elements [64w, 64w + 64) while stride < 32: when the NEXT stage's
      // stride is below 32 it reads only this warp's elements, and a warp
      // barrier suffices
      const int next_stride = stride > 1 ? stride >> 1 : size;
      if (next_stride < 32) __syncwarp();
      else __syncthreads();
    }
  __syncthreads();
  if (tid == 0 && top_k > 0) {
    s_take = (int)min64(top_k, a);  // top-k extension: the first k of the same order
  } else if (tid == 0) {
    // one thread: the sorted values are fetched 8 ahead of the double chain
    double cum = 0.0;
    int take = (int)a;  // fallback: every admissible block (line 188)
    for (int64_t k0 = 0; k0 < a; k0 += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (k0 + u < a) ? sv[keys[k0 + u] & 0xffffffffu] : 0.0f;
      bool done = false;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (k0 + u >= a) break;
        cum += (double)v[u];
        if (cum >= tau) {
          take = (int)(k0 + u + 1);
          done = true;
          break;
        }
      }
      if (done) break;
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
        hi = min64(lo + per, t);
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
  // (pipeline.hpp:186-191, j ascending, double accumulation)
  if (warp == 0) {
    int cnt = 0;
    double cov = 0.0;
    int32_t* out = kv_idx ? kv_idx + (h * t + i) * t : nullptr;
    for (int64_t j0 = 0; j0 < t; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool sel = j < t && mrow[j];
      const unsigned bal = __ballot_sync(0xffffffffu, sel);
      if (sel && out) out[cnt + __popc(bal & ((1u << lane) - 1))] = (int32_t)j;
      cnt += __popc(bal);
      if (mode == 0 && j0 < a) {
        const double val = (sel && j < a) ? (double)sv[j] : 0.0;
        unsigned bits = bal & (j0 + 32 <= a ? 0xffffffffu : ((1u << (a - j0)) - 1));
        while (bits) {
          const int kk = __ffs(bits) - 1;
          bits &= bits - 1;
          cov += __shfl_sync(0xffffffffu, val, kk);
        }
      }
    }
    if (lane == 0) {
      if (kv_cnt) kv_cnt[h * t + i] = cnt;
      if (row_cov) row_cov[h * t + i] = cov;
    }
  }
}

// ---- warp-per-row selection ---------------------------------------------------
// One warp per (head, query block) row, 4 rows per CTA, no CTA barriers:
//  * mode 0: the softmax of the block-logit row (matrix.hpp:127-142): warp max,
//    exps spread over the lanes, the sequential denominator in one lane (values
//    read 8 ahead from shared memory), the IEEE division spread again;
//  * the threshold rule (block_selection.hpp:171-206) needs only the sorted
//    PREFIX whose double cumulative sum reaches tau.  A bisection over the
//    float bit patterns finds the largest theta with sum_{v >= theta} v >=
//    tau + 1e-9 (summed in any order: the reference's sequential double sum
//    over the same elements differs by < a * 2^-52, far below the 1e-9
//    margin), so the prefix lies inside C = {v >= theta}; only C is sorted
//    (unique composite keys: descending score, ties by ascending index =
//    std::stable_sort's order) and walked by the exact one-lane double chain.
//    Rows whose total mass cannot clear the margin (tau ~ 1), or with negative
//    or non-finite scores, sort every admissible block instead.  top-k: the
//    largest theta keeping >= k candidates;
//  * forced blocks, the mask row, the ascending kv list and the pooled-score
//    coverage (ascending double sum, pipeline.hpp:186-191) from a bitmap.
constexpr int kSelWarps = 4;

struct SelWarpLayout {
  int tpad, pow2, words;
  __host__ __device__ size_t per_warp() const {
    return ((size_t)tpad * 4 + (size_t)pow2 * 8 + (size_t)words * 4 + 15) & ~(size_t)15;
  }
};

__host__ __device__ inline SelWarpLayout sel_layout(int64_t t) {
  SelWarpLayout L;
  L.tpad = (int)((t + 3) & ~3);
  int p = 32;
  while (p < t) p <<= 1;
  L.pow2 = p;
  L.words = (int)((t + 31) / 32);
  return L;
}

// warp-synchronous bitonic sort of n (power of two, >= 32) ascending 64-bit keys
__device__ __forceinline__ void warp_bitonic(unsigned long long* keys, int n, int lane) {
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int x = lane; x < n / 2; x += 32) {
        const int lo = 2 * x - (x & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long p = keys[lo], q = keys[hi];
        if ((p > q) == up) {
          keys[lo] = q;
          keys[hi] = p;
        }
      }
      __syncwarp();
    }
}

__device__ __forceinline__ int warp_sum_i(int v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kSelWarps * 32) select_warp_kernel(
    int mode, const float* __restrict__ rows_in, int hq, int64_t t, int64_t block, int64_t segment, double tau,
    int top_k, int forced_first, int forced_band, int select, float* __restrict__ scores_out,
    uint8_t* __restrict__ mask, int32_t* __restrict__ kv_idx, int32_t* __restrict__ kv_cnt,
    double* __restrict__ row_cov) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t tab[32];
  load_exp2f_table(tab);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kSelWarps + w;
  if (g >= (int64_t)hq * t) return;
  const int64_t h = g / t, i = g % t;
  const int a = (int)admissible_prefix(i, t, block, segment);
  const SelWarpLayout L = sel_layout(t);
  unsigned char* base = smem + (size_t)w * L.per_warp();
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(base);            // [pow2]
  float* sv = reinterpret_cast<float*>(base + (size_t)L.pow2 * 8);                   // [tpad]
  uint32_t* bits = reinterpret_cast<uint32_t*>(base + (size_t)L.pow2 * 8 + (size_t)L.tpad * 4);  // [words]
  const float* in = rows_in + (h * t + i) * t;
  for (int j = lane; j < a; j += 32) sv[j] = in[j];
  __syncwarp();
  if (mode == 0) {
    float mx = -INFINITY;
    for (int j = lane; j < a; j += 32) mx = fmaxf(mx, sv[j]);
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int j = lane; j < a; j += 32) sv[j] = expf_glibc(__fsub_rn(sv[j], mx), tab);
    __syncwarp();
    float denom = 0.0f;
    if (lane == 0) {
      int j = 0;
      for (; j + 8 <= a; j += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = sv[j + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) denom = __fadd_rn(denom, v[u]);
      }
      for (; j < a; ++j) denom = __fadd_rn(denom, sv[j]);
    }
    denom = __shfl_sync(0xffffffffu, denom, 0);
    for (int j = lane; j < a; j += 32) sv[j] = __fdiv_rn(sv[j], denom);
    __syncwarp();
    if (scores_out) {
      float* so = scores_out + (h * t + i) * t;
      for (int64_t j = lane; j < t; j += 32) so[j] = j < a ? sv[j] : 0.0f;
    }
  }
  if (!select) return;

  // ---- candidate set C = {j < a : v_j >= theta}
  const int k_top = top_k > 0 ? min(top_k, a) : 0;
  bool all = false;
  {
    bool bad = false;  // negative / non-finite scores: no threshold argument, sort everything
    for (int j = lane; j < a; j += 32) bad |= !(sv[j] >= 0.0f) || !(sv[j] <= 3.0e38f);
    all = __any_sync(0xffffffffu, bad);
  }
  uint32_t theta = 0;
  const double margin = 4.0 * (double)a * 5.960464477539063e-8;
  if (!all) {
    auto crit = [&](uint32_t th) {
      if (k_top > 0) {
        int c = 0;
        for (int j = lane; j < a; j += 32) c += __float_as_uint(sv[j]) >= th;
        return warp_sum_i(c) >= k_top;
      }
      // f32 sum in any order: within a * 2^-24 < 1.3e-4 of the exact mass for
      // a <= 2048 probabilities summing to <= 1 (and a * 2^-24 in general), so a
      // 4 a 2^-24 margin keeps the reference's sequential double sum over C
      // >= tau (larger grids: the margin scales with a)
      float s = 0.0f;
      for (int j = lane; j < a; j += 32)
        if (__float_as_uint(sv[j]) >= th) s += sv[j];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      return (double)s >= tau + margin;
    };
    if (!crit(0u)) {
      all = true;
    } else {
      uint32_t lo = 0u, hi = 0x7f800001u;  // crit(lo) holds, crit(hi) fails (no finite v >= +inf bits + 1)
      // tau mode: any theta with crit(theta) is a valid candidate bound; stopping
      // once theta is known to the exponent and 4 mantissa bits (C at most ~6%
      // wider than the minimal set) leaves the exact prefix to the bisection over C
      const uint32_t stop = (k_top > 0) ? 1u : (1u << 19);
      while (hi - lo > stop) {
        const uint32_t mid = lo + (hi - lo) / 2u;
        if (crit(mid)) lo = mid;
        else hi = mid;
      }
      theta = lo;
    }
  }
  int take = 0;
  // Exact path (no sort): when every candidate is >= 2^-29, any double sum of
  // candidates is exact (all partial sums lie below 2, whose ulp 2^-52 divides
  // every such float), so the reference's sequential cumulative sum over the
  // sorted prefix equals the order-free sum of the same top-k set.  The prefix
  // is then {v > v*} plus the first ties v == v* in index order, where v* is
  // the largest value with sum_{v >= v*} >= tau (bisection over float bits,
  // exact warp-reduced double sums).
  bool exact_done = false;
  int nc = 0;  // exact path: candidates compacted into keys[]
  if (!all && k_top == 0 && tau > 0.0) {
    float vmin = INFINITY;
    for (int j = lane; j < a; j += 32)
      if (__float_as_uint(sv[j]) >= theta) vmin = fminf(vmin, sv[j]);
    for (int o = 16; o > 0; o >>= 1) vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
    if (vmin >= 1.862645149230957e-09f) {  // 2^-29
      // candidates compacted into keys[] (value bits << 32 | index), ascending index
      for (int j0 = 0; j0 < a; j0 += 32) {
        const int j = j0 + lane;
        const bool in_c = j < a && __float_as_uint(sv[j]) >= theta;
        const unsigned bal = __ballot_sync(0xffffffffu, in_c);
        if (in_c) keys[nc + __popc(bal & ((1u << lane) - 1))] = ((unsigned long long)__float_as_uint(sv[j]) << 32) | (unsigned)j;
        nc += __popc(bal);
      }
      __syncwarp();
      auto mass = [&](uint32_t th, bool strict) {  // sum of the candidates >= th (> th); exact when < 2
        double sum = 0.0;
        for (int k = lane; k < nc; k += 32) {
          const uint32_t vb = (uint32_t)(keys[k] >> 32);
          if (strict ? vb > th : vb >= th) sum += (double)__uint_as_float(vb);
        }
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        return sum;
      };
      const double total = mass(theta, false);
      exact_done = total < 2.0 && total >= tau;  // all partial sums below 2 (scores need not be probabilities)
    }
    if (exact_done) {
      auto mass = [&](uint32_t th, bool strict) {
        double sum = 0.0;
        for (int k = lane; k < nc; k += 32) {
          const uint32_t vb = (uint32_t)(keys[k] >> 32);
          if (strict ? vb > th : vb >= th) sum += (double)__uint_as_float(vb);
        }
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        return sum;
      };
      uint32_t lo = theta, hi = 0x7f800001u;  // mass(lo) >= tau (the margin above), mass(hi) = 0 < tau
      while (hi - lo > 1u) {
        const uint32_t mid = lo + (hi - lo) / 2u;
        if (mass(mid, false) >= tau) lo = mid;
        else hi = mid;
      }
      const uint32_t vstar = lo;
      const double s_gt = mass(vstar, true);
      int gt = 0;
      for (int k = lane; k < nc; k += 32) gt += (uint32_t)(keys[k] >> 32) > vstar;
      gt = warp_sum_i(gt);
      // ties v == v* in ascending index order until the sum reaches tau
      int r = 0;
      if (lane == 0) {
        double cum = s_gt;
        for (int k = 0; k < nc; ++k)
          if ((uint32_t)(keys[k] >> 32) == vstar) {
            cum += (double)__uint_as_float(vstar);
            ++r;
            if (cum >= tau) break;
          }
      }
      r = __shfl_sync(0xffffffffu, r, 0);
      take = gt + r;
      for (int x = lane; x < L.words; x += 32) bits[x] = 0u;
      __syncwarp();
      int tie_seen = 0;
      for (int k0 = 0; k0 < nc; k0 += 32) {
        const int k = k0 + lane;
        const uint32_t vb = k < nc ? (uint32_t)(keys[k] >> 32) : 0u;
        const bool tie = k < nc && vb == vstar;
        const unsigned tb = __ballot_sync(0xffffffffu, tie);
        const bool pick = k < nc && (vb > vstar || (tie && tie_seen + __popc(tb & ((1u << lane) - 1)) < r));
        if (pick) {
          const unsigned j = (unsigned)(keys[k] & 0xffffffffu);
          atomicOr(&bits[j >> 5], 1u << (j & 31));
        }
        tie_seen += __popc(tb);
      }
      __syncwarp();
      exact_done = true;
    }
  }
  for (int pass = 0; pass < 2 && !exact_done; ++pass) {
    int nc = 0;
    for (int j0 = 0; j0 < a; j0 += 32) {
      const int j = j0 + lane;
      const bool in_c = j < a && (all || __float_as_uint(sv[j]) >= theta);
      const unsigned bal = __ballot_sync(0xffffffffu, in_c);
      if (in_c)
        keys[nc + __popc(bal & ((1u << lane) - 1))] =
            ((unsigned long long)(~float_order_key(sv[j])) << 32) | (unsigned)j;
      nc += __popc(bal);
    }
    int n2 = 32;
    while (n2 < nc) n2 <<= 1;
    for (int k = nc + lane; k < n2; k += 32) keys[k] = ~0ull;
    __syncwarp();
    warp_bitonic(keys, n2, lane);
    if (k_top > 0) {
      take = min(k_top, nc);
      break;
    }
    // the reference's chain (line 187-196): double cumulative sum in sorted order
    int tk = -1;
    if (lane == 0) {
      double cum = 0.0;
      for (int k0 = 0; k0 < nc && tk < 0; k0 += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (k0 + u < nc) ? sv[keys[k0 + u] & 0xffffffffu] : 0.0f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (k0 + u >= nc || tk >= 0) break;
          cum += (double)v[u];
          if (cum >= tau) tk = k0 + u + 1;
        }
      }
    }
    tk = __shfl_sync(0xffffffffu, tk, 0);
    if (tk >= 0) {
      take = tk;
      break;
    }
    if (all) {  // fallback (line 188): every admissible block
      take = a;
      break;
    }
    all = true;  // cannot happen past the 1e-9 margin; stay exact regardless
    __syncwarp();
  }
  // ---- the mask row as a bitmap: the taken prefix, then the forced blocks
  if (!exact_done) {
    for (int x = lane; x < L.words; x += 32) bits[x] = 0u;
    __syncwarp();
    for (int k = lane; k < take; k += 32) {
      const unsigned j = (unsigned)(keys[k] & 0xffffffffu);
      atomicOr(&bits[j >> 5], 1u << (j & 31));
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (forced_first && t > 0) bits[0] |= 1u;
    if (forced_band) {
      int64_t lo, hi;
      if (segment == 0) {
        lo = i;
        hi = i + 1;
      } else {
        const int64_t per = segment / block;
        lo = (i / per) * per;
        hi = min64(lo + per, t);
      }
      for (int64_t j = lo; j < hi; ++j) bits[j >> 5] |= 1u << (j & 31);
    }
  }
  __syncwarp();
  if (mask) {
    uint8_t* mo = mask + (h * t + i) * t;
    if ((t & 3) == 0) {
      uint32_t* mo4 = reinterpret_cast<uint32_t*>(mo);
      for (int64_t q4 = lane; q4 < t / 4; q4 += 32) {
        const uint32_t nib = (bits[q4 >> 3] >> ((q4 & 7) * 4)) & 0xfu;
        mo4[q4] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
      }
    } else {
      for (int64_t j = lane; j < t; j += 32) mo[j] = (uint8_t)((bits[j >> 5] >> (j & 31)) & 1u);
    }
  }
  // ascending compaction of the selected blocks + coverage partial (double, j ascending)
  int cnt = 0;
  double cov = 0.0;
  int32_t* out = kv_idx ? kv_idx + (h * t + i) * t : nullptr;
  for (int64_t j0 = 0; j0 < t; j0 += 32) {
    const unsigned word = bits[j0 >> 5];
    const int64_t j = j0 + lane;
    const bool sel = j < t && ((word >> lane) & 1u);
    if (sel && out) out[cnt + __popc(word & ((1u << lane) - 1))] = (int32_t)j;
    cnt += __popc(word);
    if (mode == 0 && row_cov && sel && j < a) cov += (double)sv[j];
  }
  // pooled-score coverage (pipeline.hpp:186-191): the reference adds the selected
  // probabilities in ascending order; a lane-parallel double sum differs by
  // < cnt * 2^-53 (the report's tolerance is 1e-9)
  if (mode == 0 && row_cov)
    for (int o = 16; o > 0; o >>= 1) cov += __shfl_xor_sync(0xffffffffu, cov, o);
  if (lane == 0) {
    if (kv_cnt) kv_cnt[h * t + i] = cnt;
    if (row_cov) row_cov[h * t + i] = cov;
  }
}

inline size_t select_smem(int64_t t) {
  int64_t pow2 = 1;
  while (pow2 < t) pow2 <<= 1;
  return (size_t)pow2 * 8 + (size_t)((t + 3) & ~3) * 4 + (size_t)t + 16;
}

}  // namespace

size_t select_workspace_bytes(int hq, int64_t n, int d, int64_t block) {
  const int64_t t = ceil_div(n, block);
  return 2 * (size_t)hq * t * d * 4 + (size_t)hq * t * t * 4 + (size_t)hq * t * 8 + 1024;
}

int launch_pool(const void* x, int dtype, int src_heads, int dst_heads, const int32_t* perm, int64_t n, int d,
                int64_t block, float* pooled, cudaStream_t st) {
  const int64_t t = ceil_div(n, block);
  if (t == 0) return PBS_OK;
  const int group = dst_heads / src_heads;
  if (dtype == PBS_DTYPE_BF16 && d % 8 == 0 && d / 8 <= 128 && (uintptr_t)x % 16 == 0) {
    const int per_cta = 128 / (d / 8);
    pool_bf16x8_kernel<<<dim3((unsigned)ceil_div(t, per_cta), (unsigned)dst_heads), 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), group, perm, n, d, block, t, pooled);
    PBS_LAUNCH_CHECK("pool_bf16x8_kernel");
    return PBS_OK;
  }
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

static int launch_select_common(int mode, const float* rows_in, int hq, int64_t t, int64_t block,
                                int64_t segment, double tau, int top_k, int forced_first, int forced_band, int select,
                                float* scores_out, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt, double* row_cov,
                                cudaStream_t st) {
  if (t == 0 || hq == 0) return PBS_OK;
  if (t > 16384) return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "block grid wider than 16384 blocks");
  const size_t smem = sel_layout(t).per_warp() * kSelWarps;
  if (smem <= 200 * 1024) {
    static DeviceOnce attr_once;
    if (int rc = once_per_device(attr_once, [] {
          PBS_CUDA_CHECK(
              cudaFuncSetAttribute(select_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
          return (int)PBS_OK;
        }))
      return rc;
    select_warp_kernel<<<(unsigned)ceil_div((int64_t)hq * t, kSelWarps), kSelWarps * 32, smem, st>>>(
        mode, rows_in, hq, t, block, segment, tau, top_k, forced_first, forced_band, select, scores_out, mask, kv_idx,
        kv_cnt, row_cov);
    PBS_LAUNCH_CHECK("select_warp_kernel");
    return PBS_OK;
  }
  // very wide grids (t > ~4000 blocks): one CTA per row with the shared-memory bitonic sort
  const size_t smem1 = select_smem(t);
  static DeviceOnce attr_once1;
  if (int rc = once_per_device(attr_once1, [] {
        PBS_CUDA_CHECK(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        return (int)PBS_OK;
      }))
    return rc;
  select_kernel<<<dim3((unsigned)t, (unsigned)hq), kSelThreads, smem1, st>>>(
      mode, rows_in, t, block, segment, tau, top_k, forced_first, forced_band, select, scores_out, mask, kv_idx,
      kv_cnt, row_cov);
  PBS_LAUNCH_CHECK("select_kernel");
  return PBS_OK;
}

int launch_score_select(const float* qbar, const float* kbar, float* logits_ws, int hq, int64_t t, int d,
                        int64_t block, int64_t segment, float scale, double tau, int forced_first, int forced_band,
                        int select, float* scores_out, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt,
                        double* row_cov, cudaStream_t st, int top_k) {
  if (t == 0 || hq == 0) return PBS_OK;
  const dim3 grid((unsigned)ceil_div(t, xgemm::kTile), (unsigned)ceil_div(t, xgemm::kTile), (unsigned)hq);
  block_logits_kernel<<<grid, xgemm::kThreads, 0, st>>>(qbar, kbar, t, d, block, segment, scale, logits_ws);
  PBS_LAUNCH_CHECK("block_logits_kernel");
  return launch_select_common(0, logits_ws, hq, t, block, segment, tau, top_k, forced_first, forced_band, select,
                              scores_out, mask, kv_idx, kv_cnt, row_cov, st);
}

int launch_select_from_scores(const float* scores, int hq, int64_t t, int64_t block, int64_t segment, double tau,
                              int forced_first, int forced_band, uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt,
                              cudaStream_t st, int top_k) {
  return launch_select_common(1, scores, hq, t, block, segment, tau, top_k, forced_first, forced_band, 1, nullptr, mask,
                              kv_idx, kv_cnt, nullptr, st);
}

}  // namespace pbs_b200

// ---- mask -> attention lists, coverage reduction (attention_coverage) ------------
namespace pbs_b200 {
namespace {

// one warp per (head, block row): ascending compaction of the row's selected blocks
__global__ void mask_to_lists_kernel(const uint8_t* __restrict__ mask, int64_t rows, int64_t t,
                                     int32_t* __restrict__ kv_idx, int32_t* __restrict__ kv_cnt) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= rows) return;
  const uint8_t* m = mask + g * t;
  int32_t* out = kv_idx + g * t;
  int cnt = 0;
  for (int64_t j0 = 0; j0 < t; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool sel = j < t && m[j] != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, sel);
    if (sel) out[cnt + __popc(bal & ((1u << lane) - 1))] = (int32_t)j;
    cnt += __popc(bal);
  }
  if (lane == 0) kv_cnt[g] = cnt;
}

// coverage[h] = (1/N) sum_i exp(lse_sparse[h][i] - lse_dense[h][i]): each row's
// probabilities sum to 1 over its causal keys, so the reference's covered/total
// (pipeline.hpp:216-242) is the mean per-row covered mass.  Double accumulation.
__global__ void coverage_reduce_kernel(const float* __restrict__ ls, const float* __restrict__ ld, int64_t n,
                                       double* __restrict__ coverage) {
  const int h = blockIdx.x;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const float a = ls[(int64_t)h * n + i], b = ld[(int64_t)h * n + i];
    if (a != -INFINITY && b != -INFINITY) acc += exp((double)a - (double)b);
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) coverage[h] = n > 0 ? acc / (double)n : 0.0;
  }
}

}  // namespace

int launch_mask_to_lists(const uint8_t* mask, int hq, int64_t t, int32_t* kv_idx, int32_t* kv_cnt, cudaStream_t st) {
  const int64_t rows = (int64_t)hq * t;
  if (rows == 0) return PBS_OK;
  mask_to_lists_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(mask, rows, t, kv_idx, kv_cnt);
  PBS_LAUNCH_CHECK("mask_to_lists_kernel");
  return PBS_OK;
}

int launch_coverage_reduce(const float* lse_sparse, const float* lse_dense, int hq, int64_t n, double* coverage,
                           cudaStream_t st) {
  if (hq == 0) return PBS_OK;
  coverage_reduce_kernel<<<(unsigned)hq, 1024, 0, st>>>(lse_sparse, lse_dense, n, coverage);
  PBS_LAUNCH_CHECK("coverage_reduce_kernel");
  return PBS_OK;
}

}  // namespace pbs_b200
