// importance.cu -- stage 1 of Algorithm 1 on sm_100a.
//
//  K1  estimate_key_importance  (permutation.hpp:143-178)   exact fp32 restatement
//  K2  build_key_permutation    (permutation.hpp:182-201)   segmented stable sort + inverse
//  K3  build_query_permutation  (permutation.hpp:206-275)   centroids, cosine argmax, group sort
//
// Exactness.  The permutations are compared bit-for-bit with the reference, so
// every floating-point value that feeds a comparison is produced by the same
// IEEE operations in the same order as the reference's scalar loops:
//  * dot products run c = 0..d-1 sequentially per output (a register-tiled
//    SIMT GEMM has exactly that per-output order).  For bf16 inputs the
//    products are exact in fp32, so FFMA equals the reference's mul-then-add;
//    f32 inputs use __fmul_rn + __fadd_rn (the reference build has no FMA).
//  * the softmax denominator is a sequential fp32 sum over all N keys (one
//    thread per query row: a dependent chain of N adds), the score
//    accumulation a sequential sum over the `take` rows per key.
//  * exp is the device port of glibc expf (expf_glibc.cuh).
// None of this is tensor-core work: the estimate is CUDA-core fp32, and the
// tensor cores are reserved for the attention kernel.
#include <algorithm>

#include "common.cuh"
#include "expf_glibc.cuh"
#include "kernels.h"

namespace pbs_b200 {

namespace {

constexpr int kTile = 128;   // rows of A and of B per CTA
constexpr int kChunk = 16;   // d-chunk staged in smem
constexpr int kPad = 4;      // smem row padding (floats)
constexpr int kThreads = 256;

// acc[a][b] = dot(A[row_a], B[row_b]) over c = 0..d-1 in order.  A rows are
// a_base[0..a_rows), B rows b_base[0..b_rows) (both row-major, stride d).
// Thread (tx, ty) owns A rows {ty*4+r, 64+ty*4+r} and B rows {tx*4+r, 64+tx*4+r}.
template <typename TA, typename TB, bool kExact>
__device__ __forceinline__ void exact_dot_tile(const TA* __restrict__ a_base, int a_rows,
                                               const TB* __restrict__ b_base, int b_rows, int d,
                                               float (&acc)[8][8], float (*As)[kTile + kPad],
                                               float (*Bs)[kTile + kPad]) {
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  const int lrow = tid >> 1;        // 0..127
  const int lcol = (tid & 1) * 8;   // 0 or 8
  for (int c0 = 0; c0 < d; c0 += kChunk) {
    const int kc = min(kChunk, d - c0);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + lcol + u;
      float av = 0.0f, bv = 0.0f;
      if (lcol + u < kc) {
        if (lrow < a_rows) av = to_f32(a_base[(int64_t)lrow * d + c]);
        if (lrow < b_rows) bv = to_f32(b_base[(int64_t)lrow * d + c]);
      }
      As[lcol + u][lrow] = av;
      Bs[lcol + u][lrow] = bv;
    }
    __syncthreads();
    for (int cc = 0; cc < kc; ++cc) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cc][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cc][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cc][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cc][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (kExact) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
          else acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
        }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int tile_row(int idx, int t) { return (idx < 4 ? 0 : 64) + t * 4 + (idx & 3); }

// K1a: E[h][j][i] = (q[r0+i] . k[j]) * scale, rowmax[h][i] = max_j.
// grid (ceil(N/128), ceil(take/128), Hq).  E is key-major so that the
// per-row denominator chains (K1c) read 128-byte lines per step.
template <typename T, bool kExact>
__global__ void __launch_bounds__(kThreads) importance_logits_kernel(
    const T* __restrict__ q, const T* __restrict__ k, int group, int64_t n, int d, int take,
    float scale, float* __restrict__ E, unsigned* __restrict__ rowmax) {
  __shared__ __align__(16) float As[kChunk][kTile + kPad];
  __shared__ __align__(16) float Bs[kChunk][kTile + kPad];
  const int h = blockIdx.z;
  const int64_t j0 = (int64_t)blockIdx.x * kTile;
  const int i0 = blockIdx.y * kTile;
  const int64_t r0 = n - take;
  const T* a_base = q + ((int64_t)h * n + r0 + i0) * d;
  const T* b_base = k + ((int64_t)(h / group) * n + j0) * d;
  const int a_rows = min(kTile, take - i0);
  const int b_rows = (int)min64(kTile, n - j0);
  float acc[8][8];
  exact_dot_tile<T, T, kExact>(a_base, a_rows, b_base, b_rows, d, acc, As, Bs);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float* Eh = E + (int64_t)h * n * take;
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) {
    const int i = tile_row(ii, ty);
    float mx = -INFINITY;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = tile_row(jj, tx);
      const float v = __fmul_rn(acc[ii][jj], scale);  // logits[j] = acc * scale (line 166)
      if (i < a_rows && j < b_rows) {
        Eh[(j0 + j) * take + i0 + i] = v;
        mx = fmaxf(mx, v);
      }
    }
    // reduce over the 16 threads sharing this row (same ty, lanes tx)
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (tx == 0 && i < a_rows) atomic_max_float(&rowmax[(int64_t)h * take + i0 + i], mx);
  }
}

// K1b: E = expf(E - mx_i) in place (lines 170-171), all heads.
template <int kTake>
__global__ void importance_exp_kernel_t(float* __restrict__ E, const unsigned* __restrict__ rowmax,
                                        int64_t n, int64_t total) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int i = (int)(e % kTake);
    const int64_t h = e / ((int64_t)kTake * n);
    const float mx = decode_order_key(rowmax[h * kTake + i]);
    E[e] = expf_glibc(__fsub_rn(E[e], mx));
  }
}

__global__ void importance_exp_generic_kernel(float* __restrict__ E, const unsigned* __restrict__ rowmax,
                                              int take, int64_t n, int64_t total) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int i = (int)(e % take);
    const int64_t h = e / ((int64_t)take * n);
    const float mx = decode_order_key(rowmax[h * take + i]);
    E[e] = expf_glibc(__fsub_rn(E[e], mx));
  }
}

// K1c: denom_i = sum_j E[j][i] in order j = 0..N-1 (lines 169-173), then
// w_i = 1 / (denom * take) (line 174).  One thread per (head, row): a
// dependent chain of N fp32 adds; consecutive lanes read consecutive i.
__global__ void importance_denom_kernel(const float* __restrict__ E, int hq, int take, int64_t n,
                                        float* __restrict__ w) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)hq * take) return;
  const int64_t h = g / take;
  const int i = (int)(g % take);
  const float* p = E + h * n * take + i;
  float denom = 0.0f;
  int64_t j = 0;
  constexpr int U = 16;
  for (; j + U <= n; j += U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(p + (j + u) * take);
#pragma unroll
    for (int u = 0; u < U; ++u) denom = __fadd_rn(denom, v[u]);
  }
  for (; j < n; ++j) denom = __fadd_rn(denom, __ldg(p + j * take));
  w[g] = __fdiv_rn(1.0f, __fmul_rn(denom, (float)take));
}

// K1d: s[j] = sum_i E[j][i] * w_i in order i = r0..N-1 (line 175), with the
// product rounded before the add (no contraction in the reference build).
// CTA = 128 keys; the [128 x 32] E tile is staged through smem so that the
// global reads are 128-byte rows and each thread then walks its key's row.
__global__ void __launch_bounds__(128) importance_scores_kernel(const float* __restrict__ E,
                                                                const float* __restrict__ w,
                                                                int take, int64_t n,
                                                                float* __restrict__ scores) {
  __shared__ float tile[128][33];
  __shared__ float ws[32];
  const int h = blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * 128;
  const int tid = threadIdx.x;
  const float* Eh = E + (int64_t)h * n * take;
  float s = 0.0f;
  for (int i0 = 0; i0 < take; i0 += 32) {
    const int ic = min(32, take - i0);
    // load rows j0..j0+127, columns i0..i0+ic: thread t loads (row t/32*.., col t%32)
    for (int e = tid; e < 128 * 32; e += 128) {
      const int r = e >> 5, c = e & 31;
      float v = 0.0f;
      if (c < ic && j0 + r < n) v = Eh[(j0 + r) * take + i0 + c];
      tile[r][c] = v;
    }
    if (tid < 32) ws[tid] = tid < ic ? w[(int64_t)h * take + i0 + tid] : 0.0f;
    __syncthreads();
    for (int c = 0; c < ic; ++c) s = __fadd_rn(s, __fmul_rn(tile[tid][c], ws[c]));
    __syncthreads();
  }
  if (j0 + tid < n) scores[(int64_t)h * n + j0 + tid] = s;
}

// ---- K2: segmented sort ------------------------------------------------------
// One CTA per (segment, head).  Keys are unique 64-bit composites
// (primary << 32 | local index), so a bitonic sort yields exactly the
// stable_sort order of the reference (ties by ascending index).
//  key_kind 0: primary = ~order(score)   -> descending scores (permutation.hpp:195-197)
//  key_kind 1: primary = group           -> ascending groups  (permutation.hpp:269-271)
__global__ void segmented_sort_kernel(const void* __restrict__ keys, int key_kind, int64_t n,
                                      int segment, int pow2, int32_t* __restrict__ perm,
                                      int32_t* __restrict__ inv) {
  extern __shared__ unsigned long long sk[];
  const int64_t h = blockIdx.y;
  const int64_t base = (int64_t)blockIdx.x * segment;
  for (int t = threadIdx.x; t < pow2; t += blockDim.x) {
    unsigned long long key = ~0ull;
    if (t < segment) {
      uint32_t prim;
      if (key_kind == 0) prim = ~float_order_key(static_cast<const float*>(keys)[h * n + base + t]);
      else prim = static_cast<const uint32_t*>(keys)[h * n + base + t];
      key = ((unsigned long long)prim << 32) | (unsigned)t;
    }
    sk[t] = key;
  }
  __syncthreads();
  for (int size = 2; size <= pow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < pow2 / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long a = sk[lo], b = sk[hi];
        if ((a > b) == up) {
          sk[lo] = b;
          sk[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < segment; t += blockDim.x) {
    const int local = (int)(sk[t] & 0xffffffffu);
    perm[h * n + base + t] = (int32_t)(base + local);
    if (inv) inv[h * n + base + local] = (int32_t)(base + t);
  }
}

__global__ void identity_tail_kernel(int32_t* __restrict__ perm, int32_t* __restrict__ inv, int heads,
                                     int64_t n, int64_t start) {
  const int64_t span = n - start;
  const int64_t total = span * heads;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = e / span, p = start + e % span;
    if (perm) perm[h * n + p] = (int32_t)p;
    if (inv) inv[h * n + p] = (int32_t)p;
  }
}

// ---- K3: query groups (build_query_permutation, permutation.hpp:218-260) ----
// centroids of key blocks: sequential row sums, /= cc, then sq in c order.
template <typename T>
__global__ void centroid_kernel(const T* __restrict__ k, int64_t n, int d, int64_t block, int64_t tc,
                                float* __restrict__ cent, float* __restrict__ cnorm) {
  extern __shared__ float sdst[];
  const int64_t h = blockIdx.y;
  const int64_t j = blockIdx.x;
  const int64_t c0 = j * block;
  const int64_t cc = min(block, n - c0);
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.0f;
    for (int64_t r = c0; r < c0 + cc; ++r) acc = __fadd_rn(acc, to_f32(k[(h * n + r) * d + c]));
    acc = __fdiv_rn(acc, (float)cc);
    sdst[c] = acc;
    cent[(h * tc + j) * d + c] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float sq = 0.0f;
    for (int c = 0; c < d; ++c) sq = __fadd_rn(sq, __fmul_rn(sdst[c], sdst[c]));
    cnorm[h * tc + j] = __fsqrt_rn(sq);
  }
}

template <typename T>
__global__ void qnorm_kernel(const T* __restrict__ q, int64_t rows, int d, float* __restrict__ qn) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= rows) return;
  const T* p = q + g * d;
  float s = 0.0f;
  for (int c = 0; c < d; ++c) {
    const float x = to_f32(p[c]);
    s = __fadd_rn(s, __fmul_rn(x, x));
  }
  qn[g] = __fsqrt_rn(s);
}

// sims = dot / (qnorm * cnorm) over [N x tc] tiles; per-row argmax with the
// first index winning ties, through a packed 64-bit atomicMax
// (order(sim) << 32 | ~j).  Only sims > -1 can win (best_sim starts at -1).
template <typename T>
__global__ void __launch_bounds__(kThreads) query_group_kernel(
    const T* __restrict__ q, const float* __restrict__ cent, const float* __restrict__ qn,
    const float* __restrict__ cn, int k_group, int64_t n, int d, int64_t tc,
    unsigned long long* __restrict__ best) {
  __shared__ __align__(16) float As[kChunk][kTile + kPad];
  __shared__ __align__(16) float Bs[kChunk][kTile + kPad];
  const int h = blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.x * kTile;
  const int64_t j0 = (int64_t)blockIdx.y * kTile;
  const int hk = h / k_group;
  const int a_rows = (int)min64(kTile, n - i0);
  const int b_rows = (int)min64(kTile, tc - j0);
  float acc[8][8];
  // centroids are f32 (not bf16-exact): always the non-fused mul + add path
  exact_dot_tile<T, float, false>(q + ((int64_t)h * n + i0) * d, a_rows,
                                  cent + ((int64_t)hk * tc + j0) * d, b_rows, d, acc, As, Bs);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) {
    const int i = tile_row(ii, ty);
    unsigned long long bk = 0ull;
    const float qv = (i < a_rows) ? qn[(int64_t)h * n + i0 + i] : 0.0f;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = tile_row(jj, tx);
      if (i < a_rows && j < b_rows) {
        const float cv = cn[(int64_t)hk * tc + j0 + j];
        float sim = -1.0f;
        if (qv > 0.0f && cv > 0.0f) sim = __fdiv_rn(acc[ii][jj], __fmul_rn(qv, cv));
        if (sim > -1.0f) {  // NaN and <= -1 never win
          const unsigned long long key =
              ((unsigned long long)float_order_key(sim) << 32) | (0xffffffffu - (unsigned)(j0 + j));
          bk = key > bk ? key : bk;
        }
      }
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, bk, o);
      bk = other > bk ? other : bk;
    }
    if (tx == 0 && i < a_rows && bk) atomicMax(&best[(int64_t)h * n + i0 + i], bk);
  }
}

__global__ void query_group_finalize_kernel(const unsigned long long* __restrict__ best, int64_t total,
                                            int64_t tc, uint32_t* __restrict__ groups) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= total) return;
  const unsigned long long b = best[g];
  groups[g] = b ? (0xffffffffu - (uint32_t)(b & 0xffffffffu)) : (uint32_t)tc;
}

inline int grid_for(int64_t total, int threads) {
  const int64_t b = (total + threads - 1) / threads;
  return (int)min64(b, 148 * 32);
}

}  // namespace

size_t importance_workspace_bytes(int hq, int64_t n, int64_t block) {
  const int64_t take = min64(block, n);
  return (size_t)hq * n * take * 4 + (size_t)hq * take * 8 + 256;
}

int launch_importance(const void* q, const void* k, int dtype, int hq, int hkv, int64_t n, int d,
                      int64_t block, float scale, float* scores, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
  const int take = (int)min64(block, n);
  if (ws_bytes < importance_workspace_bytes(hq, n, block))
    return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "importance workspace too small");
  float* E = static_cast<float*>(ws);
  unsigned* rowmax = reinterpret_cast<unsigned*>(E + (size_t)hq * n * take);
  float* w = reinterpret_cast<float*>(rowmax + (size_t)hq * take);
  PBS_CUDA_CHECK(cudaMemsetAsync(rowmax, 0, sizeof(unsigned) * hq * take, st));
  const int group = hq / hkv;
  dim3 grid((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(take, kTile), (unsigned)hq);
  if (dtype == PBS_DTYPE_BF16)
    importance_logits_kernel<__nv_bfloat16, true><<<grid, kThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), group, n, d, take,
        scale, E, rowmax);
  else
    importance_logits_kernel<float, false><<<grid, kThreads, 0, st>>>(
        static_cast<const float*>(q), static_cast<const float*>(k), group, n, d, take, scale, E, rowmax);
  PBS_LAUNCH_CHECK("importance_logits_kernel");
  const int64_t total = (int64_t)hq * n * take;
  if (take == 128)
    importance_exp_kernel_t<128><<<grid_for(total, 256), 256, 0, st>>>(E, rowmax, n, total);
  else
    importance_exp_generic_kernel<<<grid_for(total, 256), 256, 0, st>>>(E, rowmax, take, n, total);
  PBS_LAUNCH_CHECK("importance_exp_kernel");
  const int64_t rows = (int64_t)hq * take;
  importance_denom_kernel<<<(unsigned)ceil_div(rows, 32), 32, 0, st>>>(E, hq, take, n, w);
  PBS_LAUNCH_CHECK("importance_denom_kernel");
  importance_scores_kernel<<<dim3((unsigned)ceil_div(n, 128), (unsigned)hq), 128, 0, st>>>(E, w, take, n,
                                                                                         scores);
  PBS_LAUNCH_CHECK("importance_scores_kernel");
  return PBS_OK;
}

int launch_identity(int32_t* perm, int heads, int64_t n, cudaStream_t st) {
  if (n == 0 || heads == 0) return PBS_OK;
  identity_tail_kernel<<<grid_for(n * heads, 256), 256, 0, st>>>(perm, nullptr, heads, n, 0);
  PBS_LAUNCH_CHECK("identity_tail_kernel");
  return PBS_OK;
}

int launch_segmented_sort(const void* keys, int key_kind, int heads, int64_t n, int64_t segment,
                          int32_t* perm, int32_t* inv, cudaStream_t st) {
  if (segment <= 0) return fail(PBS_ERR_CONFIG, "E_CONFIG", "segment size must be >= 1");
  const int64_t groups = n / segment;
  if (groups > 0) {
    if (segment > 8192)
      return fail(PBS_ERR_CONFIG, "E_CONFIG", "segment size > 8192 is not supported by the device sort");
    int pow2 = 1;
    while (pow2 < segment) pow2 <<= 1;
    const int threads = std::max(32, std::min(1024, pow2 / 2));
    const size_t smem = sizeof(unsigned long long) * pow2;
    segmented_sort_kernel<<<dim3((unsigned)groups, (unsigned)heads), threads, smem, st>>>(
        keys, key_kind, n, (int)segment, pow2, perm, inv);
    PBS_LAUNCH_CHECK("segmented_sort_kernel");
  }
  const int64_t start = groups * segment;
  if (start < n) {
    identity_tail_kernel<<<grid_for((n - start) * heads, 256), 256, 0, st>>>(perm, inv, heads, n, start);
    PBS_LAUNCH_CHECK("identity_tail_kernel");
  }
  return PBS_OK;
}

size_t query_perm_workspace_bytes(int hq, int64_t n, int d, int64_t block) {
  const int64_t tc = ceil_div(n, block);
  return (size_t)hq * tc * d * 4 + (size_t)hq * tc * 4 + (size_t)hq * n * 4 + (size_t)hq * n * 8 + 1024;
}

int launch_query_groups(const void* q, const void* k, int dtype, int hq, int k_heads, int64_t n, int d,
                        int64_t block, uint32_t* groups, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < query_perm_workspace_bytes(hq, n, d, block))
    return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "query permutation workspace too small");
  const int64_t tc = ceil_div(n, block);
  char* p = static_cast<char*>(ws);
  float* cent = reinterpret_cast<float*>(p);
  p += (size_t)hq * tc * d * 4;
  float* cn = reinterpret_cast<float*>(p);
  p += (size_t)hq * tc * 4;
  float* qn = reinterpret_cast<float*>(p);
  p += (size_t)hq * n * 4;
  p = reinterpret_cast<char*>(((uintptr_t)p + 15) & ~(uintptr_t)15);
  unsigned long long* best = reinterpret_cast<unsigned long long*>(p);
  PBS_CUDA_CHECK(cudaMemsetAsync(best, 0, sizeof(unsigned long long) * hq * n, st));
  const size_t csmem = sizeof(float) * d;
  if (dtype == PBS_DTYPE_BF16) {
    centroid_kernel<__nv_bfloat16><<<dim3((unsigned)tc, (unsigned)k_heads), 128, csmem, st>>>(
        static_cast<const __nv_bfloat16*>(k), n, d, block, tc, cent, cn);
    PBS_LAUNCH_CHECK("centroid_kernel");
    qnorm_kernel<__nv_bfloat16><<<(unsigned)ceil_div((int64_t)hq * n, 128), 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(q), (int64_t)hq * n, d, qn);
    PBS_LAUNCH_CHECK("qnorm_kernel");
    query_group_kernel<__nv_bfloat16>
        <<<dim3((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(tc, kTile), (unsigned)hq), kThreads, 0,
           st>>>(static_cast<const __nv_bfloat16*>(q), cent, qn, cn, hq / k_heads, n, d, tc, best);
  } else {
    centroid_kernel<float><<<dim3((unsigned)tc, (unsigned)k_heads), 128, csmem, st>>>(
        static_cast<const float*>(k), n, d, block, tc, cent, cn);
    PBS_LAUNCH_CHECK("centroid_kernel");
    qnorm_kernel<float><<<(unsigned)ceil_div((int64_t)hq * n, 128), 128, 0, st>>>(
        static_cast<const float*>(q), (int64_t)hq * n, d, qn);
    PBS_LAUNCH_CHECK("qnorm_kernel");
    query_group_kernel<float>
        <<<dim3((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(tc, kTile), (unsigned)hq), kThreads, 0,
           st>>>(static_cast<const float*>(q), cent, qn, cn, hq / k_heads, n, d, tc, best);
  }
  PBS_LAUNCH_CHECK("query_group_kernel");
  query_group_finalize_kernel<<<(unsigned)ceil_div((int64_t)hq * n, 256), 256, 0, st>>>(
      best, (int64_t)hq * n, tc, groups);
  PBS_LAUNCH_CHECK("query_group_finalize_kernel");
  return PBS_OK;
}

namespace {
__global__ void debug_expf_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = expf_glibc(x[i]);
}
}  // namespace

int launch_debug_expf(const float* x, float* y, int64_t n, cudaStream_t st) {
  if (n <= 0) return PBS_OK;
  debug_expf_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, y, n);
  PBS_LAUNCH_CHECK("debug_expf_kernel");
  return PBS_OK;
}

}  // namespace pbs_b200
