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
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include <cstdio>

#include "common.cuh"
#include "exact_gemm.cuh"
#include "expf_glibc.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "tc.cuh"

namespace pbs_b200 {

namespace {

using xgemm::kTile;
using xgemm::tile_row;

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ptx::smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// K1a: L[h][j][i] = (q[r0+i] . k[j]) * scale and rowmax[h][i] = max_j L.
// grid (ceil(N/128), ceil(take/128), Hq).  L is key-major ([j][i]) so that the
// per-row denominator chains (K1c) read 128-byte lines per step.
// kWide (bf16, d % 32 == 0): xgemm::tile_bf16_wide with dynamic shared memory.
template <typename T, bool kExact, bool kVec, bool kWide = false>
__global__ void __launch_bounds__(xgemm::kThreads, 2) importance_logits_kernel(
    const T* __restrict__ q, const T* __restrict__ k, int group, int64_t n, int64_t q_rows, int d, int take,
    float scale, float* __restrict__ L, unsigned* __restrict__ rowmax, int h0) {
  const int h = h0 + blockIdx.z;
  const int64_t j0 = (int64_t)blockIdx.x * kTile;
  const int i0 = blockIdx.y * kTile;
  // q holds q_rows rows per head (N, or just the last `take` rows), the
  // estimate reads its last `take`
  const int64_t r0 = q_rows - take;
  const T* a_base = q + ((int64_t)h * q_rows + r0 + i0) * d;
  const T* b_base = k + ((int64_t)(h / group) * n + j0) * d;
  const int a_rows = min(kTile, take - i0);
  const int b_rows = (int)min64(kTile, n - j0);
  float acc[8][8];
  if constexpr (kWide) {
    extern __shared__ __align__(16) unsigned char sm_dyn[];
    xgemm::tile_bf16_wide(a_base, a_rows, b_base, b_rows, d, acc, *reinterpret_cast<xgemm::SmemWide*>(sm_dyn));
  } else {
    __shared__ __align__(16) xgemm::Smem sm;
    xgemm::tile<T, T, kExact, kVec>(a_base, a_rows, b_base, b_rows, d, acc, sm);
  }
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float* Lh = L + (int64_t)h * n * take;
  float rmax[8];
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) rmax[ii] = -INFINITY;
  const bool vec_store = (take % 4 == 0);
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = tile_row(jj, tx);
    if (j >= b_rows) continue;
    float v[8];
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) {
      v[ii] = __fmul_rn(acc[ii][jj], scale);  // logits[j] = acc * scale (permutation.hpp:166)
      if (tile_row(ii, ty) < a_rows) rmax[ii] = fmaxf(rmax[ii], v[ii]);
    }
    float* dst = Lh + (j0 + j) * take + i0;
    if (vec_store && ty * 4 + 3 < a_rows && 64 + ty * 4 + 3 < a_rows) {
      *reinterpret_cast<float4*>(dst + ty * 4) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(dst + 64 + ty * 4) = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
        if (tile_row(ii, ty) < a_rows) dst[tile_row(ii, ty)] = v[ii];
    }
  }
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) {
    float mx = rmax[ii];
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int i = tile_row(ii, ty);
    if (tx == 0 && i < a_rows) atomic_max_float(&rowmax[(int64_t)h * take + i0 + i], mx);
  }
}

// K1b: E[j][i] = expf(L[j][i] - mx_i) in place (permutation.hpp:171), every
// element once, on the whole GPU (the sequential passes below only stream E).
// CTA = kExpKeys keys of one head; the row maxima are decoded into smem.
constexpr int kExpKeys = 128;
__global__ void __launch_bounds__(256) importance_exp_kernel(float* __restrict__ L, const unsigned* __restrict__ rowmax,
                                                             int take, int64_t n, int h0) {
  __shared__ float mx[1024];
  __shared__ uint64_t tab[32];
  load_exp2f_table(tab);
  const int h = h0 + blockIdx.y;
  for (int i = threadIdx.x; i < take && i < 1024; i += blockDim.x) mx[i] = decode_order_key(rowmax[(int64_t)h * take + i]);
  __syncthreads();
  const int64_t j0 = (int64_t)blockIdx.x * kExpKeys;
  const int64_t cnt = min64(kExpKeys, n - j0) * take;
  float* base = L + ((int64_t)h * n + j0) * take;
  if (take % 4 == 0 && take <= 1024) {
    // four 16-byte loads in flight per thread before any exp.  When take
    // divides 4 x blockDim (take = B = 128), a thread's row offset i never
    // changes (the CTA starts on a key boundary): its four maxima are hoisted.
    float4* b4 = reinterpret_cast<float4*>(base);
    const int64_t n4 = cnt / 4;
    if ((4 * (int)blockDim.x) % take == 0) {
      const int i = (4 * (int)threadIdx.x) % take;
      const float m0 = mx[i], m1 = mx[i + 1], m2 = mx[i + 2], m3 = mx[i + 3];
      for (int64_t e0 = threadIdx.x; e0 < n4; e0 += 4 * (int64_t)blockDim.x) {
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t e = e0 + (int64_t)u * blockDim.x;
          if (e < n4) x[u] = b4[e];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t e = e0 + (int64_t)u * blockDim.x;
          if (e >= n4) break;
          x[u].x = expf_glibc(__fsub_rn(x[u].x, m0), tab);
          x[u].y = expf_glibc(__fsub_rn(x[u].y, m1), tab);
          x[u].z = expf_glibc(__fsub_rn(x[u].z, m2), tab);
          x[u].w = expf_glibc(__fsub_rn(x[u].w, m3), tab);
          b4[e] = x[u];
        }
      }
      return;
    }
    for (int64_t e0 = threadIdx.x; e0 < n4; e0 += 4 * (int64_t)blockDim.x) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + (int64_t)u * blockDim.x;
        if (e < n4) x[u] = b4[e];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + (int64_t)u * blockDim.x;
        if (e >= n4) break;
        const int i = (int)((e * 4) % take);
        x[u].x = expf_glibc(__fsub_rn(x[u].x, mx[i]), tab);
        x[u].y = expf_glibc(__fsub_rn(x[u].y, mx[i + 1]), tab);
        x[u].z = expf_glibc(__fsub_rn(x[u].z, mx[i + 2]), tab);
        x[u].w = expf_glibc(__fsub_rn(x[u].w, mx[i + 3]), tab);
        b4[e] = x[u];
      }
    }
  } else {
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
      const int i = (int)(e % take);
      const float m = i < 1024 ? mx[i] : decode_order_key(rowmax[(int64_t)h * take + i]);
      base[e] = expf_glibc(__fsub_rn(base[e], m), tab);
    }
  }
}

// K1c: denom_i = sequential fp32 sum of E[j][i] over j = 0..N-1 (line 172), then
// w_i = 1 / (denom * take) (line 174).  One CTA per (head, 32 rows): warp 1
// streams 128-key x 32-row tiles of E into a shared-memory ring, one 2-D TMA
// copy per tile (the whole ring in flight), warp 0 is the adder, one dependent
// chain of N adds per lane.  Shapes whose row groups are not whole 16-byte
// pieces (take % 4 != 0 or a partial row group) take 4-byte cp.async copies.
constexpr int kJT = 256;    // keys per ring tile (one barrier round trip per 256 adds)
constexpr int kRing = 4;    // 4 tiles = 128 KB in flight

__device__ __forceinline__ void tma_load_3d_f32(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(ptx::smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(ptx::smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(64, 1) importance_denom_kernel(const __grid_constant__ CUtensorMap tm_e, bool tma,
                                                              const float* __restrict__ E, int take, int64_t n,
                                                              int h0, float* __restrict__ w) {
  extern __shared__ __align__(128) unsigned char dsm[];
  float (*ring)[kJT][32] = reinterpret_cast<float (*)[kJT][32]>(dsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + sizeof(float) * kRing * kJT * 32);
  uint64_t* empty = full + kRing;
  const int h = h0 + blockIdx.y;
  const int i0 = blockIdx.x * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rows = min(32, take - i0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      ptx::mbar_init(&full[s], tma ? 1 : 32);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int64_t ntiles = (n + kJT - 1) / kJT;
  const float* Eh = E + (int64_t)h * n * take;
  if (warp == 1) {
    for (int64_t t = 0; t < ntiles; ++t) {
      const int slot = (int)(t % kRing);
      ptx::mbar_wait(&empty[slot], (uint32_t)(((t / kRing) & 1) ^ 1));
      const int64_t jb = t * kJT;
      const int cnt = (int)min64(kJT, n - jb);
      if (tma) {
        // keys past N are zero-filled by the TMA unit; the box is always 4 KB
        if (lane == 0) {
          ptx::mbar_expect_tx(&full[slot], kJT * 32 * 4);
          tma_load_3d_f32(&ring[slot][0][0], &tm_e, &full[slot], i0, (int)jb, h);
        }
      } else {
        for (int jj = 0; jj < cnt; ++jj)
          if (lane < rows) cp_async4(&ring[slot][jj][lane], Eh + (jb + jj) * take + i0 + lane);
        cp_async_wait_all();
        ptx::mbar_arrive(&full[slot]);
      }
    }
  } else {
    float denom = 0.0f;
    for (int64_t t = 0; t < ntiles; ++t) {
      const int slot = (int)(t % kRing);
      ptx::mbar_wait(&full[slot], (uint32_t)((t / kRing) & 1));
      const int cnt = (int)min64(kJT, n - t * kJT);
      if (cnt == kJT) {
#pragma unroll
        for (int j0 = 0; j0 < kJT; j0 += 128) {
          float v[128];
#pragma unroll
          for (int jj = 0; jj < 128; ++jj) v[jj] = ring[slot][j0 + jj][lane];
#pragma unroll
          for (int jj = 0; jj < 128; ++jj) denom = __fadd_rn(denom, v[jj]);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[slot]);
      } else {
        for (int jj = 0; jj < cnt; ++jj) denom = __fadd_rn(denom, ring[slot][jj][lane]);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[slot]);
      }
    }
    if (lane < rows) w[(int64_t)h * take + i0 + lane] = __fdiv_rn(1.0f, __fmul_rn(denom, (float)take));
  }
}

// K1d: s[j] = sum_i E[j][i] * w_i in order i = 0..take-1 (line 175), the product
// rounded before the add.  CTA = 128 keys, one per thread; 32-row chunks of the
// keys' E rows double-buffered through smem (16-byte cp.async, rows padded to 36
// floats so each thread's 16-byte reads are bank-conflict free).
constexpr int kSK = 128;
constexpr int kSPad = 36;
__global__ void __launch_bounds__(kSK) importance_scores_kernel(const float* __restrict__ E,
                                                                const float* __restrict__ w, int take, int64_t n,
                                                                int h0, float* __restrict__ scores) {
  __shared__ __align__(16) float tile[2][kSK][kSPad];
  __shared__ float ws[2][32];
  const int h = h0 + blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * kSK;
  const int tid = threadIdx.x;
  const int keys = (int)min64(kSK, n - j0);
  const float* Eh = E + (int64_t)h * n * take;
  const bool vec = (take % 4 == 0);
  auto stage = [&](int buf, int i0) {
    const int ic = min(32, take - i0);
    if (tid < 32) ws[buf][tid] = tid < ic ? w[(int64_t)h * take + i0 + tid] : 0.0f;
    if (vec) {
      // ic is a multiple of 4 here: ic / 4 pieces per key
      const int pk = ic >> 2;
      for (int c = tid; c < keys * pk; c += kSK) {
        const int r = c / pk, q = c - r * pk;
        cp_async16(&tile[buf][r][4 * q], Eh + (j0 + r) * take + i0 + 4 * q);
      }
    } else {
      for (int c = tid; c < keys * ic; c += kSK) {
        const int r = c / ic, q = c - r * ic;
        cp_async4(&tile[buf][r][q], Eh + (j0 + r) * take + i0 + q);
      }
    }
    cp_async_commit();
  };
  float s = 0.0f;
  stage(0, 0);
  int buf = 0;
  for (int i0 = 0; i0 < take; i0 += 32, buf ^= 1) {
    const bool more = i0 + 32 < take;
    if (more) stage(buf ^ 1, i0 + 32);
    if (more) cp_async_wait_group1();
    else cp_async_wait_all();
    __syncthreads();
    const int ic = min(32, take - i0);
    if (ic == 32) {
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 e = *reinterpret_cast<const float4*>(&tile[buf][tid][c]);
        s = __fadd_rn(s, __fmul_rn(e.x, ws[buf][c]));
        s = __fadd_rn(s, __fmul_rn(e.y, ws[buf][c + 1]));
        s = __fadd_rn(s, __fmul_rn(e.z, ws[buf][c + 2]));
        s = __fadd_rn(s, __fmul_rn(e.w, ws[buf][c + 3]));
      }
    } else {
      for (int c = 0; c < ic; ++c) s = __fadd_rn(s, __fmul_rn(tile[buf][tid][c], ws[buf][c]));
    }
    __syncthreads();  // buf is refilled two chunks later
  }
  if (tid < keys) scores[(int64_t)h * n + j0 + tid] = s;
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

// |q_i| = sqrt(sum_c q_ic^2), sequential c (permutation.hpp:238-243).  One
// thread per row; rows are read 16 bytes at a time when d and the base allow
// (a row per lane: scalar 2-byte loads made every warp load touch 32 lines).
template <typename T>
__global__ void qnorm_kernel(const T* __restrict__ q, int64_t rows, int d, float* __restrict__ qn) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= rows) return;
  const T* p = q + g * d;
  float s = 0.0f;
  constexpr int kPer = 16 / (int)sizeof(T);
  if (d % kPer == 0 && (uintptr_t)q % 16 == 0) {
    for (int c = 0; c < d; c += kPer) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p + c));
      const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const float x = to_f32(e[u]);
        s = __fadd_rn(s, __fmul_rn(x, x));
      }
    }
  } else {
    for (int c = 0; c < d; ++c) {
      const float x = to_f32(p[c]);
      s = __fadd_rn(s, __fmul_rn(x, x));
    }
  }
  qn[g] = __fsqrt_rn(s);
}

// sims = dot / (qnorm * cnorm) over [N x tc] tiles; per-row argmax with the
// first index winning ties, through a packed 64-bit atomicMax
// (order(sim) << 32 | ~j).  Only sims > -1 can win (best_sim starts at -1).
template <typename T, bool kVec>
__global__ void __launch_bounds__(xgemm::kThreads) query_group_kernel(
    const T* __restrict__ q, const float* __restrict__ cent, const float* __restrict__ qn,
    const float* __restrict__ cn, int k_group, int64_t n, int d, int64_t tc,
    unsigned long long* __restrict__ best) {
  __shared__ __align__(16) xgemm::Smem sm;
  const int h = blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.x * kTile;
  const int64_t j0 = (int64_t)blockIdx.y * kTile;
  const int hk = h / k_group;
  const int a_rows = (int)min64(kTile, n - i0);
  const int b_rows = (int)min64(kTile, tc - j0);
  float acc[8][8];
  // centroids are f32 (not bf16-exact): always the non-fused mul + add path
  xgemm::tile<T, float, false, kVec>(q + ((int64_t)h * n + i0) * d, a_rows, cent + ((int64_t)hk * tc + j0) * d,
                                     b_rows, d, acc, sm);
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

// ---- K3 screen (bf16, d = 128): tensor-core cosine screen + exact re-check ----
// The assignment only needs each query's argmax.  The centroids (f32) are split
// into bf16 hi + lo parts, so q . (c_hi + c_lo) on the tensor cores (tcgen05,
// f32 accumulation in TMEM) is within 4.3e-5 |q||c| of the reference's
// sequential f32 dot (split residual 2^-18, accumulation 256 x 2^-23, the
// reference's own rounding 128 x 2^-24).  With delta = 1e-4 (2.3x that bound):
//  1. screen: a row whose best screened cosine beats every other centroid by
//     more than 2 delta has the reference's argmax; the other rows are listed
//     per KV head with their best screened score;
//  2. the listed rows are screened again (the same MMA sequence, so identical
//     scores): every centroid within 2 delta of the best is a candidate;
//  3. the candidates' cosines are computed exactly as the reference does
//     (sequential c, rounded products, IEEE division), argmax with the first
//     index on ties; a row with more than kScrCand candidates scans every
//     centroid exactly.
constexpr int kScrPad = 136;               // bf16 per padded centroid row (272 B; the TMA box reads the first 128)
constexpr int kScrCand = 16;               // candidates kept per listed row
constexpr float kScrDelta = 1e-4f;

// grid (tcp, k_heads): centroid j of KV head blockIdx.y; the column scales are
// padded to tcp (a multiple of the screen's 128-centroid chunk) with rinv 0 and
// pen -inf, so every chunk's scales are one aligned 512-byte bulk copy
__global__ void centroid_split_kernel(const float* __restrict__ cent, const float* __restrict__ cn, int64_t tc,
                                      int64_t tcp, __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo,
                                      float* __restrict__ rinv, float* __restrict__ pen) {
  const int64_t j = blockIdx.x;
  if (j >= tc) {
    if (threadIdx.x == 0) {
      rinv[blockIdx.y * tcp + j] = 0.0f;
      pen[blockIdx.y * tcp + j] = -INFINITY;
    }
    return;
  }
  const int64_t r = blockIdx.y * tc + j;
  for (int c = threadIdx.x; c < kScrPad; c += blockDim.x) {
    const float x = c < 128 ? cent[r * 128 + c] : 0.0f;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    hi[r * kScrPad + c] = h;
    lo[r * kScrPad + c] = __float2bfloat16_rn(x - __bfloat162float(h));
  }
  if (threadIdx.x == 0) {
    const float v = cn[r];
    rinv[blockIdx.y * tcp + j] = v > 0.0f ? 1.0f / v : 0.0f;
    pen[blockIdx.y * tcp + j] = v > 0.0f ? 0.0f : -INFINITY;
  }
}

struct Best2 {
  float m, s2;  // best and second-best scaled score
  int j;        // index of the best
};
__device__ __forceinline__ void best2_push(Best2& b, float v, int j) {
  if (v > b.m) {
    b.s2 = b.m;
    b.m = v;
    b.j = j;
  } else {
    b.s2 = fmaxf(b.s2, v);
  }
}
__device__ __forceinline__ Best2 best2_merge(Best2 a, Best2 o) {
  const bool ob = o.m > a.m || (o.m == a.m && o.j < a.j);
  Best2 r;
  r.m = ob ? o.m : a.m;
  r.j = ob ? o.j : a.j;
  r.s2 = ob ? fmaxf(o.s2, a.m) : fmaxf(a.s2, o.m);
  return r;
}

struct ScreenLists {
  int32_t* count;  // [k_heads] listed rows per KV head
  int32_t* rows;   // [k_heads][k_group * n] global row index h * n + i
  float* best;     // [k_heads][k_group * n] best screened (scaled) score of the row
  int32_t* cand;   // [k_heads][k_group * n][kScrCand]
  int32_t* cand_n; // [k_heads][k_group * n]
};

// K3 screen on the 5th-generation tensor cores.  Persistent CTAs (one per SM)
// walk tiles of 256 query rows (two 128-row sub-tiles) -- rows r0.. of one
// head (kListed = false: decide or list), or 256 of the rows listed for one KV
// head (kListed = true: emit candidates) -- and score each against every
// centroid of its KV head in chunks of 128 (N):
//   S_u = Q_u C_hi^T + Q_u C_lo^T  (per sub-tile u: 16 tcgen05.mma, K = 128 +
//   128, f32 in TMEM; two accumulator sets, so a chunk's MMAs run while the
//   epilogue reads the previous one)
// giving the scaled scores cos * |q| = S * rinv_j + pen_j.  Both sub-tiles
// share each centroid chunk: the chunks are the kernel's L2 traffic (a 128-row
// tile re-reads 512 KB of centroids), which bounded the 128-row version.
// Warp 0 loads (the Q tile by TMA, or the listed rows gathered by cp.async
// into the same SW128 layout; centroid chunks hi + lo by TMA, two stages, with
// their column scales), warp 1 owns TMEM and issues the MMAs, warps 2-17 read
// the accumulators: four warps per TMEM lane quadrant, each taking 32 of a
// chunk's 128 columns of both sub-tiles, with four independent (best, second
// best) pairs per row (first index on ties) merged per row at the end of the
// tile, or the rows' candidates.  Every output element depends only on its own
// row and column, so both passes compute bit-identical scores for a listed row.
constexpr int kQsChunk = 128;  // centroids per chunk (MMA N)
constexpr int kQsRows = 256;   // query rows per tile (two MMA M = 128 sub-tiles)
constexpr int kQsEpiWarps = 16;
constexpr int kQsThreads = 64 + 32 * kQsEpiWarps;
struct QsSmem {
  static constexpr int q = 0;                             // [sub-tile 0..1][128 rows x 128 bf16] (two SW128 panels each)
  static constexpr int c = 2 * 32768;                     // [stage 0..1][hi, lo] x 32 KB
  static constexpr int ri = c + 2 * 2 * 32768;            // [stage][rinv, pen][128] f32
  static constexpr int xch = ri + 2 * 2 * kQsChunk * 4;   // [256 rows][4] Best2 partials
  static constexpr int bars = xch + kQsRows * 4 * 12;
  static constexpr int total = bars + 256 + 1024;         // + alignment slack
};

// tile index -> (head, or KV head when listed; first row); listed: each KV head's list in turn
template <bool kListed>
__device__ __forceinline__ bool qs_tile(int64_t t, int heads, int64_t n, const int32_t* count, int& h, int64_t& r0) {
  if (!kListed) {
    const int64_t per = (n + kQsRows - 1) / kQsRows;
    h = (int)(t / per);
    r0 = (t % per) * kQsRows;
    return h < heads;
  }
  for (h = 0; h < heads; ++h) {
    const int64_t per = ((int64_t)count[h] + kQsRows - 1) / kQsRows;
    if (t < per) {
      r0 = t * kQsRows;
      return true;
    }
    t -= per;
  }
  return false;
}

template <bool kListed>
__global__ void __launch_bounds__(kQsThreads, 1) query_group_screen_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_chi,
    const __grid_constant__ CUtensorMap tm_clo, const __nv_bfloat16* __restrict__ q, const float* __restrict__ rinv,
    const float* __restrict__ pen, const float* __restrict__ qn, int heads, int k_group, int64_t n, int64_t tc,
    int64_t tcp, uint32_t* __restrict__ groups, ScreenLists L) {
  extern __shared__ __align__(1024) unsigned char qs_raw[];
  // 1024-byte aligned by pointer arithmetic on the shared array (a round trip
  // through an integer would turn the scale reads below into generic loads)
  unsigned char* sm = qs_raw + ((1024u - (ptx::smem_u32(qs_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + QsSmem::bars);
  uint64_t* q_full = bar;        // the tile's Q rows loaded
  uint64_t* q_empty = bar + 1;   // every MMA reading them complete
  uint64_t* c_full = bar + 2;    // [2] centroid stage (and its scales) loaded
  uint64_t* c_empty = bar + 4;   // [2] its MMAs complete and its scales read
  uint64_t* s_full = bar + 6;    // [2] accumulator set b holds a chunk's scores
  uint64_t* s_free = bar + 8;    // [2] the epilogue read accumulator set b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);
  float* sri = reinterpret_cast<float*>(sm + QsSmem::ri);
  Best2* xch = reinterpret_cast<Best2*>(sm + QsSmem::xch);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunks = (int)((tc + kQsChunk - 1) / kQsChunk);
  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&c_full[b], 1);                 // TMA tiles + scales (expect_tx)
      ptx::mbar_init(&c_empty[b], 1 + kQsEpiWarps);  // MMA commit + every epilogue warp past the scales
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&s_free[b], kQsEpiWarps);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(ptx::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    // ---- loads: per tile Q, then the centroid chunks (the chunk stages run ahead of Q)
    uint32_t it = 0, cit = 0;
    int h;
    int64_t r0;
    for (int64_t t = blockIdx.x; qs_tile<kListed>(t, heads, n, L.count, h, r0); t += gridDim.x, ++it) {
      const int hk = kListed ? h : h / k_group;
      ptx::mbar_wait(q_empty, (it & 1) ^ 1);
      if (!kListed) {
        if (lane == 0) {
          ptx::mbar_expect_tx(q_full, 65536);  // rows past n zero-filled
          for (int u = 0; u < 2; ++u)
            for (int p = 0; p < 2; ++p)
              tc::tma_load_3d(sm + QsSmem::q + u * 32768 + p * 16384, &tm_q, q_full, p * 64,
                              (int)(r0 + u * 128), h);
        }
      } else {
        // the listed rows (global row h * n + i) gathered into the SW128 K-major
        // layout the TMA would write: 16-byte chunk cc of row rr at panel cc / 8,
        // rr * 128 + ((cc % 8) ^ (rr % 8)) * 16; half a warp per 256-byte row
        const int64_t nrows = L.count[h];
        const int64_t lb = (int64_t)h * k_group * n;
        const int hb = lane >> 4, cc = lane & 15, c8 = cc & 7;
        for (int u = 0; u < 2; ++u) {
          int src[4];
#pragma unroll
          for (int jr = 0; jr < 4; ++jr) src[jr] = L.rows[lb + min64(r0 + u * 128 + 32 * jr + lane, nrows - 1)];
          const uint32_t base = ptx::smem_u32(sm + QsSmem::q + u * 32768) + (uint32_t)(cc >> 3) * 16384u;
#pragma unroll
          for (int jr = 0; jr < 4; ++jr)
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
              const int rr = 32 * jr + 2 * i + hb;
              const int gi = __shfl_sync(0xffffffffu, src[jr], (2 * i + hb) & 31);
              const uint32_t dst = base + (uint32_t)rr * 128u + ((uint32_t)(c8 ^ (rr & 7)) << 4);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                           "l"(q + (int64_t)gi * 128 + cc * 8)
                           : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the MMA's operand reads
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(q_full);
      }
      for (int c = 0; c < nchunks; ++c, ++cit) {
        const int st = cit & 1;
        ptx::mbar_wait(&c_empty[st], ((cit >> 1) & 1) ^ 1);
        if (lane == 0) {
          // centroids past tc zero-filled; the chunk's column scales (padded:
          // rinv 0, pen -inf past tc, never a winner) by two bulk copies
          ptx::mbar_expect_tx(&c_full[st], 65536 + 2 * kQsChunk * 4);
          unsigned char* dst = sm + QsSmem::c + st * 65536;
          for (int p = 0; p < 2; ++p) {
            tc::tma_load_3d(dst + p * 16384, &tm_chi, &c_full[st], p * 64, c * kQsChunk, hk);
            tc::tma_load_3d(dst + 32768 + p * 16384, &tm_clo, &c_full[st], p * 64, c * kQsChunk, hk);
          }
          const int64_t j0 = (int64_t)hk * tcp + (int64_t)c * kQsChunk;
          tc::bulk_load(sri + st * 2 * kQsChunk, rinv + j0, kQsChunk * 4, &c_full[st]);
          tc::bulk_load(sri + st * 2 * kQsChunk + kQsChunk, pen + j0, kQsChunk * 4, &c_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    const uint32_t idesc = tc::idesc_bf16(kQsChunk);
    const uint64_t qdesc0 = tc::sdesc_sw128(ptx::smem_u32(sm + QsSmem::q));
    const uint64_t qdesc1 = tc::sdesc_sw128(ptx::smem_u32(sm + QsSmem::q + 32768));
    uint32_t it = 0, cit = 0;
    int h;
    int64_t r0;
    for (int64_t t = blockIdx.x; qs_tile<kListed>(t, heads, n, L.count, h, r0); t += gridDim.x, ++it) {
      ptx::mbar_wait(q_full, it & 1);
      for (int c = 0; c < nchunks; ++c, ++cit) {
        const int st = cit & 1, b = cit & 1;
        ptx::mbar_wait(&c_full[st], (cit >> 1) & 1);
        ptx::mbar_wait(&s_free[b], ((cit >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t cb = ptx::smem_u32(sm + QsSmem::c + st * 65536);
        const uint32_t acc = tmem + b * 2 * kQsChunk;
        tc::mma_k128(acc, qdesc0, tc::sdesc_sw128(cb), idesc, false);                      // Q_0 C_hi^T
        tc::mma_k128(acc, qdesc0, tc::sdesc_sw128(cb + 32768), idesc, true);               // + Q_0 C_lo^T
        tc::mma_k128(acc + kQsChunk, qdesc1, tc::sdesc_sw128(cb), idesc, false);           // Q_1 C_hi^T
        tc::mma_k128(acc + kQsChunk, qdesc1, tc::sdesc_sw128(cb + 32768), idesc, true);    // + Q_1 C_lo^T
        tc::commit(&c_empty[st]);
        tc::commit(&s_full[b]);
      }
      tc::commit(q_empty);  // every MMA reading this Q tile issued
    }
  } else {
    // ---- epilogue: warp e reads TMEM lane quadrant e % 4 (rows 32 (e % 4).. of
    // both sub-tiles) and columns 32 (e / 4).. of each chunk
    const int e = warp - 2, quad = warp & 3, cq = e >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    uint32_t cit = 0;
    int h;
    int64_t r0;
    for (int64_t t = blockIdx.x; qs_tile<kListed>(t, heads, n, L.count, h, r0); t += gridDim.x) {
      const int hk = kListed ? h : h / k_group;
      const int64_t lb = (int64_t)hk * k_group * n;
      const int64_t nrows = kListed ? (int64_t)L.count[h] : n;
      bool valid[2];
      int64_t rc[2], gi[2];
      float thr[2] = {0.0f, 0.0f};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t r = r0 + u * 128 + row;
        valid[u] = r < nrows;
        rc[u] = min64(r, nrows - 1);
        gi[u] = kListed ? (int64_t)L.rows[lb + rc[u]] : (int64_t)h * n + rc[u];
        if (kListed) thr[u] = L.best[lb + rc[u]] - 2.0f * kScrDelta * qn[gi[u]];
      }
      // four independent running (best, second) pairs per row over j % 4 (a
      // dependent compare chain per element would serialise the epilogue),
      // merged with the first index on ties -- the pair a j-ascending scan gives
      Best2 bp[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int x = 0; x < 4; ++x) bp[u][x] = Best2{-INFINITY, -INFINITY, 0};
      for (int c = 0; c < nchunks; ++c, ++cit) {
        const int st = cit & 1, b = cit & 1;
        ptx::mbar_wait(&s_full[b], (cit >> 1) & 1);
        ptx::mbar_wait(&c_full[st], (cit >> 1) & 1);  // the scales (complete: the MMAs waited on it)
        tc::fence_after();
        const float* scl = sri + st * 2 * kQsChunk + cq * 32;
        const int j0 = c * kQsChunk + cq * 32;
#pragma unroll
        for (int u = 0; u < 2; ++u) {  // one sub-tile at a time: 32 scores live per thread
          uint32_t v[32];
          PBS_TC_LD32(tmem + lane_off + (uint32_t)(b * 2 * kQsChunk + u * kQsChunk + cq * 32), v);
          tc::wait_ld();
          if (u == 1) {  // both sub-tiles' scores are in registers: the accumulator set may be rewritten
            tc::fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&s_free[b]);
          }
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const float x = fmaf(__uint_as_float(v[jj]), scl[jj], scl[kQsChunk + jj]);  // padding: pen -inf
            if (!kListed) {
              best2_push(bp[u][jj & 3], x, j0 + jj);
            } else if (x >= thr[u] && valid[u] && j0 + jj < tc) {
              const int slot = atomicAdd(&L.cand_n[lb + rc[u]], 1);
              if (slot < kScrCand) L.cand[(lb + rc[u]) * kScrCand + slot] = j0 + jj;
            }
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&c_empty[st]);  // the scales of this stage read
      }
      if (kListed) continue;
      // each row's four column groups (the warps of its quadrant) merged in shared memory
#pragma unroll
      for (int u = 0; u < 2; ++u)
        xch[(u * 128 + row) * 4 + cq] = best2_merge(best2_merge(bp[u][0], bp[u][1]), best2_merge(bp[u][2], bp[u][3]));
      ptx::named_bar_sync(1, 32 * kQsEpiWarps);
      if (cq < 2 && valid[cq]) {  // warps cq = 0 / 1 decide the rows of sub-tile 0 / 1
        const int u = cq;
        Best2 best = xch[(u * 128 + row) * 4];
#pragma unroll
        for (int x = 1; x < 4; ++x) best = best2_merge(best, xch[(u * 128 + row) * 4 + x]);
        const float qv = qn[gi[u]];
        // scaled scores are cos * |q|; the screen decides only with a clear 2 delta margin
        const float dq = kScrDelta * qv;
        if (!(qv > 0.0f)) {
          groups[gi[u]] = (uint32_t)tc;  // no positive-norm match (permutation.hpp:246-258)
        } else if (best.m > -INFINITY && best.s2 < best.m - 2.0f * dq && best.m > -qv + dq) {
          groups[gi[u]] = (uint32_t)best.j;
        } else {
          const int slot = atomicAdd(&L.count[hk], 1);
          L.rows[lb + slot] = (int32_t)gi[u];
          L.best[lb + slot] = best.m;
        }
      }
      ptx::named_bar_sync(1, 32 * kQsEpiWarps);  // xch may be rewritten after this
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// stage 3: exact cosines (permutation.hpp:244-258) of each listed row's
// candidates, one warp per row (lane = candidate); a row with more candidates
// than kept (or none: the best was -inf) scans every centroid, lanes taking
// j = lane, lane + 32, ... in increasing order.  Argmax with the first index on
// ties, over sims > -1 only.
__global__ void __launch_bounds__(256) query_group_exact_kernel(
    const __nv_bfloat16* __restrict__ q, const float* __restrict__ cent, const float* __restrict__ qn,
    const float* __restrict__ cn, int k_group, int64_t n, int64_t tc, ScreenLists L, uint32_t* __restrict__ groups) {
  const int hk = blockIdx.y;
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t list_base = (int64_t)hk * k_group * n;
  const int64_t rows = L.count[hk];
  for (int64_t w = (int64_t)blockIdx.x * 8 + wl; w < rows; w += (int64_t)gridDim.x * 8) {
    const int64_t gi = L.rows[list_base + w];
    const int nc = L.cand_n[list_base + w];
    const __nv_bfloat16* qi = q + gi * 128;
    const float qv = qn[gi];
    float best = -1.0f;
    int bj = -1;
    auto consider = [&](int64_t j) {
      const float cv = cn[hk * tc + j];
      float sim = -1.0f;
      if (qv > 0.0f && cv > 0.0f) {
        const float* cj = cent + ((int64_t)hk * tc + j) * 128;
        float dot = 0.0f;
        for (int c = 0; c < 128; ++c) dot = __fadd_rn(dot, __fmul_rn(__bfloat162float(qi[c]), __ldg(cj + c)));
        sim = __fdiv_rn(dot, __fmul_rn(qv, cv));
      }
      if (sim > best || (sim == best && bj >= 0 && (int)j < bj && sim > -1.0f)) {
        best = sim;
        bj = (int)j;
      }
    };
    if (nc >= 1 && nc <= kScrCand) {
      if (lane < nc) consider(L.cand[(list_base + w) * kScrCand + lane]);
    } else {
      for (int64_t j = lane; j < tc; j += 32) consider(j);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (oj >= 0 && (bj < 0 || ob > best || (ob == best && oj < bj))) {
        best = ob;
        bj = oj;
      }
    }
    if (lane == 0) groups[gi] = bj < 0 ? (uint32_t)tc : (uint32_t)bj;
  }
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

namespace {
struct ImpWs {
  float* L;
  unsigned* rowmax;
  float* w;
};
ImpWs imp_ws(void* ws, int hq, int64_t n, int take) {
  ImpWs r;
  r.L = static_cast<float*>(ws);
  r.rowmax = reinterpret_cast<unsigned*>(r.L + (size_t)hq * n * take);
  r.w = reinterpret_cast<float*>(r.rowmax + (size_t)hq * take);
  return r;
}
}  // namespace

int launch_importance_logits(const void* q, const void* k, int dtype, int hq, int hkv, int h0, int nh, int64_t n,
                             int d, int64_t block, float scale, void* ws, size_t ws_bytes, cudaStream_t st,
                             int64_t q_rows) {
  const int take = (int)min64(block, n);
  if (q_rows <= 0) q_rows = n;
  if (q_rows < take) return fail(PBS_ERR_CONFIG, "E_SHAPE", "importance: q holds fewer rows than the estimate reads");
  if (ws_bytes < importance_workspace_bytes(hq, n, block))
    return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "importance workspace too small");
  if (h0 < 0 || nh < 0 || h0 + nh > hq) return fail(PBS_ERR_CONFIG, "E_SHAPE", "importance: head range");
  if (nh == 0) return PBS_OK;
  const ImpWs W = imp_ws(ws, hq, n, take);
  PBS_CUDA_CHECK(cudaMemsetAsync(W.rowmax + (size_t)h0 * take, 0, sizeof(unsigned) * nh * take, st));
  const int group = hq / hkv;
  const bool vec = (d % 16 == 0) && ((uintptr_t)q % 16 == 0) && ((uintptr_t)k % 16 == 0);
  dim3 grid((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(take, kTile), (unsigned)nh);
  if (dtype == PBS_DTYPE_BF16) {
    auto qq = static_cast<const __nv_bfloat16*>(q);
    auto kk = static_cast<const __nv_bfloat16*>(k);
    if (vec && d % xgemm::kChunkW == 0) {
      auto kern = importance_logits_kernel<__nv_bfloat16, true, true, true>;
      static DeviceOnce attr_once;
      if (int rc = once_per_device(attr_once, [&] {
            PBS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)sizeof(xgemm::SmemWide)));
            return (int)PBS_OK;
          }))
        return rc;
      kern<<<grid, xgemm::kThreads, sizeof(xgemm::SmemWide), st>>>(qq, kk, group, n, q_rows, d, take, scale, W.L,
                                                                   W.rowmax, h0);
    } else if (vec) importance_logits_kernel<__nv_bfloat16, true, true><<<grid, xgemm::kThreads, 0, st>>>(qq, kk, group, n, q_rows, d, take, scale, W.L, W.rowmax, h0);
    else importance_logits_kernel<__nv_bfloat16, true, false><<<grid, xgemm::kThreads, 0, st>>>(qq, kk, group, n, q_rows, d, take, scale, W.L, W.rowmax, h0);
  } else {
    auto qq = static_cast<const float*>(q);
    auto kk = static_cast<const float*>(k);
    if (vec) importance_logits_kernel<float, false, true><<<grid, xgemm::kThreads, 0, st>>>(qq, kk, group, n, q_rows, d, take, scale, W.L, W.rowmax, h0);
    else importance_logits_kernel<float, false, false><<<grid, xgemm::kThreads, 0, st>>>(qq, kk, group, n, q_rows, d, take, scale, W.L, W.rowmax, h0);
  }
  PBS_LAUNCH_CHECK("importance_logits_kernel");
  return PBS_OK;
}

int launch_importance_finish(int hq, int h0, int nh, int64_t n, int64_t block, float* scores, void* ws,
                             size_t ws_bytes, cudaStream_t st) {
  const int take = (int)min64(block, n);
  if (ws_bytes < importance_workspace_bytes(hq, n, block))
    return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "importance workspace too small");
  if (h0 < 0 || nh < 0 || h0 + nh > hq) return fail(PBS_ERR_CONFIG, "E_SHAPE", "importance: head range");
  if (nh == 0) return PBS_OK;
  const ImpWs W = imp_ws(ws, hq, n, take);
  float* L = W.L;
  // E = expf(L - mx) once per element on the whole GPU (the glibc port is
  // FP64 work: computing it once and streaming E twice beats recomputing it
  // inside the two sequential passes, measured 1.46 vs 2.6 ms at C3)
  importance_exp_kernel<<<dim3((unsigned)ceil_div(n, kExpKeys), (unsigned)nh), 256, 0, st>>>(L, W.rowmax, take, n,
                                                                                             h0);
  PBS_LAUNCH_CHECK("importance_exp_kernel");
  const size_t smem = sizeof(float) * kRing * kJT * 32 + 2 * kRing * sizeof(uint64_t);
  static DeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, [&] {
        PBS_CUDA_CHECK(
            cudaFuncSetAttribute(importance_denom_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        return (int)PBS_OK;
      }))
    return rc;
  alignas(64) CUtensorMap tm_e;
  const bool tma = (take % 4 == 0) && (take % 32 == 0);  // every CTA's 32 rows are whole 16-byte pieces
  if (tma) {
    if (int rc = make_f32_map_3d(&tm_e, L, take, n, hq, 32, kJT)) return rc;
  } else {
    memset(&tm_e, 0, sizeof(tm_e));
  }
  importance_denom_kernel<<<dim3((unsigned)ceil_div(take, 32), (unsigned)nh), 64, smem, st>>>(tm_e, tma, L, take, n,
                                                                                              h0, W.w);
  PBS_LAUNCH_CHECK("importance_denom_kernel");
  importance_scores_kernel<<<dim3((unsigned)ceil_div(n, kSK), (unsigned)nh), kSK, 0, st>>>(L, W.w, take, n, h0,
                                                                                         scores);
  PBS_LAUNCH_CHECK("importance_scores_kernel");
  return PBS_OK;
}

int launch_importance(const void* q, const void* k, int dtype, int hq, int hkv, int64_t n, int d,
                      int64_t block, float scale, float* scores, void* ws, size_t ws_bytes,
                      cudaStream_t st, int64_t q_rows) {
  if (int rc = launch_importance_logits(q, k, dtype, hq, hkv, 0, hq, n, d, block, scale, ws, ws_bytes, st, q_rows))
    return rc;
  return launch_importance_finish(hq, 0, hq, n, block, scores, ws, ws_bytes, st);
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
    // segments of 4097..8192 keys need 64 KB of shared memory
    static DeviceOnce attr_once;
    if (int rc = once_per_device(attr_once, [] {
          PBS_CUDA_CHECK(cudaFuncSetAttribute(segmented_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)(sizeof(unsigned long long) * 8192)));
          return (int)PBS_OK;
        }))
      return rc;
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
  // centroids, their norms, |q|, the per-query best keys (exact path) or the
  // fallback list (screen path), then the screen's split centroids and scales
  return (size_t)hq * tc * d * 4 + (size_t)hq * tc * 4 + (size_t)hq * n * 4 + (size_t)hq * n * 8 +
         (size_t)hq * n * 4 * (kScrCand + 2) + (size_t)hq * tc * kScrPad * 4 +
         (size_t)hq * (tc + 128) * 8 + 4096;
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
  const size_t csmem = sizeof(float) * d;
  if (dtype == PBS_DTYPE_BF16) {
    centroid_kernel<__nv_bfloat16><<<dim3((unsigned)tc, (unsigned)k_heads), 128, csmem, st>>>(
        static_cast<const __nv_bfloat16*>(k), n, d, block, tc, cent, cn);
    PBS_LAUNCH_CHECK("centroid_kernel");
    qnorm_kernel<__nv_bfloat16><<<(unsigned)ceil_div((int64_t)hq * n, 128), 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(q), (int64_t)hq * n, d, qn);
    PBS_LAUNCH_CHECK("qnorm_kernel");
    if (d == 128 && (uintptr_t)q % 16 == 0 && !getenv("PBS_QGROUP_EXACT")) {
      // screen on the tensor cores, exact re-check of the undecided rows' candidates
      const int kg = hq / k_heads;
      char* p2 = reinterpret_cast<char*>(best);  // the exact path's per-row keys are not used here
      ScreenLists SL;
      SL.count = reinterpret_cast<int32_t*>(p2);
      p2 += 1024;
      SL.rows = reinterpret_cast<int32_t*>(p2);
      p2 += (size_t)hq * n * 4;
      SL.best = reinterpret_cast<float*>(p2);
      p2 += (size_t)hq * n * 4;
      SL.cand_n = reinterpret_cast<int32_t*>(p2);
      p2 += (size_t)hq * n * 4;
      SL.cand = reinterpret_cast<int32_t*>(p2);
      p2 += (size_t)hq * n * 4 * kScrCand;
      p2 = reinterpret_cast<char*>(((uintptr_t)p2 + 255) & ~(uintptr_t)255);
      __nv_bfloat16* chi = reinterpret_cast<__nv_bfloat16*>(p2);
      __nv_bfloat16* clo = chi + (size_t)k_heads * tc * kScrPad;
      const int64_t tcp = (tc + kQsChunk - 1) / kQsChunk * kQsChunk;
      float* rinv = reinterpret_cast<float*>(
          ((uintptr_t)(clo + (size_t)k_heads * tc * kScrPad) + 15) & ~(uintptr_t)15);
      float* pen = rinv + (size_t)k_heads * tcp;
      PBS_CUDA_CHECK(cudaMemsetAsync(SL.count, 0, sizeof(int32_t) * k_heads, st));
      PBS_CUDA_CHECK(cudaMemsetAsync(SL.cand_n, 0, sizeof(int32_t) * hq * n, st));
      centroid_split_kernel<<<dim3((unsigned)tcp, (unsigned)k_heads), 128, 0, st>>>(cent, cn, tc, tcp, chi, clo,
                                                                                   rinv, pen);
      PBS_LAUNCH_CHECK("centroid_split_kernel");
      static DeviceOnce scr_once;
      if (int rc = once_per_device(scr_once, [] {
            PBS_CUDA_CHECK(cudaFuncSetAttribute(query_group_screen_kernel<false>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, QsSmem::total));
            PBS_CUDA_CHECK(cudaFuncSetAttribute(query_group_screen_kernel<true>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, QsSmem::total));
            return (int)PBS_OK;
          }))
        return rc;
      const auto* qb = static_cast<const __nv_bfloat16*>(q);
      alignas(64) CUtensorMap tm_q, tm_chi, tm_clo;
      if (int rc = make_bf16_sw128_map_3d(&tm_q, qb, 128, n, hq, 128, 64, 128)) return rc;
      if (int rc = make_bf16_sw128_map_3d(&tm_chi, chi, 128, tc, k_heads, kScrPad, 64, 128)) return rc;
      if (int rc = make_bf16_sw128_map_3d(&tm_clo, clo, 128, tc, k_heads, kScrPad, 64, 128)) return rc;
      const int grid = num_sms();
      query_group_screen_kernel<false><<<grid, kQsThreads, QsSmem::total, st>>>(tm_q, tm_chi, tm_clo, qb, rinv, pen,
                                                                              qn, hq, kg, n, tc, tcp, groups, SL);
      PBS_LAUNCH_CHECK("query_group_screen_kernel");
      // the listed rows of every KV head (tile counts read on the device)
      query_group_screen_kernel<true><<<grid, kQsThreads, QsSmem::total, st>>>(tm_q, tm_chi, tm_clo, qb, rinv, pen,
                                                                             qn, k_heads, kg, n, tc, tcp, groups, SL);
      PBS_LAUNCH_CHECK("query_group_screen_kernel");
      query_group_exact_kernel<<<dim3((unsigned)num_sms() * 4, (unsigned)k_heads), 256, 0, st>>>(qb, cent, qn, cn, kg,
                                                                                             n, tc, SL, groups);
      PBS_LAUNCH_CHECK("query_group_exact_kernel");
      if (getenv("PBS_QGROUP_STATS")) {  // debug: rows the screen left to the exact re-check
        std::vector<int32_t> c(k_heads);
        cudaMemcpyAsync(c.data(), SL.count, 4 * k_heads, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        long long tot = 0;
        for (int x : c) tot += x;
        fprintf(stderr, "query groups: %lld of %lld rows re-checked exactly\n", tot, (long long)hq * n);
      }
      return PBS_OK;
    }
    PBS_CUDA_CHECK(cudaMemsetAsync(best, 0, sizeof(unsigned long long) * hq * n, st));
    const dim3 g3((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(tc, kTile), (unsigned)hq);
    if (d % 16 == 0)
      query_group_kernel<__nv_bfloat16, true><<<g3, xgemm::kThreads, 0, st>>>(
          static_cast<const __nv_bfloat16*>(q), cent, qn, cn, hq / k_heads, n, d, tc, best);
    else
      query_group_kernel<__nv_bfloat16, false><<<g3, xgemm::kThreads, 0, st>>>(
          static_cast<const __nv_bfloat16*>(q), cent, qn, cn, hq / k_heads, n, d, tc, best);
  } else {
    centroid_kernel<float><<<dim3((unsigned)tc, (unsigned)k_heads), 128, csmem, st>>>(
        static_cast<const float*>(k), n, d, block, tc, cent, cn);
    PBS_LAUNCH_CHECK("centroid_kernel");
    qnorm_kernel<float><<<(unsigned)ceil_div((int64_t)hq * n, 128), 128, 0, st>>>(
        static_cast<const float*>(q), (int64_t)hq * n, d, qn);
    PBS_LAUNCH_CHECK("qnorm_kernel");
    PBS_CUDA_CHECK(cudaMemsetAsync(best, 0, sizeof(unsigned long long) * hq * n, st));
    const dim3 g3((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(tc, kTile), (unsigned)hq);
    if (d % 16 == 0)
      query_group_kernel<float, true><<<g3, xgemm::kThreads, 0, st>>>(static_cast<const float*>(q), cent, qn, cn,
                                                                      hq / k_heads, n, d, tc, best);
    else
      query_group_kernel<float, false><<<g3, xgemm::kThreads, 0, st>>>(static_cast<const float*>(q), cent, qn, cn,
                                                                       hq / k_heads, n, d, tc, best);
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
