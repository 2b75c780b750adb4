// exact_gemm.cuh -- register-tiled SIMT "GEMM" whose every output is the
// reference's sequential dot product: acc = 0; for c in 0..d-1: acc += a[c]*b[c]
// (matrix.hpp:87-94, permutation.hpp:165, block_selection.hpp:151).
//
// A 128 x 128 output tile per 256-thread CTA, 8 x 8 outputs per thread, the
// d axis staged through shared memory in chunks of 16 with register
// double-buffering.  Each output accumulates strictly in c order, so the
// result is bit-identical to the scalar loop:
//   kExact = true  : fmaf (valid when every product is exact in fp32, e.g.
//                    bf16 x bf16 with |product| >= 2^-126)
//   kExact = false : rounded product then add (the reference's un-contracted
//                    x86-64 code for arbitrary fp32 operands), packed f32x2
#pragma once

#include "common.cuh"

namespace pbs_b200 {
namespace xgemm {

constexpr int kTile = 128;
constexpr int kChunk = 16;
constexpr int kPad = 4;
constexpr int kThreads = 256;

struct Smem {
  float a[2][kChunk][kTile + kPad];
  float b[2][kChunk][kTile + kPad];
};

__device__ __forceinline__ int tile_row(int idx, int t) { return (idx < 4 ? 0 : 64) + t * 4 + (idx & 3); }

// Two independent outputs per instruction (Blackwell f32x2 SIMD, FFMA2) for
// the exact-product path: each lane is an ordinary IEEE round-to-nearest FMA,
// so every output keeps its own sequential accumulation order.
__device__ __forceinline__ uint64_t pk2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}
// {-0.0f, -0.0f}.  Kept in constant memory so that ptxas cannot see the value:
// ptxas contracts mul.rn.f32x2 + add.rn.f32x2 (and an fma with a literal -0
// addend + add) into one FFMA2, which would skip the product's rounding.
static __constant__ uint64_t kNegZero2 = 0x8000000080000000ull;

template <bool kExact>
__device__ __forceinline__ void acc2(float& c0, float& c1, float a, float b0, float b1) {
  uint64_t rc = pk2(c0, c1);
  const uint64_t ra = pk2(a, a), rb = pk2(b0, b1);
  if (kExact) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(rc) : "l"(ra), "l"(rb));
  } else {
    // product rounded on its own (fma with a -0 addend == mul, bit for bit,
    // signed zeros included), then the add: the reference's un-contracted
    // mul-then-add, two outputs per instruction
    uint64_t rp;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rp) : "l"(ra), "l"(rb), "l"(kNegZero2));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(rc) : "l"(rp));
  }
  upk2(rc, c0, c1);
}

// load 8 consecutive elements [c, c+8) of row `row` (zero beyond rows/d)
template <typename T, bool kVec>
__device__ __forceinline__ void load8(const T* __restrict__ base, int rows, int d, int row, int c, float (&v)[8]) {
  if (row >= rows) {
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = 0.0f;
    return;
  }
  const T* p = base + (int64_t)row * d + c;
  if constexpr (kVec) {
    if constexpr (sizeof(T) == 2) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f = __bfloat1622float2(h[u]);
        v[2 * u] = f.x;
        v[2 * u + 1] = f.y;
      }
    } else {
      const float4 x0 = __ldg(reinterpret_cast<const float4*>(p));
      const float4 x1 = __ldg(reinterpret_cast<const float4*>(p) + 1);
      v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
      v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (c + u < d) ? to_f32(p[u]) : 0.0f;
  }
}

// acc[ii][jj] = dot(A[tile_row(ii, ty)], B[tile_row(jj, tx)]) over c = 0..d-1 in order.
template <typename TA, typename TB, bool kExact, bool kVec>
__device__ __forceinline__ void tile(const TA* __restrict__ a_base, int a_rows, const TB* __restrict__ b_base,
                                     int b_rows, int d, float (&acc)[8][8], Smem& sm) {
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int lrow = tid >> 1;
  const int lcol = (tid & 1) * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  const int nchunks = (d + kChunk - 1) / kChunk;
  float ra[8], rb[8];
  load8<TA, kVec>(a_base, a_rows, d, lrow, lcol, ra);
  load8<TB, kVec>(b_base, b_rows, d, lrow, lcol, rb);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    sm.a[0][lcol + u][lrow] = ra[u];
    sm.b[0][lcol + u][lrow] = rb[u];
  }
  __syncthreads();
  for (int kc = 0; kc < nchunks; ++kc) {
    const int buf = kc & 1;
    const bool more = kc + 1 < nchunks;
    if (more) {
      load8<TA, kVec>(a_base, a_rows, d, lrow, (kc + 1) * kChunk + lcol, ra);
      load8<TB, kVec>(b_base, b_rows, d, lrow, (kc + 1) * kChunk + lcol, rb);
    }
    const int kcount = min(kChunk, d - kc * kChunk);
#pragma unroll 4
    for (int cc = 0; cc < kcount; ++cc) {
      const float4 a0 = *reinterpret_cast<const float4*>(&sm.a[buf][cc][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&sm.a[buf][cc][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&sm.b[buf][cc][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&sm.b[buf][cc][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; j += 2) acc2<kExact>(acc[i][j], acc[i][j + 1], a[i], b[j], b[j + 1]);
    }
    if (more) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sm.a[buf ^ 1][lcol + u][lrow] = ra[u];
        sm.b[buf ^ 1][lcol + u][lrow] = rb[u];
      }
    }
    __syncthreads();
  }
}

// bf16 operands with d % 32 == 0: the same per-output order, d staged in
// chunks of 32 (half the CTA barriers of tile()), the next chunk held in
// registers as raw bf16 (8 x 32-bit per operand per thread) and widened to f32
// on its way into shared memory.  Needs sizeof(SmemWide) of dynamic smem.
constexpr int kChunkW = 32;
struct SmemWide {
  float a[2][kChunkW][kTile + kPad];
  float b[2][kChunkW][kTile + kPad];
};

__device__ __forceinline__ void load16_bf16(const __nv_bfloat16* __restrict__ base, int rows, int d, int row, int c,
                                            uint4 (&v)[2]) {
  if (row >= rows) {
    v[0] = make_uint4(0u, 0u, 0u, 0u);
    v[1] = v[0];
    return;
  }
  const uint4* p = reinterpret_cast<const uint4*>(base + (int64_t)row * d + c);
  v[0] = __ldg(p);
  v[1] = __ldg(p + 1);
}

__device__ __forceinline__ void store16_widened(float (*dst)[kTile + kPad], int col0, int row, const uint4 (&v)[2]) {
  const uint32_t w[8] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w};
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    dst[col0 + 2 * u][row] = __uint_as_float(w[u] << 16);             // bf16 -> f32 is exact
    dst[col0 + 2 * u + 1][row] = __uint_as_float(w[u] & 0xffff0000u);
  }
}

__device__ __forceinline__ void tile_bf16_wide(const __nv_bfloat16* __restrict__ a_base, int a_rows,
                                               const __nv_bfloat16* __restrict__ b_base, int b_rows, int d,
                                               float (&acc)[8][8], SmemWide& sm) {
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int lrow = tid >> 1;
  const int lcol = (tid & 1) * 16;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  const int nchunks = d / kChunkW;
  uint4 ra[2], rb[2];
  load16_bf16(a_base, a_rows, d, lrow, lcol, ra);
  load16_bf16(b_base, b_rows, d, lrow, lcol, rb);
  store16_widened(sm.a[0], lcol, lrow, ra);
  store16_widened(sm.b[0], lcol, lrow, rb);
  __syncthreads();
  for (int kc = 0; kc < nchunks; ++kc) {
    const int buf = kc & 1;
    const bool more = kc + 1 < nchunks;
    if (more) {
      load16_bf16(a_base, a_rows, d, lrow, (kc + 1) * kChunkW + lcol, ra);
      load16_bf16(b_base, b_rows, d, lrow, (kc + 1) * kChunkW + lcol, rb);
    }
#pragma unroll 8
    for (int cc = 0; cc < kChunkW; ++cc) {
      const float4 a0 = *reinterpret_cast<const float4*>(&sm.a[buf][cc][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&sm.a[buf][cc][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&sm.b[buf][cc][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&sm.b[buf][cc][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; j += 2) acc2<true>(acc[i][j], acc[i][j + 1], a[i], b[j], b[j + 1]);
    }
    if (more) {
      store16_widened(sm.a[buf ^ 1], lcol, lrow, ra);
      store16_widened(sm.b[buf ^ 1], lcol, lrow, rb);
    }
    __syncthreads();
  }
}

}  // namespace xgemm
}  // namespace pbs_b200
