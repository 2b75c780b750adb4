// Micro-benchmark (debug tool, not part of the library): cycles per softmax
// "exp pass" -- p = 2^(s*c - m) -> bf16 -> tcgen05.st, plus the row sum -- for
// kCols keys per thread, kPoly of every 16 keys on the FMA-pipe polynomial,
// W warps per SM sub-partition.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint64_t pk2(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ void upk2(uint64_t r, float& x, float& y) { asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ void exp2_poly2(float y0, float y1, float& p0, float& p1) {
  const uint64_t x = pk2(fmaxf(y0, -126.5f), fmaxf(y1, -126.5f));
  const uint64_t t = fadd2(x, pk2(12582912.0f, 12582912.0f));
  const uint64_t jf = fadd2(t, pk2(-12582912.0f, -12582912.0f));
  const uint64_t f = fadd2(x, jf ^ 0x8000000080000000ull);
  uint64_t p = ffma2(pk2(0.055219680070877075f, 0.055219680070877075f), f, pk2(0.2426094114780426f, 0.2426094114780426f));
  p = ffma2(p, f, pk2(0.6932516694068909f, 0.6932516694068909f));
  p = ffma2(p, f, pk2(0.9999279975891113f, 0.9999279975891113f));
  float q0, q1, t0, t1; upk2(p, q0, q1); upk2(t, t0, t1);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}
#define TMEM_ST16(taddr, r) asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory")

template <int kCols, int kPoly>
__device__ __forceinline__ float emit(const float (&r)[kCols], float sc, float nm, uint32_t tP) {
  const uint64_t sc2 = pk2(sc, sc), nm2 = pk2(nm, nm);
  uint64_t sum2[2] = {0, 0};
#pragma unroll
  for (int c = 0; c < kCols / 32; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int jp = 0; jp < 16; ++jp) {
      const int j = c * 32 + 2 * jp;
      float y0, y1, p0, p1;
      upk2(ffma2(pk2(r[j], r[j + 1]), sc2, nm2), y0, y1);
      if ((j & 15) >= 16 - kPoly) exp2_poly2(y0, y1, p0, p1);
      else { p0 = ex2(y0); p1 = ex2(y1); }
      sum2[jp & 1] = fadd2(sum2[jp & 1], pk2(p0, p1));
      __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
      pk[jp] = *reinterpret_cast<uint32_t*>(&b2);
    }
    TMEM_ST16(tP + c * 16, pk);
  }
  float a, b, cc, d; upk2(sum2[0], a, b); upk2(sum2[1], cc, d);
  return (a + b) + (cc + d);
}

template <int kCols, int kPoly>
__global__ void bench(float* out, long long* cyc, int iters) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * (kCols / 2);
  float r[kCols];
#pragma unroll
  for (int j = 0; j < kCols; ++j) r[j] = -0.01f * ((threadIdx.x * 7 + j * 13) % 97);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    acc += emit<kCols, kPoly>(r, 1.4427f, -0.5f - acc * 1e-30f, tmem);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

template <int kCols, int kPoly>
void run(int warps) {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  bench<kCols, kPoly><<<148, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  bench<kCols, kPoly><<<148, warps * 32>>>(out, cyc, iters);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("cols %3d poly %2d/16 warps/SMSP %d: %7.1f cycles per pass (%s)\n", kCols, kPoly, warps / 4,
         (double)h / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<128, 0>(4); run<128, 4>(4); run<128, 6>(4); run<128, 8>(4);
  run<64, 0>(4); run<64, 6>(4);
  run<64, 0>(8); run<64, 4>(8); run<64, 6>(8); run<64, 8>(8);
  run<128, 0>(8); run<128, 6>(8);
  return 0;
}
