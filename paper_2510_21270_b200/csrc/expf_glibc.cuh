// expf_glibc.cuh -- device restatement of glibc 2.39's expf.
//
// The reference calls std::exp(float) (permutation.hpp:171,
// matrix.hpp:136, attention.hpp:108-114), which on x86-64 Linux is glibc's
// expf (sysdeps/ieee754/flt-32/e_expf.c, the ARM optimized-routines
// algorithm: a 32-entry 2^(i/32) table and a cubic in double precision).
// glibc dispatches to an FMA build of it on FMA-capable hosts; that build
// contracts z = InvLn2N*x into both uses (kd = fma(InvLn2N, x, SHIFT),
// r = fma(InvLn2N, x, -kd)) and evaluates the polynomial with FMAs.
//
// Pinning: this exact sequence was compared against host expf for all 2^32
// float inputs with 0 mismatches (tests/test_expf.py reproduces it on the box
// that runs the oracle, on device and on host).  Double FMA is IEEE on the
// GPU and the final double->float conversion is round-to-nearest with
// subnormals preserved (no FTZ), so the device result is bit-identical.
//
// Measured alternative (round 2): the two conversions done in integer ops
// instead of F2F (exact, also 0 mismatches over all 2^32 inputs) made the exp
// passes 1.3-2.7x SLOWER on B200 (64-bit shifts and adds cost more issue
// slots than the two F2F); the FP64 arithmetic bounds the port either way, so
// the pipeline computes each exponential once (importance.cu).
#pragma once

#include <stdint.h>

namespace pbs_b200 {

// __exp2f_data.tab (N = 32): asuint64(2^(i/32)) - (i << 47); identical to the
// table found in this image's libm.so.6 (checked by oracle tests).
static __device__ const uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

// `tab` is the 2^(i/32) table: a shared-memory copy in the hot kernels (the
// per-lane index makes constant-cache reads serialise), else the global one.
__device__ __forceinline__ float expf_glibc(float x, const uint64_t* tab) {
  // glibc evaluates the table + cubic formula for every x in [-103.97, 88.72]
  // (including the subnormal-result range) and special-cases the rest; here
  // the formula runs unconditionally and the special cases are selects, so
  // independent calls interleave (no branches).
  const double xd = (double)x;
  const double kInvLn2N = 0x1.71547652b82fep+5;  // 32 / ln 2
  const double kShift = 0x1.8p+52;
  double kd = __fma_rn(kInvLn2N, xd, kShift);
  const uint64_t ki = (uint64_t)__double_as_longlong(kd);
  kd -= kShift;
  const double r = __fma_rn(kInvLn2N, xd, -kd);
  uint64_t t = tab[ki & 31u];
  t += ki << 47;
  const double s = __longlong_as_double((long long)t);
  const double z = __fma_rn(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);  // C0/N^3, C1/N^2
  const double r2 = r * r;
  double y = __fma_rn(0x1.62e42ff0c52d6p-6, r, 1.0);  // C2/N
  y = __fma_rn(z, r2, y);
  y = y * s;
  float res = __double2float_rn(y);
  // special cases of e_expf.c (|x| >= 88 branch)
  res = (x > 0x1.62e42ep6f) ? __int_as_float(0x7f800000) : res;  // overflow -> +inf
  res = (x < -0x1.9fe368p6f) ? 0.0f : res;                        // underflow (and -inf) -> +0
  res = (x != x) ? x + x : res;                                   // nan
  return res;
}

__device__ __forceinline__ float expf_glibc(float x) { return expf_glibc(x, kExp2fTab); }

// stage the table in shared memory (call with all threads, then __syncthreads)
__device__ __forceinline__ void load_exp2f_table(uint64_t* smem_tab) {
  for (int i = threadIdx.x; i < 32; i += blockDim.x) smem_tab[i] = kExp2fTab[i];
}

}  // namespace pbs_b200
