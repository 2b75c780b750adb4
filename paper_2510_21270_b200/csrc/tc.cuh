// tc.cuh -- tcgen05 / TMEM / TMA wrappers for the non-attention tensor-core
// kernels (the query-grouping screen).  Warp-collective forms: the whole warp
// executes them and one elected lane issues, so descriptors stay uniform.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "ptx.cuh"

namespace pbs_b200 {
namespace tc {

// SW128 K-major shared-memory matrix descriptor (sm100: version 1 at bit 46, layout 2)
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((16u >> 4) & 0x3FFFu) << 16;    // LBO (unused for SW128 K-major)
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;  // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::f16: f32 accumulate, bf16 A and B, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(ptx::smem_u32(bar))
      : "memory");
}

// D (+)= A B^T over K = 128 (two 64-column SW128 panels of 16 KB, 4 K-steps of
// 16 each): 8 MMAs from one elected lane; the first one overwrites D unless acc.
__device__ __forceinline__ void mma_k128(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n"
      ".reg .pred e, t, f;\n"
      ".reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
      "setp.ne.b32 t, 1, 0;\n"
      "setp.ne.b32 f, %4, 0;\n"
      "add.s64 a1, %1, 2;    add.s64 b1, %2, 2;\n"
      "add.s64 a2, %1, 4;    add.s64 b2, %2, 4;\n"
      "add.s64 a3, %1, 6;    add.s64 b3, %2, 6;\n"
      "add.s64 a4, %1, 1024; add.s64 b4, %2, 1024;\n"
      "add.s64 a5, %1, 1026; add.s64 b5, %2, 1026;\n"
      "add.s64 a6, %1, 1028; add.s64 b6, %2, 1028;\n"
      "add.s64 a7, %1, 1030; add.s64 b7, %2, 1030;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, f;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, t;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc ? 1u : 0u)
      : "memory");
}

#define PBS_TC_LD32(taddr, r)                                                                                  \
  asm volatile(                                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "   \
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),        \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),  \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),             \
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),             \
        "=r"(r[30]), "=r"(r[31])                                                                               \
      : "r"(taddr))
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(ptx::smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(ptx::smem_u32(bar))
      : "memory");
}

// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completing on `bar` like a tensor copy
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          ptx::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
      : "memory");
}

}  // namespace tc
}  // namespace pbs_b200
