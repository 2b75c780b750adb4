// Micro-benchmark (debug tool, not part of the library): tcgen05.mma kind::f16
// M=128 N=128 K=16 issue/execution rate, SS (A and B from shared memory) vs TS
// (A from TMEM), one CTA per SM, one issuing warp.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(uint32_t n, uint32_t bmn = 0) { return (1u << 4) | (1u << 7) | (1u << 10) | (bmn << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24); }
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
}

// kLoad: 0 none; 1: warps 1.. stream tcgen05.ld over TMEM columns [256, 384);
// 2: warps 1.. stream tcgen05.st; 3: warps 1.. stream st.shared into a 64 KB region
template <int kMode, int kN, int kLoad, bool kRandom = false, int kCommit = 0>
__global__ void bench(long long* out, int iters, volatile int* stop) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2[2];
  __shared__ uint32_t tbase;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[0]))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[1]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t a = smem_u32(s), b = smem_u32(s + 32768);
  if (kRandom) {  // random bf16 operands (switching power like real data)
    uint32_t x = 12345u + threadIdx.x * 7919u + blockIdx.x * 104729u;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
      x = x * 1664525u + 1013904223u;
      const uint32_t lo = 0x3f80u ^ ((x >> 9) & 0x807fu), hi = 0x3f80u ^ ((x >> 20) & 0x807fu);
      reinterpret_cast<uint32_t*>(s)[i] = lo | (hi << 16);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  __shared__ int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (threadIdx.x >= 32) {
    const int w = threadIdx.x >> 5;
    const uint32_t t = tm + (((uint32_t)(w & 3) * 32) << 16) + 256 + ((w >> 2) & 1) * 64;
    uint32_t r[32] = {};
    int n = 0;
    while (!*(volatile int*)&done) {
      if (kLoad == 1) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(t));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        n += r[n & 31];
      } else if (kLoad == 2) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
          :: "r"(t), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        ++n;
      } else if (kLoad == 3) {
        int4* dst = reinterpret_cast<int4*>(s + 65536) + ((threadIdx.x - 32 + n * 224) & 4095);
        *dst = make_int4(n, n, n, n);
        ++n;
      } else break;
    }
    if (n == 12345678) out[1000] = n;
  } else {
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (kCommit == 3) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (kCommit == 4) { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); __syncwarp(); asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
    if (kCommit == 5) { uint32_t ok; asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar2[1])), "r"(1u) : "memory"); asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t bd = sdesc(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      if (kMode == 0) mma_ss(tm, sdesc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), bd, idesc(kN), k > 0);
      else if (kMode == 1) mma_ts(tm, tm + 256 + k * 8, bd, idesc(kN), k > 0);
      else if (kMode == 2) mma_ts(tm, tm + 256 + k * 8, sdesc(b + k * 16 * 128, 16384, 1024), idesc(kN, 1), k > 0);  // B MN-major (V)
      else {  // 3: the attention step mix, QK^T (SS) into cols 0.. then PV (TS, B MN-major) into cols 384..
        mma_ss(tm, sdesc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), bd, idesc(kN), k > 0);
      }
    }
    if (kMode == 3) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_ts(tm + 384, tm + 128 + k * 8, sdesc(b + k * 16 * 128, 16384, 1024), idesc(kN, 1), k > 0);
    }
    if (kCommit == 1) commit(&bar2[it & 1]);  // a commit after every 8 MMAs (nobody waits)
    if (kCommit == 2) { commit(&bar2[0]); wait(&bar2[0], it & 1); }  // and wait for it
  }
  commit(&bar);
  wait(&bar, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (threadIdx.x == 0) *(volatile int*)&done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int kMode, int kN, int kLoad, bool kRandom = false, int kCommit = 0>
void run(int warps) {
  long long* d; cudaMalloc(&d, 148 * 8);
  auto k = bench<kMode, kN, kLoad, kRandom, kCommit>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int iters = 20000;
  k<<<148, 32 * warps, 140 * 1024>>>(d, iters, nullptr);
  cudaDeviceSynchronize();
  k<<<148, 32 * warps, 140 * 1024>>>(d, iters, nullptr);
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * (kMode == 3 ? 16.0 : 8.0));
  printf("commit %d %s%s N=%d load %d warps %d: %.1f cycles per 128x%dx16 MMA (ideal %d) %s\n", kCommit, kMode == 3 ? "QK+PV" : kMode == 2 ? "TS-Bmn" : kMode ? "TS" : "SS", kRandom ? " random" : "", kN, kLoad, warps, per, kN, kN / 2,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main(int argc, char**) {
  if (argc > 1) {  // N sweep: does a narrow MMA cost proportionally less?
    run<0, 256, 0, true>(1); run<0, 128, 0, true>(1); run<0, 64, 0, true>(1); run<0, 32, 0, true>(1); run<0, 16, 0, true>(1);
    run<1, 64, 0, true>(1); run<1, 32, 0, true>(1);
    return 0;
  }
  run<0, 128, 0>(1); run<1, 128, 0>(1); run<2, 128, 0>(1); run<2, 128, 0, false, 2>(1);
  run<1, 128, 0, false, 3>(1); run<1, 128, 0, false, 4>(1); run<1, 128, 0, false, 5>(1);
  run<0, 128, 0, true>(1); run<0, 256, 0, true>(1);
  run<0, 128, 0, false, 1>(1); run<1, 128, 0, false, 1>(1); run<0, 128, 0, false, 2>(1); run<1, 128, 0, false, 2>(1);
  run<0, 128, 1>(9); run<1, 128, 1>(9); run<1, 128, 1>(5);
  run<0, 128, 2>(9); run<1, 128, 2>(9);
  run<0, 128, 3>(9); run<1, 128, 3>(9);
  run<3, 128, 0, true>(1); run<3, 128, 0, true, 1>(1); run<3, 128, 3, true>(9); run<3, 128, 1, true>(9); run<0, 128, 3, true>(9); run<0, 128, 3, true>(5);
  return 0;
}
