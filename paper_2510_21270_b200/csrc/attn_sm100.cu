// attn_sm100.cu -- K6/K8: tcgen05/TMEM FlashAttention forward for sm_100a.
//
// One kernel serves both the permuted block-sparse attention
// (attention_block_sparse, attention.hpp:259-310, with the ElementMask of
// attention.hpp:41-73) and the project's dense causal comparator
// (attention_tiled with causal = true, attention.hpp:314-321): they differ only
// in the list of key blocks a query block visits.
//
// Tile: B = 128 query rows x 128 keys, d = 128, bf16 in, fp32 accumulate.
// Work item: a PAIR of query tiles of one head, query blocks 2p and 2p + 1
// (under B = 128, S = 256 the two blocks of one segment).  The CTA streams the
// union of the two tiles' visited key blocks once through shared memory and
// each K/V tile feeds both query tiles, so the K/V bytes moved per tensor-core
// FLOP halve against one tile per item, and the two tiles' softmax phases
// interleave on each SM sub-partition (one tile's exponentials run while the
// other's scores load; DESIGN.md §4 has the chain this sets and the
// alternatives measured).  Persistent CTAs (one per SM) take items from a global
// counter (warp 3 publishes them through an mbarrier ring), ordered one KV
// source at a time for L2 locality, heaviest pairs first.
// Warp roles (384 threads; setmaxnreg gives the softmax 208 registers):
//   warp 0       TMA producer for Q_0, Q_1 (once per item) and K (ring)
//   warp 2       TMA producer for V (ring)
//                (cp.async.bulk.tensor through 3-D [H, N, d] maps, SW128)
//   warp 3       item scheduler
//   warp 1       TMEM owner + MMA issuer (warp-collective, one elected lane).
//                Per union entry u, for tile w = 0 then 1:
//                  O_w (+)= P_w(u-1) V_{u-1}  (TS: P over S_w in TMEM, V MN-major)
//                  S_w = Q_w K_u^T            (SS: Q_w, K K-major in smem)
//                each only where tile w visits the block; the PV of keys 0-63
//                starts when the group signals that half of P (p_half).
//   warps 4..7   softmax group 0: query tile 0 (block 2p)
//   warps 8..11  softmax group 1: query tile 1 (block 2p + 1)
// TMEM holds S_0 | S_1 | O_0 | O_1.  A softmax thread owns one query row (one
// TMEM lane) and all 128 keys of each block its tile visits, with its own
// running max, sum and accumulator; the two warps of an SM sub-partition
// belong to different tiles, so one's exponentials overlap the other's loads.
// Per block: 4 x tcgen05.ld 32x32b.x32 (partial blocks masked in TMEM first),
// row max (3-input FMNMX), online softmax in the exp2 domain with lazy
// rescaling (O_w rescaled only when the max grows by more than 8),
// p = 2^(s c - m) on the MUFU written back over S_w as bf16 (tcgen05.st), then
// p_full.  The epilogue writes O_w / l straight to row out_rows[i] (the fused
// un-permute, pipeline.hpp:178); the tiles finish independently (no merge).
// Block classes follow AdmissibilityIndex::classify (attention.hpp:167-174):
// per-block [min, max] of original positions; `none` blocks are skipped by
// every role (an exact no-op, attention.hpp:286), `full` blocks skip the
// per-element test, `partial` ones compare k_orig[j] <= q_orig[i].  A small
// pre-pass (visit_pair_kernel) writes, per item, the ascending union of the
// two tiles' visited key blocks with both tiles' classes packed in; every
// role prefetches it 32 entries at a time and broadcasts entries by warp
// shuffle, so the hot loop has no dependent global loads.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace pbs_b200 {
namespace {

constexpr int kBM = 128;      // query rows per tile (= block size B)
constexpr int kBN = 128;      // keys per tile (= block size B)
constexpr int kD = 128;       // head dim
#ifndef PBS_ATTN_K_STAGES
#define PBS_ATTN_K_STAGES 2
#define PBS_ATTN_V_STAGES 2
#endif
constexpr int kKStages = PBS_ATTN_K_STAGES;  // K ring depth (freed once both tiles' QK^T complete)
constexpr int kVStages = PBS_ATTN_V_STAGES;  // V ring depth (freed once both tiles' PV complete)
constexpr int kGroups = 2;                   // softmax warpgroups = query tiles per item
constexpr int kCols = kBN;                   // key columns per softmax thread
constexpr int kSoftmaxThreads = 128 * kGroups;
constexpr int kThreads = 128 + kSoftmaxThreads;
constexpr int kRegsControl = 88;                  // setmaxnreg: producers / MMA issuer / scheduler
constexpr int kRegsSoftmax = 208;                 //             softmax warpgroups
static_assert((168 - kRegsControl) * 128 >= (kRegsSoftmax - 168) * kSoftmaxThreads, "register file split");
// keys of every 16 whose exp2 runs on the FMA pipe (polynomial) instead of the
// MUFU; 0: with two groups working on different tiles the MUFU keeps up
// (round 1 A/B on the box: 0 / 2 / 4 of 16 -> 61 / 62 / 66 ms x GHz at 128K)
#ifndef PBS_PRODUCER_SLEEP_NS
#define PBS_PRODUCER_SLEEP_NS 64
#endif
#ifndef PBS_POLY_PER16
#define PBS_POLY_PER16 0
#endif
constexpr int kPolyPer16 = PBS_POLY_PER16;
#ifndef PBS_ITEM_RING
#define PBS_ITEM_RING 1
#endif
// items claimed ahead of the consumers: a deep ring let the first CTAs to reach
// a head's heavy items each hoard several of them (CTA end times spread over
// 1.4 ms of a 5 ms 4-head launch with 4 slots, 0.6 ms with 2, 0.17 ms with 1;
// e2e at C3 50.1 / 49.1 / 48.1 ms)
constexpr int kItemRing = PBS_ITEM_RING;
constexpr int kItemConsumers = 3 + kSoftmaxThreads / 32;  // warps 0, 1, 2 and the softmax warps
constexpr int kPanelBytes = kBM * 128;            // 128 rows x 64 bf16 (SW128 panel)
constexpr int kTileBytes = 2 * kPanelBytes;       // 128 x 128 bf16 = 32 KB
constexpr uint32_t kTmemCols = 512;               // S0 | S1 | O0 | O1
__host__ __device__ constexpr uint32_t col_s(int w) { return (uint32_t)w * 128u; }
__host__ __device__ constexpr uint32_t col_o(int w) { return 256u + (uint32_t)w * 128u; }
// union entry: kb | class of tile 0 << 26 | class of tile 1 << 28
constexpr int kKbBits = 26;
constexpr uint32_t kKbMask = (1u << kKbBits) - 1u;

struct __align__(8) Barriers {
  uint64_t q_full[kGroups], q_empty[kGroups];
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[kGroups];  // S_w = Q_w K^T complete (and every earlier MMA: tile w's previous PV)
  uint64_t p_half[kGroups];  // P_w's first 64 keys written (the PV of those keys may start)
  uint64_t p_full[kGroups];  // P_w written into TMEM over S_w by the group's 128 threads
  uint64_t o_full[kGroups];  // tile w's last PV of the item complete
  uint64_t o_free[kGroups];  // group w's epilogue read O_w
  uint64_t drained;  // every tcgen05 operation of the MMA issuer complete (before dealloc)
  // dynamic work distribution: warp 3 claims items from a global counter and
  // publishes them through this ring to the 11 consumer warps
  uint64_t item_full[kItemRing], item_empty[kItemRing];
  int32_t item_ring[kItemRing];
  uint32_t tmem_base;
};

struct SmemLayout {
  // 1024-byte aligned tiles (SW128 atoms)
  static constexpr int q = 0;                              // Q_0 | Q_1
  static constexpr int k = q + kGroups * kTileBytes;
  static constexpr int v = k + kKStages * kTileBytes;
  static constexpr int korig = v + kVStages * kTileBytes;  // int [kGroups][128]
  static constexpr int bars = korig + kGroups * 128 * 4;
  static constexpr int total = bars + sizeof(Barriers) + 1024;  // + alignment slack
};
static_assert(SmemLayout::total <= 232448, "shared memory budget");

// ---- PTX wrappers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Softmax -> MMA signals: one arrival per warp (the barrier counts 4 per group)
// after the warp's lanes have fenced their TMEM accesses, instead of 128 lane
// arrivals serialised on one shared-memory word.
#ifdef PBS_LANE_ARRIVE
constexpr int kGroupArrivals = 128;
__device__ __forceinline__ void group_arrive(uint64_t* bar) { mbar_arrive(bar); }
#else
constexpr int kGroupArrivals = 4;
__device__ __forceinline__ void group_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
#endif
// Bounded wait: a deadlock becomes a trap (~10 s at 2 GHz; the launch then fails
// with an illegal-instruction error) instead of a hung GPU.  The trap is inline:
// a call (e.g. to printf) would make every wait site an ABI call boundary and
// force the softmax's 128 live scores into local memory.
__device__ __forceinline__ bool mbar_try(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(addr, parity))
    if (clock64() - t0 > 20000000000ll) asm volatile("trap;");
}

// Producer-side wait (slot free): the TMA warps run ahead of the consumers, so
// they poll with a short sleep instead of spinning.  A spinning producer
// re-issued its try_wait loop ~65 times per tile and took issue slots from the
// softmax warps of its SM sub-partition (ncu source page).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try(addr, parity)) return;
  const long long t0 = clock64();
  do {
    __nanosleep(PBS_PRODUCER_SLEEP_NS);
    if (clock64() - t0 > 20000000000ll) asm volatile("trap;");
  } while (!mbar_try(addr, parity));
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Warp-collective forms: the whole (converged) warp executes these and one
// elected lane issues.  Keeping the issuing code warp-uniform lets the
// descriptors live in uniform registers; a `lane == 0` branch instead makes the
// compiler wrap every tcgen05.mma in a waterfall loop of R2UR conversions.
__device__ __forceinline__ void tc_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// QK^T of one tile, K = d = 128 as 8 MMAs from ONE elected lane, descriptors
// advanced inside the asm block (start address field = byte address >> 4):
// k-step k reads bytes (k & 3) * 32 + (k >> 2) * kPanelBytes past the bases.
// One election and one register->uniform move per operand for the 8 MMAs
// .
__device__ __forceinline__ void tc_mma_qk8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n"
      ".reg .pred e, t, f;\n"
      ".reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
      "setp.ne.b32 t, 1, 0;\n"
      "setp.ne.b32 f, 0, 0;\n"
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
      "l"(adesc), "l"(bdesc), "r"(idesc)
      : "memory");
}

// PV over 64 keys: 4 MMAs (K = 16 keys each), A = P in TMEM (+8 columns per
// step), B = V rows advancing 16 x 128 bytes (encoded +128) per step.
__device__ __forceinline__ void tc_mma_pv4(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred e, t, p;\n"
      ".reg .b32 a1, a2, a3;\n"
      ".reg .b64 b1, b2, b3;\n"
      "setp.ne.b32 t, 1, 0;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "add.s32 a1, %1, 8;   add.s64 b1, %2, 128;\n"
      "add.s32 a2, %1, 16;  add.s64 b2, %2, 256;\n"
      "add.s32 a3, %1, 24;  add.s64 b3, %2, 384;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, t;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#define TMEM_ST16(taddr, r)                                                                                     \
  asm volatile(                                                                                                 \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "  \
      "%14, %15, %16};" ::"r"(taddr),                                                                          \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),        \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])                         \
      : "memory")

#define TMEM_LD32(taddr, r)                                                                                     \
  asm volatile(                                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "    \
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"       \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),         \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),   \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),              \
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),              \
        "=r"(r[30]), "=r"(r[31])                                                                                \
      : "r"(taddr))

#define TMEM_ST32(taddr, r)                                                                                     \
  asm volatile(                                                                                                 \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "  \
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"        \
      ::"r"(taddr),                                                                                             \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),        \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),            \
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),           \
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                        \
      : "memory")

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// 2^x on the FMA/ALU pipes (Cody-Waite split + degree-3 minimax on [-1/2, 1/2],
// max relative error 7.7e-5, far below bf16 P's 2^-9): offloads the MUFU unit.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -126.5f);
  const float t = x + 12582912.0f;  // 1.5 * 2^23: round-to-nearest integer in the low bits
  const float jf = t - 12582912.0f;
  const float f = x - jf;
  float p = fmaf(0.055219680070877075f, f, 0.2426094114780426f);
  p = fmaf(p, f, 0.6932516694068909f);
  p = fmaf(p, f, 0.9999279975891113f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// SW128 shared-memory matrix descriptor (sm100: version 1 at bit 46, layout 2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16 instruction descriptor: f32 accumulate, bf16 A/B, M=128, N=128
__host__ __device__ constexpr uint32_t make_idesc(uint32_t a_mn_major, uint32_t b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn_major << 15) | (b_mn_major << 16) | ((uint32_t)(kBN >> 3) << 17) |
         ((uint32_t)(kBM >> 4) << 24);
}

struct KernelArgs {
  int hq, kv_heads, group;
  int64_t n, t;    // t = ceil(n / block): query / key blocks of the selection
  int64_t block;   // B: 128, or 64 (sub-blocked tiles, below)
  int sub;         // B = 64: a 128 x 128 tile holds 2 x 2 selection blocks with their own classes
  int64_t t128;    // ceil(n / 128): tiles per head
  int64_t npairs;  // ceil(t128 / 2): items are (head, pair of query tiles 2p, 2p + 1)
  int64_t p_lo, p_hi;  // pairs [p_lo, p_hi) of every head (a shard's query-block range)
  float scale_log2;
  const int32_t* kv_idx;
  const int32_t* kv_cnt;
  const int32_t* q_orig;
  const int32_t* k_orig;
  const int32_t* out_rows;
  const int2* q_mm;  // [hq][t] min/max of q_orig per block (nullptr: identity)
  const int2* k_mm;  // [hq][t] min/max of k_orig per block
  int32_t* status;
  float* lse;  // [hq][n] in output-row order, or nullptr
  __nv_bfloat16* out;
  int causal;   // identity element mask when q_orig/k_orig are null
  int dense;    // dense causal lists (kb = 0..qb)
  int64_t items;
  const int32_t* vis;   // [hq][npairs][t] union lists (kb | c0 << 26 | c1 << 28), sparse mode
  const int32_t* nvis;  // [hq][npairs]
  int32_t* item_counter;  // zeroed before the launch; items are claimed in order (heaviest first)
  unsigned long long* trace;  // span sums (-DPBS_ATTN_SPANS with PBS_ATTN_TRACE), else nullptr
};

// Span accounting (-DPBS_ATTN_SPANS, debug): every CTA sums the clock64 time
// its MMA warp and one thread per softmax group spend in each pipeline phase
// and adds the totals into a.trace[0..32) at exit; no per-event stores, so the
// timings are those of the product build.
#ifdef PBS_ATTN_SPANS
#define SPAN_DECL unsigned long long sp_[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long sp_t_ = clock64();
#define SPAN(i) do { const long long n_ = clock64(); sp_[i] += (unsigned long long)(n_ - sp_t_); sp_t_ = n_; } while (0)
#define SPAN_COUNT(i) (++sp_[i])
#define SPAN_FLUSH(cond, base) do { if ((cond) && a.trace) for (int i_ = 0; i_ < 8; ++i_) atomicAdd(a.trace + (base) + i_, sp_[i_]); } while (0)
#else
#define SPAN_DECL
#define SPAN(i) do { } while (0)
#define SPAN_COUNT(i) do { } while (0)
#define SPAN_FLUSH(cond, base) do { } while (0)
#endif
// Event timeline (-DPBS_ATTN_EVENTS, debug): CTA 0's first 1024 steps, clock64
// stamps into a.trace[32 + step * 8 + k] (MMA warp) and a.trace[8224 + ...] (softmax)
#ifdef PBS_ATTN_EVENTS
#define EVT(cond, idx, k) do { if ((cond) && blockIdx.x == 0 && a.trace && (idx) < 2048) a.trace[32 + (idx) * 8 + (k)] = clock64(); } while (0)
#else
#define EVT(cond, idx, k) do { } while (0)
#endif

struct Item {
  int h;
  int64_t p;  // query blocks 2p (tile 0) and 2p + 1 (tile 1, when < t)
};

__device__ __forceinline__ Item item_of(const KernelArgs& a, int64_t idx) {
  // L2 locality: all CTAs sweep one KV source at a time (per q head for the
  // per-head permuted K'/V', per GQA group for shared K/V), heaviest pairs
  // first inside it.
  Item it;
  const int64_t np = a.p_hi - a.p_lo;
  const int64_t per = np * (a.kv_heads == a.hq ? 1 : a.group);
  const int64_t grp = idx / per, rem = idx % per;
  if (a.kv_heads == a.hq) {
    it.h = (int)grp;
    it.p = a.p_hi - 1 - rem;
  } else {
    it.h = (int)(grp * a.group + rem % a.group);
    it.p = a.p_hi - 1 - rem / a.group;
  }
  return it;
}

__device__ __forceinline__ int2 q_range(const KernelArgs& a, int h, int64_t qb) {
  if (a.q_mm) return a.q_mm[(int64_t)h * a.t + qb];
  const int64_t lo = qb * a.block;
  return make_int2((int)lo, (int)(min64(a.n, lo + a.block) - 1));
}
__device__ __forceinline__ int2 k_range(const KernelArgs& a, int h, int64_t kb) {
  if (a.k_mm) return a.k_mm[(int64_t)h * a.t + kb];
  const int64_t lo = kb * a.block;
  return make_int2((int)lo, (int)(min64(a.n, lo + a.block) - 1));
}

// 0 none, 1 partial, 2 full (AdmissibilityIndex::classify); a ragged key block is
// treated as partial so that keys past N are masked.
__device__ __forceinline__ int block_class(const KernelArgs& a, int h, int64_t qb, int64_t kb) {
  const bool masked = a.causal || a.q_orig || a.k_orig;
  const bool ragged = (kb + 1) * a.block > a.n;
  if (!masked) return ragged ? 1 : 2;
  const int2 qr = q_range(a, h, qb), kr = k_range(a, h, kb);
  if (kr.y <= qr.x) return ragged ? 1 : 2;
  if (kr.x > qr.y) return 0;
  return 1;
}

// visited-block cursor over an item's union list: dense causal lists are
// computed, sparse lists come from the pre-pass, prefetched 32 entries per warp.
struct Visit {
  const int32_t* list;
  int len;
  int base;
  uint32_t cache;
};

__device__ __forceinline__ Visit visit_begin(const KernelArgs& a, const Item& it) {
  Visit v;
  v.base = -64;
  v.cache = 0;
  if (a.dense) {
    v.list = nullptr;
    v.len = (int)(min64(2 * it.p + 1, a.t - 1) + 1);  // 0 .. last query block of the pair
  } else {
    v.list = a.vis + ((int64_t)it.h * a.npairs + it.p) * a.t128;
    v.len = a.nvis[(int64_t)it.h * a.npairs + it.p];
  }
  return v;
}

// Sub-blocked entries (B = 64): kt | sc << 16, sc = 2-bit classes of the 8
// selection blocks of the entry, bit 2 * (4 w + 2 a + b) for tile w, query half
// a (rows 64a..) and key half b (keys 64b..)
constexpr int kSubShift = 16;
__device__ __forceinline__ int sub_class(uint32_t sc, int w, int a_half, int b_half) {
  return (int)((sc >> (2 * (4 * w + 2 * a_half + b_half))) & 3u);
}
// tile w's class from its four blocks: 0 none visited, 2 all four full, else 1
__device__ __forceinline__ int tile_class(uint32_t sc, int w) {
  const uint32_t q = (sc >> (8 * w)) & 0xffu;
  return q == 0 ? 0 : (q == 0xaau ? 2 : 1);
}

// all 32 lanes of the warp must call this with the same e (e non-decreasing);
// c0 / c1: the block's class for tile 0 / tile 1 (0 = not visited by that tile);
// sc: the sub-blocked classes (B = 64), else 0
__device__ __forceinline__ void visit_get(const KernelArgs& a, const Item& it, Visit& v, int e, int lane,
                                          int64_t& kb, int& c0, int& c1, uint32_t& sc) {
  sc = 0;
  if (a.dense) {
    kb = e;
    const bool ragged = (kb + 1) * kBN > a.n;
    const int64_t qb0 = 2 * it.p, qb1 = qb0 + 1;
    c0 = kb < qb0 ? (ragged ? 1 : 2) : (kb == qb0 ? 1 : 0);
    c1 = qb1 < a.t ? ((kb < qb1 && !ragged) ? 2 : 1) : 0;
    return;
  }
  if (e >= v.base + 32) {
    v.base = e & ~31;
    v.cache = (v.base + lane < v.len) ? (uint32_t)__ldg(v.list + v.base + lane) : 0u;
  }
  const uint32_t x = __shfl_sync(0xffffffffu, v.cache, e - v.base);
  if (a.sub) {
    kb = x & ((1u << kSubShift) - 1u);
    sc = x >> kSubShift;
    c0 = tile_class(sc, 0);
    c1 = tile_class(sc, 1);
    return;
  }
  kb = x & kKbMask;
  c0 = (int)((x >> kKbBits) & 3u);
  c1 = (int)((x >> (kKbBits + 2)) & 3u);
}

// overload for the roles that only need the tiles' classes
__device__ __forceinline__ void visit_get(const KernelArgs& a, const Item& it, Visit& v, int e, int lane,
                                          int64_t& kb, int& c0, int& c1) {
  uint32_t sc;
  visit_get(a, it, v, e, lane, kb, c0, c1, sc);
}

__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint64_t pk2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair on the FMA/ALU pipes (packed f32x2): the Cody-Waite split and
// degree-3 minimax of exp2_poly.  Offloads the MUFU, whose 16 ex2/clk/SM take
// as long as the block's two MMAs.
__device__ __forceinline__ void exp2_poly2(float y0, float y1, float& p0, float& p1) {
  const uint64_t x = pk2(fmaxf(y0, -126.5f), fmaxf(y1, -126.5f));
  const uint64_t t = fadd2(x, pk2(12582912.0f, 12582912.0f));
  const uint64_t jf = fadd2(t, pk2(-12582912.0f, -12582912.0f));
  const uint64_t f = fadd2(x, jf ^ 0x8000000080000000ull);
  uint64_t p = ffma2(pk2(0.055219680070877075f, 0.055219680070877075f), f,
                     pk2(0.2426094114780426f, 0.2426094114780426f));
  p = ffma2(p, f, pk2(0.6932516694068909f, 0.6932516694068909f));
  p = ffma2(p, f, pk2(0.9999279975891113f, 0.9999279975891113f));
  float q0, q1, t0, t1;
  upk2(p, q0, q1);
  upk2(t, t0, t1);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

// Pass 1 (per visited block): this thread's kCols scores and their max
// (3-input FMNMX, eight independent chains).
__device__ __forceinline__ float load_scores(uint32_t tS, uint32_t (&r)[kCols]) {
#pragma unroll
  for (int c = 0; c < kCols / 32; ++c) TMEM_LD32(tS + c * 32, (r + c * 32));
  tmem_wait_ld();
  float mx[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) mx[u] = __uint_as_float(r[u]);
#pragma unroll
  for (int j = 8; j + 16 <= kCols; j += 16) {
#pragma unroll
    for (int u = 0; u < 8; ++u) mx[u] = max3(mx[u], __uint_as_float(r[j + u]), __uint_as_float(r[j + 8 + u]));
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) mx[u] = fmaxf(mx[u], __uint_as_float(r[kCols - 8 + u]));
  return max3(max3(mx[0], mx[1], mx[2]), max3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7]));
}

// Pass 2: p = 2^(s * scale_log2 - m) -> bf16 pairs written into TMEM over the
// consumed S columns (two keys per 32-bit column: the A-operand layout of the
// PV MMA), one 32-key chunk at a time; returns sum p.  Packed f32x2 FMA/add;
// kPolyPer16 of every 16 keys take the FMA-pipe polynomial.
template <int kPolyPer16>
__device__ __forceinline__ float emit_p(const uint32_t (&r)[kCols], float sc, float neg_m, uint32_t tP,
                                        uint64_t* half_bar) {
  const uint64_t sc2 = pk2(sc, sc), nm2 = pk2(neg_m, neg_m);
  uint64_t sum2[2] = {0ull, 0ull};
#pragma unroll
  for (int c = 0; c < kCols / 32; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int jp = 0; jp < 16; ++jp) {
      const int j = c * 32 + 2 * jp;
      float y0, y1, p0, p1;
      upk2(ffma2(pk2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), sc2, nm2), y0, y1);
      if ((j & 15) >= 16 - kPolyPer16) {
        exp2_poly2(y0, y1, p0, p1);
      } else {
#ifdef PBS_EXP_FAKE  // timing experiment only (wrong results): no MUFU work
        p0 = fmaxf(fmaf(y0, 0.001f, 1.0f), 0.0f);
        p1 = fmaxf(fmaf(y1, 0.001f, 1.0f), 0.0f);
#else
        p0 = ex2(y0);
        p1 = ex2(y1);
#endif
      }
      sum2[jp & 1] = fadd2(sum2[jp & 1], pk2(p0, p1));
      __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
      pk[jp] = *reinterpret_cast<uint32_t*>(&b2);
    }
    TMEM_ST16(tP + c * 16, pk);
    if (c == 1) {  // keys 0..63 are in TMEM: their half of the PV may start
      tmem_wait_st();
      tc_fence_before();
      group_arrive(half_bar);
    }
  }
  float s0, s1, s2, s3;
  upk2(sum2[0], s0, s1);
  upk2(sum2[1], s2, s3);
  return (s0 + s1) + (s2 + s3);
}

// The item sequence of this CTA, as published by the scheduler warp: every
// consumer warp reads the same sequence in order; -1 ends it.
struct ItemStream {
  uint32_t n = 0;
  __device__ __forceinline__ int64_t next(Barriers* bar, int lane) {
    const int slot = (int)(n % kItemRing);
    mbar_wait(&bar->item_full[slot], (n / kItemRing) & 1);
    // atomic access: the slot hand-over is ordered by the mbarriers, which
    // compute-sanitizer's racecheck does not model for plain shared accesses
    const int32_t idx = atomicOr(&bar->item_ring[slot], 0);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar->item_empty[slot]);
    ++n;
    return idx;
  }
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const KernelArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Barriers* bar = reinterpret_cast<Barriers*>(smem + SmemLayout::bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int w = 0; w < kGroups; ++w) {
      mbar_init(&bar->q_full[w], 1);
      mbar_init(&bar->q_empty[w], 1);
      mbar_init(&bar->s_full[w], 1);
      mbar_init(&bar->p_half[w], kGroupArrivals);
      mbar_init(&bar->p_full[w], kGroupArrivals);
      mbar_init(&bar->o_full[w], 1);
      mbar_init(&bar->o_free[w], kGroupArrivals);
    }
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&bar->k_full[s], 1);
      mbar_init(&bar->k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&bar->v_full[s], 1);
      mbar_init(&bar->v_empty[s], 1);
    }
    mbar_init(&bar->drained, 1);
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(&bar->item_full[i], 1);
      mbar_init(&bar->item_empty[i], kItemConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&bar->tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar->tmem_base;
#ifdef PBS_ATTN_EVENTS
  if (threadIdx.x == 0 && a.trace) {  // per-CTA start time (global ns)
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.trace[32 + 2048 * 8 + 512 + blockIdx.x] = gt;
  }
#endif

  if (warp < 4) {
   asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsControl));
   if (warp == 0 || warp == 2) {
    // ===================== TMA producers (lane 0 issues) =====================
    // warp 0: Q_0, Q_1 + the K ring; warp 2: the V ring.  Both walk the union list.
    const bool kp = (warp == 0);
    uint32_t q_it = 0, it_k = 0;
    ItemStream items;
    for (int64_t idx; (idx = items.next(bar, lane)) >= 0;) {
      const Item it = item_of(a, idx);
      const int kvh = it.h / a.group;
      Visit vis = visit_begin(a, it);
      if (kp && lane == 0) {
        for (int w = 0; w < kGroups; ++w) {
          int64_t qb = 2 * it.p + w;
          if (qb >= a.t128) qb = 2 * it.p;  // a lone last tile: tile 1's buffer gets tile 0's rows (never read)
          mbar_wait_backoff(&bar->q_empty[w], (q_it & 1) ^ 1);
          mbar_expect_tx(&bar->q_full[w], kTileBytes);
          for (int p = 0; p < 2; ++p)
            tma_load_3d(smem + SmemLayout::q + w * kTileBytes + p * kPanelBytes, &tm_q, &bar->q_full[w], p * 64,
                        (int)(qb * kBM), it.h);
        }
      }
      ++q_it;
      for (int e = 0; e < vis.len; ++e) {
        int64_t kb;
        int c0, c1;
        visit_get(a, it, vis, e, lane, kb, c0, c1);
        if (lane == 0) {
          const int nst = kp ? kKStages : kVStages;
          const int s = (int)(it_k % nst);
          uint64_t* empty = kp ? &bar->k_empty[s] : &bar->v_empty[s];
          uint64_t* full = kp ? &bar->k_full[s] : &bar->v_full[s];
          mbar_wait_backoff(empty, ((it_k / nst) & 1) ^ 1);
#ifdef PBS_NO_KV_LOAD  // timing experiment only (wrong results): K/V tiles loaded once per ring slot
          if (it_k >= (uint32_t)nst) {
            mbar_arrive(full);
            ++it_k;
            continue;
          }
#endif
          mbar_expect_tx(full, kTileBytes);
          unsigned char* dst = smem + (kp ? SmemLayout::k : SmemLayout::v) + s * kTileBytes;
          for (int p = 0; p < 2; ++p)
            tma_load_3d(dst + p * kPanelBytes, kp ? &tm_k : &tm_v, full, p * 64, (int)(kb * kBN), kvh);
        }
        ++it_k;
      }
    }
   } else if (warp == 1) {
    // ===================== MMA issuer (warp-collective, one elected lane) ========
    // Union entry u, tile w = 0 then 1:
    //   O_w (+)= P_w(u-1) V_{u-1}  if tile w visited entry u-1 (its softmax wrote P over S_w)
    //   S_w = Q_w K_u^T            if tile w visits entry u (after that PV in issue
    //                              order: it overwrites P_w)
    // so K_u and V_{u-1} are each consumed within one step and free right after.
    const uint32_t idesc_qk = make_idesc(0, 0);  // Q K-major, K K-major
    const uint32_t idesc_pv = make_idesc(0, 1);  // P K-major (TMEM), V MN-major
    const uint32_t q_base = smem_u32(smem + SmemLayout::q);
    uint32_t q_it = 0, k_it = 0, v_it = 0, o_no[kGroups] = {0, 0}, p_cnt[kGroups] = {0, 0};
    uint32_t gs = 0;  // CTA step counter (events)
    SPAN_DECL
    ItemStream items;
    for (int64_t idx; (idx = items.next(bar, lane)) >= 0;) {
      const Item it = item_of(a, idx);
      Visit vis = visit_begin(a, it);
      for (int w = 0; w < kGroups; ++w) mbar_wait(&bar->q_full[w], q_it & 1);
      ++q_it;
      SPAN(7);
      if (vis.len == 0) {
        for (int w = 0; w < kGroups; ++w) tc_commit_w(&bar->q_empty[w]);
        continue;
      }
      bool pend[kGroups] = {false, false}, first[kGroups] = {true, true};
      for (int u = 0; u <= vis.len; ++u, ++gs) {
        int64_t kb = 0;
        int cls[kGroups] = {0, 0};
        EVT(lane == 0 && gs < 1024, gs, 0);
        if (u < vis.len) visit_get(a, it, vis, u, lane, kb, cls[0], cls[1]);
        uint32_t v_base = 0;
        if (u > 0) {
          const uint32_t vs = v_it % kVStages;
          mbar_wait(&bar->v_full[vs], (v_it / kVStages) & 1);
          v_base = smem_u32(smem + SmemLayout::v + vs * kTileBytes);
        }
        const uint32_t ks = k_it % kKStages;
        const uint32_t k_base = smem_u32(smem + SmemLayout::k + ks * kTileBytes);
        bool k_seen = false;
        EVT(lane == 0 && gs < 1024, gs, 1);
        // the tile whose PV is the last reader of V_{u-1}: the V slot is released
        // right after it, before the following QK^T (a commit covers every
        // earlier MMA, so a later commit would hold the slot for one more QK^T)
        const int last_pv = pend[1] ? 1 : 0;
        SPAN(0);
#pragma unroll
        for (int w = 0; w < kGroups; ++w) {
          if (pend[w]) {
            // A = P [128 q x 128 kv] in TMEM (64 columns over S_w); B = V [128 kv x 128 d] MN-major SW128.
            // Keys 0..63 go as soon as the group wrote them, keys 64..127 after the rest.
            static_assert(kBN == 128, "two 64-key PV halves");
            if (first[w]) mbar_wait(&bar->o_free[w], (o_no[w] & 1) ^ 1);  // the previous epilogue read O_w
            mbar_wait(&bar->p_half[w], p_cnt[w] & 1);
            SPAN(1);
            tc_fence_after();
            tc_mma_pv4(tmem + col_o(w), tmem + col_s(w), sdesc(v_base, kPanelBytes, 1024), idesc_pv,
                       first[w] ? 0u : 1u);
            SPAN(2);
            mbar_wait(&bar->p_full[w], p_cnt[w] & 1);
            EVT(lane == 0 && gs < 1024, gs, 2 + 2 * w);
            SPAN(1);
            ++p_cnt[w];
            tc_fence_after();
            tc_mma_pv4(tmem + col_o(w), tmem + col_s(w) + 32, sdesc(v_base + 64 * 128, kPanelBytes, 1024), idesc_pv,
                       1u);
            SPAN(3);
            first[w] = false;
            pend[w] = false;
#ifndef PBS_LATE_V_RELEASE
            if (w == last_pv) {
              tc_commit_w(&bar->v_empty[v_it % kVStages]);
              ++v_it;
            }
#endif
          }
          if (cls[w]) {
            if (!k_seen) {
              mbar_wait(&bar->k_full[ks], (k_it / kKStages) & 1);
              SPAN(5);
              k_seen = true;
            }
            tc_fence_after();
            static_assert(kD == 128 && kPanelBytes == 1024 * 16, "tc_mma_qk8 descriptor steps");
            tc_mma_qk8(tmem + col_s(w), sdesc(q_base + w * kTileBytes, 16, 1024), sdesc(k_base, 16, 1024),
                       idesc_qk);
            tc_commit_w(&bar->s_full[w]);
            EVT(lane == 0 && gs < 1024, gs, 3 + 2 * w);
            SPAN(6);
            pend[w] = true;
          }
        }
#ifdef PBS_LATE_V_RELEASE
        if (u > 0) {
          tc_commit_w(&bar->v_empty[v_it % kVStages]);
          ++v_it;
        }
#endif
        if (u < vis.len) {
          tc_commit_w(&bar->k_empty[ks]);
          ++k_it;
          SPAN_COUNT(4);
        }
        EVT(lane == 0 && gs < 1024, gs, 6);
        if (u + 1 == vis.len)  // every QK^T of the item issued: Q_0, Q_1 are free once they complete
          for (int w = 0; w < kGroups; ++w) tc_commit_w(&bar->q_empty[w]);
      }
      for (int w = 0; w < kGroups; ++w)
        if (!first[w]) {
          tc_commit_w(&bar->o_full[w]);
          ++o_no[w];
        }
      SPAN(3);
    }
    // nothing may still write TMEM when it is released
    tc_commit_w(&bar->drained);
    mbar_wait(&bar->drained, 0);
    SPAN_FLUSH(lane == 0, 0);
   } else {
    // ===================== scheduler: claim items in order, publish them =========
    if (lane == 0) {
      for (uint32_t n = 0;; ++n) {
        const int slot = (int)(n % kItemRing);
        mbar_wait(&bar->item_empty[slot], ((n / kItemRing) & 1) ^ 1);
        int32_t idx = atomicAdd(a.item_counter, 1);
        if ((int64_t)idx >= a.items) idx = -1;
        atomicExch(&bar->item_ring[slot], idx);
        mbar_arrive(&bar->item_full[slot]);  // release: the consumers' wait orders the read after the write
        if (idx < 0) break;
      }
    }
   }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
    // ===================== softmax: group w owns query tile w of the item ==========
    // One thread per query row (TMEM lane) and all 128 keys of each visited block,
    // with the row's running max m, sum l and accumulator O_w.  O_w is stable when
    // S_w is ready: the tile's previous PV was issued before this QK^T, whose
    // commit covers it, so the lazy rescale needs no wait.
    const int w = (warp - 4) >> 2;     // softmax group = query tile
    const int quad = warp & 3;         // TMEM lane quadrant of this warp
    const int row = quad * 32 + lane;  // query row within the tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + lane_off + col_s(w);
    const uint32_t tO = tmem + lane_off + col_o(w);
    int* ko = reinterpret_cast<int*>(smem + SmemLayout::korig) + w * 128;
    const float sc = a.scale_log2;
    const bool any_mask = a.causal || a.q_orig || a.k_orig;
    uint32_t s_cnt = 0, o_cnt = 0;
    SPAN_DECL
    ItemStream items;
    for (int64_t idx; (idx = items.next(bar, lane)) >= 0;) {
      const Item it = item_of(a, idx);
      Visit vis = visit_begin(a, it);
      const int64_t qb = 2 * it.p + w;  // query tile (128 rows)
      const int64_t i = qb * kBM + row;
      const bool valid = qb < a.t128 && i < a.n;
      // the selection block of this thread's row (degenerate-row reports)
      const int64_t qsel = a.sub ? 2 * qb + (row >> 6) : qb;
      const int qo = valid ? (a.q_orig ? a.q_orig[(int64_t)it.h * a.n + i] : (int)i) : -1;
      float m = -INFINITY;  // running max (log2 domain)
      float l = 0.0f;       // running sum
      bool any = false;
      for (int e = 0; e < vis.len; ++e) {
        int64_t kb;
        int c0, c1;
        uint32_t scl;
        EVT(row == 0 && w == 0 && s_cnt < 1024, 1024 + s_cnt, 0);
        visit_get(a, it, vis, e, lane, kb, c0, c1, scl);
        const int cls = w ? c1 : c0;
        if (cls == 0) continue;  // warp-uniform: a block's class is the tile's
        any = true;
        if (cls == 1) {  // original positions of the block's keys, for this tile
          const int64_t j = kb * kBN + row;
          int v = 0x7fffffff;
          if (j < a.n) v = a.k_orig ? a.k_orig[(int64_t)it.h * a.n + j] : (int)j;
          if (!any_mask && j < a.n) v = -1;  // unmasked: only the ragged tail
          ko[row] = v;
          named_bar_sync(1 + w, 128);
        }
        SPAN(0);
        EVT(row == 0 && w == 0 && s_cnt < 1024, 1024 + s_cnt, 1);
        mbar_wait(&bar->s_full[w], s_cnt & 1);
        EVT(row == 0 && w == 0 && s_cnt < 1024, 1024 + s_cnt, 2);
        SPAN(1);
        SPAN_COUNT(7);
        ++s_cnt;
        tc_fence_after();
#if defined(PBS_SOFTMAX_NOP) || defined(PBS_SOFTMAX_LOADONLY)  // timing experiments only (wrong results)
        {
#ifdef PBS_SOFTMAX_LOADONLY
          uint32_t r[kCols];
          const float hm = load_scores(tS, r);
          m = fmaxf(m, hm * sc);
#endif
          l = 1.0f;
          tc_fence_before();
          group_arrive(&bar->p_half[w]);
          group_arrive(&bar->p_full[w]);
          SPAN(4);
          continue;
        }
#endif
        uint32_t r[kCols];
        if (cls == 1) {
          // ElementMask (attention.hpp:41-73) applied in TMEM, 32 columns at a
          // time, so the 128 scores below are loaded already masked
#pragma unroll 1
          for (int c = 0; c < kCols / 32; ++c) {
            // B = 64: this warp's query half against key half c / 2 -- a block
            // not selected for it is masked whole, a full one not at all
            const int bc = a.sub ? sub_class(scl, w, quad >> 1, c >> 1) : 1;
            if (bc == 2) continue;
            uint32_t t32[32];
            TMEM_LD32(tS + c * 32, t32);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (bc == 0 || ko[c * 32 + j] > qo) t32[j] = 0xff800000u;  // -inf: inadmissible (attention.hpp:298-300)
            TMEM_ST32(tS + c * 32, t32);
          }
          tmem_wait_st();
          named_bar_sync(1 + w, 128);  // ko may be refilled after this
        }
        const float hmax = load_scores(tS, r);
        EVT(row == 0 && w == 0 && s_cnt <= 1024, 1023 + s_cnt, 3);
        SPAN(2);
        // online softmax (absorb, attention.hpp:96-126) in the log2 domain with
        // lazy rescaling: O_w is rescaled only when the max grows by more than 8
        const float m_new = fmaxf(m, hmax * sc);
        float factor = 1.0f;
        bool rescale = false;
        if (m_new != -INFINITY) {
          if (m == -INFINITY) {
            m = m_new;  // nothing accumulated for this row in O_w yet (exactly 0)
          } else if (m_new > m + 8.0f) {
            factor = ex2(m - m_new);
            rescale = true;
            m = m_new;
          }
        }
        const float neg_m = (m == -INFINITY) ? 0.0f : -m;
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
          for (int c = 0; c < kD / 32; ++c) {
            uint32_t o[32];
            TMEM_LD32(tO + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * factor);
            TMEM_ST32(tO + c * 32, o);
          }
        }
        SPAN(3);
        EVT(row == 0 && w == 0 && s_cnt <= 1024, 1023 + s_cnt, 4);
        const float rs = emit_p<kPolyPer16>(r, sc, neg_m, tS, &bar->p_half[w]);
        l = l * factor + rs;
        tmem_wait_st();
        tc_fence_before();
        group_arrive(&bar->p_full[w]);
        EVT(row == 0 && w == 0 && s_cnt <= 1024, 1023 + s_cnt, 5);
        SPAN(4);
      }
      // ---- epilogue (OnlineSoftmaxState::finalize, attention.hpp:130-138):
      // O_w / l -> out[out_rows[i]] (the fused un-permute, pipeline.hpp:178)
      if (!any) {  // the tile visits no block: no PV ran, O_w is not ours to read
        if (valid && a.status) {
          a.status[0] = 1;
          atomicMin(&a.status[1], (int)(it.h * a.t + qsel));
        }
        continue;
      }
      mbar_wait(&bar->o_full[w], o_cnt & 1);  // the tile's last PV
      ++o_cnt;
      tc_fence_after();
      if (valid && !(l > 0.0f) && a.status) {
        a.status[0] = 1;
        atomicMin(&a.status[1], (int)(it.h * a.t + qsel));
      }
      const int64_t orow = valid ? (a.out_rows ? (int64_t)a.out_rows[(int64_t)it.h * a.n + i] : i) : 0;
      if (a.lse && valid)  // natural-log LSE: l = sum 2^(s c - m), c = scale log2(e)
        a.lse[(int64_t)it.h * a.n + orow] = (l > 0.0f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
      const float inv = (l > 0.0f) ? 1.0f / l : 0.0f;
      __nv_bfloat16* dst = a.out + ((int64_t)it.h * a.n + orow) * kD;
#pragma unroll 1
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t o[32];
        TMEM_LD32(tO + c * 32, o);
        tmem_wait_ld();
        if (valid && l > 0.0f) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t pk[4];
#pragma unroll
            for (int w2 = 0; w2 < 4; ++w2) {
              const int j = u * 8 + 2 * w2;
              __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(o[j]) * inv, __uint_as_float(o[j + 1]) * inv);
              pk[w2] = *reinterpret_cast<uint32_t*>(&b2);
            }
            *reinterpret_cast<uint4*>(dst + c * 32 + u * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
      }
      tc_fence_before();
      group_arrive(&bar->o_free[w]);
      SPAN(5);
    }
    SPAN(6);
    SPAN_FLUSH(row == 0, 16 + 8 * w);
  }
  tc_fence_before();
  __syncthreads();
#ifdef PBS_ATTN_EVENTS
  if (threadIdx.x == 0 && a.trace) {  // per-CTA end time (global ns) for the launch's tail
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.trace[32 + 2048 * 8 + blockIdx.x] = gt;
  }
#endif
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// per item (head, pair of query blocks): the ascending union of the two tiles'
// selected key blocks, each with both tiles' classes (AdmissibilityIndex::
// classify; blocks of class none for both tiles dropped).  One warp per item:
// the two lists become bitmaps in shared memory, then each lane walks 32 words.
constexpr int kVisitWarps = 4;
__global__ void visit_pair_kernel(KernelArgs a, int words, int32_t* __restrict__ vis, int32_t* __restrict__ nvis) {
  extern __shared__ uint32_t bm_smem[];
  const int wip = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kVisitWarps + wip;
  if (g >= (int64_t)a.hq * a.npairs) return;
  uint32_t* bm0 = bm_smem + (size_t)wip * 2 * words;
  uint32_t* bm1 = bm0 + words;
  for (int x = lane; x < 2 * words; x += 32) bm0[x] = 0u;
  __syncwarp();
  const int h = (int)(g / a.npairs);
  const int64_t p = g % a.npairs;
  const int64_t qb0 = 2 * p, qb1 = qb0 + 1;
  for (int w = 0; w < kGroups; ++w) {
    const int64_t qb = qb0 + w;
    if (qb >= a.t) break;
    const int cnt = a.kv_cnt[(int64_t)h * a.t + qb];
    const int32_t* list = a.kv_idx + ((int64_t)h * a.t + qb) * a.t;
    uint32_t* bm = w ? bm1 : bm0;
    for (int e = lane; e < cnt; e += 32) {
      const int kb = list[e];
      atomicOr(&bm[kb >> 5], 1u << (kb & 31));
    }
  }
  __syncwarp();
  int32_t* out = vis + g * a.t128;
  int total = 0;
  for (int w0 = 0; w0 < words; w0 += 32) {
    const int wi = w0 + lane;
    const uint32_t m0 = wi < words ? bm0[wi] : 0u, m1 = wi < words ? bm1[wi] : 0u;
    uint32_t keep = 0u;
    for (uint32_t u = m0 | m1; u; u &= u - 1) {
      const int bit = __ffs(u) - 1;
      const int64_t kb = (int64_t)wi * 32 + bit;
      const int c0 = ((m0 >> bit) & 1u) ? block_class(a, h, qb0, kb) : 0;
      const int c1 = ((m1 >> bit) & 1u) ? block_class(a, h, qb1, kb) : 0;
      if (c0 | c1) keep |= 1u << bit;
    }
    const int cnt = __popc(keep);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = total + incl - cnt;
    for (uint32_t u = keep; u; u &= u - 1) {
      const int bit = __ffs(u) - 1;
      const int64_t kb = (int64_t)wi * 32 + bit;
      const int c0 = ((m0 >> bit) & 1u) ? block_class(a, h, qb0, kb) : 0;
      const int c1 = ((m1 >> bit) & 1u) ? block_class(a, h, qb1, kb) : 0;
      out[pos++] = (int32_t)((uint32_t)kb | ((uint32_t)c0 << kKbBits) | ((uint32_t)c1 << (kKbBits + 2)));
    }
    total += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) nvis[g] = total;
}

// B = 64 (sub-blocked tiles): per item (head, pair of query tiles = query
// blocks 4p .. 4p + 3) the ascending union of the 128-key tiles that hold any
// selected block of the four query blocks, each with the eight blocks' classes
// (kt | sc << 16, sub_class layout).  One warp per item, one bitmap per
// (tile, query half, key half) in shared memory.
__global__ void visit_quad_kernel(KernelArgs a, int words, int32_t* __restrict__ vis, int32_t* __restrict__ nvis) {
  extern __shared__ uint32_t bm_smem[];
  const int wip = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kVisitWarps + wip;
  if (g >= (int64_t)a.hq * a.npairs) return;
  uint32_t* bm = bm_smem + (size_t)wip * 8 * words;
  for (int x = lane; x < 8 * words; x += 32) bm[x] = 0u;
  __syncwarp();
  const int h = (int)(g / a.npairs);
  const int64_t p = g % a.npairs;
  for (int q = 0; q < 4; ++q) {
    const int64_t qb = 4 * p + q;
    if (qb >= a.t) break;
    const int cnt = a.kv_cnt[(int64_t)h * a.t + qb];
    const int32_t* list = a.kv_idx + ((int64_t)h * a.t + qb) * a.t;
    for (int e = lane; e < cnt; e += 32) {
      const int kb = list[e], kt = kb >> 1, s = 2 * q + (kb & 1);  // s = 4 w + 2 a + b
      atomicOr(&bm[s * words + (kt >> 5)], 1u << (kt & 31));
    }
  }
  __syncwarp();
  auto classes = [&](const uint32_t (&m)[8], int bit, int64_t kt) {
    uint32_t sc = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if ((m[s] >> bit) & 1u) sc |= (uint32_t)block_class(a, h, 4 * p + (s >> 1), 2 * kt + (s & 1)) << (2 * s);
    return sc;
  };
  int32_t* out = vis + g * a.t128;
  int total = 0;
  for (int w0 = 0; w0 < words; w0 += 32) {
    const int wi = w0 + lane;
    uint32_t m[8], any = 0u;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      m[s] = wi < words ? bm[s * words + wi] : 0u;
      any |= m[s];
    }
    uint32_t keep = 0u;
    for (uint32_t u = any; u; u &= u - 1) {
      const int bit = __ffs(u) - 1;
      if (classes(m, bit, (int64_t)wi * 32 + bit)) keep |= 1u << bit;
    }
    const int cnt = __popc(keep);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = total + incl - cnt;
    for (uint32_t u = keep; u; u &= u - 1) {
      const int bit = __ffs(u) - 1;
      const int64_t kt = (int64_t)wi * 32 + bit;
      out[pos++] = (int32_t)((uint32_t)kt | (classes(m, bit, kt) << kSubShift));
    }
    total += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) nvis[g] = total;
}

// per-block [min, max] of an original-position map (AdmissibilityIndex::build)
__global__ void block_minmax_kernel(const int32_t* __restrict__ orig, int heads, int64_t n, int64_t t,
                                    int64_t block, int2* __restrict__ mm) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= (int64_t)heads * t) return;
  const int64_t h = g / t, b = g % t;
  const int64_t lo = b * block, hi = min64(n, lo + block);
  int mn = 0x7fffffff, mx = -1;
  for (int64_t p = lo + lane; p < hi; p += 32) {
    const int v = orig[h * n + p];
    mn = min(mn, v);
    mx = max(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) mm[g] = make_int2(mn, mx);
}

// ---- host side -----------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_map(CUtensorMap* map, const void* base, int heads, int64_t n) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(PBS_ERR_CUDA, "E_CUDA", "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)kD, (cuuint64_t)n, (cuuint64_t)heads};
  const cuuint64_t strides[2] = {(cuuint64_t)kD * 2, (cuuint64_t)n * kD * 2};
  const cuuint32_t box[3] = {64, (cuuint32_t)kBM, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PBS_ERR_CUDA, "E_CUDA", "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return PBS_OK;
}

// Library-owned scratch for calls that pass none (the block-sparse / dense C-ABI
// entries): one grow-only device buffer per stream, so back-to-back calls never
// go through the allocator (a stream-ordered malloc/free per call showed up as
// occasional 10-30 ms stalls when the pool returned memory to the driver).
// Work on one stream is ordered, so the buffer is reused safely by that stream.
void* stream_scratch(cudaStream_t st, size_t bytes) {
  struct Entry {
    int device;
    cudaStream_t stream;
    void* ptr;
    size_t bytes;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  // keyed by (device, stream): the legacy default stream (handle 0) exists once per device
  for (auto& e : cache) {
    if (e.device != dev || e.stream != st) continue;
    if (e.bytes >= bytes) return e.ptr;
    cudaStreamSynchronize(st);  // the old buffer may still be in use by this stream
    cudaFree(e.ptr);
    e.ptr = nullptr;
    e.bytes = 0;
    if (cudaMalloc(&e.ptr, bytes) != cudaSuccess) return nullptr;
    e.bytes = bytes;
    return e.ptr;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  cache.push_back({dev, st, p, bytes});
  return p;
}

}  // namespace

bool attention_sm100_supported(const AttnParams& p) {
  if (p.dtype != PBS_DTYPE_BF16 || p.d != kD) return false;
  // B = 128 tiles; B = 64 block-sparse lists as 2 x 2 blocks per tile
  if (p.block != kBM && !(p.block == 64 && p.kv_idx)) return false;
  if ((uintptr_t)p.q % 16 || (uintptr_t)p.k % 16 || (uintptr_t)p.v % 16 || (uintptr_t)p.out % 16) return false;
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return false;
  if (major != 10) return false;
  if (getenv("PBS_FORCE_SIMT")) return false;
  return true;
}

size_t attention_sm100_workspace_bytes(int hq, int64_t n, int64_t block) {
  const int64_t t = ceil_div(n, block);
  // the item counter, block min/max of sigma and pi, then the visit lists and counts
  return 256 + (size_t)2 * hq * t * sizeof(int2) + ((size_t)hq * t * t + (size_t)hq * t) * 4 + 256;
}

// fp32 [d2, d1, d0] row-major map with a [1, box1, box0] box, no swizzle
// (importance.cu streams the estimate's exps with it)
int make_f32_map_3d(void* map, const float* base, int64_t d0, int64_t d1, int64_t d2, int box0, int box1) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(PBS_ERR_CUDA, "E_CUDA", "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  const cuuint64_t strides[2] = {(cuuint64_t)d0 * 4, (cuuint64_t)d1 * d0 * 4};
  const cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PBS_ERR_CUDA, "E_CUDA", "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return PBS_OK;
}

int make_bf16_sw128_map_3d(void* map, const void* base, int64_t d0, int64_t d1, int64_t d2, int64_t row_elems,
                           int box0, int box1) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(PBS_ERR_CUDA, "E_CUDA", "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  const cuuint64_t strides[2] = {(cuuint64_t)row_elems * 2, (cuuint64_t)d1 * row_elems * 2};
  const cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PBS_ERR_CUDA, "E_CUDA", "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return PBS_OK;
}

int launch_attention_sm100(const AttnParams& p, void* sched_ws, cudaStream_t st) {
  const int64_t t = ceil_div(p.n, p.block);
  if (t == 0) return PBS_OK;
  CUtensorMap mq, mk, mv;
  if (int rc = make_map(&mq, p.q, p.hq, p.n)) return rc;
  if (int rc = make_map(&mk, p.k, p.kv_heads, p.n)) return rc;
  if (int rc = make_map(&mv, p.v, p.kv_heads, p.n)) return rc;
  KernelArgs a{};
  a.hq = p.hq;
  a.kv_heads = p.kv_heads;
  a.group = p.hq / p.kv_heads;
  a.n = p.n;
  a.t = t;
  a.block = p.block;
  a.sub = p.block == 64 ? 1 : 0;
  a.t128 = ceil_div(p.n, (int64_t)kBM);
  a.scale_log2 = p.scale * 1.4426950408889634f;
  a.kv_idx = p.kv_idx;
  a.kv_cnt = p.kv_cnt;
  a.q_orig = p.q_orig;
  a.k_orig = p.k_orig;
  a.out_rows = p.out_rows;
  a.status = p.status;
  a.lse = p.lse;
  a.out = static_cast<__nv_bfloat16*>(p.out);
  a.causal = p.causal;
  a.dense = p.kv_idx == nullptr;
  if (a.dense && !p.causal) return fail(PBS_ERR_CONFIG, "E_CONFIG", "attention without a block list must be causal");
  a.npairs = ceil_div(a.t128, 2);
  {
    // items are pairs of 128-row tiles: 2 query blocks at B = 128, 4 at B = 64
    const int64_t per = a.sub ? 4 : 2;
    const int64_t qb_end = p.qb_end > 0 ? min64(p.qb_end, t) : t;
    if (p.qb_begin < 0 || p.qb_begin >= qb_end || (p.qb_begin % per))
      return fail(PBS_ERR_CONFIG, "E_CONFIG", "query-block range must be non-empty and start on a whole tile pair");
    a.p_lo = p.qb_begin / per;
    a.p_hi = ceil_div(qb_end, per);
    if (qb_end != t && (qb_end % per))
      return fail(PBS_ERR_CONFIG, "E_CONFIG", "query-block range must end on a whole tile pair or at the last block");
  }
  a.items = (int64_t)p.hq * (a.p_hi - a.p_lo);
  // scratch: block min/max of the original positions + visit lists
  if (!sched_ws) {
    sched_ws = stream_scratch(st, a.dense ? 256 : attention_sm100_workspace_bytes(p.hq, p.n, p.block));
    if (!sched_ws) return fail(PBS_ERR_RESOURCE, "E_RESOURCE", "attention scratch allocation failed");
  }
  a.item_counter = static_cast<int32_t*>(sched_ws);
  PBS_CUDA_CHECK(cudaMemsetAsync(a.item_counter, 0, sizeof(int32_t), st));
  sched_ws = static_cast<char*>(sched_ws) + 256;
  if (p.q_orig || p.k_orig) {
    int2* mm = static_cast<int2*>(sched_ws);
    const int64_t rows = (int64_t)p.hq * t;
    if (p.q_orig) {
      block_minmax_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(p.q_orig, p.hq, p.n, t, p.block, mm);
      PBS_LAUNCH_CHECK("block_minmax_kernel");
      a.q_mm = mm;
    }
    if (p.k_orig) {
      block_minmax_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(p.k_orig, p.hq, p.n, t, p.block, mm + rows);
      PBS_LAUNCH_CHECK("block_minmax_kernel");
      a.k_mm = mm + rows;
    }
  }
  if (!a.dense) {
    int32_t* vis = static_cast<int32_t*>(sched_ws) + (2 * (size_t)p.hq * t * sizeof(int2)) / sizeof(int32_t);
    int32_t* nvis = vis + (size_t)p.hq * a.npairs * a.t128;
    const int words = (int)ceil_div(a.t128, 32);
    const size_t smem = (size_t)kVisitWarps * (a.sub ? 8 : 2) * words * sizeof(uint32_t);
    // the pre-pass keeps one bitmap row per key tile in shared memory, and a
    // sub-blocked entry packs the tile index into 16 bits
    if (smem > 200 * 1024 || (a.sub && a.t128 > 0xffff))
      return fail(PBS_ERR_CONFIG, "E_CONFIG",
                  "block-sparse attention on the tensor cores: sequence too long for the visit lists (N = " +
                      std::to_string(p.n) + ", B = " + std::to_string(p.block) + ")");
    if (smem > 48 * 1024) {
      static DeviceOnce vis_once;
      if (int rc = once_per_device(vis_once, [] {
            PBS_CUDA_CHECK(cudaFuncSetAttribute(visit_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                200 * 1024));
            PBS_CUDA_CHECK(cudaFuncSetAttribute(visit_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                200 * 1024));
            return (int)PBS_OK;
          }))
        return rc;
    }
    // every pair of every head (the items may be a query-block range of them)
    if (a.sub) {
      visit_quad_kernel<<<(unsigned)ceil_div((int64_t)p.hq * a.npairs, kVisitWarps), kVisitWarps * 32, smem, st>>>(
          a, words, vis, nvis);
      PBS_LAUNCH_CHECK("visit_quad_kernel");
    } else {
      visit_pair_kernel<<<(unsigned)ceil_div((int64_t)p.hq * a.npairs, kVisitWarps), kVisitWarps * 32, smem, st>>>(
          a, words, vis, nvis);
      PBS_LAUNCH_CHECK("visit_pair_kernel");
    }
    a.vis = vis;
    a.nvis = nvis;
  }
  static DeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, [] {
        PBS_CUDA_CHECK(cudaFuncSetAttribute(attn_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            SmemLayout::total));
        return (int)PBS_OK;
      }))
    return rc;
  int grid = (int)min64(a.items, num_sms());
  if (const char* e = getenv("PBS_ATTN_GRID")) grid = (int)min64(grid, atoi(e) > 0 ? atoi(e) : grid);  // debug
  // debug (-DPBS_ATTN_SPANS builds): per-phase cycle sums of every CTA, dumped to $PBS_ATTN_TRACE
  const char* trace_path = getenv("PBS_ATTN_TRACE");
  constexpr int kSpanWords = 32 + 2048 * 8 + 1024;
  if (trace_path) {
    PBS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&a.trace), kSpanWords * 8, st));
    PBS_CUDA_CHECK(cudaMemsetAsync(a.trace, 0, kSpanWords * 8, st));
  }
  attn_sm100_kernel<<<grid, kThreads, SmemLayout::total, st>>>(mq, mk, mv, a);
  PBS_LAUNCH_CHECK("attn_sm100_kernel");
  if (trace_path) {  // debug only: synchronous dump
    std::vector<unsigned long long> h(kSpanWords);
    PBS_CUDA_CHECK(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
    PBS_CUDA_CHECK(cudaStreamSynchronize(st));
    PBS_CUDA_CHECK(cudaFree(a.trace));
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  return PBS_OK;
}

}  // namespace pbs_b200
