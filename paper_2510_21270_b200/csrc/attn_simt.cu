// attn_simt.cu -- CUDA-core block-sparse attention for the shapes the
// tensor-core kernel does not take (f32 inputs, d != 128, block sizes other
// than 128, tiny problems).  Same semantics as attention_block_sparse
// (attention.hpp:259-310): selected key blocks in ascending order, the
// original-position element mask k_orig[j] <= q_orig[i] (attention.hpp:60),
// l == 0 => DegenerateRowError(query block) (attention.hpp:132), and the
// optional fused un-permute of the output rows (pipeline.hpp:178-180).
// Numerics: f32 online softmax per key; tolerance parity, not bit parity.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pbs_b200 {
namespace {

constexpr int kRows = 32;     // query rows per CTA
constexpr int kLanes = 4;     // threads per row (split over d)
constexpr int kKeys = 32;     // keys staged per step

template <typename T>
__global__ void __launch_bounds__(kRows* kLanes) attn_simt_kernel(AttnParams p, int64_t t, int subtiles) {
  extern __shared__ float sm[];
  const int d = p.d;
  float* ks = sm;                 // [kKeys][d]
  float* vs = ks + kKeys * d;     // [kKeys][d]
  int* kor = reinterpret_cast<int*>(vs + kKeys * d);  // [kKeys]
  const int h = blockIdx.y;
  const int64_t qb = p.qb_begin + blockIdx.x / subtiles;
  const int sub = blockIdx.x % subtiles;
  const int tid = threadIdx.x;
  const int rl = tid / kLanes, lane = tid % kLanes;
  const int64_t r0 = qb * p.block;
  const int64_t rows_in_block = min(p.block, p.n - r0);
  const int64_t row_local = (int64_t)sub * kRows + rl;
  const bool active = row_local < rows_in_block;
  const int64_t i = r0 + row_local;
  const int kvh = p.kv_heads == p.hq ? h : h / (p.hq / p.kv_heads);
  const T* q = static_cast<const T*>(p.q) + (int64_t)h * p.n * d;
  const T* k = static_cast<const T*>(p.k) + (int64_t)kvh * p.n * d;
  const T* v = static_cast<const T*>(p.v) + (int64_t)kvh * p.n * d;
  const int64_t qo = active ? (p.q_orig ? (int64_t)p.q_orig[(int64_t)h * p.n + i] : i) : 0;
  const int per = (d + kLanes - 1) / kLanes;
  float qr[64];
  float o[64];
  for (int c = 0; c < 64; ++c) {
    const int cc = lane * per + c;
    qr[c] = (c < per && cc < d && active) ? to_f32(q[i * d + cc]) : 0.0f;
    o[c] = 0.0f;
  }
  float m = -INFINITY, l = 0.0f;
  int64_t nkb;
  if (p.kv_idx) nkb = p.kv_cnt[(int64_t)h * t + qb];
  else if (p.causal) nkb = qb + 1;
  else nkb = t;
  for (int64_t e = 0; e < nkb; ++e) {
    const int64_t kb = p.kv_idx ? p.kv_idx[((int64_t)h * t + qb) * t + e] : e;
    const int64_t c0 = kb * p.block;
    const int64_t cc = min(p.block, p.n - c0);
    for (int64_t j0 = 0; j0 < cc; j0 += kKeys) {
      const int kc = (int)min64(kKeys, cc - j0);
      __syncthreads();
      for (int x = tid; x < kc * d; x += blockDim.x) {
        const int jj = x / d, c = x % d;
        const int64_t j = c0 + j0 + jj;
        ks[jj * d + c] = to_f32(k[j * d + c]);
        vs[jj * d + c] = to_f32(v[j * d + c]);
      }
      for (int jj = tid; jj < kc; jj += blockDim.x) {
        const int64_t j = c0 + j0 + jj;
        kor[jj] = p.k_orig ? p.k_orig[(int64_t)h * p.n + j] : (int)j;
      }
      __syncthreads();
      for (int jj = 0; jj < kc; ++jj) {
        float part = 0.0f;
        for (int c = 0; c < per; ++c) {
          const int col = lane * per + c;
          if (col < d) part = fmaf(qr[c], ks[jj * d + col], part);
        }
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        const int64_t j = c0 + j0 + jj;
        bool adm = active;
        if (p.q_orig || p.k_orig) adm = adm && (int64_t)kor[jj] <= qo;
        else if (p.causal) adm = adm && j <= i;
        if (!adm) continue;
        const float s = part * p.scale;
        const float m_new = fmaxf(m, s);
        const float factor = expf(m - m_new);
        const float pj = expf(s - m_new);
        l = l * factor + pj;
        for (int c = 0; c < per; ++c) {
          const int col = lane * per + c;
          if (col < d) o[c] = fmaf(pj, vs[jj * d + col], o[c] * factor);
        }
        m = m_new;
      }
    }
  }
  if (!active) return;
  const int64_t orow = p.out_rows ? (int64_t)p.out_rows[(int64_t)h * p.n + i] : i;
  if (p.lse && lane == 0) p.lse[(int64_t)h * p.n + orow] = l > 0.0f ? m + logf(l) : -INFINITY;
  if (l == 0.0f) {
    if (p.status && lane == 0) {
      p.status[0] = 1;
      atomicMin(&p.status[1], (int)(h * t + qb));
    }
    return;
  }
  const float inv = 1.0f / l;
  T* out = static_cast<T*>(p.out) + ((int64_t)h * p.n + orow) * d;
  for (int c = 0; c < per; ++c) {
    const int col = lane * per + c;
    if (col < d) out[col] = from_f32<T>(o[c] * inv);
  }
}

}  // namespace

int launch_attention_simt(const AttnParams& p, cudaStream_t st) {
  if (p.d > 64 * kLanes) return fail(PBS_ERR_CONFIG, "E_CONFIG", "head dim > 256 is not supported");
  const int64_t t = ceil_div(p.n, p.block);
  if (t == 0) return PBS_OK;
  const int subtiles = (int)ceil_div(p.block, kRows);
  const int64_t qb_end = p.qb_end > 0 ? min64(p.qb_end, t) : t;
  if (p.qb_begin < 0 || p.qb_begin >= qb_end) return fail(PBS_ERR_CONFIG, "E_CONFIG", "empty query-block range");
  const size_t smem = (size_t)2 * kKeys * p.d * 4 + kKeys * 4;
  // head dims above 192 need more than the 48 KB default (d = 256: 64 KB + 128 B)
  static DeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, [] {
        const int most = (int)((size_t)2 * kKeys * 64 * kLanes * 4 + kKeys * 4);
        PBS_CUDA_CHECK(cudaFuncSetAttribute(attn_simt_kernel<__nv_bfloat16>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, most));
        PBS_CUDA_CHECK(cudaFuncSetAttribute(attn_simt_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, most));
        return (int)PBS_OK;
      }))
    return rc;
  dim3 grid((unsigned)((qb_end - p.qb_begin) * subtiles), (unsigned)p.hq);
  if (p.dtype == PBS_DTYPE_BF16)
    attn_simt_kernel<__nv_bfloat16><<<grid, kRows * kLanes, smem, st>>>(p, t, subtiles);
  else
    attn_simt_kernel<float><<<grid, kRows * kLanes, smem, st>>>(p, t, subtiles);
  PBS_LAUNCH_CHECK("attn_simt_kernel");
  return PBS_OK;
}

}  // namespace pbs_b200
