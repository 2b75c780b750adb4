/*
 * pbs_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference PBS-Attn hot path (the headers under
 * /root/reference/proj/include/pbs/) in plain C, one head per call, in the reference's own
 * element types (float and double; suffixes _f32 / _f64).  It is the parity
 * checker for the CUDA path and nothing else: only tests/, the smoke() hook
 * and bench.py's cpu_baseline leg may load it.  The product library never
 * links it.
 *
 * Parity pinning: every function is checked bit-for-bit against the
 * reference headers compiled unmodified into oracle/_ref/libpbsref.so
 * (oracle/ref_shim.cpp, oracle/Makefile) and against the reference's own
 * known-answer tests and tests/golden/pipeline256.json (tests/test_oracle.py).
 *
 * Float semantics follow the reference build (proj/CMakeLists.txt:3-8:
 * -O3, no -march, so x86-64 baseline SSE2 with no FMA contraction); this file
 * is compiled with -ffp-contract=off to make that explicit.  std::exp(float)
 * in the reference is glibc expf, which this file calls directly.
 */
#ifndef PBS_ORACLE_H_
#define PBS_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/pbs_cabi.h"

#ifdef __cplusplus
extern "C" {
#endif

#define PBSO_DECL(REAL, SFX)                                                                   \
  int pbso_estimate_key_importance_##SFX(const REAL* q, size_t n, const REAL* k, size_t m,     \
                                         size_t d, size_t block, double scale, REAL* scores,   \
                                         size_t* source_query_block);                          \
  int pbso_build_key_permutation_##SFX(const REAL* scores, size_t n, size_t segment,           \
                                       int32_t* perm);                                         \
  int pbso_build_query_permutation_##SFX(const REAL* q, size_t n, const REAL* k, size_t m,     \
                                         size_t d, size_t block, size_t segment,               \
                                         int32_t* perm);                                       \
  void pbso_apply_rows_##SFX(const int32_t* perm, const REAL* src, size_t rows, size_t cols,   \
                             REAL* dst);                                                       \
  int pbso_block_causal_mask_##SFX(size_t t_r, size_t t_c, size_t block, size_t segment,       \
                                   REAL* causal);                                              \
  int pbso_meanpool_block_scores_##SFX(const REAL* qp, size_t n, const REAL* kp, size_t m,     \
                                       size_t d, size_t block, const REAL* causal,             \
                                       double scale, REAL* scores);                            \
  int pbso_select_blocks_##SFX(const REAL* scores, const REAL* causal, size_t t_r,             \
                               size_t t_c, size_t block, size_t segment, double tau,           \
                               int forced_first, int forced_band, uint8_t* mask);              \
  int pbso_select_blocks_top_k_##SFX(const REAL* scores, const REAL* causal, size_t t_r,       \
                                     size_t t_c, size_t block, size_t segment, size_t top_k,   \
                                     int forced_first, int forced_band, uint8_t* mask);        \
  int pbso_attention_block_sparse_##SFX(const REAL* q, size_t n, const REAL* k,                \
                                        const REAL* v, size_t m, size_t d, size_t dv,          \
                                        size_t block, double scale, int causal,                \
                                        const uint8_t* mask, const int32_t* q_orig,            \
                                        const int32_t* k_orig, REAL* out,                      \
                                        size_t* degenerate_block);                             \
  int pbso_attention_oracle_##SFX(const REAL* q, size_t n, const REAL* k, const REAL* v,       \
                                  size_t m, size_t d, size_t dv, size_t block, double scale,   \
                                  int causal, const int32_t* q_orig, const int32_t* k_orig,    \
                                  REAL* out);                                                  \
  int pbso_pbs_attention_##SFX(const REAL* q, const REAL* k, const REAL* v, size_t n,          \
                               size_t d, const pbs_pipeline_config* cfg, REAL* out,            \
                               int32_t* sigma, int32_t* pi, uint8_t* mask, pbs_report* rep);   \
  int pbso_attention_coverage_##SFX(const REAL* q, const REAL* k, size_t n, size_t d,          \
                                    const uint8_t* mask, size_t block, const int32_t* sigma,   \
                                    const int32_t* pi, double scale, double* coverage);

PBSO_DECL(float, f32)
PBSO_DECL(double, f64)

void pbso_inverse(const int32_t* perm, size_t n, int32_t* inv);
const char* pbso_last_error(void);
/* the reference's scalar exp for float: glibc expf (exposed for the device-port check) */
void pbso_expf(const float* x, float* y, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* PBS_ORACLE_H_ */
