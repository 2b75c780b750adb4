/*
 * pbs_cabi.h — C ABI of the B200-native PBS-Attn prefill path.
 *
 * This is the drop-in boundary for the reference's operator API
 * (the headers under /root/reference/proj/include/pbs/, header-only C++20 templates in
 * namespace pbs).  Every entry point below replaces one reference operator;
 * the citation on each names the function it stands in for.  The signatures
 * use only plain pointers, sizes and PODs (no torch, no C++ types) so that
 * ctypes / cgo / JNI / N-API bindings can call them directly.
 *
 * Conventions
 *  - Tensors are head-major [H, N, d] row-major device buffers (the layout of
 *    a PBST 3-D stack, tensor_io.hpp:23-29, 120-124).  dtype is bf16 or f32.
 *  - Permutations are int32 with the reference meaning map[new_pos] = old_pos
 *    (permutation.hpp:19-22), one length-N map per query head.
 *  - Block masks are uint8 row-major T x T grids (block_selection.hpp:26-81),
 *    one per query head; T = ceil(N / B).
 *  - GQA: query head h reads kv head h / (Hq / Hkv).  The reference has no
 *    GQA (pbs_main.cpp:86-89); with Hq == Hkv every call is the reference's.
 *  - All device entry points are stream-ordered on `stream` (a cudaStream_t,
 *    NULL = legacy default stream) and never allocate: callers provide the
 *    workspace sized by pbs_workspace_size().
 *  - Status codes mirror pbs::ErrorCode (errors.hpp:11-16) plus PBS_ERR_CUDA.
 *    pbs_last_error() returns the single-line "E_*: message" text of the
 *    calling thread's last failure (the CLI's stderr format, README.md:105-111).
 */
#ifndef PBS_CABI_H_
#define PBS_CABI_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PBS_API __attribute__((visibility("default")))
#else
#define PBS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:11-16) ---------------------------------- */
#define PBS_OK 0
#define PBS_ERR_CUDA 1       /* CUDA runtime / launch failure (no ref equivalent) */
#define PBS_ERR_CONFIG 2     /* ConfigError / ShapeError  (errors.hpp:32-40) */
#define PBS_ERR_IO 3         /* IoError / FormatError     (errors.hpp:42-59) */
#define PBS_ERR_RESOURCE 4   /* ResourceError             (errors.hpp:61-73) */
#define PBS_ERR_DEGENERATE 5 /* DegenerateRowError        (errors.hpp:75-89) */

/* ---- enums ------------------------------------------------------------ */
/* PermutationStrategy, pipeline.hpp:19 */
enum pbs_strategy {
  PBS_STRATEGY_NONE = 0,
  PBS_STRATEGY_KEY_PERMUTE = 1,
  PBS_STRATEGY_QUERY_PERMUTE = 2,
  PBS_STRATEGY_BOTH = 3
};

/* element type of Q/K/V/O buffers */
enum pbs_dtype { PBS_DTYPE_F32 = 0, PBS_DTYPE_BF16 = 1 };

/* ---- PODs ------------------------------------------------------------- */
/* PipelineConfig (pipeline.hpp:30-49) + ForcedPolicy (block_selection.hpp:163-166) */
typedef struct pbs_pipeline_config {
  int64_t block_size;   /* B >= 1 */
  int64_t segment_size; /* S == 0 or (S >= B and S % B == 0) */
  double tau;           /* [0, 1] */
  int32_t strategy;     /* enum pbs_strategy */
  int32_t forced_first_block;
  int32_t forced_diagonal_band;
  int32_t top_k;        /* 0: cumulative threshold tau (the reference); > 0: keep the top_k admissible
                           blocks per row by pooled score (extension: no reference oracle) */
  double scale; /* 0 => 1/sqrt(d) (attention.hpp:32-34) */
} pbs_pipeline_config;

/* problem shape (the reference is one head per call; this adds Hq/Hkv) */
typedef struct pbs_shape {
  int32_t dtype;        /* enum pbs_dtype */
  int32_t num_q_heads;  /* Hq */
  int32_t num_kv_heads; /* Hkv, Hq % Hkv == 0 */
  int32_t head_dim;     /* d; the tensor-core path needs d == 128 */
  int64_t seq_len;      /* N (self-attention, N == M, pipeline.hpp:112-113) */
} pbs_shape;

/* PipelineReport (pipeline.hpp:63-74), aggregated over heads.
 * density fields are per-head averages; counts are sums over heads. */
typedef struct pbs_report {
  double block_density;
  double causal_density_baseline;
  double pooled_score_coverage;
  int64_t selected_blocks;
  int64_t total_admissible_blocks;
  /* StageTimings (pipeline.hpp:51-61) in microseconds, from CUDA events */
  double estimate_us;
  double permute_us;
  double select_us;
  double attention_us;
  double unpermute_us;
} pbs_report;

/* ---- library ---------------------------------------------------------- */
PBS_API const char* pbs_last_error(void);
PBS_API const char* pbs_version(void);
/* number of kernels this library has launched in the process (diagnostics) */
PBS_API int64_t pbs_kernel_launches(void);

/* Device scratch needed by pbs_attention / the estimate and select stages. */
PBS_API size_t pbs_workspace_size(const pbs_shape* shape, const pbs_pipeline_config* cfg);

/* ---- stage 1: importance + permutations -------------------------------- */

/* estimate_key_importance (permutation.hpp:143-178): scores[h][j] = mean over
 * the last min(B, N) query rows of softmax(scale * q_i K^T)_j, no causal mask.
 * Bit-exact restatement of the reference's fp32 arithmetic on the
 * (bf16-upcast) inputs.  scores: f32 [Hq, N]. */
PBS_API int pbs_estimate_key_importance(const void* q, const void* k, const pbs_shape* shape,
                                int64_t block_size, double scale, float* scores,
                                void* workspace, size_t workspace_bytes, void* stream);

/* build_key_permutation + SegmentedPermutation::flatten + Permutation::inverse
 * (permutation.hpp:182-201, 118-126, 51-55): per segment a stable descending
 * argsort of the scores (ties by ascending index); the trailing N mod S keys
 * map to themselves.  perm, inv: int32 [H, N]; inv may be NULL. */
PBS_API int pbs_build_key_permutation(const float* scores, int32_t num_heads, int64_t seq_len,
                              int64_t segment_size, int32_t* perm, int32_t* inv,
                              void* stream);

/* build_query_permutation (permutation.hpp:206-275): key-block centroids,
 * cosine argmax group per query, stable sort by group within each segment.
 * k may be the already key-permuted K' (strategy both, pipeline.hpp:144-153);
 * k_heads gives its head count (Hkv for raw K, Hq for a per-q-head K'). */
PBS_API int pbs_build_query_permutation(const void* q, const void* k, int32_t k_heads,
                                const pbs_shape* shape, int64_t block_size,
                                int64_t segment_size, int32_t* perm, int32_t* inv,
                                void* workspace, size_t workspace_bytes, void* stream);

/* Device workspace bytes pbs_build_query_permutation needs for this shape and
 * block size (0 on a bad shape). */
PBS_API size_t pbs_query_permutation_workspace_size(const pbs_shape* shape, int64_t block_size);

/* ---- stage 2: gathers --------------------------------------------------- */

/* apply_rows (permutation.hpp:79-89), batched with a GQA broadcast:
 * dst[h][i][:] = src[h / (dst_heads / src_heads)][perm[h][i]][:].
 * perm may be NULL (identity).  Also serves the stage-5 un-permute
 * (pipeline.hpp:178-180) when called with sigma^{-1}. */
PBS_API int pbs_apply_rows(const int32_t* perm, const void* src, int32_t src_heads, int32_t dst_heads,
                   int64_t rows, int32_t cols, int32_t dtype, void* dst, void* stream);

/* Stage 5, the un-permute (pipeline.hpp:178-180, O = apply_rows(sigma^-1, O')):
 * dst[h][sigma[h][i]] = src[h][i] over [H, rows, cols] buffers.  The fused
 * pipeline does this in the attention epilogue (out_rows); this is the
 * standalone operator. */
PBS_API int pbs_unpermute(const int32_t* sigma, const void* src, int32_t num_heads, int64_t rows, int32_t cols,
                  int32_t dtype, void* dst, void* stream);

/* ---- stage 3: block scores + selection ---------------------------------- */

/* meanpool_block_scores (block_selection.hpp:120-161) under the
 * segment-band causal mask (build_block_causal_mask, block_selection.hpp:86-97):
 * scores f32 [Hq, T, T]; entries above the band are 0 (softmax of -inf). */
PBS_API int pbs_meanpool_block_scores(const void* qp, const void* kp, const pbs_shape* shape,
                              int64_t block_size, int64_t segment_size, double scale,
                              float* scores, void* workspace, size_t workspace_bytes,
                              void* stream);

/* select_blocks (block_selection.hpp:171-206): cumulative-tau prefix of the
 * descending scores (double accumulation), plus forced block 0 and the
 * diagonal segment band.  mask: uint8 [H, T, T].  kv_idx/kv_cnt (optional):
 * per (head, query block) the selected key blocks in ascending order,
 * kv_idx [H, T, T] (row-padded CSR), kv_cnt [H, T]. */
PBS_API int pbs_select_blocks(const float* scores, int32_t num_heads, int64_t num_blocks,
                      int64_t block_size, int64_t segment_size, double tau,
                      int32_t forced_first_block, int32_t forced_diagonal_band,
                      uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt, void* stream);
/* Top-k selection (extension, the reference selects by threshold only): per row
 * the top_k admissible blocks in the same stable descending order (ties by
 * ascending index), plus the forced blocks. */
PBS_API int pbs_select_blocks_top_k(const float* scores, int32_t num_heads, int64_t num_blocks,
                      int64_t block_size, int64_t segment_size, int32_t top_k,
                      int32_t forced_first_block, int32_t forced_diagonal_band,
                      uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt, void* stream);

/* ---- stage 4: attention ------------------------------------------------- */

/* attention_block_sparse (attention.hpp:259-310) with the original-position
 * ElementMask (attention.hpp:41-73): permuted query row i may see permuted key
 * j iff k_orig[j] <= q_orig[i].  q_orig = sigma, k_orig = pi; one of them NULL
 * = identity on that side; both NULL = no element mask (em == nullptr with
 * cfg.causal false, attention.hpp:262: every key of a selected block).
 * kv_idx/kv_cnt from pbs_select_blocks (block-level skip, attention.hpp:284-286).
 * kp/vp hold kv_heads heads (kv_heads == Hq for per-q-head permuted K'/V',
 * == Hkv for unpermuted shared K/V).  out_rows (optional) scatters output row
 * i of head h to row out_rows[h][i] -- the fused stage-5 un-permute (pass
 * sigma).  status (optional, device int32[2]): {degenerate flag, first
 * degenerate (head * T + query block)}.  out has the dtype of q. */
PBS_API int pbs_block_sparse_attention_fwd(const void* qp, const void* kp, const void* vp,
                                   int32_t kv_heads, const pbs_shape* shape,
                                   int64_t block_size, double scale, const int32_t* kv_idx,
                                   const int32_t* kv_cnt, const int32_t* q_orig,
                                   const int32_t* k_orig, const int32_t* out_rows, void* out,
                                   int32_t* status, void* stream);

/* The project's dense causal FlashAttention (the comparator; attention_tiled
 * with causal = true, attention.hpp:314-321).  GQA via kv head h/G. */
PBS_API int pbs_dense_causal_attention_fwd(const void* q, const void* k, const void* v,
                                   const pbs_shape* shape, double scale, void* out,
                                   void* stream);

/* Read back a status buffer written by the attention kernels; returns
 * PBS_ERR_DEGENERATE (with "E_DEGENERATE: query block ..." text) if set. */
PBS_API int pbs_check_status(const int32_t* status, int64_t num_blocks, void* stream);

/* ---- fused pipeline (pbs_attention, pipeline.hpp:107-193) ---------------- */

/* Algorithm 1 end to end for all heads on device buffers.  sigma, pi
 * (int32 [Hq, N]) and mask (uint8 [Hq, T, T]) are optional outputs.  When
 * report != NULL the call synchronises `stream` and fills it. */
PBS_API int pbs_attention(const void* q, const void* k, const void* v, const pbs_shape* shape,
                  const pbs_pipeline_config* cfg, void* out, int32_t* sigma, int32_t* pi,
                  uint8_t* mask, void* workspace, size_t workspace_bytes, pbs_report* report,
                  void* stream);

/* Same, on HOST buffers (the reference-facing call: Matrix<T> in, Matrix<T>
 * out).  Copies in, runs, copies out, synchronises.  Uses a library-owned
 * device arena on the current device. */
PBS_API int pbs_attention_host(const void* q, const void* k, const void* v, const pbs_shape* shape,
                       const pbs_pipeline_config* cfg, void* out, int32_t* sigma,
                       int32_t* pi, uint8_t* mask, pbs_report* report);

/* ---- multi-GPU: head-parallel shards ----------------------
 * Replaces the reference CLI's per-head fan-out (for_each_head,
 * tools/pbs_main.cpp:99-122: heads share nothing) with one process
 * per GPU.  Work units are (query head, pair of query blocks), weighted by
 * their causal key blocks; rank r owns the contiguous unit range holding the
 * r-th 1/world of the work (whole heads when Hq % world == 0, otherwise a cut
 * inside a head), so every rank's output rows are ONE contiguous range of the
 * flattened [Hq * N] output rows.  A rank needs its query heads
 * [head_begin, head_end) and KV heads [kv_begin, kv_end) only. */
typedef struct pbs_shard {
  int32_t head_begin, head_end; /* query heads touched */
  int32_t kv_begin, kv_end;     /* KV heads needed */
  int64_t qb_begin;             /* first query block of head_begin (even) */
  int64_t qb_end;               /* end query block of head_end - 1 (T = all) */
  int64_t out_row_begin;        /* the rank's rows of the flattened [Hq * N] output */
  int64_t out_rows;
} pbs_shard;
PBS_API int pbs_shard_plan(const pbs_shape* global_shape, int64_t block_size, int32_t world_size, int32_t rank,
                           pbs_shard* shard);
PBS_API size_t pbs_shard_workspace_size(const pbs_shape* global_shape, const pbs_pipeline_config* cfg,
                                        int32_t world_size, int32_t rank);
/* Rank `rank`'s share of pbs_attention, compute only (no collective):
 * q_local [head_end - head_begin, N, d], k_local / v_local
 * [kv_end - kv_begin, N, d]; writes only the shard's rows of out_full
 * [Hq, N, d].  Running every rank's shard into one buffer reproduces
 * pbs_attention's output bit for bit.  report (optional) covers the shard's
 * rows, densities averaged over the GLOBAL Hq (sum them over ranks). */
PBS_API int pbs_attention_shard(const void* q_local, const void* k_local, const void* v_local,
                                const pbs_shape* global_shape, const pbs_pipeline_config* cfg, int32_t world_size,
                                int32_t rank, void* out_full, void* workspace, size_t workspace_bytes,
                                pbs_report* report, void* stream);

/* Per-rank handle owning an NCCL communicator (NCCL is loaded at run time).
 * Rank 0 makes the id, the ranks share it out of band (e.g. torch.distributed
 * or MPI), every rank creates its handle on its own device. */
#define PBS_NCCL_UNIQUE_ID_BYTES 128
typedef struct pbs_dist pbs_dist;
PBS_API int pbs_dist_unique_id(uint8_t id[PBS_NCCL_UNIQUE_ID_BYTES]);
PBS_API int pbs_dist_create(const uint8_t id[PBS_NCCL_UNIQUE_ID_BYTES], int32_t world_size, int32_t rank,
                            pbs_dist** handle);
PBS_API int pbs_dist_destroy(pbs_dist* handle);
PBS_API size_t pbs_dist_workspace_size(const pbs_dist* handle, const pbs_shape* global_shape,
                                       const pbs_pipeline_config* cfg);
/* pbs_attention_shard on this rank, then the one exchange: every rank's rows
 * broadcast in place into out_full on all ranks (one NCCL group of
 * ncclBroadcast calls = an all-gather-v over NVLink).  Collective: every rank
 * calls it with the same global shape and config; report (global counts) is
 * collective too -- all ranks pass one or none. */
PBS_API int pbs_dist_attention(pbs_dist* handle, const void* q_local, const void* k_local, const void* v_local,
                               const pbs_shape* global_shape, const pbs_pipeline_config* cfg, void* out_full,
                               void* workspace, size_t workspace_bytes, pbs_report* report, void* stream);

/* ---- diagnostics (pipeline.hpp:195-295) --------------------------------- */

/* Device scratch for pbs_attention_coverage. */
PBS_API size_t pbs_coverage_workspace_size(const pbs_shape* shape, int64_t block_size);

/* attention_coverage (pipeline.hpp:198-243): per query head, the fraction of
 * the true causal attention probability mass (on the original, unpermuted
 * q, k) that falls inside the selected blocks of the permuted grid: key j
 * counts for query i iff mask[h][sigma^{-1}(i)/B][pi^{-1}(j)/B].  The
 * reference streams rows in double and caps N^2 at 2^26; here each row's mass
 * is exp(lse_selected - lse_causal) from two attention passes (block-sparse
 * over the permuted grid, dense causal over the original order), so it runs at
 * full length.  sigma / pi may be NULL (identity).  coverage: device double
 * [Hq].  Tolerance vs the reference: 1e-5 on f32 inputs, 1e-3 on bf16 (the
 * tensor-core pass uses approximate exp2). */
PBS_API int pbs_attention_coverage(const void* q, const void* k, const pbs_shape* shape, int64_t block_size,
                                   const uint8_t* mask, const int32_t* sigma, const int32_t* pi, double scale,
                                   double* coverage, void* workspace, size_t workspace_bytes, void* stream);

/* ---- PBST tensor files (tensor_io.hpp) ------------------------------------ */
/* Header of a PBST file: read_tensor's checks (tensor_io.hpp:98-146), same
 * E_IO / E_FORMAT texts and byte offsets. */
typedef struct pbs_tensor_info {
  int32_t file_dtype;     /* Dtype (tensor_io.hpp:31): 0 = f32, 1 = f64 */
  int32_t ndim;           /* 2 (rows, cols) or 3 (heads, rows, cols) */
  int64_t heads;          /* 1 for a 2-D file */
  int64_t rows;
  int64_t cols;
  int64_t payload_offset; /* bytes */
} pbs_tensor_info;
PBS_API int pbs_tensor_info_read(const char* path, pbs_tensor_info* info);
/* read_tensor (tensor_io.hpp:98-146) into device memory: dst holds
 * heads x rows x cols elements of dst_dtype (f32, or bf16 rounded to nearest).
 * A non-finite payload element fails with E_FORMAT at its byte offset
 * (tensor_io.hpp:80-81).  Synchronous with respect to `stream`. */
PBS_API int pbs_tensor_load(const char* path, void* dst, int32_t dst_dtype, void* stream);
/* write_tensor / write_tensor_stack (tensor_io.hpp:155-193) from device
 * memory: src [heads, rows, cols] of src_dtype, file_dtype 0 = f32 / 1 = f64,
 * as_stack = 0 writes a 2-D file (heads must be 1). */
PBS_API int pbs_tensor_save(const char* path, const void* src, int32_t src_dtype, int64_t heads, int64_t rows,
                            int64_t cols, int32_t file_dtype, int32_t as_stack, void* stream);

/* ---- synthetic workloads (workload.hpp, rng.hpp) -------------------------- */
/* WorkloadSpec (workload.hpp:21-38) for run manifests that name a `workload`
 * (manifest.hpp:26-39) instead of input files. */
enum pbs_workload_kind {
  PBS_WORKLOAD_GAUSSIAN = 0,
  PBS_WORKLOAD_VERTICAL_LINES = 1,
  PBS_WORKLOAD_BLOCK_DIAG = 2,
  PBS_WORKLOAD_MIXED = 3
};
enum pbs_line_scatter { PBS_SCATTER_CLUSTERED = 0, PBS_SCATTER_SCATTERED = 1 };
enum pbs_host_dtype { PBS_HOST_F32 = 0, PBS_HOST_F64 = 1 };
typedef struct pbs_workload_spec {
  int32_t kind;         /* pbs_workload_kind (default gaussian) */
  int32_t scatter;      /* pbs_line_scatter (default scattered) */
  int64_t n, d, heads;  /* defaults 1024, 64, 1 */
  uint64_t seed;        /* default 0 */
  int64_t line_count;   /* default 8 */
  double line_strength; /* default 150 */
} pbs_workload_spec;
/* generate_head (workload.hpp:145-198) on the HOST: head `head` of the
 * workload into row-major [n, d] host buffers q, k, v of host_dtype (the
 * manifest's precision), bit-identical to the reference generator; the planted
 * line positions go to `planted` (capacity line_count, may be NULL) and their
 * number to *planted_count.  Validation and error texts of
 * WorkloadSpec::validate. */
PBS_API int pbs_generate_workload_head(const pbs_workload_spec* spec, int64_t head, int64_t block_size,
                                       int64_t segment_size, int32_t host_dtype, void* q, void* k, void* v,
                                       int64_t* planted, int64_t* planted_count);

/* ---- device memory (for FFI callers without the CUDA runtime) ------------ */
#define PBS_COPY_H2D 0
#define PBS_COPY_D2H 1
#define PBS_COPY_D2D 2
PBS_API int pbs_malloc(size_t bytes, void** ptr);
PBS_API int pbs_free(void* ptr);
/* stream-ordered copy; kind = PBS_COPY_*; host memory should be pinned for overlap */
PBS_API int pbs_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream);
PBS_API int pbs_stream_synchronize(void* stream);

/* ---- test hooks ---------------------------------------------------------- */
/* y[i] = the device port of glibc expf (the reference's std::exp(float)). */
PBS_API int pbs_debug_expf(const float* x, float* y, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PBS_CABI_H_ */
