"""ctypes binding of libpbs_b200.so (the C ABI in include/pbs_cabi.h).

The library is loaded from this package directory (built in-tree by
paper_2510_21270_b200/build.py).  There is no fallback: if the .so is missing
or fails to load, importing the op layer raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libpbs_b200.so")

PBS_OK = 0
PBS_ERR_CUDA = 1
PBS_ERR_CONFIG = 2
PBS_ERR_IO = 3
PBS_ERR_RESOURCE = 4
PBS_ERR_DEGENERATE = 5

DTYPE_F32 = 0
DTYPE_BF16 = 1

STRATEGIES = {"none": 0, "key_permute": 1, "query_permute": 2, "both": 3}

# every symbol include/pbs_cabi.h declares
EXPORTS = [
    "pbs_last_error", "pbs_generate_workload_head", "pbs_version", "pbs_kernel_launches", "pbs_workspace_size", "pbs_estimate_key_importance",
    "pbs_build_key_permutation", "pbs_build_query_permutation", "pbs_query_permutation_workspace_size", "pbs_apply_rows", "pbs_unpermute",
    "pbs_meanpool_block_scores", "pbs_select_blocks", "pbs_select_blocks_top_k", "pbs_block_sparse_attention_fwd",
    "pbs_dense_causal_attention_fwd", "pbs_check_status", "pbs_attention", "pbs_attention_host",
    "pbs_coverage_workspace_size", "pbs_attention_coverage", "pbs_tensor_info_read", "pbs_tensor_load",
    "pbs_tensor_save", "pbs_debug_expf", "pbs_shard_plan", "pbs_shard_workspace_size", "pbs_attention_shard",
    "pbs_dist_unique_id", "pbs_dist_create", "pbs_dist_destroy", "pbs_dist_workspace_size", "pbs_dist_attention",
    "pbs_malloc", "pbs_free", "pbs_memcpy", "pbs_stream_synchronize",
]


class Shape(C.Structure):
    """pbs_shape."""

    _fields_ = [("dtype", C.c_int32), ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("seq_len", C.c_int64)]


class PipelineConfig(C.Structure):
    """pbs_pipeline_config == PipelineConfig (pipeline.hpp:30-49) + ForcedPolicy."""

    _fields_ = [("block_size", C.c_int64), ("segment_size", C.c_int64), ("tau", C.c_double),
                ("strategy", C.c_int32), ("forced_first_block", C.c_int32),
                ("forced_diagonal_band", C.c_int32), ("top_k", C.c_int32), ("scale", C.c_double)]


class Report(C.Structure):
    """pbs_report == PipelineReport (pipeline.hpp:63-74) + StageTimings (51-61)."""

    _fields_ = [("block_density", C.c_double), ("causal_density_baseline", C.c_double),
                ("pooled_score_coverage", C.c_double), ("selected_blocks", C.c_int64),
                ("total_admissible_blocks", C.c_int64), ("estimate_us", C.c_double),
                ("permute_us", C.c_double), ("select_us", C.c_double), ("attention_us", C.c_double),
                ("unpermute_us", C.c_double)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class Shard(C.Structure):
    """pbs_shard: one rank's share of the head-parallel split."""

    _fields_ = [("head_begin", C.c_int32), ("head_end", C.c_int32), ("kv_begin", C.c_int32), ("kv_end", C.c_int32),
                ("qb_begin", C.c_int64), ("qb_end", C.c_int64), ("out_row_begin", C.c_int64),
                ("out_rows", C.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class TensorInfo(C.Structure):
    """pbs_tensor_info: a PBST header (tensor_io.hpp:23-29)."""

    _fields_ = [("file_dtype", C.c_int32), ("ndim", C.c_int32), ("heads", C.c_int64), ("rows", C.c_int64),
                ("cols", C.c_int64), ("payload_offset", C.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class WorkloadSpec(C.Structure):
    """pbs_workload_spec == WorkloadSpec (workload.hpp:21-38), the reference's defaults."""

    _fields_ = [("kind", C.c_int32), ("scatter", C.c_int32), ("n", C.c_int64), ("d", C.c_int64),
                ("heads", C.c_int64), ("seed", C.c_uint64), ("line_count", C.c_int64), ("line_strength", C.c_double)]

    def __init__(self, **kw):
        super().__init__(kind=0, scatter=1, n=1024, d=64, heads=1, seed=0, line_count=8, line_strength=150.0)
        for key, value in kw.items():
            setattr(self, key, value)


WORKLOAD_KINDS = {"gaussian": 0, "vertical_lines": 1, "block_diag": 2, "mixed": 3}
LINE_SCATTER = {"clustered": 0, "scattered": 1}


class PbsError(RuntimeError):
    """Raised for any non-zero status; `code` mirrors pbs::ErrorCode (errors.hpp:11-16)."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class ConfigError(PbsError):
    pass


class ResourceError(PbsError):
    pass


class DegenerateRowError(PbsError):
    pass


class IoError(PbsError):
    """E_IO / E_FORMAT (errors.hpp:42-59)."""


class CudaError(PbsError):
    pass


_ERRORS = {PBS_ERR_CONFIG: ConfigError, PBS_ERR_RESOURCE: ResourceError, PBS_ERR_IO: IoError,
           PBS_ERR_DEGENERATE: DegenerateRowError, PBS_ERR_CUDA: CudaError}

_lib = None

VP = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
SZ = C.c_size_t
DBL = C.c_double

_SIGS = {
    "pbs_last_error": (C.c_char_p, []),
    "pbs_version": (C.c_char_p, []),
    "pbs_kernel_launches": (C.c_int64, []),
    "pbs_workspace_size": (SZ, [C.POINTER(Shape), C.POINTER(PipelineConfig)]),
    "pbs_estimate_key_importance": (C.c_int, [VP, VP, C.POINTER(Shape), I64, DBL, VP, VP, SZ, VP]),
    "pbs_build_key_permutation": (C.c_int, [VP, I32, I64, I64, VP, VP, VP]),
    "pbs_build_query_permutation": (C.c_int, [VP, VP, I32, C.POINTER(Shape), I64, I64, VP, VP, VP, SZ, VP]),
    "pbs_query_permutation_workspace_size": (SZ, [C.POINTER(Shape), I64]),
    "pbs_apply_rows": (C.c_int, [VP, VP, I32, I32, I64, I32, I32, VP, VP]),
    "pbs_unpermute": (C.c_int, [VP, VP, I32, I64, I32, I32, VP, VP]),
    "pbs_meanpool_block_scores": (C.c_int, [VP, VP, C.POINTER(Shape), I64, I64, DBL, VP, VP, SZ, VP]),
    "pbs_select_blocks": (C.c_int, [VP, I32, I64, I64, I64, DBL, I32, I32, VP, VP, VP, VP]),
    "pbs_select_blocks_top_k": (C.c_int, [VP, I32, I64, I64, I64, I32, I32, I32, VP, VP, VP, VP]),
    "pbs_block_sparse_attention_fwd": (C.c_int, [VP, VP, VP, I32, C.POINTER(Shape), I64, DBL, VP, VP, VP, VP,
                                                 VP, VP, VP, VP]),
    "pbs_dense_causal_attention_fwd": (C.c_int, [VP, VP, VP, C.POINTER(Shape), DBL, VP, VP]),
    "pbs_check_status": (C.c_int, [VP, I64, VP]),
    "pbs_attention": (C.c_int, [VP, VP, VP, C.POINTER(Shape), C.POINTER(PipelineConfig), VP, VP, VP, VP, VP, SZ,
                                C.POINTER(Report), VP]),
    "pbs_attention_host": (C.c_int, [VP, VP, VP, C.POINTER(Shape), C.POINTER(PipelineConfig), VP, VP, VP, VP,
                                     C.POINTER(Report)]),
    "pbs_coverage_workspace_size": (SZ, [C.POINTER(Shape), I64]),
    "pbs_attention_coverage": (C.c_int, [VP, VP, C.POINTER(Shape), I64, VP, VP, VP, DBL, VP, VP, SZ, VP]),
    "pbs_tensor_info_read": (C.c_int, [C.c_char_p, C.POINTER(TensorInfo)]),
    "pbs_tensor_load": (C.c_int, [C.c_char_p, VP, I32, VP]),
    "pbs_tensor_save": (C.c_int, [C.c_char_p, VP, I32, I64, I64, I64, I32, I32, VP]),
    "pbs_debug_expf": (C.c_int, [VP, VP, I64, VP]),
    "pbs_generate_workload_head": (C.c_int, [C.POINTER(WorkloadSpec), I64, I64, I64, I32, VP, VP, VP, VP, VP]),
    "pbs_malloc": (C.c_int, [SZ, C.POINTER(VP)]),
    "pbs_free": (C.c_int, [VP]),
    "pbs_memcpy": (C.c_int, [VP, VP, SZ, I32, VP]),
    "pbs_stream_synchronize": (C.c_int, [VP]),
    "pbs_shard_plan": (C.c_int, [C.POINTER(Shape), I64, I32, I32, C.POINTER(Shard)]),
    "pbs_shard_workspace_size": (SZ, [C.POINTER(Shape), C.POINTER(PipelineConfig), I32, I32]),
    "pbs_attention_shard": (C.c_int, [VP, VP, VP, C.POINTER(Shape), C.POINTER(PipelineConfig), I32, I32, VP, VP, SZ,
                                      C.POINTER(Report), VP]),
    "pbs_dist_unique_id": (C.c_int, [VP]),
    "pbs_dist_create": (C.c_int, [VP, I32, I32, C.POINTER(VP)]),
    "pbs_dist_destroy": (C.c_int, [VP]),
    "pbs_dist_workspace_size": (SZ, [VP, C.POINTER(Shape), C.POINTER(PipelineConfig)]),
    "pbs_dist_attention": (C.c_int, [VP, VP, VP, VP, C.POINTER(Shape), C.POINTER(PipelineConfig), VP, VP, SZ,
                                     C.POINTER(Report), VP]),
}


def load(path: str | None = None):
    """Load libpbs_b200.so (raises if it is missing: there is no CPU fallback).
    PBS_B200_LIB names another build of the same library (A/B timing only)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PBS_B200_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing; build it with `python -m paper_2510_21270_b200.build` "
                          "(the PBS-Attn path has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc != PBS_OK:
        msg = _lib.pbs_last_error().decode()
        raise _ERRORS.get(rc, PbsError)(rc, msg)
