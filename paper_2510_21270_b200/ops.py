"""Host-side mirror of the reference operator API over device tensors.

Function names, argument meaning and error behaviour follow the reference
headers (/root/reference/proj/include/pbs/); every call goes through the C
ABI of libpbs_b200.so (include/pbs_cabi.h) on the current CUDA stream.
Tensors use the head-major [H, N, d] layout; permutations are int32
``map[new] = old``; masks uint8 [H, T, T].  PyTorch is only the device-memory
and stream plumbing here.

    estimate_key_importance   permutation.hpp:143-178
    build_key_permutation     permutation.hpp:182-201 (+ flatten, inverse)
    build_query_permutation   permutation.hpp:206-275
    apply_rows                permutation.hpp:79-89
    unpermute                 pipeline.hpp:178-180
    meanpool_block_scores     block_selection.hpp:120-161
    select_blocks             block_selection.hpp:171-206
    attention_block_sparse    attention.hpp:259-310
    dense_causal_attention    attention.hpp:314-321 (causal comparator)
    pbs_attention             pipeline.hpp:107-193
    attention_coverage        pipeline.hpp:198-243
    density_sweep             pipeline.hpp:245-295
    tensor_info / load_tensor / save_tensor   tensor_io.hpp (PBST files)
    shard_plan / attention_shard / DistContext  head-parallel multi-GPU (the
                              per-head fan-out of pbs_main.cpp:99-122)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import PipelineConfig, Report, Shape, Shard, check

_WS: dict = {}


def lib():
    return _lib.load()


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, f"E_CONFIG: dtype {t.dtype} (need bfloat16 or float32)")


def _check_dev(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_SHAPE: tensors must be contiguous CUDA tensors")


def make_shape(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor | None = None) -> Shape:
    """pbs_shape of [Hq, N, d] queries over [Hkv, N, d] keys (and values).
    The C ABI carries one N and one d, so mismatched inputs are refused here
    with the reference's texts (pipeline.hpp:111-116) before any kernel could
    read past a shorter tensor."""
    for name, x in (("Q", q), ("K", k), ("V", v)):
        if x is not None and x.dim() != 3:
            raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, f"E_SHAPE: {name} must be a [heads, rows, cols] stack")
    if q.dtype != k.dtype or (v is not None and v.dtype != k.dtype):
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_CONFIG: Q, K and V must share one dtype")
    hq, n, d = q.shape
    hkv = k.shape[0]
    if k.shape[1] != n:
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG,
                               f"E_CONFIG: pipeline expects self-attention: N == M, got {n} vs {k.shape[1]}")
    if k.shape[2] != d or (v is not None and tuple(v.shape) != tuple(k.shape)):
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_SHAPE: pipeline inputs have inconsistent shapes")
    if hkv <= 0 or hq % hkv != 0:
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG,
                               "E_SHAPE: num_q_heads must be a positive multiple of num_kv_heads")
    return Shape(_dtype_code(q), hq, hkv, d, n)


def make_config(block_size=128, segment_size=256, tau=0.9, strategy="key_permute",
                forced_first_block=True, forced_diagonal_band=True, scale=0.0, top_k=0) -> PipelineConfig:
    """PipelineConfig defaults of the reference (pipeline.hpp:30-38).
    top_k > 0 selects the top_k admissible blocks per row instead of the tau
    threshold (an extension: the reference has no top-k mode)."""
    if isinstance(strategy, str):
        strategy = _lib.STRATEGIES[strategy]
    return PipelineConfig(block_size, segment_size, tau, strategy, int(forced_first_block),
                          int(forced_diagonal_band), int(top_k), scale)


def workspace(nbytes: int, device=None) -> torch.Tensor:
    """A cached device scratch buffer of at least nbytes."""
    device = torch.device(device or "cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (device.type, device.index)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def estimate_key_importance(q, k, block_size, scale=0.0):
    """scores [Hq, N] f32 (exact restatement of the reference's fp32 arithmetic)."""
    _check_dev(q, k)
    shape = make_shape(q, k)
    n = q.shape[1]
    take = min(block_size, n)
    ws = workspace(q.shape[0] * n * take * 4 + q.shape[0] * take * 8 + 4096, q.device)
    out = torch.empty(q.shape[0], n, dtype=torch.float32, device=q.device)
    check(lib().pbs_estimate_key_importance(_ptr(q), _ptr(k), C.byref(shape), block_size, scale, _ptr(out),
                                            _ptr(ws), ws.numel(), _stream()))
    return out


def build_key_permutation(scores, segment_size, with_inverse=True):
    """(perm, inv) int32 [H, N]."""
    _check_dev(scores)
    h, n = scores.shape
    perm = torch.empty(h, n, dtype=torch.int32, device=scores.device)
    inv = torch.empty_like(perm) if with_inverse else None
    check(lib().pbs_build_key_permutation(_ptr(scores), h, n, segment_size, _ptr(perm), _ptr(inv), _stream()))
    return perm, inv


def build_query_permutation(q, k, block_size, segment_size, with_inverse=True):
    _check_dev(q, k)
    shape = make_shape(q, k)
    hq, n, d = q.shape
    need = lib().pbs_query_permutation_workspace_size(C.byref(shape), block_size)
    if need == 0:
        check(lib().pbs_build_query_permutation(None, None, 0, C.byref(shape), block_size, segment_size,
                                                None, None, None, 0, _stream()))
    ws = workspace(need, q.device)
    perm = torch.empty(hq, n, dtype=torch.int32, device=q.device)
    inv = torch.empty_like(perm) if with_inverse else None
    check(lib().pbs_build_query_permutation(_ptr(q), _ptr(k), k.shape[0], C.byref(shape), block_size,
                                            segment_size, _ptr(perm), _ptr(inv), _ptr(ws), ws.numel(),
                                            _stream()))
    return perm, inv


def apply_rows(perm, src, dst_heads=None):
    """dst[h][i] = src[h // G][perm[h][i]] (perm None = identity broadcast)."""
    _check_dev(perm, src)
    hs, n, d = src.shape
    hd = dst_heads or (perm.shape[0] if perm is not None else hs)
    dst = torch.empty(hd, n, d, dtype=src.dtype, device=src.device)
    check(lib().pbs_apply_rows(_ptr(perm), _ptr(src), hs, hd, n, d, _dtype_code(src), _ptr(dst), _stream()))
    return dst


def unpermute(sigma, src):
    """The stage-5 un-permute (pipeline.hpp:178-180): out[h][sigma[h][i]] = src[h][i],
    i.e. apply_rows(sigma^-1, src) without forming the inverse."""
    _check_dev(sigma, src)
    h, n, d = src.shape
    out = torch.empty_like(src)
    check(lib().pbs_unpermute(_ptr(sigma), _ptr(src), h, n, d, _dtype_code(src), _ptr(out), _stream()))
    return out


def meanpool_block_scores(qp, kp, block_size, segment_size, scale=0.0):
    """Block scores [Hq, T, T] f32 under the segment-band causal mask."""
    _check_dev(qp, kp)
    shape = make_shape(qp, kp)
    hq, n, d = qp.shape
    t = -(-n // block_size)
    ws = workspace(2 * (hq * t * d * 4 + 256) + hq * t * t * 4 + 8192, qp.device)
    out = torch.empty(hq, t, t, dtype=torch.float32, device=qp.device)
    check(lib().pbs_meanpool_block_scores(_ptr(qp), _ptr(kp), C.byref(shape), block_size, segment_size, scale,
                                          _ptr(out), _ptr(ws), ws.numel(), _stream()))
    return out


def select_blocks(scores, block_size, segment_size, tau, forced_first_block=True, forced_diagonal_band=True,
                  top_k=0):
    """(mask uint8 [H,T,T], kv_idx int32 [H,T,T], kv_cnt int32 [H,T]); top_k > 0
    keeps the top_k admissible blocks per row instead of the tau prefix."""
    _check_dev(scores)
    h, t, _ = scores.shape
    mask = torch.empty(h, t, t, dtype=torch.uint8, device=scores.device)
    kv_idx = torch.empty(h, t, t, dtype=torch.int32, device=scores.device)
    kv_cnt = torch.empty(h, t, dtype=torch.int32, device=scores.device)
    if top_k:
        check(lib().pbs_select_blocks_top_k(_ptr(scores), h, t, block_size, segment_size, int(top_k),
                                            int(forced_first_block), int(forced_diagonal_band), _ptr(mask),
                                            _ptr(kv_idx), _ptr(kv_cnt), _stream()))
    else:
        check(lib().pbs_select_blocks(_ptr(scores), h, t, block_size, segment_size, tau, int(forced_first_block),
                                      int(forced_diagonal_band), _ptr(mask), _ptr(kv_idx), _ptr(kv_cnt), _stream()))
    return mask, kv_idx, kv_cnt


def attention_block_sparse(qp, kp, vp, block_size, kv_idx, kv_cnt, q_orig=None, k_orig=None, out_rows=None,
                           scale=0.0, check_status=True, out=None, status=None):
    """Permuted block-sparse attention; raises DegenerateRowError like finalize_into.
    `out` / `status` (int32 [2]) may be preallocated: the call then allocates
    nothing and never synchronises (check_status=False)."""
    _check_dev(qp, kp, vp, kv_idx, kv_cnt, q_orig, k_orig, out_rows)
    shape = make_shape(qp, kp, vp)
    out = torch.empty_like(qp) if out is None else out
    if status is None:
        status = torch.empty(2, dtype=torch.int32, device=qp.device)
    status[0] = 0
    status[1] = 0x7FFFFFFF
    check(lib().pbs_block_sparse_attention_fwd(_ptr(qp), _ptr(kp), _ptr(vp), kp.shape[0], C.byref(shape),
                                               block_size, scale, _ptr(kv_idx), _ptr(kv_cnt), _ptr(q_orig),
                                               _ptr(k_orig), _ptr(out_rows), _ptr(out), _ptr(status), _stream()))
    if check_status:
        t = -(-qp.shape[1] // block_size)
        check(lib().pbs_check_status(_ptr(status), t, _stream()))
    return out


def dense_causal_attention(q, k, v, scale=0.0, out=None):
    """The project's dense causal FlashAttention (GQA: kv head h // G)."""
    _check_dev(q, k, v)
    shape = make_shape(q, k, v)
    out = torch.empty_like(q) if out is None else out
    check(lib().pbs_dense_causal_attention_fwd(_ptr(q), _ptr(k), _ptr(v), C.byref(shape), scale, _ptr(out),
                                               _stream()))
    return out


@dataclass
class PipelineResult:
    """PipelineResult (pipeline.hpp:76-83) with per-head device tensors."""

    output: torch.Tensor
    sigma: torch.Tensor
    pi: torch.Tensor
    mask: torch.Tensor
    report: dict | None


def workspace_size(q, k, cfg: PipelineConfig) -> int:
    shape = make_shape(q, k)
    return int(lib().pbs_workspace_size(C.byref(shape), C.byref(cfg)))


def pbs_attention(q, k, v, cfg: PipelineConfig | None = None, report=True, out=None, return_perms=True,
                  ws=None):
    """Algorithm 1 on device tensors q [Hq,N,d], k/v [Hkv,N,d] (pipeline.hpp:107-193).

    With report=True the call synchronises and fills the PipelineReport; with
    report=False it is fully stream-ordered (graph-capturable)."""
    cfg = cfg or make_config()
    _check_dev(q, k, v)
    shape = make_shape(q, k, v)
    hq, n, d = q.shape
    t = -(-n // max(int(cfg.block_size), 1))
    need = lib().pbs_workspace_size(C.byref(shape), C.byref(cfg))
    if need == 0:
        check(_lib.PBS_ERR_CONFIG)
    ws = workspace(need, q.device) if ws is None else ws
    out = torch.empty_like(q) if out is None else out
    sigma = pi = mask = None
    if return_perms:
        sigma = torch.empty(hq, n, dtype=torch.int32, device=q.device)
        pi = torch.empty(hq, n, dtype=torch.int32, device=q.device)
        mask = torch.empty(hq, t, t, dtype=torch.uint8, device=q.device)
    rep = Report() if report else None
    check(lib().pbs_attention(_ptr(q), _ptr(k), _ptr(v), C.byref(shape), C.byref(cfg), _ptr(out), _ptr(sigma),
                              _ptr(pi), _ptr(mask), _ptr(ws), ws.numel(), C.byref(rep) if rep else None,
                              _stream()))
    return PipelineResult(out, sigma, pi, mask, rep.as_dict() if rep else None)


def pbs_attention_host(q, k, v, cfg: PipelineConfig | None = None, return_perms=False, out=None, report=True):
    """The reference-facing call on HOST (CPU) tensors: copies in, runs, copies out.
    Pass pinned host tensors (and a pinned `out`) for full PCIe bandwidth."""
    cfg = cfg or make_config()
    for x in (q, k, v):
        if x.is_cuda or not x.is_contiguous():
            raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_SHAPE: host tensors must be contiguous CPU tensors")
    shape = make_shape(q, k, v)
    hq, n, d = q.shape
    t = -(-n // max(int(cfg.block_size), 1))
    out = torch.empty_like(q) if out is None else out
    sigma = pi = mask = None
    if return_perms:
        sigma = torch.empty(hq, n, dtype=torch.int32)
        pi = torch.empty(hq, n, dtype=torch.int32)
        mask = torch.empty(hq, t, t, dtype=torch.uint8)
    rep = Report() if report else None
    check(lib().pbs_attention_host(_ptr(q), _ptr(k), _ptr(v), C.byref(shape), C.byref(cfg), _ptr(out),
                                   _ptr(sigma), _ptr(pi), _ptr(mask), C.byref(rep) if rep else None))
    return PipelineResult(out, sigma, pi, mask, rep.as_dict() if rep else None)


def attention_coverage(q, k, mask, sigma=None, pi=None, block_size=128, scale=0.0):
    """attention_coverage (pipeline.hpp:198-243) per query head: the fraction of
    the true causal probability mass of the ORIGINAL q, k that falls inside the
    selected blocks of the permuted grid.  Returns a float64 CPU tensor [Hq].
    (No N^2 <= 2^26 cap: the mass is computed from two attention passes.)"""
    _check_dev(q, k, mask, sigma, pi)
    shape = make_shape(q, k)
    need = lib().pbs_coverage_workspace_size(C.byref(shape), int(block_size))
    if need == 0:
        check(_lib.PBS_ERR_CONFIG)
    ws = workspace(need, q.device)
    cov = torch.empty(q.shape[0], dtype=torch.float64, device=q.device)
    check(lib().pbs_attention_coverage(_ptr(q), _ptr(k), C.byref(shape), int(block_size), _ptr(mask), _ptr(sigma),
                                       _ptr(pi), float(scale), _ptr(cov), _ptr(ws), ws.numel(), _stream()))
    return cov.cpu()


@dataclass
class SweepRow:
    """SweepRow (pipeline.hpp:234-243); density / coverage averaged over heads."""

    tau: float
    segment_size: int
    strategy: str
    density: float
    coverage: float
    max_err: float
    mean_err: float
    time_us: float


_STRATEGY_NAMES = {0: "none", 1: "key_permute", 2: "query_permute", 3: "both"}


def density_sweep(q, k, v, base: PipelineConfig, taus, segment_sizes):
    """density_sweep (pipeline.hpp:245-295): one pipeline run per (tau, segment
    size), against the dense causal attention of the same inputs; rows sorted by
    (segment size, tau).  Errors compare with this library's dense causal
    attention (the reference compares with its attention_oracle)."""
    if not taus or not segment_sizes:
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_CONFIG: density_sweep needs at least one tau and one segment size")
    oracle = dense_causal_attention(q, k, v, scale=base.scale).float()
    rows = []
    for s in sorted(segment_sizes):
        for tau in sorted(taus):
            cfg = make_config(block_size=int(base.block_size), segment_size=int(s), tau=float(tau),
                              strategy=_STRATEGY_NAMES[int(base.strategy)], scale=float(base.scale),
                              forced_first_block=bool(base.forced_first_block),
                              forced_diagonal_band=bool(base.forced_diagonal_band))
            res = pbs_attention(q, k, v, cfg)
            cov = attention_coverage(q, k, res.mask, res.sigma, res.pi, int(cfg.block_size), float(cfg.scale))
            err = (res.output.float() - oracle).abs()
            r = res.report
            rows.append(SweepRow(tau=float(tau), segment_size=int(s), strategy=_STRATEGY_NAMES[int(cfg.strategy)],
                                 density=r["block_density"], coverage=float(cov.mean()),
                                 max_err=float(err.max()), mean_err=float(err.mean()),
                                 time_us=r["estimate_us"] + r["permute_us"] + r["select_us"] + r["attention_us"]
                                 + r["unpermute_us"]))
    return rows


def tensor_info(path) -> dict:
    """The header of a PBST file (read_tensor's checks, tensor_io.hpp:98-146):
    file_dtype (0 f32 / 1 f64), ndim, heads, rows, cols, payload_offset."""
    info = _lib.TensorInfo()
    check(lib().pbs_tensor_info_read(str(path).encode(), C.byref(info)))
    return info.as_dict()


def load_tensor(path, dtype=torch.bfloat16, device=None) -> torch.Tensor:
    """read_tensor (tensor_io.hpp:98-146) straight into device memory: a 3-D
    file gives [heads, rows, cols], a 2-D file [rows, cols], as bf16 (rounded
    to nearest) or f32.  Non-finite payload elements raise E_FORMAT with their
    byte offset (tensor_io.hpp:80-81)."""
    info = tensor_info(path)
    shape = (info["heads"], info["rows"], info["cols"]) if info["ndim"] == 3 else (info["rows"], info["cols"])
    out = torch.empty(shape, dtype=dtype, device=device or torch.device("cuda", torch.cuda.current_device()))
    check(lib().pbs_tensor_load(str(path).encode(), _ptr(out), _dtype_code(out), _stream()))
    return out


def save_tensor(path, t: torch.Tensor, file_dtype="f32", as_stack=None):
    """write_tensor / write_tensor_stack (tensor_io.hpp:155-193) from a device
    tensor ([heads, rows, cols] or [rows, cols], bf16 or f32).  as_stack
    defaults to the tensor's rank (3-D -> stack)."""
    _check_dev(t)
    if t.dim() not in (2, 3):
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, "E_SHAPE: write_tensor takes a 2-D matrix or a 3-D stack")
    heads, rows, cols = (t.shape if t.dim() == 3 else (1, *t.shape))
    stack = (t.dim() == 3) if as_stack is None else bool(as_stack)
    code = {"f32": 0, "f64": 1}[file_dtype]
    check(lib().pbs_tensor_save(str(path).encode(), _ptr(t), _dtype_code(t), heads, rows, cols, code, int(stack),
                                _stream()))


def workload_spec(kind="gaussian", n=1024, d=64, heads=1, seed=0, line_count=8, line_strength=150.0,
                  scatter="scattered") -> "_lib.WorkloadSpec":
    """WorkloadSpec (workload.hpp:21-38) with the reference's defaults; kind and
    scatter by their manifest names (workload_kind_from_name, scatter_from_name)."""
    if kind not in _lib.WORKLOAD_KINDS:
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, f"E_CONFIG: unknown workload kind '{kind}'")
    if scatter not in _lib.LINE_SCATTER:
        raise _lib.ConfigError(_lib.PBS_ERR_CONFIG, f"E_CONFIG: unknown scatter mode '{scatter}'")
    return _lib.WorkloadSpec(kind=_lib.WORKLOAD_KINDS[kind], scatter=_lib.LINE_SCATTER[scatter], n=n, d=d,
                             heads=heads, seed=seed, line_count=line_count, line_strength=line_strength)


def generate_workload_head(spec, head, block_size, segment_size, precision="f32"):
    """generate_head (workload.hpp:145-198) on the host, bit-identical to the
    reference: numpy q, k, v [n, d] in the manifest precision (f32 / f64) and
    the planted line positions."""
    import numpy as np

    dt = {"f32": np.float32, "f64": np.float64}[precision]
    q, k, v = (np.empty((spec.n, spec.d), dtype=dt) for _ in range(3))
    planted = np.zeros(max(int(spec.line_count), 1), dtype=np.int64)
    cnt = C.c_int64(0)
    check(lib().pbs_generate_workload_head(C.byref(spec), head, block_size, segment_size,
                                           0 if precision == "f32" else 1, q.ctypes.data, k.ctypes.data,
                                           v.ctypes.data, planted.ctypes.data, C.byref(cnt)))
    return q, k, v, planted[:cnt.value]


def debug_expf(x: torch.Tensor) -> torch.Tensor:
    _check_dev(x)
    y = torch.empty_like(x)
    check(lib().pbs_debug_expf(_ptr(x), _ptr(y), x.numel(), _stream()))
    return y


# ---------------------------------------------------------------- multi-GPU
def shard_plan(num_q_heads, num_kv_heads, seq_len, head_dim, block_size, world_size, rank, dtype=torch.bfloat16):
    """pbs_shard_plan: rank's contiguous share of the (query head, query-block
    pair) work units, weighted by causal key blocks.  Pure host arithmetic."""
    code = _lib.DTYPE_BF16 if dtype == torch.bfloat16 else _lib.DTYPE_F32
    shape = Shape(code, num_q_heads, num_kv_heads, head_dim, seq_len)
    s = Shard()
    check(lib().pbs_shard_plan(C.byref(shape), block_size, world_size, rank, C.byref(s)))
    return s.as_dict()


def _global_shape(q_local, num_q_heads, num_kv_heads):
    _, n, d = q_local.shape
    return Shape(_dtype_code(q_local), num_q_heads, num_kv_heads, d, n)


def attention_shard(q_local, k_local, v_local, num_q_heads, num_kv_heads, cfg, world_size, rank, out_full,
                    ws=None, report=False):
    """Rank `rank`'s share of pbs_attention, compute only, into its rows of
    out_full [Hq, N, d] (q_local: the shard's query heads, k/v_local: its KV heads)."""
    _check_dev(q_local, k_local, v_local, out_full)
    shape = _global_shape(q_local, num_q_heads, num_kv_heads)
    need = lib().pbs_shard_workspace_size(C.byref(shape), C.byref(cfg), world_size, rank)
    if need == 0:
        check(_lib.PBS_ERR_CONFIG)
    ws = workspace(need, q_local.device) if ws is None else ws
    rep = Report() if report else None
    check(lib().pbs_attention_shard(_ptr(q_local), _ptr(k_local), _ptr(v_local), C.byref(shape), C.byref(cfg),
                                    world_size, rank, _ptr(out_full), _ptr(ws), ws.numel(),
                                    C.byref(rep) if rep else None, _stream()))
    return rep.as_dict() if rep else None


def dist_unique_id() -> bytes:
    """pbs_dist_unique_id: the NCCL id rank 0 shares with the other ranks."""
    buf = (C.c_uint8 * 128)()
    check(lib().pbs_dist_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class DistContext:
    """pbs_dist: a per-rank handle owning the NCCL communicator of the
    head-parallel path; attention() computes the rank's share and all-gathers
    every rank's rows into out_full (the one exchange)."""

    def __init__(self, unique_id: bytes, world_size: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self.world, self.rank = world_size, rank
        self._h = C.c_void_p()
        check(lib().pbs_dist_create(C.cast(buf, C.c_void_p), world_size, rank, C.byref(self._h)))

    def workspace_size(self, q_local, num_q_heads, num_kv_heads, cfg):
        shape = _global_shape(q_local, num_q_heads, num_kv_heads)
        return int(lib().pbs_dist_workspace_size(self._h, C.byref(shape), C.byref(cfg)))

    def attention(self, q_local, k_local, v_local, num_q_heads, num_kv_heads, cfg, out_full, ws=None, report=False):
        _check_dev(q_local, k_local, v_local, out_full)
        shape = _global_shape(q_local, num_q_heads, num_kv_heads)
        if ws is None:
            ws = workspace(self.workspace_size(q_local, num_q_heads, num_kv_heads, cfg), q_local.device)
        rep = Report() if report else None
        check(lib().pbs_dist_attention(self._h, _ptr(q_local), _ptr(k_local), _ptr(v_local), C.byref(shape),
                                       C.byref(cfg), _ptr(out_full), _ptr(ws), ws.numel(),
                                       C.byref(rep) if rep else None, _stream()))
        return rep.as_dict() if rep else None

    def close(self):
        if self._h:
            lib().pbs_dist_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
