"""TEST INFRASTRUCTURE ONLY -- the parity checker, never the product path.

ctypes bindings for
  * ``oracle/_build/libpbs_oracle.so`` -- the plain-C restatement of the
    reference hot path (oracle/pbs_oracle_impl.inc, each function citing the
    reference file:line it follows), and
  * ``oracle/_ref/libpbsref.so`` -- the unmodified reference headers compiled
    in place from /root/reference by oracle/Makefile (present wherever it was
    built; it travels to the GPU box as a prebuilt binary).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2510_21270_b200) never imports it and has no CPU fallback.

Both libraries expose the same per-head API; ``Oracle(kind)`` wraps either
with numpy in / numpy out, mirroring the reference's function names.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libpbs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpbsref.so")
REF_INCLUDE = "/root/reference/proj/include"

STRATEGIES = {"none": 0, "key_permute": 1, "query_permute": 2, "both": 3}


class PipelineConfig(C.Structure):
    """pbs_pipeline_config (include/pbs_cabi.h) == PipelineConfig (pipeline.hpp:30-49)."""

    _fields_ = [
        ("block_size", C.c_int64),
        ("segment_size", C.c_int64),
        ("tau", C.c_double),
        ("strategy", C.c_int32),
        ("forced_first_block", C.c_int32),
        ("forced_diagonal_band", C.c_int32),
        ("top_k", C.c_int32),
        ("scale", C.c_double),
    ]


class Report(C.Structure):
    """pbs_report (include/pbs_cabi.h) == PipelineReport (pipeline.hpp:63-74)."""

    _fields_ = [
        ("block_density", C.c_double),
        ("causal_density_baseline", C.c_double),
        ("pooled_score_coverage", C.c_double),
        ("selected_blocks", C.c_int64),
        ("total_admissible_blocks", C.c_int64),
        ("estimate_us", C.c_double),
        ("permute_us", C.c_double),
        ("select_us", C.c_double),
        ("attention_us", C.c_double),
        ("unpermute_us", C.c_double),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


def make_config(block_size=128, segment_size=256, tau=0.9, strategy="key_permute",
                forced_first_block=True, forced_diagonal_band=True, scale=0.0, top_k=0) -> PipelineConfig:
    if isinstance(strategy, str):
        strategy = STRATEGIES[strategy]
    return PipelineConfig(block_size, segment_size, tau, strategy, int(forced_first_block),
                          int(forced_diagonal_band), int(top_k), scale)


class OracleError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the restatement (and the reference shim when /root/reference exists)."""
    targets = ["oracle"]
    if ref and os.path.exists(os.path.join(REF_INCLUDE, "pbs", "pipeline.hpp")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


_SZ = C.c_size_t
_F = {np.float32: C.c_float, np.float64: C.c_double}
_SFX = {np.float32: "f32", np.float64: "f64"}


@dataclass
class PipelineResult:
    output: np.ndarray
    sigma: np.ndarray
    pi: np.ndarray
    mask: np.ndarray
    report: dict


class Oracle:
    """kind = "oracle" (C restatement) or "ref" (compiled reference headers)."""

    def __init__(self, kind: str = "oracle"):
        path = ORACLE_SO if kind == "oracle" else REF_SO
        if not os.path.exists(path):
            build(ref=(kind == "ref"))
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} is missing (reference not built here)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.prefix = "pbso_" if kind == "oracle" else "pbsref_"
        self._last_error = getattr(self.lib, self.prefix + "last_error")
        self._last_error.restype = C.c_char_p

    @staticmethod
    def available(kind: str) -> bool:
        return os.path.exists(ORACLE_SO if kind == "oracle" else REF_SO)

    def _fn(self, name, dtype):
        return getattr(self.lib, f"{self.prefix}{name}_{_SFX[dtype]}")

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._last_error().decode())

    @staticmethod
    def _arr(x, dtype):
        return np.ascontiguousarray(x, dtype=dtype)

    # ---- a1 estimate_key_importance (permutation.hpp:143-178)
    def estimate_key_importance(self, q, k, block_size, scale=0.0):
        dt = q.dtype.type
        q, k = self._arr(q, dt), self._arr(k, dt)
        n, d = q.shape
        m = k.shape[0]
        out = np.zeros(m, dtype=dt)
        src = _SZ(0)
        self._check(self._fn("estimate_key_importance", dt)(
            _p(q, _F[dt]), _SZ(n), _p(k, _F[dt]), _SZ(m), _SZ(d), _SZ(block_size), C.c_double(scale),
            _p(out, _F[dt]), C.byref(src)))
        return out, src.value

    # ---- a2 build_key_permutation + flatten (permutation.hpp:182-201, 118-126)
    def build_key_permutation(self, scores, segment_size):
        dt = scores.dtype.type
        scores = self._arr(scores, dt)
        perm = np.zeros(scores.shape[0], dtype=np.int32)
        self._check(self._fn("build_key_permutation", dt)(
            _p(scores, _F[dt]), _SZ(scores.shape[0]), _SZ(segment_size), _p(perm, C.c_int32)))
        return perm

    # ---- a4 build_query_permutation (permutation.hpp:206-275)
    def build_query_permutation(self, q, k, block_size, segment_size):
        dt = q.dtype.type
        q, k = self._arr(q, dt), self._arr(k, dt)
        perm = np.zeros(q.shape[0], dtype=np.int32)
        self._check(self._fn("build_query_permutation", dt)(
            _p(q, _F[dt]), _SZ(q.shape[0]), _p(k, _F[dt]), _SZ(k.shape[0]), _SZ(q.shape[1]),
            _SZ(block_size), _SZ(segment_size), _p(perm, C.c_int32)))
        return perm

    # ---- a6 build_block_causal_mask (block_selection.hpp:86-97)
    def build_block_causal_mask(self, t, block_size, segment_size, dtype=np.float32):
        out = np.zeros((t, t), dtype=dtype)
        self._check(self._fn("block_causal_mask", dtype)(
            _SZ(t), _SZ(t), _SZ(block_size), _SZ(segment_size), _p(out, _F[dtype])))
        return out

    # ---- a7 meanpool_block_scores (block_selection.hpp:120-161)
    def meanpool_block_scores(self, qp, kp, block_size, causal, scale=0.0):
        dt = qp.dtype.type
        qp, kp, causal = self._arr(qp, dt), self._arr(kp, dt), self._arr(causal, dt)
        out = np.zeros(causal.shape, dtype=dt)
        self._check(self._fn("meanpool_block_scores", dt)(
            _p(qp, _F[dt]), _SZ(qp.shape[0]), _p(kp, _F[dt]), _SZ(kp.shape[0]), _SZ(qp.shape[1]),
            _SZ(block_size), _p(causal, _F[dt]), C.c_double(scale), _p(out, _F[dt])))
        return out

    # ---- a8 select_blocks (block_selection.hpp:171-206)
    def select_blocks(self, scores, causal, block_size, segment_size, tau,
                      forced_first_block=True, forced_diagonal_band=True, top_k=0):
        """top_k > 0: the top-k extension (the C restatement only; the reference has none)."""
        dt = scores.dtype.type
        scores, causal = self._arr(scores, dt), self._arr(causal, dt)
        t_r, t_c = scores.shape
        mask = np.zeros((t_r, t_c), dtype=np.uint8)
        if top_k:
            assert self.kind == "oracle", "the reference has no top-k selection"
            self._check(self._fn("select_blocks_top_k", dt)(
                _p(scores, _F[dt]), _p(causal, _F[dt]), _SZ(t_r), _SZ(t_c), _SZ(block_size),
                _SZ(segment_size), _SZ(top_k), int(forced_first_block), int(forced_diagonal_band),
                _p(mask, C.c_uint8)))
            return mask
        self._check(self._fn("select_blocks", dt)(
            _p(scores, _F[dt]), _p(causal, _F[dt]), _SZ(t_r), _SZ(t_c), _SZ(block_size),
            _SZ(segment_size), C.c_double(tau), int(forced_first_block), int(forced_diagonal_band),
            _p(mask, C.c_uint8)))
        return mask

    # ---- a10 attention_block_sparse (attention.hpp:259-310)
    def attention_block_sparse(self, q, k, v, block_size, mask=None, q_orig=None, k_orig=None,
                               causal=False, scale=0.0):
        dt = q.dtype.type
        q, k, v = self._arr(q, dt), self._arr(k, dt), self._arr(v, dt)
        mask = None if mask is None else self._arr(mask, np.uint8)
        q_orig = None if q_orig is None else self._arr(q_orig, np.int32)
        k_orig = None if k_orig is None else self._arr(k_orig, np.int32)
        out = np.zeros((q.shape[0], v.shape[1]), dtype=dt)
        deg = _SZ(0)
        rc = self._fn("attention_block_sparse", dt)(
            _p(q, _F[dt]), _SZ(q.shape[0]), _p(k, _F[dt]), _p(v, _F[dt]), _SZ(k.shape[0]),
            _SZ(q.shape[1]), _SZ(v.shape[1]), _SZ(block_size), C.c_double(scale), int(causal),
            _p(mask, C.c_uint8), _p(q_orig, C.c_int32), _p(k_orig, C.c_int32), _p(out, _F[dt]),
            C.byref(deg))
        if rc != 0:
            err = OracleError(rc, self._last_error().decode())
            err.query_block = deg.value
            raise err
        return out

    # ---- a13 attention_oracle (attention.hpp:226-255)
    def attention_oracle(self, q, k, v, block_size=1, causal=False, q_orig=None, k_orig=None,
                         scale=0.0):
        dt = q.dtype.type
        q, k, v = self._arr(q, dt), self._arr(k, dt), self._arr(v, dt)
        q_orig = None if q_orig is None else self._arr(q_orig, np.int32)
        k_orig = None if k_orig is None else self._arr(k_orig, np.int32)
        out = np.zeros((q.shape[0], v.shape[1]), dtype=dt)
        self._check(self._fn("attention_oracle", dt)(
            _p(q, _F[dt]), _SZ(q.shape[0]), _p(k, _F[dt]), _p(v, _F[dt]), _SZ(k.shape[0]),
            _SZ(q.shape[1]), _SZ(v.shape[1]), _SZ(block_size), C.c_double(scale), int(causal),
            _p(q_orig, C.c_int32), _p(k_orig, C.c_int32), _p(out, _F[dt])))
        return out

    # ---- attention_coverage (pipeline.hpp:198-243)
    def attention_coverage(self, q, k, mask, block_size, sigma=None, pi=None, scale=0.0):
        dt = q.dtype.type
        q, k = self._arr(q, dt), self._arr(k, dt)
        mask = self._arr(mask, np.uint8)
        sigma = None if sigma is None else self._arr(sigma, np.int32)
        pi = None if pi is None else self._arr(pi, np.int32)
        out = C.c_double(0.0)
        self._check(self._fn("attention_coverage", dt)(
            _p(q, _F[dt]), _p(k, _F[dt]), _SZ(q.shape[0]), _SZ(q.shape[1]), _p(mask, C.c_uint8),
            _SZ(block_size), _p(sigma, C.c_int32), _p(pi, C.c_int32), C.c_double(scale), C.byref(out)))
        return out.value

    # ---- a12 pbs_attention (pipeline.hpp:107-193)
    def pbs_attention(self, q, k, v, cfg: PipelineConfig) -> PipelineResult:
        dt = q.dtype.type
        q, k, v = self._arr(q, dt), self._arr(k, dt), self._arr(v, dt)
        n, d = q.shape
        b = max(int(cfg.block_size), 1)
        t = (n + b - 1) // b
        out = np.zeros((n, d), dtype=dt)
        sigma = np.zeros(n, dtype=np.int32)
        pi = np.zeros(n, dtype=np.int32)
        mask = np.zeros((t, t), dtype=np.uint8)
        rep = Report()
        self._check(self._fn("pbs_attention", dt)(
            _p(q, _F[dt]), _p(k, _F[dt]), _p(v, _F[dt]), _SZ(n), _SZ(d), C.byref(cfg),
            _p(out, _F[dt]), _p(sigma, C.c_int32), _p(pi, C.c_int32), _p(mask, C.c_uint8),
            C.byref(rep)))
        return PipelineResult(out, sigma, pi, mask, rep.as_dict())

    # ---- PBST files through the reference's tensor_io.hpp (reference only)
    def write_tensor(self, path, a, as_stack=None):
        """write_tensor / write_tensor_stack (tensor_io.hpp:155-193)."""
        assert self.kind == "ref"
        a = np.ascontiguousarray(a)
        heads, rows, cols = (a.shape if a.ndim == 3 else (1, *a.shape))
        stack = (a.ndim == 3) if as_stack is None else bool(as_stack)
        fn = self.lib[f"pbsref_write_tensor_{_SFX[a.dtype.type]}"]
        fn.argtypes = [C.c_char_p, C.c_void_p, _SZ, _SZ, _SZ, C.c_int]
        self._check(fn(str(path).encode(), a.ctypes.data, heads, rows, cols, int(stack)))

    def read_tensor(self, path):
        """read_tensor (tensor_io.hpp:98-146): (values as float64 [heads, rows, cols]
        or [rows, cols], file dtype code, ndim); errors raise with the E_* text."""
        assert self.kind == "ref"
        fn = self.lib["pbsref_read_tensor"]
        fn.argtypes = [C.c_char_p, C.c_void_p, _SZ, C.c_void_p, C.c_void_p, C.c_void_p]
        dims = np.zeros(3, dtype=np.int64)
        fdt, nd = C.c_int(0), C.c_int(0)
        self._check(fn(str(path).encode(), None, 0, dims.ctypes.data, C.addressof(fdt), C.addressof(nd)))
        out = np.zeros(int(np.prod(dims)), dtype=np.float64)
        self._check(fn(str(path).encode(), out.ctypes.data, out.size, dims.ctypes.data, C.addressof(fdt),
                       C.addressof(nd)))
        shape = tuple(int(x) for x in dims) if nd.value == 3 else (int(dims[1]), int(dims[2]))
        return out.reshape(shape), fdt.value, nd.value

    # ---- multi-head CPU run (reference only; pbs_main.cpp:99-122)
    def pbs_attention_heads(self, q, k, v, cfg: PipelineConfig, threads: int):
        assert self.kind == "ref"
        q = self._arr(q, np.float32)
        k = self._arr(k, np.float32)
        v = self._arr(v, np.float32)
        hq, n, d = q.shape
        hkv = k.shape[0]
        out = np.zeros_like(q)
        rep = Report()
        fn = self.lib["pbsref_pbs_attention_heads_f32"]
        self._check(fn(_p(q, C.c_float), _p(k, C.c_float), _p(v, C.c_float), C.c_int(hq),
                       C.c_int(hkv), _SZ(n), _SZ(d), C.byref(cfg), _p(out, C.c_float),
                       C.c_int(threads), C.byref(rep)))
        return out, rep.as_dict()


def inverse(perm: np.ndarray) -> np.ndarray:
    """Permutation::inverse (permutation.hpp:51-55)."""
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0], dtype=perm.dtype)
    return inv


def host_expf(x: np.ndarray) -> np.ndarray:
    """glibc expf on this host -- the reference's std::exp(float)."""
    lib = Oracle("oracle").lib
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    lib.pbso_expf(_p(x, C.c_float), _p(y, C.c_float), _SZ(x.size))
    return y
