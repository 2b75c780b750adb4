#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY -- regenerate tests/golden/ from the reference.

Runs in the build container, where /root/reference exists and
oracle/_ref/libpbsref.so (the unmodified reference headers, compiled in
place by oracle/Makefile) can be built.  The fixtures it writes are small,
committed, and let the oracle be pinned on machines without the reference:

* pipeline256.npz -- the inputs of the reference's GoldenRun256 test
  (pipeline_test.cpp:79-103): generate_workload<double>(gaussian, n=256,
  d=16, seed=13) with B=32, S=64.  tests/golden/pipeline256.json (copied
  from proj/tests/golden/, 3 numbers) holds the expected max/mean error and
  density.
* attn4.npz -- the golden attention case of attention_test.cpp:50-73
  (gaussian n=4, d=2, seed 42, f64) with expected full and causal outputs
  computed by the formula of proj/tests/golden/make_golden.py (NumPy f64,
  full materialisation).  The reference ships only the generator; its .pbst
  inputs are missing, so they are regenerated here.
* ref_pipeline_f32_<kind>.npz -- f32 Algorithm-1 runs of the compiled
  reference on its own synthetic workloads (vertical_lines / mixed /
  gaussian), with sigma, pi, mask, importance, block scores and outputs.

Usage:  python oracle/gen_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import Oracle, build, make_config  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_GOLDEN = "/root/reference/proj/tests/golden"
KINDS = {"gaussian": 0, "vertical_lines": 1, "block_diag": 2, "mixed": 3}


def generate_head(ref: Oracle, kind, n, d, seed, block, segment, head=0, line_count=8,
                  line_strength=150.0, scatter=1, dtype=np.float64):
    """pbs::generate_head (workload.hpp:145-198) through the reference shim."""
    sfx = "f64" if dtype == np.float64 else "f32"
    ct = C.c_double if dtype == np.float64 else C.c_float
    q = np.zeros((n, d), dtype=dtype)
    k = np.zeros((n, d), dtype=dtype)
    v = np.zeros((n, d), dtype=dtype)
    planted = np.zeros(max(line_count, 1), dtype=np.int64)
    fn = ref.lib[f"pbsref_generate_head_{sfx}"]
    rc = fn(C.c_int(KINDS[kind]), C.c_size_t(n), C.c_size_t(d), C.c_uint64(seed),
            C.c_size_t(line_count), C.c_double(line_strength), C.c_int(scatter),
            C.c_size_t(head), C.c_size_t(block), C.c_size_t(segment),
            q.ctypes.data_as(C.POINTER(ct)), k.ctypes.data_as(C.POINTER(ct)),
            v.ctypes.data_as(C.POINTER(ct)), planted.ctypes.data_as(C.POINTER(C.c_int64)))
    if rc < 0:
        raise RuntimeError(ref.lib["pbsref_last_error"]())
    return q, k, v, planted[:rc]


def np_attention(q, k, v, causal):
    """make_golden.py:45-55, verbatim formula."""
    d = q.shape[1]
    scores = q @ k.T / np.sqrt(d)
    if causal:
        n, m = scores.shape
        scores = np.where(np.arange(m)[None, :] <= np.arange(n)[:, None], scores, -np.inf)
    scores = scores - scores.max(axis=1, keepdims=True)
    weights = np.exp(scores)
    weights /= weights.sum(axis=1, keepdims=True)
    return weights @ v


def main():
    build(ref=True)
    ref = Oracle("ref")
    os.makedirs(GOLDEN, exist_ok=True)
    shutil.copy(os.path.join(REF_GOLDEN, "pipeline256.json"), os.path.join(GOLDEN, "pipeline256.json"))

    q, k, v, _ = generate_head(ref, "gaussian", 256, 16, 13, 32, 64)
    np.savez_compressed(os.path.join(GOLDEN, "pipeline256.npz"), q=q, k=k, v=v)

    q, k, v, _ = generate_head(ref, "gaussian", 4, 2, 42, 1, 1)
    np.savez_compressed(os.path.join(GOLDEN, "attn4.npz"), q=q, k=k, v=v,
                        expected_full=np_attention(q, k, v, False),
                        expected_causal=np_attention(q, k, v, True))

    cases = [
        ("vertical_lines", dict(n=512, d=64, seed=1, block=64, segment=128, line_count=8,
                                line_strength=150.0, tau=0.9, strategy="key_permute")),
        ("mixed", dict(n=384, d=32, seed=7, block=32, segment=64, line_count=6,
                       line_strength=40.0, tau=0.8, strategy="both")),
        ("gaussian", dict(n=300, d=16, seed=3, block=16, segment=32, line_count=0,
                          line_strength=1.0, tau=0.7, strategy="query_permute")),
    ]
    meta = {}
    for kind, c in cases:
        q, k, v, planted = generate_head(ref, kind, c["n"], c["d"], c["seed"], c["block"],
                                         c["segment"], line_count=c["line_count"],
                                         line_strength=c["line_strength"], dtype=np.float32)
        cfg = make_config(block_size=c["block"], segment_size=c["segment"], tau=c["tau"],
                          strategy=c["strategy"])
        res = ref.pbs_attention(q, k, v, cfg)
        imp, _ = ref.estimate_key_importance(q, k, c["block"])
        t = (c["n"] + c["block"] - 1) // c["block"]
        causal = ref.build_block_causal_mask(t, c["block"], c["segment"])
        qp = q[res.sigma]
        kp = k[res.pi]
        scores = ref.meanpool_block_scores(qp, kp, c["block"], causal)
        np.savez_compressed(os.path.join(GOLDEN, f"ref_pipeline_f32_{kind}.npz"), q=q, k=k, v=v,
                            output=res.output, sigma=res.sigma, pi=res.pi, mask=res.mask,
                            importance=imp, block_scores=scores, planted=planted)
        rep = {key: val for key, val in res.report.items() if not key.endswith("_us")}
        meta[kind] = {**c, "report": rep}
    with open(os.path.join(GOLDEN, "ref_pipeline_f32.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(GOLDEN)))


if __name__ == "__main__":
    main()
