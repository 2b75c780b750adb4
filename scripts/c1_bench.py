"""BASELINE configs[0] (C1): one head, N = 4096, d = 128, B = 64, S = 256, fp32,
the reference's own CPU-runnable case, end to end on both sides with no
extrapolation.

Inputs come from the reference's generator (pbs::generate_head, vertical lines,
seed 1, 16 lines of strength 150) through the compiled reference
shim.  The reference side is the unmodified reference pbs_attention on one host
thread (one head); ours is pbs_attention_host (host buffers in and out: the f32
path, SIMT attention since B = 64) and the device entry with inputs resident.
Prints one JSON line; outputs are checked against the reference (f32 tolerance).

    python scripts/c1_bench.py [--steps 10]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch  # noqa: E402

import oracle  # noqa: E402
from gen_golden import generate_head  # noqa: E402
from paper_2510_21270_b200 import ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    n, d, b, s, tau = 4096, 128, 64, 256, 0.9
    ref = oracle.Oracle("ref")
    q, k, v, _ = generate_head(ref, "vertical_lines", n, d, 1, b, s, line_count=16, line_strength=150.0,
                               dtype=np.float32)
    rcfg = oracle.make_config(block_size=b, segment_size=s, tau=tau, strategy="key_permute")
    t0 = time.perf_counter()
    rr = ref.pbs_attention(q, k, v, rcfg)
    ref_ms = (time.perf_counter() - t0) * 1e3

    cfg = ops.make_config(block_size=b, segment_size=s, tau=tau, strategy="key_permute")
    hq, hk, hv = (torch.from_numpy(x[None].copy()).pin_memory() for x in (q, k, v))
    hout = torch.empty_like(hq).pin_memory()
    for _ in range(3):
        res = ops.pbs_attention_host(hq, hk, hv, cfg, out=hout, return_perms=True)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ops.pbs_attention_host(hq, hk, hv, cfg, out=hout, report=False)
        ts.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = float(np.median(ts))
    dq, dk, dv = (x.cuda() for x in (hq, hk, hv))
    for _ in range(3):
        ops.pbs_attention(dq, dk, dv, cfg, report=False, return_perms=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        ops.pbs_attention(dq, dk, dv, cfg, report=False, return_perms=False)
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / args.steps

    err = np.abs(res.output[0].numpy() - rr.output)
    line = {
        "workload": "c1_single_head_4k_b64_f32", "config": {"n": n, "d": d, "block": b, "segment": s, "tau": tau,
                                                           "strategy": "key_permute", "dtype": "f32",
                                                           "data": "pbs::generate_head vertical_lines seed 1, "
                                                                   "16 lines x 150"},
        "reference_cpu_ms": ref_ms, "reference_threads": 1,
        "e2e_ms": e2e_ms, "device_ms": dev_ms, "speedup_e2e": ref_ms / e2e_ms,
        "pi_bitexact": bool(np.array_equal(res.pi[0].numpy(), rr.pi)),
        "mask_bitexact": bool(np.array_equal(res.mask[0].numpy(), rr.mask)),
        "max_abs_err": float(err.max()), "mean_abs_err": float(err.mean()),
        "block_density": float(rr.report["block_density"]),
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
