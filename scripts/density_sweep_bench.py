#!/usr/bin/env python3
"""BASELINE.json configs[4] / SURVEY.md §8d C5: block-density sweep (5%-50% of
the causal blocks kept) at 64K, Llama-3.1-8B attention shape (32 q / 8 kv heads,
d = 128, bf16), the tcgen05 block-sparse attention against the project's dense
causal FlashAttention (same kernel, full causal lists).

Masks are the acceptance suite's deterministic hash (acceptance_main.cpp:386-391),
here (i * 31 + j * 17) % 20 < k on the causal grid j <= i, plus the diagonal
block, so the kept fraction of the causal blocks is exact to within a few
blocks.  Kernel-only: Q/K/V resident, unpermuted (identity sigma / pi: the
element mask is the causal one).  One JSON line per density; times are CUDA
events over >= --min-ms of launches after 2 warm-ups.

    python scripts/density_sweep_bench.py [--seq 65536] [--reps 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_21270_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=65536)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--min-ms", type=float, default=400.0)
args = ap.parse_args()
HQ, HKV, D, B = 32, 8, 128, 128
n = args.seq
t = n // B
torch.manual_seed(0)
q = torch.randn(HQ, n, D, device="cuda").to(torch.bfloat16)
k = torch.randn(HKV, n, D, device="cuda").to(torch.bfloat16)
v = torch.randn(HKV, n, D, device="cuda").to(torch.bfloat16)


def timed(fn):
    """CUDA-event time per launch over at least --min-ms of back-to-back launches
    (GPU clocks under the power cap move on ~100 ms scales; short windows are noisy)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    reps = max(args.reps, int(args.min_ms / max(e0.elapsed_time(e1), 1e-3)) + 1)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = torch.empty_like(q)
dense_ms = timed(lambda: ops.dense_causal_attention(q, k, v, out=out))
causal_blocks = t * (t + 1) // 2
ii = torch.arange(t, device="cuda")[:, None]
jj = torch.arange(t, device="cuda")[None, :]
for keep in (1, 2, 4, 6, 7, 8, 9, 10):  # 5% .. 50%
    sel = (((ii * 31 + jj * 17) % 20) < keep) & (jj <= ii)
    sel |= ii == jj
    cnt = sel.sum(1).to(torch.int32)
    # ascending lists: the sorted column indices of each row, padded
    order = torch.where(sel, jj.expand(t, t), torch.full_like(jj.expand(t, t), t)).sort(1).values
    kv_idx = order.to(torch.int32).clamp_max(t - 1).unsqueeze(0).expand(HQ, t, t).contiguous()
    kv_cnt = cnt.unsqueeze(0).expand(HQ, t).contiguous()
    st = torch.empty(2, dtype=torch.int32, device="cuda")
    ms = timed(lambda: ops.attention_block_sparse(q, k, v, B, kv_idx, kv_cnt, check_status=False, out=out, status=st))
    sparse_out = ops.attention_block_sparse(q, k, v, B, kv_idx, kv_cnt)
    assert torch.isfinite(sparse_out.float()).all()
    frac = cnt.sum().item() / causal_blocks
    flops = 4.0 * B * B * D * cnt.sum().item() * HQ
    print(json.dumps({"workload": f"llama31_8b_attn_{n // 1024}k_density_sweep", "kept_of_causal": round(frac, 4),
                      "block_density": round(cnt.sum().item() / (t * t), 4), "sparse_ms": ms, "dense_ms": dense_ms,
                      "speedup_vs_dense_fa": dense_ms / ms, "executed_tflops": flops / (ms * 1e-3) / 1e12,
                      "dense_tflops": 4.0 * D * n * (n + 1) / 2 * HQ / (dense_ms * 1e-3) / 1e12}), flush=True)
