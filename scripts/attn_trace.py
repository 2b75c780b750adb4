"""Debug: CTA 0's attention pipeline timeline on the C3 bench workload.

Needs a build with the trace events compiled in:
    PBS_NVCC_EXTRA=-DPBS_ATTN_TRACE_EVENTS python -m paper_2510_21270_b200.build --force
then PBS_ATTN_TRACE (set below) dumps clock64 stamps of CTA 0.  Events,
indexed by the CTA-cumulative visited block g (group g % 2 within an item):
  0 MMA sees P(g) complete   1 PV(g) issued      2 QK(g) issued      3 MMA starts waiting for V(g)
  4 S(g) ready (softmax)     5 max(g) done       6 P(g) written      7 softmax starts waiting for S(g)
  10 MMA starts waiting for K(g)   11 MMA sees V(g)   12 MMA sees K(g)

    python scripts/attn_trace.py [N]          # record and analyse
    python scripts/attn_trace.py --analyse F  # analyse a recorded dump

A -DPBS_ATTN_SPANS build instead sums, over every CTA, the clock64 time the
MMA warp and one thread per softmax group spend in each phase (no per-event
stores, so the product's timing); `--spans F` prints the per-block averages.
"""
import os
import sys

import numpy as np


def analyse(path):
    t = np.fromfile(path, dtype=np.uint64).reshape(16, 4096).astype(np.int64)
    mma_p, pv, qk, mma_w, sr, md, pd, sw = (t[i] for i in range(8))
    kw, vs, ks = t[10], t[11], t[12]
    if not (sr > 0).any():
        sys.exit("no events: rebuild with PBS_NVCC_EXTRA=-DPBS_ATTN_TRACE_EVENTS")
    g = np.arange(200, 3000)
    ok = np.all([x[g] > 0 for x in (mma_p, pv, mma_w, sr, md, pd, sw, vs)], axis=0) & (sr[g + 2] > 0) & (qk[g + 2] > 0)
    g = g[ok]
    med = lambda x: float(np.median(x))  # noqa: E731
    span = (sr[g[-1]] - sr[g[0]]) / max(1, g[-1] - g[0])
    print(f"CTA 0: {len(g)} blocks; mean period per block {span:.0f} clk (ideal 1024: MMA 2 x 512, exp 16384 / 16)")
    print("  softmax waits for S(g)                 ", med(sr[g] - sw[g]))
    print("  S(g) ready -> max done (load + max)    ", med(md[g] - sr[g]))
    print("  max done -> P(g) written (exp + store) ", med(pd[g] - md[g]))
    print("  P(g) written -> MMA sees it            ", med(mma_p[g] - pd[g]))
    print("  MMA waits for V(g)                     ", med(vs[g] - mma_w[g]))
    print("  MMA sees P(g) -> PV(g) second half out ", med(pv[g] - mma_p[g]))
    print("  PV(g) issued -> QK(g+2) issued         ", med(qk[g + 2] - pv[g]))
    print("  MMA waits for K(g+2)                   ", med(ks[g + 2] - kw[g + 2]))
    print("  QK(g+2) issued -> S(g+2) ready         ", med(sr[g + 2] - qk[g + 2]))
    print("  P(g) written -> S(g+2) ready           ", med(sr[g + 2] - pd[g]))


MMA_SPANS = ["wait V (+ O free)", "wait P half/full", "PV keys 0-63 issue", "PV keys 64-127 issue + commits",
             None, "wait K", "QK issue + commits", "item fetch + wait Q"]
SM_SPANS = ["visit / item", "wait S", "mask + load + max", "rescale", "exp + P store + arrive", "epilogue", "tail"]


def spans(path):
    t = np.fromfile(path, dtype=np.uint64)[:32].astype(np.float64)
    nb = t[4]
    print(f"MMA warp, per block ({nb:.0f} blocks over all CTAs), SM cycles:")
    for i, name in enumerate(MMA_SPANS):
        if name:
            print(f"  {name:34s} {t[i] / nb:8.0f}")
    print(f"  {'total':34s} {sum(t[i] for i in range(8) if MMA_SPANS[i]) / nb:8.0f}")
    for w in range(2):
        b = 16 + 8 * w
        n = t[b + 7]
        print(f"softmax group {w}, per own block ({n:.0f}):")
        for i, name in enumerate(SM_SPANS):
            print(f"  {name:34s} {t[b + i] / n:8.0f}")
        print(f"  {'total':34s} {sum(t[b + i] for i in range(7)) / n:8.0f}")


def record(n):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    import bench
    from paper_2510_21270_b200 import ops
    q, k, v = bench.make_inputs(torch, n, 0, 32, list(range(8)), "cuda")
    cfg = ops.make_config(block_size=128, segment_size=256, tau=0.9, strategy="key_permute")
    path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "attn_trace.bin")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    for _ in range(2):
        ops.pbs_attention(q, k, v, cfg, report=False)
    torch.cuda.synchronize()
    os.environ["PBS_ATTN_TRACE"] = path
    ops.pbs_attention(q, k, v, cfg, report=False)
    torch.cuda.synchronize()
    return path


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--analyse":
        analyse(sys.argv[2])
    elif len(sys.argv) > 1 and sys.argv[1] == "--spans":
        spans(sys.argv[2] if len(sys.argv) > 2 else record(131072))
    else:
        analyse(record(int(sys.argv[1]) if len(sys.argv) > 1 else 131072))
