"""Debug: record CTA 0's attention pipeline timeline (PBS_ATTN_TRACE) on the
C3 bench workload and print per-block phase latencies (SM clocks)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_21270_b200 import ops  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
dense = len(sys.argv) > 2 and sys.argv[2] == "dense"
q, k, v = bench.make_inputs(torch, n, 0, 32, list(range(8)), "cuda")
cfg = ops.make_config(block_size=128, segment_size=256, tau=0.9, strategy="key_permute")
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "attn_trace.bin")
os.makedirs(os.path.dirname(path), exist_ok=True)
for _ in range(2):
    (ops.dense_causal_attention(q, k, v) if dense else ops.pbs_attention(q, k, v, cfg, report=False))
torch.cuda.synchronize()
os.environ["PBS_ATTN_TRACE"] = path
(ops.dense_causal_attention(q, k, v) if dense else ops.pbs_attention(q, k, v, cfg, report=False))
torch.cuda.synchronize()
t = np.fromfile(path, dtype=np.uint64).reshape(12, 4096).astype(np.int64)
names = ["mma_sees_p0", "mma_sees_p1", "pv_issue0", "pv_issue1", "qk_issue0", "qk_issue1", "s_ready0", "s_ready1",
         "p_done0", "p_done1", "max_done0", "max_done1"]
t0 = t[t > 0].min()
lo, hi = 100, 1500
sr, pd, md, qk, pv, ms, pvd = (t[6], t[8], t[10], t[4], t[2], t[0], t[3])
b = np.arange(lo, hi)
ok = (sr[b] > 0) & (pd[b] > 0) & (qk[b] > 0) & (pv[b] > 0) & (ms[b] > 0) & (sr[b + 2] > 0)
b = b[ok]
med = lambda x: float(np.median(x))
print(f"CTA 0: blocks {len(b)}   (order per block b: QK(b+1) issued, PV(b-1)... see below)")
print("  softmax: S(b) ready -> max done      ", med(md[b] - sr[b]))
print("  softmax: max done -> P(b) written    ", med(pd[b] - md[b]))
print("  P(b) written -> MMA sees P(b)        ", med(ms[b] - pd[b]))
print("  MMA sees P(b) -> PV(b) issued        ", med(pv[b] - ms[b]))
print("  PV(b) issued -> PV(b) complete       ", med(pvd[b] - pv[b]))
print("  PV(b) issued -> QK(b+2) issued       ", med(qk[b + 2] - pv[b]))
print("  QK(b+2) issued -> S(b+2) ready       ", med(sr[b + 2] - qk[b + 2]))
print("  PV(b) complete -> S(b+2) ready       ", med(sr[b + 2] - pvd[b]))
print("  P(b) written -> S(b+1) ready         ", med(sr[b + 1] - pd[b]))
print("  period S(b) -> S(b+1)                ", med(sr[b + 1] - sr[b]))
kf, vf, top = t[1], t[5], t[7]
print("  PV(b) issued -> MMA at QK(b+2)       ", med(top[b + 2] - pv[b]))
print("  MMA at QK(b+2) -> K(b+2) present     ", med(kf[b + 2] - top[b + 2]))
print("  K(b+2) present -> QK(b+2) issued     ", med(qk[b + 2] - kf[b + 2]))
print("  MMA sees P(b) -> V(b) present        ", med(vf[b] - ms[b]))
lt, vg = t[9], t[11]
print("  P(b) written -> loop top (b+1)       ", med(lt[b + 1] - pd[b]))
print("  loop top -> visit entry (b+1)        ", med(vg[b + 1] - lt[b + 1]))
print("  visit entry -> S(b+1) passed         ", med(sr[b + 1] - vg[b + 1]))
print("  QK(b+1) issued -> PV(b) complete (>0: QK done before)", med(pvd[b] - qk[b + 1]))
