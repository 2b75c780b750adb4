"""Debug: wall time of the host-buffer entry at C3 (128K), with / without the report."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2510_21270_b200 import ops
q, k, v = bench.make_inputs(torch, 131072, 0, 32, list(range(8)), "cuda")
hq_, hk_, hv_ = (x.cpu().pin_memory() for x in (q, k, v))
hout = torch.empty_like(hq_).pin_memory()
cfg = ops.make_config()
for rep in (True, False, True):
    for _ in range(2):
        ops.pbs_attention_host(hq_, hk_, hv_, cfg, out=hout, report=rep)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        ops.pbs_attention_host(hq_, hk_, hv_, cfg, out=hout, report=rep)
        ts.append((time.perf_counter() - t0) * 1e3)
    print("report", rep, [round(x, 1) for x in ts])
r = ops.pbs_attention_host(hq_, hk_, hv_, cfg, out=hout, report=True).report
print("host-entry stage sums (ms):", {k: round(r[k] / 1e3, 2) for k in ("estimate_us", "permute_us", "select_us", "attention_us")})
d = ops.pbs_attention(q, k, v, cfg).report
print("device-entry stages (ms):  ", {k: round(d[k] / 1e3, 2) for k in ("estimate_us", "permute_us", "select_us", "attention_us")})
# one traced call (PBS_HOST_TRACE: CUDA-event timeline of the three streams, on stderr)
os.environ["PBS_HOST_TRACE"] = "1"
ops.pbs_attention_host(hq_, hk_, hv_, cfg, out=hout, report=False)
