import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import bench
from paper_2510_21270_b200 import ops
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = bench.make_inputs(torch, n, 0, 32, list(range(8)), "cuda")
hq_, hk_, hv_ = (x.cpu().pin_memory() for x in (q, k, v))
hout = torch.empty_like(hq_).pin_memory()
cfg = ops.make_config()
for _ in range(3):
    ops.pbs_attention_host(hq_, hk_, hv_, cfg, out=hout, report=False)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); ops.pbs_attention_host(hq_, hk_, hv_, cfg, out=hout, report=False); ts.append((time.perf_counter() - t0) * 1e3)
print("e2e", [round(x, 2) for x in ts])
os.environ["PBS_HOST_TRACE"] = "1"
ops.pbs_attention_host(hq_, hk_, hv_, cfg, out=hout, report=False)
