"""Debug (-DPBS_ATTN_EVENTS build): per-CTA start / end times of one attention
launch, for the full C3 problem and for one 4-head group (the host entry's chunk)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2510_21270_b200 import ops
q, k, v = bench.make_inputs(torch, 131072, 0, 32, list(range(8)), "cuda")
cfg = ops.make_config()
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "tail.bin")
for name, args in (("full", (q, k, v)), ("chunk", (q[:4].contiguous(), k[:1].contiguous(), v[:1].contiguous()))):
    for _ in range(2):
        ops.pbs_attention(*args, cfg, report=False)
    torch.cuda.synchronize()
    os.environ["PBS_ATTN_TRACE"] = path
    ops.pbs_attention(*args, cfg, report=False)
    torch.cuda.synchronize()
    del os.environ["PBS_ATTN_TRACE"]
    t = np.fromfile(path, dtype=np.uint64).astype(np.int64)
    end = t[32 + 16384:32 + 16384 + 148]
    st = t[32 + 16384 + 512:32 + 16384 + 512 + 148]
    t0 = st.min()
    e = np.sort(end - t0) / 1e3
    print(f"{name}: start spread {(st.max() - t0) / 1e3:.1f} us; end times (us after first start): "
          f"min {e[0]:.0f} p10 {e[14]:.0f} p50 {e[74]:.0f} p90 {e[133]:.0f} max {e[-1]:.0f}")
