"""ncu helper: one full pipeline launch, then the 8 per-group chunks (C3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2510_21270_b200 import ops
q, k, v = bench.make_inputs(torch, 131072, 0, 32, list(range(8)), "cuda")
cfg = ops.make_config()
ops.pbs_attention(q, k, v, cfg, report=False)
chunks = [(q[4 * c:4 * c + 4].contiguous(), k[c:c + 1].contiguous(), v[c:c + 1].contiguous()) for c in range(8)]
for a, b, c_ in chunks:
    ops.pbs_attention(a, b, c_, cfg, report=False)
torch.cuda.synchronize()
