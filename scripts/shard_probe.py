"""Debug: device time of one rank's share (Llama 128K) for 1/2/4/8-way head splits on one GPU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2510_21270_b200 import ops
cfg = ops.make_config()
for world in (1, 2, 4, 8):
    q0, q1, kv, _ = bench.shard_of(0, world)
    q, k, v = bench.make_inputs(torch, 131072, q0, q1, kv, "cuda")
    ws = ops.workspace(ops.workspace_size(q, k, cfg))
    out = torch.empty_like(q)
    for _ in range(2):
        ops.pbs_attention(q, k, v, cfg, report=False, out=out, return_perms=False, ws=ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5):
        ops.pbs_attention(q, k, v, cfg, report=False, out=out, return_perms=False, ws=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    r = ops.pbs_attention(q, k, v, cfg, report=True, out=out, return_perms=False, ws=ws).report
    print(f"world {world}: {q1 - q0} heads {ms:.2f} ms (1-GPU time / world: see world 1)",
          {kk: round(r[kk] / 1e3, 2) for kk in ("estimate_us", "permute_us", "select_us", "attention_us")})
    del q, k, v, out
