"""Debug: the device pipeline over 4-head chunks (one KV group each, as the host
entry runs it) vs one launch over all 32 heads, no host copies (C3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2510_21270_b200 import ops
q, k, v = bench.make_inputs(torch, 131072, 0, 32, list(range(8)), "cuda")
cfg = ops.make_config()
def timed(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
full = timed(lambda: ops.pbs_attention(q, k, v, cfg, report=False))
chunks = [(q[4 * c:4 * c + 4].contiguous(), k[c:c + 1].contiguous(), v[c:c + 1].contiguous()) for c in range(8)]
ch = timed(lambda: [ops.pbs_attention(a, b, c_, cfg, report=False) for a, b, c_ in chunks])
r = ops.pbs_attention(q, k, v, cfg).report
rs = [ops.pbs_attention(a, b, c_, cfg).report for a, b, c_ in chunks]
print(f"full launch {full:.2f} ms, 8 chunks {ch:.2f} ms")
for key in ("estimate_us", "permute_us", "select_us", "attention_us"):
    print(key, round(r[key] / 1e3, 2), "vs chunks", round(sum(x[key] for x in rs) / 1e3, 2))
if os.environ.get("PBS_CHUNK_ONCE"):
    pass
