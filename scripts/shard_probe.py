"""Debug: device time of rank 0's share (Llama 128K, or --model qwen at 256K) for
1/2/4/8-way head-parallel splits (pbs_shard_plan), run on one GPU without the
exchange: how close each rank's compute comes to 1/world of the whole."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_21270_b200 import ops  # noqa: E402

model = sys.argv[sys.argv.index("--model") + 1] if "--model" in sys.argv else "llama"
bench.HQ, bench.HKV, bench.N, bench.PREFIX = bench.MODELS[model]
cfg = ops.make_config()
n = bench.N
base = None
for world in (1, 2, 4, 8):
    worst = 0.0
    for rank in range(world):
        s = ops.shard_plan(bench.HQ, bench.HKV, n, 128, 128, world, rank)
        q, k, v = bench.make_inputs(torch, n, s["head_begin"], s["head_end"], list(range(s["kv_begin"], s["kv_end"])),
                                    "cuda")
        out = torch.zeros(bench.HQ, n, 128, dtype=torch.bfloat16, device="cuda")
        for _ in range(2):
            ops.attention_shard(q, k, v, bench.HQ, bench.HKV, cfg, world, rank, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            ops.attention_shard(q, k, v, bench.HQ, bench.HKV, cfg, world, rank, out)
        e1.record()
        torch.cuda.synchronize()
        worst = max(worst, e0.elapsed_time(e1) / 3)
        del q, k, v, out
        if world == 8 and rank >= 1 and model == "llama":
            break  # Llama's ranks are identical by construction
    base = base or worst
    print(f"{model} world {world}: slowest rank {worst:.2f} ms, {base / world / worst * 100:.1f}% of linear")
