"""How much K/V traffic a two-query-tiles-per-CTA attention would save at C3:
for every head, pair query blocks (2s, 2s + 1) (one segment) and compare the
union of their selected key blocks with the two lists' total.

    python scripts/pair_union.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_21270_b200 import ops  # noqa: E402

n = 131072
q, k, v = bench.make_inputs(torch, n, 0, 32, list(range(8)), "cuda")
cfg = ops.make_config(block_size=128, segment_size=256, tau=0.9, strategy="key_permute")
res = ops.pbs_attention(q, k, v, cfg, report=True, return_perms=True)
m = res.mask.bool()  # [hq, t, t]
a, b = m[:, 0::2], m[:, 1::2]
both = int((a & b).sum())
union = int((a | b).sum())
total = int(m.sum())
# adjacent q heads of one KV group share K only when pi matches: report both pairings
print(json.dumps({"selected": total, "pair_union": union, "pair_both": both,
                  "kv_tiles_saved_frac": 1 - union / total, "tensor_work": total,
                  "mean_list": total / (m.shape[0] * m.shape[1])}))
