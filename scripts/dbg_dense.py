import os, sys
import torch
sys.path.insert(0, '.')
from paper_2510_21270_b200 import ops
cases = [(32, 8, 2048), (1, 1, 4096), (2, 1, 2048), (32, 8, 16384)]
for (hq, hkv, n) in cases:
    torch.manual_seed(2)
    d = 128
    q = torch.randn(hq, n, d, device="cuda").to(torch.bfloat16)
    k = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    out = ops.dense_causal_attention(q, k, v)
    g = hq // hkv
    ref = torch.nn.functional.scaled_dot_product_attention(q[None], k.repeat_interleave(g, 0)[None], v.repeat_interleave(g, 0)[None], is_causal=True)[0]
    err = (out.float() - ref.float()).abs().amax(-1)
    bad = (err > 0.05).nonzero()
    print(os.environ.get("PBS_ATTN_GRID"), hq, hkv, n, "max", round(err.max().item(), 3), "bad rows", bad.shape[0], bad[:6].tolist(),
          "blocks", torch.unique(bad[:, 1] // 128).tolist()[:12])
