import os, sys
import torch
sys.path.insert(0, '.')
from paper_2510_21270_b200 import ops
torch.manual_seed(2)
for (hq, hkv, n) in [(1, 1, 1024), (2, 1, 1024), (1, 1, 2048), (2, 1, 2048)]:
    d = 128
    q = torch.randn(hq, n, d, device="cuda").to(torch.bfloat16)
    k = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(hkv, n, d, device="cuda").to(torch.bfloat16)
    g = hq // hkv
    kk, vv = k.repeat_interleave(g, 0).float(), v.repeat_interleave(g, 0).float()
    s = (q.float() @ kk.transpose(1, 2)) / d ** 0.5
    mask = torch.ones(n, n, device="cuda").tril().bool()
    ref = torch.softmax(s.masked_fill(~mask, float("-inf")), -1) @ vv
    for trial in range(3):
        out = ops.dense_causal_attention(q, k, v).float()
        err = (out - ref).abs().amax(-1)
        bad = (err > 0.03).nonzero()
        msg = f"{os.environ.get('PBS_ATTN_GRID')} {hq} {n} trial {trial} max {err.max().item():.3f} bad {bad.shape[0]}"
        if bad.shape[0]:
            h, r = bad[0].tolist()
            qb = r // 128
            # which hypothesis matches: attention over blocks [0, qb] minus one block?
            best = None
            for drop in range(qb + 1):
                keep = torch.zeros(n, dtype=torch.bool, device="cuda")
                keep[:(qb + 1) * 128] = True
                keep[drop * 128:(drop + 1) * 128] = False
                m2 = mask[r] & keep
                o2 = torch.softmax(s[h, r].masked_fill(~m2, float("-inf")), -1) @ vv[h]
                e2 = (out[h, r] - o2).abs().max().item()
                if best is None or e2 < best[0]:
                    best = (e2, drop)
            msg += f" | first bad (h {h}, row {r}, qb {qb}) err {err[h, r].item():.3f}; best 'missing block' {best[1]} err {best[0]:.4f}"
            msg += f" | bad rows in qb: {sorted(set((x // 128) for x in bad[:, 1].tolist()))[:10]} rows%128 {sorted(set(x % 128 for x in bad[:, 1].tolist()))[:16]}"
        print(msg)
