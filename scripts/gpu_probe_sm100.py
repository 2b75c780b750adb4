"""Quick standalone probe of the tcgen05 attention kernel (run under `timeout`).

python scripts/gpu_probe_sm100.py   -> prints max errors vs SDPA and vs the SIMT path
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_21270_b200 import ops  # noqa: E402


def sdpa_causal(q, k, v):
    g = q.shape[0] // k.shape[0]
    kk = k.float().repeat_interleave(g, 0)
    vv = v.float().repeat_interleave(g, 0)
    return torch.nn.functional.scaled_dot_product_attention(q.float()[None], kk[None], vv[None], is_causal=True)[0]


def main():
    torch.manual_seed(0)
    for (hq, hkv, n) in [(1, 1, 128), (1, 1, 256), (2, 1, 1024), (4, 2, 1000), (8, 2, 4096)]:
        q = torch.randn(hq, n, 128, device="cuda").to(torch.bfloat16)
        k = torch.randn(hkv, n, 128, device="cuda").to(torch.bfloat16)
        v = torch.randn(hkv, n, 128, device="cuda").to(torch.bfloat16)
        out = ops.dense_causal_attention(q, k, v)
        torch.cuda.synchronize()
        ref = sdpa_causal(q, k, v)
        err = (out.float() - ref).abs()
        print(f"dense hq={hq} hkv={hkv} n={n}: max {err.max().item():.3e} mean {err.mean().item():.3e}", flush=True)
    # sparse pipeline: tcgen05 vs SIMT path on the same selection
    hq, hkv, n = 4, 2, 2048
    q = torch.randn(hq, n, 128, device="cuda")
    k = torch.randn(hkv, n, 128, device="cuda")
    u = torch.nn.functional.normalize(torch.randn(128, device="cuda"), dim=0)
    q += 128 ** 0.5 * u
    k[:, torch.randperm(n)[:16]] += 20 * u
    q, k, v = q.to(torch.bfloat16), k.to(torch.bfloat16), torch.randn(hkv, n, 128, device="cuda").to(torch.bfloat16)
    for strategy in ["key_permute", "none", "query_permute", "both"]:
        cfg = ops.make_config(strategy=strategy, segment_size=0 if strategy == "none" else 256)
        a = ops.pbs_attention(q, k, v, cfg)
        os.environ["PBS_FORCE_SIMT"] = "1"
        b = ops.pbs_attention(q, k, v, cfg)
        del os.environ["PBS_FORCE_SIMT"]
        torch.cuda.synchronize()
        err = (a.output.float() - b.output.float()).abs()
        print(f"sparse {strategy}: density {a.report['block_density']:.3f} tc-vs-simt max {err.max().item():.3e} "
              f"mean {err.mean().item():.3e} masks equal {torch.equal(a.mask, b.mask)}", flush=True)


if __name__ == "__main__":
    main()
