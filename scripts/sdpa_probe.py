"""Debug: torch SDPA (cuDNN backend) dense causal attention on the C3 shapes
(32 q / 8 kv heads, N = 131072 or --seq, d = 128, bf16), for an ncu capture
of the outside anchor next to our own attention kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

n = int(sys.argv[sys.argv.index("--seq") + 1]) if "--seq" in sys.argv else 131072
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, 32, n, 128, device="cuda", generator=g, dtype=torch.bfloat16)
k = torch.randn(1, 8, n, 128, device="cuda", generator=g, dtype=torch.bfloat16)
v = torch.randn(1, 8, n, 128, device="cuda", generator=g, dtype=torch.bfloat16)
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    for _ in range(2):
        torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
torch.cuda.synchronize()
print("ok")
