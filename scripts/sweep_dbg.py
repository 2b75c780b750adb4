import os, sys, torch
sys.path.insert(0, '.')
from paper_2510_21270_b200 import ops
HQ, HKV, D, B = 32, 8, 128, 128
n = 65536; t = n // B
torch.manual_seed(0)
q = torch.randn(HQ, n, D, device="cuda").to(torch.bfloat16)
k = torch.randn(HKV, n, D, device="cuda").to(torch.bfloat16)
v = torch.randn(HKV, n, D, device="cuda").to(torch.bfloat16)
ii = torch.arange(t, device="cuda")[:, None]; jj = torch.arange(t, device="cuda")[None, :]
for keep in (1, 2, 4):
    sel = (((ii * 31 + jj * 17) % 20) < keep) & (jj <= ii); sel |= ii == jj
    cnt = sel.sum(1).to(torch.int32)
    order = torch.where(sel, jj.expand(t, t), torch.full_like(jj.expand(t, t), t)).sort(1).values
    kv_idx = order.to(torch.int32).clamp_max(t - 1).unsqueeze(0).expand(HQ, t, t).contiguous()
    kv_cnt = cnt.unsqueeze(0).expand(HQ, t).contiguous()
    ts = []
    for r in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ops.attention_block_sparse(q, k, v, B, kv_idx, kv_cnt, check_status=False); e1.record()
        torch.cuda.synchronize(); ts.append(round(e0.elapsed_time(e1), 2))
    print(keep, ts)
print("back-to-back, events between launches, no host sync:")
for keep in (1, 2):
    sel = (((ii * 31 + jj * 17) % 20) < keep) & (jj <= ii); sel |= ii == jj
    cnt = sel.sum(1).to(torch.int32)
    order = torch.where(sel, jj.expand(t, t), torch.full_like(jj.expand(t, t), t)).sort(1).values
    kv_idx = order.to(torch.int32).clamp_max(t - 1).unsqueeze(0).expand(HQ, t, t).contiguous()
    kv_cnt = cnt.unsqueeze(0).expand(HQ, t).contiguous()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(31)]
    import time
    t0 = time.perf_counter()
    for r in range(30):
        evs[r].record(); ops.attention_block_sparse(q, k, v, B, kv_idx, kv_cnt, check_status=False)
    evs[30].record(); host = time.perf_counter() - t0
    torch.cuda.synchronize()
    print(keep, "host enqueue s", round(host, 3), [round(evs[r].elapsed_time(evs[r + 1]), 2) for r in range(30)])
