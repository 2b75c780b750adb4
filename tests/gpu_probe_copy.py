"""Probe pinned host <-> device copy bandwidth on this box (context for the e2e number)."""
import time

import torch

x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(2):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
h2d = 5 * (1 << 30) / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(5):
    x.copy_(y, non_blocking=True)
torch.cuda.synchronize()
d2h = 5 * (1 << 30) / (time.perf_counter() - t) / 1e9
print(f"pinned H2D {h2d:.1f} GB/s  D2H {d2h:.1f} GB/s")
