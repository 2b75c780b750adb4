"""Debug: pinned H2D / D2H bandwidth alone and concurrent (the host entry's transfer budget)."""
import torch, time
n = 1 << 30
h_in = torch.empty(3 * n // 2, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(3 * n // 2, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3
for _ in range(2):
    a = t(lambda: d_in.copy_(h_in, non_blocking=True))
    b = t(lambda: h_out.copy_(d_out, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    c = t(both)
    print(f"H2D 1.5 GiB {a:.1f} ms ({1.5*1.074/a*1e3:.0f} GB/s)  D2H 1 GiB {b:.1f} ms ({1.074/b*1e3:.0f} GB/s)  concurrent {c:.1f} ms")
