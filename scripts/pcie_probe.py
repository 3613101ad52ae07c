"""Pinned host <-> device copy bandwidth (one direction, and both at once):
the bound for bench.py's e2e figure.  python scripts/pcie_probe.py"""
import torch, time
n = 4 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d1.copy_(h1, non_blocking=True)),
                 ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(name, n / dt / 1e9, "GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("duplex", n / dt / 1e9, "GB/s each way")
