"""Pinned host<->device copy bandwidth on this box: H2D and D2H alone and concurrently
(the ceiling of bench.py e2e, which moves ~2.88 GB in and ~0.91 GB out per C3 step)."""
import torch, time
n = 2_880_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(910_000_000, dtype=torch.uint8).pin_memory()
d2 = torch.empty(910_000_000, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); a = time.perf_counter() - t
t = time.perf_counter(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); b = time.perf_counter() - t
t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); c = time.perf_counter() - t
print(f"H2D {n/a/1e9:.1f} GB/s ({a*1e3:.1f} ms)  D2H {910e6/b/1e9:.1f} GB/s ({b*1e3:.1f} ms)  both {c*1e3:.1f} ms")
