"""PCIe floor for bench.py e2e: 2.5 GB pinned H2D alone, then concurrently with a
0.83 GB D2H (the per-step transfer volumes of a C3 xsp_run_host call)."""
import torch, time
n = 2_500_000_000
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print("H2D GB/s", n / ms / 1e6)
d2 = torch.empty(n // 3, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n // 3, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
e0.record()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record()
torch.cuda.synchronize()
print("H2D 2.5 GB + D2H 0.83 GB concurrent ms", e0.elapsed_time(e1))
