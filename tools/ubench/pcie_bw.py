"""Pinned host <-> device copy bandwidth on this box (the e2e lines' copy bound)."""
import torch
n = 1 << 27  # 1 GiB of fp64
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
for name, f in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {n * 8 / ms / 1e6:.1f} GB/s ({ms:.1f} ms per GiB)")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"both directions concurrently: {2 * n * 8 / (e0.elapsed_time(e1) / 5) / 1e6:.1f} GB/s total")
