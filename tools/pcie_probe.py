#!/usr/bin/env python3
"""Raw PCIe probe: pinned H2D, D2H and simultaneous H2D+D2H copy bandwidth (the e2e ceiling)."""
import torch
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n // 4, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    print(f"{name}: {n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter() - t0
print(f"H2D {n/1e9:.2f} GB + D2H {n/4/1e9:.2f} GB concurrently: {t*1e3:.1f} ms -> H2D {n/t/1e9:.1f} GB/s")
