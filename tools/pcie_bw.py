#!/usr/bin/env python3
"""Pinned host<->device copy bandwidth (context for the e2e numbers)."""
import time
import torch

n = 1 << 28  # 2 GiB of float64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(name, round(3 * n * 8 / (time.perf_counter() - t) / 1e9, 1), "GB/s")
