#!/usr/bin/env python3
"""femgpu_assemble_host throughput (pinned host buffers, H2D + kernel + D2H) for one
config: e2e_time.py <cfg> (development aid; FEMGPU_LIB selects an A/B build)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

if os.environ.get("FEMGPU_LIB"):
    femgpu.LIB_PATH = os.environ["FEMGPU_LIB"]
cfg = fe.CONFIGS[sys.argv[1]]
coords, coeffs = fe.cell_inputs(cfg)
E = coords.shape[0]
form = femgpu.Form.from_config(cfg)
hx = torch.from_numpy(coords).pin_memory()
hc = torch.from_numpy(coeffs).pin_memory()
hA = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64).pin_memory()
form.assemble_host_ptr(E, hx.data_ptr(), hc.data_ptr(), hA.data_ptr())
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    form.assemble_host_ptr(E, hx.data_ptr(), hc.data_ptr(), hA.data_ptr())
    ts.append(time.perf_counter() - t0)
t = sorted(ts)[2]
print(f"{sys.argv[1]} e2e {E / t:.3g} elem/s, {(hx.numel() + hc.numel() + hA.numel()) * 8 / t / 1e9:.1f} GB/s")
