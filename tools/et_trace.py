#!/usr/bin/env python3
"""Elasticity tensor-kernel timeline of CTA 0 (tools/build_trace.sh; development aid).
Slots: 0 producer inputs landed, 1 producer past EMPTY, 2 producer FULL,
3 compute past FULL, 4 GEMM done, 5 issuer wait_read done, 6 first barrier,
7 second barrier (slabs written)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1604_05872_b200 import femgpu  # noqa: E402

femgpu.LIB_PATH = os.path.join(ROOT, "tools", "libfemgpu_trace.so")
import torch  # noqa: E402

from paper_1604_05872_b200 import fe  # noqa: E402

cfg = fe.CONFIGS["c3"]
coords, coeffs = fe.cell_inputs(cfg)
form = femgpu.Form.from_config(cfg)
dev = torch.device("cuda:0")
x = torch.from_numpy(coords).to(dev)
c = torch.from_numpy(coeffs).to(dev)
out = torch.empty((coords.shape[0], cfg.n, cfg.n), dtype=torch.float64, device=dev)
for _ in range(3):
    form.assemble(x, c, out)
torch.cuda.synchronize()
L = femgpu.lib()
buf = (C.c_ulonglong * (256 * 8))()
L.femgpu_debug_trace_et(buf)
T = np.array(buf, dtype=np.float64).reshape(256, 8)
n = int((T[:, 3] > 0).sum())
t0 = T[0, 0]
print("tile prodIn prodEmpty prodFull | compFull gemm wait_read bar1 bar2 (cycles rel. to compFull)")
for it in range(10, 22):
    r = T[it]
    print(f"{it:3d} {(r[0]-t0)/1e3:8.2f} {(r[1]-t0)/1e3:8.2f} {(r[2]-t0)/1e3:8.2f} | {(r[3]-t0)/1e3:8.2f}"
          f" {r[4]-r[3]:6.0f} {r[5]-r[4]:6.0f} {r[6]-r[5]:6.0f} {r[7]-r[6]:6.0f}")
per = np.diff(T[5:n - 5, 3])
print(f"mean tile period {per.mean():.0f} cycles; gemm {np.mean(T[5:n-5,4]-T[5:n-5,3]):.0f},"
      f" wait_read {np.mean(T[5:n-5,5]-T[5:n-5,4]):.0f}, bar1 {np.mean(T[5:n-5,6]-T[5:n-5,5]):.0f},"
      f" epilogue+bar2 {np.mean(T[5:n-5,7]-T[5:n-5,6]):.0f}; producer per tile"
      f" {np.mean(np.diff(T[5:n-5,2])):.0f}, prod in-wait {np.mean(T[6:n-5,0]-T[5:n-6,2]):.0f}")
