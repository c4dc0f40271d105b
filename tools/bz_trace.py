#!/usr/bin/env python3
"""Burgers pipeline timeline of CTA 0 (needs tools/build_trace.sh; development aid).
Slots: 0 producer inputs landed, 1 producer past EMPTY, 2 producer A1 done (A2 start),
3 producer FULL, 4 compute past FULL, 5 GEMM-2 done, 6..14 (c,d) barriers,
15 issuer cycles in wait_group.read."""
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

cfg = fe.CONFIGS["c5"]
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
buf = (C.c_ulonglong * (128 * 20))()
L.femgpu_debug_trace(buf)
T = np.array(buf, dtype=np.float64).reshape(128, 20)
ntile = int((T[:, 4] > 0).sum())
t0 = T[0, 0]
print(f"tiles traced {ntile}")
print("tile  prodIn prodEmp prodA2 prodFull | compFull gemm2 | steps(9) ... | issuer_wait")
for it in range(min(ntile, 12)):
    r = T[it]
    steps = " ".join(f"{(r[6 + k] - r[5 + k if k else 5]) / 1e3:5.2f}" for k in range(9))
    print(f"{it:3d} {(r[0]-t0)/1e3:8.1f} {(r[1]-t0)/1e3:7.1f} {(r[2]-t0)/1e3:7.1f} {(r[3]-t0)/1e3:7.1f} |"
          f" {(r[4]-t0)/1e3:7.1f} {(r[5]-r[4])/1e3:5.2f} | {steps} | {r[15]/1e3:6.2f}")
per_tile = np.diff(T[:ntile, 4])
print(f"mean tile period (kcycles) {per_tile[2:].mean()/1e3:.2f}; gemm2 {np.mean(T[2:ntile,5]-T[2:ntile,4])/1e3:.2f};"
      f" steps {np.mean(T[2:ntile,14]-T[2:ntile,5])/1e3:.2f}; producer A1 {np.mean(T[2:ntile,2]-T[2:ntile,1])/1e3:.2f},"
      f" A2 {np.mean(T[2:ntile,3]-T[2:ntile,2])/1e3:.2f}; issuer wait {np.mean(T[2:ntile,15])/1e3:.2f}")
print("ring (per tile, kcycles after compFull): first stage landed, last stage landed; issuer at tile end: wait_read1 start/end (after the tile's last step)")
for it in range(2, min(ntile, 10)):
    r = T[it]
    print(f"{it:3d} first {(r[16]-r[4])/1e3:6.2f} last {(r[19]-r[4])/1e3:6.2f} gemm2 {(r[5]-r[4])/1e3:6.2f} | wait_read1 {(r[17]-r[14])/1e3:6.2f} -> {(r[18]-r[14])/1e3:6.2f}  next compFull {(T[it+1][4]-r[14])/1e3:6.2f}")
