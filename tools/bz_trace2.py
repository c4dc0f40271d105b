#!/usr/bin/env python3
"""Burgers pipeline timeline of CTA 0 for the interleaved schedule (BZ_SCHED 1;
needs tools/build_trace.sh; development aid).
Slots: 0 producer inputs landed, 1 producer past EMPTY, 2 producer A1 done,
3 producer FULL, 4 compute past FULL, 6..11 off-diagonal block b written (before
its GEMM-2 chunk), 5 GEMM-2 done, 12..14 diagonal blocks, 16/19 first/last ring
stage landed, 15 issuer cycles waiting for slabs full, 18 issuer cycles in
wait_group.read, 17 next-tile ring refill issued."""
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
k = lambda v: v / 1e3  # noqa: E731
print(f"tiles traced {ntile}  (kcycles; columns relative to the tile's compute start)")
print("tile  start | prodIn prodA1 prodFull | off1..off6 (end of block) | gemm2done | diag1..3 | ring0 ring16 | issuerFullWait readWait")
for it in range(min(ntile, 14)):
    r = T[it]
    s = r[4]
    offs = " ".join(f"{k(r[6 + b] - s):5.1f}" for b in range(6))
    diags = " ".join(f"{k(r[12 + b] - s):5.1f}" for b in range(3))
    print(f"{it:3d} {k(s - t0):7.1f} | {k(r[0]-s):6.1f} {k(r[2]-s):6.1f} {k(r[3]-s):6.1f} | {offs} | {k(r[5]-s):5.1f} |"
          f" {diags} | {k(r[16]-s):5.1f} {k(r[19]-s):5.1f} | {k(r[15]):5.2f} {k(r[18]):5.2f}")
per = np.diff(T[:ntile, 4])[2:]
print(f"mean tile period {k(per.mean()):.2f} kcycles; producer A1 {k(np.mean(T[2:ntile,2]-T[2:ntile,1])):.2f},"
      f" A2 {k(np.mean(T[2:ntile,3]-T[2:ntile,2])):.2f}; issuer full-wait {k(np.mean(T[2:ntile,15])):.2f},"
      f" read-wait {k(np.mean(T[2:ntile,18])):.2f}")
