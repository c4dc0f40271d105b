#!/usr/bin/env python3
"""Run one config's element-vector kernel a few times (target for ncu): prof_vector.py <cfg> [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = fe.CONFIGS[name]
coords, coeffs = fe.cell_inputs(cfg)
form = femgpu.Form.from_config(cfg)
dev = torch.device("cuda:0")
x = torch.from_numpy(coords).to(dev)
c = torch.from_numpy(coeffs).to(dev)
out = torch.empty((coords.shape[0], cfg.n), dtype=torch.float64, device=dev)
for _ in range(reps):
    form.assemble_vector(x, c, out)
torch.cuda.synchronize()
print("ok", name)
