#!/usr/bin/env python3
"""Run femopt's c2 tensor plan once through the generic backend's GEMM mapping (ncu target)."""
import gzip, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1604_05872_b200 import emit_cuda, fe, ir  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c2_tensor"
d = json.load(gzip.open(os.path.join(ROOT, "tests", "golden", "ir_full", case + ".json.gz"), "rt"))
cfg = fe.CONFIGS[d["config"]]
E = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.ncells
coords, coeffs = fe.cell_inputs(cfg, ncells=E)
dev = torch.device("cuda:0")
et = {k: torch.from_numpy(v).to(dev) for k, v in ir.e_tables(cfg, coords, coeffs).items()}
for kk in d["kernels"][:1]:
    k = kk["ir"]
    K = emit_cuda.IRKernel(k, "gemm")
    inputs = {n: et[n] if n in et else torch.tensor(np.asarray(k["tables"][n]["values"]), device=dev)
              for n in K.inputs}
    (o,) = K.outputs
    out = torch.zeros(K.size(0, o, E), dtype=torch.float64, device=dev)
    for _ in range(2):
        K.run({o: out}, inputs, k.get("constants", {}), E)
    torch.cuda.synchronize()
print("ok")
