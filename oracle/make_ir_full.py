#!/usr/bin/env python3
"""femopt's own optimized element kernels of the BASELINE configs, as IR.

TEST / MEASUREMENT INFRASTRUCTURE (container only: needs the reference built by
oracle/Makefile).  For every config and femopt plan of oracle/refkernel.py
(the plans the reference arm times), the config's IR (ir.py, built on E = 8
cells: the e-loop extent is a literal of the IR, the per-cell tables are
supplied at run time) goes through femopt_optimize (zero-skip off, SURVEY.md
§0.5b) and femopt_kernel_to_json (json_io.cpp:287-304).  The result is what a
femopt user hands to a backend: tools/bench_generic.py --femopt runs it on the
full BASELINE meshes through the generic B200 backend (femgpu_ir_*), and
tests/test_emit_cuda.py checks it against the hand-written kernels.

Writes tests/golden/ir_full/<cfg>_<plan>.json.gz (kernels + flop counts).
"""
import gzip
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
import refbridge as rb  # noqa: E402
import refkernel  # noqa: E402

from paper_1604_05872_b200 import fe, ir  # noqa: E402

E = 8
OUT = os.path.join(ROOT, "tests", "golden", "ir_full")


def make(cfg, plan):
    enc, th, _ = refkernel.PLANS[plan]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=E)
    res = {"config": cfg.name, "plan": plan, "encoding": enc, "memory_limit": th, "ncells": E,
           "kernels": []}
    for out, k in ir.build(cfg, coords, coeffs, tabs, enc):
        K = rb.Kernel(ir.dumps(k))
        raw = K.flops()
        t0 = time.time()
        Ko, rep = K.optimize(memory_limit=th, preeval=True, zero_skip=False)
        res["kernels"].append({"output": out, "flops_raw_per_cell": raw / E,
                               "flops_per_cell": Ko.flops() / E,
                               "ir": json.loads(Ko.to_json())})
        print(f"{cfg.name}/{plan} {out}: {raw / E:.0f} -> {Ko.flops() / E:.0f} flops/cell "
              f"({time.time() - t0:.1f}s)", flush=True)
    res["flops_per_cell"] = sum(k["flops_per_cell"] for k in res["kernels"])
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"{cfg.name}_{plan}.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(res, f, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


def main(names):
    for name in names:
        cfg = fe.CONFIGS[name]
        for plan in refkernel.plans_for(cfg):
            make(cfg, plan)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
