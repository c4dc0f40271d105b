#!/usr/bin/env python3
"""Generate tests/golden/ fixtures and the reference-arm sources from the reference.

TEST INFRASTRUCTURE -- runs only where /root/reference exists (the build
container).  For every BASELINE config it

  1. emits femopt's optimized element kernels (oracle/refkernel.py) for the
     bench's reference arm (chunk = 512 cells) and for the fixture (chunk =
     the fixture's cell count);
  2. runs the fixture cells through (a) the compiled optimized emitted C and
     (b) femopt's interpreter on the *raw* IR (proj/src/interp.cpp:125-154);
  3. writes tests/golden/<cfg>.npz (tables, coords, coeffs, both results) and
     tests/golden/<cfg>.json (flop counts, agreement, plans).

Usage: python oracle/make_golden.py [c1 c2 ...]   (default: all five)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import refbridge as rb  # noqa: E402
import refkernel as rk  # noqa: E402
from paper_1604_05872_b200 import fe, ir  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
# fixture cells per config, and how many of them the (slow) interpreter checks
CELLS = {"c1": (512, 512), "c2": (128, 8), "c3": (128, 16), "c4": (64, 4), "c5": (32, 4)}


def frob_rel(a, b):
    a = a.reshape(a.shape[0], -1)
    b = b.reshape(b.shape[0], -1)
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)))


def main(names):
    os.makedirs(GOLDEN, exist_ok=True)
    for name in names:
        cfg = fe.CONFIGS[name]
        E, Ei = CELLS[name]
        tabs = fe.tables(cfg)
        coords, coeffs = fe.cell_inputs(cfg, ncells=E)
        meta = {"config": name, "description": cfg.description, "cells": E,
                "interp_cells": Ei, "plans": {}}
        results = {}
        for plan in rk.plans_for(cfg):
            if not rk.available(cfg, plan, rk.CHUNK):
                rk.emit(cfg, plan, rk.CHUNK)
            m = rk.emit(cfg, plan, E)
            K = rk.RefKernel(cfg, plan, E)
            t = time.time()
            results[plan] = K.run(coords, coeffs, 1)
            meta["plans"][plan] = {
                "flops_per_cell": m["flops_per_cell"],
                "flops_raw_per_cell": sum(k["flops_raw_per_cell"] for k in m["kernels"]),
                "status": [k["status"] for k in m["kernels"]],
                "run_seconds": round(time.time() - t, 3)}
        # femopt's interpreter on the raw IR for the first Ei cells
        t = time.time()
        blocks = {o: rb.interpret(ir.dumps(k), o)
                  for o, k in ir.build(cfg, coords[:Ei], coeffs[:Ei], tabs, "ufl")}
        A_interp = ir.assemble_blocks(cfg, blocks, Ei)
        meta["interp_seconds"] = round(time.time() - t, 2)
        A = results["quad"]
        meta["emitted_vs_interp_frob_rel"] = frob_rel(A[:Ei], A_interp)
        for plan, R in results.items():
            meta["plans"][plan]["vs_quad_frob_rel"] = frob_rel(R, A)
        np.savez_compressed(
            os.path.join(GOLDEN, f"{name}.npz"), W=tabs.W, B=tabs.B, D=tabs.D, P=tabs.P, X=tabs.X,
            coords=coords, coeffs=coeffs, A=A, A_interp=A_interp,
            **{f"A_{p}": r for p, r in results.items() if p != "quad"})
        with open(os.path.join(GOLDEN, f"{name}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(fe.CONFIGS))
