#!/usr/bin/env python3
"""Throughput of the generic IR backend (emit_cuda) on the BASELINE meshes.

The raw femopt IR of each config (ir.py, built on 4 cells for its code) is
compiled by emit_cuda and run on the full config mesh with the per-cell
e-tables supplied at run time; device-timed with CUDA events.  The hand-written
kernels (bench.py) are the fast path; this is the thread-per-cell generic one.
usage: bench_generic.py [cfg ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1604_05872_b200 import emit_cuda, fe, ir  # noqa: E402


def e_tables(cfg, coords, coeffs):
    """SoA per-cell tables of ir.py's naming for the whole mesh."""
    E = coords.shape[0]
    x = coords.reshape(E, 4, 3)
    t = {f"x{v}{c}": x[:, v, c] for v in range(4) for c in range(3)}
    ns = cfg.ns
    if cfg.kind == fe.HELMHOLTZ:
        t.update({f"f{m:02d}": coeffs[:, m] for m in range(coeffs.shape[1])})
    elif cfg.kind == fe.ELASTICITY:
        t.update({f"mu{m}": coeffs[:, m] for m in range(4)})
        t.update({f"lam{m}": coeffs[:, 4 + m] for m in range(4)})
    elif cfg.kind == fe.HYPERELASTICITY:
        t.update({f"w{c}{m:02d}": coeffs[:, c * ns + m] for c in range(3) for m in range(ns)})
        t.update({f"mu{m}": coeffs[:, 3 * ns + m] for m in range(4)})
        t.update({f"lam{m}": coeffs[:, 3 * ns + 4 + m] for m in range(4)})
    else:
        t.update({f"u{c}{m:02d}": coeffs[:, c * ns + m] for c in range(3) for m in range(ns)})
    return t


def main(names):
    dev = torch.device("cuda:0")
    for name in names:
        cfg = fe.CONFIGS[name]
        tabs = fe.tables(cfg)
        c4, f4 = fe.cell_inputs(cfg, ncells=4)
        kernels = ir.build(cfg, c4, f4, tabs=tabs)
        coords, coeffs = fe.cell_inputs(cfg)
        E = coords.shape[0]
        et = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
              for k, v in e_tables(cfg, coords, coeffs).items()}
        total_ms = 0.0
        for oname, k in kernels:
            K = emit_cuda.IRKernel(k)
            inputs = {}
            for n in K.inputs:
                if n in et:
                    inputs[n] = et[n]
                else:
                    inputs[n] = torch.tensor(np.asarray(k["tables"][n]["values"]), device=dev)
            outs = {o: torch.zeros(K.size(0, o, E), dtype=torch.float64, device=dev)
                    for o in K.outputs}
            K.run(outs, inputs, k.get("constants", {}), E)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                K.run(outs, inputs, k.get("constants", {}), E)
            e1.record()
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1) / reps
        print(json.dumps({"config": name, "cells": E, "kernels": len(kernels), "ir": "raw (ufl)",
                          "ms": round(total_ms, 3), "elem_per_s": E / (total_ms / 1e3)}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
