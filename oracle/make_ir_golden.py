#!/usr/bin/env python3
"""Golden fixtures for the generic IR backend (paper_1604_05872_b200/emit_cuda.py).

TEST INFRASTRUCTURE (container only: needs the reference built by oracle/Makefile).
For each case the kernel IR -- raw (ir.py) or femopt-optimized (femopt_optimize,
zero-skip off) -- is stored as JSON with its tables, together with the outputs
of the reference itself on that IR:
  * ``emitc_<out>``: femopt's emitted C (emit_c.cpp:108-174) compiled with
    ``cc -O3 -ffp-contract=off`` and run through the uniform argv wrapper
    (test_backend.cpp:62-98), outputs zero-initialised (emit_c's += contract);
  * ``interp_<out>``: femopt's interpreter (interp.cpp:125-154).
Writes tests/golden/ir/<case>.json + <case>.npz.
"""
import ctypes as C
import json
import os
import sys
import tempfile
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
import refbridge as rb  # noqa: E402

from paper_1604_05872_b200 import fe, ir  # noqa: E402

E = 5
OUT = os.path.join(ROOT, "tests", "golden", "ir")


def cases():
    c1, c2, c3, c4, c5 = (fe.CONFIGS[k] for k in ("c1", "c2", "c3", "c4", "c5"))
    c2s = replace(c2, quad_degree=6)   # smaller tables; exactness is not the point here
    c5s = replace(c5, quad_degree=4)

    def mat(cfg, enc="ufl", block=None):
        def f(coords, coeffs, tabs):
            ks = ir.build(cfg, coords, coeffs, tabs=tabs, encoding=enc)
            return dict(ks)[block] if block else ks[0][1]
        return cfg, f

    def vec(cfg):
        return cfg, lambda coords, coeffs, tabs: ir.build_vector(cfg, coords, coeffs, tabs)[1]

    return {
        "c1_matrix": (*mat(c1), ("raw", "opt")),
        "c1_matrix_gfac": (*mat(c1, "gfac"), ("opt",)),
        "c1_load": (*vec(c1), ("raw", "opt")),
        "c2_matrix_gfac": (*mat(c2s, "gfac"), ("opt",)),
        "c2_load": (*vec(c2s), ("opt",)),
        "c3_matrix": (*mat(c3), ("opt",)),
        "c4_matrix": (*mat(c4), ("raw",)),
        "c4_residual": (*vec(c4), ("raw", "opt")),
        "c5_block01": (*mat(c5s, block="A01"), ("opt",)),
        "c5_block11": (*mat(c5s, block="A11"), ("opt",)),
        "c5_residual": (*vec(c5s), ("opt",)),
    }


def run_emitted_c(irjson: str, outputs):
    k = rb.Kernel(irjson)
    src = k.emit_c("kfn")
    d = json.loads(irjson)
    tabs = d["tables"]
    inputs = sorted(n for n, t in tabs.items() if t.get("provenance", "input") != "preevaluated")
    consts = sorted((d.get("constants") or {}).keys())
    outs = sorted(outputs)
    src += rb.argv_wrapper("kfn", len(outs), len(inputs), len(consts))
    with tempfile.TemporaryDirectory() as tmp:
        so = rb.compile_c(src, os.path.join(tmp, "k.so"))
        lib = C.CDLL(so)
        fn = lib.kfn_argv
        fn.restype = None
        # output sizes from the interpreter
        res = {o: np.zeros_like(rb.interpret(irjson, o)) for o in outs}
        tarr = [np.ascontiguousarray(np.asarray(tabs[n]["values"], dtype=np.float64))
                for n in inputs]
        carr = np.asarray([float(d["constants"][c]) for c in consts] or [0.0])
        dp = C.POINTER(C.c_double)
        o_ptrs = (dp * len(outs))(*[res[o].ctypes.data_as(dp) for o in outs])
        t_ptrs = (dp * max(1, len(inputs)))(*[t.ctypes.data_as(dp) for t in tarr])
        fn(o_ptrs, t_ptrs, carr.ctypes.data_as(dp))
    return res


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, (cfg, build, variants) in cases().items():
        tabs = fe.tables(cfg)
        coords, coeffs = fe.cell_inputs(cfg, ncells=E)
        raw = build(coords, coeffs, tabs)
        for var in variants:
            if var == "raw":
                d = raw
            else:
                K = rb.Kernel(ir.dumps(raw))
                Ko, _ = K.optimize(memory_limit=262144, preeval=True, zero_skip=False)
                d = json.loads(Ko.to_json())
            js = json.dumps(d, separators=(",", ":"))
            outs = d["outputs"]
            arrays = {}
            for o, v in run_emitted_c(js, outs).items():
                arrays[f"emitc_{o}"] = v
            for o in outs:
                arrays[f"interp_{o}"] = rb.interpret(js, o)
            case = f"{name}_{var}"
            with open(os.path.join(OUT, case + ".json"), "w") as f:
                f.write(js)
            np.savez_compressed(os.path.join(OUT, case + ".npz"), **arrays)
            dev = max(float(np.max(np.abs(arrays[f"emitc_{o}"] - arrays[f"interp_{o}"]))
                            / max(1e-300, np.max(np.abs(arrays[f"interp_{o}"])))) for o in outs)
            print(f"{case}: {len(js) / 1024:.0f} KB, outputs {outs}, emit_c vs interp {dev:.1e}")


if __name__ == "__main__":
    main()
