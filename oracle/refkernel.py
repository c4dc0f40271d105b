"""The reference's CPU path for a config: femopt-optimized emitted C, threaded.

TEST / BASELINE INFRASTRUCTURE.  This is what bench.py's reference arm and
``cpu_baseline`` time, and what tests/golden/ is generated from:

  IR (paper_1604_05872_b200/ir.py)
    -> femopt_optimize (zero-skip OFF: proj/src/zeroskip.cpp miscompiles
       vector elements)               [proj/src/driver.cpp:35-143]
    -> femopt_emit_c                                   [proj/src/emit_c.cpp:108-174]
    -> cc -O3 -march=native -ffp-contract=off          (SURVEY.md §8d CPU baseline)
    -> oracle/refrun.c: chunks of E=chunk cells, one contiguous range per thread.

Two stages, because /root/reference exists only in the build container:
  * ``emit(cfg, plan)`` (container only) runs the reference optimizer and writes
    oracle/_ref/src/<cfg>_<plan>.c + .json (git-ignored, shipped to the box);
  * ``RefKernel(cfg, plan)`` compiles that source for the *current* host CPU
    (cached under oracle/_ref/host-<cpu>/) and runs it.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_1604_05872_b200 import fe, ir  # noqa: E402

SRC_DIR = os.path.join(HERE, "_ref", "src")
CHUNK = 512  # divides 6*N^3 for N = 32, 48, 64

# plan name -> (encoding, femopt memory_limit T_H, optimize?)
PLANS = {
    "quad": ("ufl", 262144, True),        # femopt defaults (driver.hpp:8-13), UFL encoding
    "unbounded": ("ufl", 1 << 40, True),  # UFL encoding, T_H unbounded (paper's T_H=L3 runs)
    "tensor": ("gfac", 1 << 40, True),    # G-factored, T_H unbounded: full pre-evaluation
    "raw": ("ufl", 0, False),             # as written (no optimization)
}


def plans_for(cfg) -> list[str]:
    if cfg.kind == fe.HELMHOLTZ:
        return ["quad", "tensor"]
    if cfg.kind == fe.BURGERS:
        return ["quad", "unbounded"]
    return ["quad"]


def src_path(cfg, plan, chunk=CHUNK):
    return os.path.join(SRC_DIR, f"{cfg.name}_{plan}_{chunk}")


def emit(cfg, plan: str, chunk: int = CHUNK, verbose=True) -> dict:
    """Run the reference optimizer/emitter for ``cfg``; write .c/.json sources."""
    import refbridge as rb

    enc, th, do_opt = PLANS[plan]
    tabs = fe.tables(cfg)
    coords, coeffs = fe.cell_inputs(cfg, ncells=chunk)
    kernels = ir.build(cfg, coords, coeffs, tabs, enc)
    meta = {"config": cfg.name, "plan": plan, "encoding": enc, "memory_limit": th,
            "chunk": chunk, "kernels": []}
    srcs = ["#include <math.h>\n"]
    for ki, (out, k) in enumerate(kernels):
        K = rb.Kernel(ir.dumps(k))
        raw = K.flops()
        t0 = time.time()
        status = "optimized"
        rep = None
        if do_opt:
            try:
                Ko, rep = K.optimize(memory_limit=th, preeval=True, zero_skip=False)
            except rb.FemoptError as e:  # fall back to the raw nest (always valid)
                Ko, status = K, f"raw ({e})"
        else:
            Ko, status = K, "raw"
        kj = json.loads(Ko.to_json())
        fn = f"k{ki}"
        srcs.append(Ko.emit_c(fn).replace("#include <math.h>\n", ""))
        outs, tabl, cons = ir.argument_order(kj)
        srcs.append(rb_argv(fn, len(outs), len(tabl), len(cons)))
        meta["kernels"].append({
            "fn": fn, "outputs": outs, "tables": tabl, "constants": cons,
            "e_tables": [t for t in tabl if kj["tables"][t]["dims"] == ["e"]],
            "flops_raw_per_cell": raw / chunk, "flops_per_cell": Ko.flops() / chunk,
            "status": status, "seconds": round(time.time() - t0, 2),
            "report_flops": {kk: v for kk, v in (rep or {}).items() if kk.startswith("flops")},
        })
        if verbose:
            print(f"[emit] {cfg.name}/{plan} {out}: {raw / chunk:.0f} -> "
                  f"{Ko.flops() / chunk:.0f} flops/cell ({status}, {time.time() - t0:.1f}s)",
                  flush=True)
    meta["flops_per_cell"] = sum(k["flops_per_cell"] for k in meta["kernels"])
    os.makedirs(SRC_DIR, exist_ok=True)
    base = src_path(cfg, plan, chunk)
    with open(base + ".c", "w") as f:
        f.write("".join(srcs))
    with open(base + ".json", "w") as f:
        json.dump(meta, f, indent=1)
    return meta


def rb_argv(fn, no, nt, nc):
    import refbridge as rb
    return rb.argv_wrapper(fn, no, nt, nc)


def available(cfg, plan, chunk=CHUNK) -> bool:
    b = src_path(cfg, plan, chunk)
    return os.path.exists(b + ".c") and os.path.exists(b + ".json")


def host_tag() -> str:
    cpu = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return hashlib.sha1(cpu.encode()).hexdigest()[:10]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class RefKernel:
    """femopt's emitted C for one config+plan, compiled for this host."""

    def __init__(self, cfg, plan: str, chunk: int = CHUNK):
        self.cfg, self.plan, self.chunk = cfg, plan, chunk
        base = src_path(cfg, plan, chunk)
        if not available(cfg, plan, chunk):
            raise FileNotFoundError(f"{base}.c missing: run oracle/make_golden.py (needs "
                                    "/root/reference) or `python -c 'import __graft_entry__ as g; "
                                    "g.build()'`")
        with open(base + ".json") as f:
            self.meta = json.load(f)
        outdir = os.path.join(HERE, "_ref", f"host-{host_tag()}")
        os.makedirs(outdir, exist_ok=True)
        so = os.path.join(outdir, os.path.basename(base) + ".so")
        srcs = [base + ".c", os.path.join(HERE, "refrun.c")]
        if not os.path.exists(so) or any(os.path.getmtime(s) > os.path.getmtime(so) for s in srcs):
            tmp = so + f".{os.getpid()}.tmp"
            subprocess.run(["cc", "-O3", "-march=native", "-ffp-contract=off", "-shared", "-fPIC",
                            "-o", tmp, *srcs, "-lm", "-lpthread"], check=True)
            os.replace(tmp, so)
        self.lib = C.CDLL(so)
        ks = self.meta["kernels"]
        self.out_names = sorted({o for k in ks for o in k["outputs"]})
        self.tab_names = sorted({t for k in ks for t in k["tables"]})
        self.con_names = sorted({c for k in ks for c in k["constants"]})
        idx = []
        for k in ks:
            idx += [self.out_names.index(o) for o in k["outputs"]]
            idx += [self.tab_names.index(t) for t in k["tables"]]
            idx += [self.con_names.index(c) for c in k["constants"]]
        nk = len(ks)
        self._fns = (C.c_void_p * nk)(*[C.cast(getattr(self.lib, k["fn"] + "_argv"), C.c_void_p)
                                        for k in ks])
        self._nout = (C.c_int * nk)(*[len(k["outputs"]) for k in ks])
        self._ntab = (C.c_int * nk)(*[len(k["tables"]) for k in ks])
        self._ncon = (C.c_int * nk)(*[len(k["constants"]) for k in ks])
        self._idx = (C.c_int * len(idx))(*idx)
        e_tabs = {t for k in ks for t in k["e_tables"]}
        self._is_e = (C.c_int * len(self.tab_names))(*[int(t in e_tabs) for t in self.tab_names])
        self.lib.refrun.restype = C.c_int
        self.flops_per_cell = self.meta["flops_per_cell"]

    def prepare(self, coords, coeffs):
        """Cell-major inputs -> the SoA tables the emitted C reads (not timed)."""
        cfg = self.cfg
        E = coords.shape[0]
        assert E % self.chunk == 0, "sample must be a multiple of the chunk"
        tabs = fe.tables(cfg)
        full = ir.build(cfg, coords[:1], coeffs[:1], tabs, PLANS[self.plan][0])
        tables = {}
        for _, k in full:
            for name, t in k["tables"].items():
                if t["dims"] == ["e"]:
                    continue
                tables[name] = np.ascontiguousarray(np.array(t["values"], dtype=np.float64))
        for v in range(4):
            for c in range(3):
                tables[f"x{v}{c}"] = np.ascontiguousarray(coords[:, v, c])
        for name, t in _coef_soa(cfg, coeffs).items():
            tables[name] = t
        missing = [t for t in self.tab_names if t not in tables]
        if missing:
            raise KeyError(f"no data for tables {missing[:5]}")
        consts = {"nu": cfg.consts[0], "dt": cfg.consts[1]} if cfg.consts else {}
        outs = {}
        for o in self.out_names:
            per = (cfg.ns * cfg.ns) if cfg.kind == fe.BURGERS else cfg.n * cfg.n
            outs[o] = np.zeros((E, per))
        return {"E": E, "tables": [tables[t] for t in self.tab_names],
                "consts": np.array([consts[c] for c in self.con_names] or [0.0]), "outs": outs}

    def run_prepared(self, st, nthreads: int):
        E = st["E"]
        outs = [st["outs"][o] for o in self.out_names]
        optr = (C.POINTER(C.c_double) * len(outs))(
            *[o.ctypes.data_as(C.POINTER(C.c_double)) for o in outs])
        per = (C.c_long * len(outs))(*[o.shape[1] for o in outs])
        tptr = (C.POINTER(C.c_double) * len(st["tables"]))(
            *[t.ctypes.data_as(C.POINTER(C.c_double)) for t in st["tables"]])
        cptr = st["consts"].ctypes.data_as(C.POINTER(C.c_double))
        rc = self.lib.refrun(len(self.meta["kernels"]), self._fns, self._nout, self._ntab,
                             self._ncon, self._idx, C.c_long(E), C.c_long(self.chunk), optr, per,
                             tptr, self._is_e, cptr, int(nthreads))
        if rc != 0:
            raise RuntimeError("refrun failed")
        return st["outs"]

    def run(self, coords, coeffs, nthreads: int = 1) -> np.ndarray:
        st = self.prepare(coords, coeffs)
        outs = self.run_prepared(st, nthreads)
        return ir.assemble_blocks(self.cfg, outs, st["E"])


def _coef_soa(cfg, coeffs):
    """Cell-major coefficient dofs -> per-dof e-tables named as in ir.py."""
    out = {}
    col = 0
    for (name, nd, nc, *_rest) in cfg.coef_ranges:
        for c in range(nc):
            for m in range(nd):
                if name == "f":
                    key = f"f{m:02d}"
                elif name in ("mu", "lam"):
                    key = f"{name}{m}"
                else:  # vector coefficient w / u
                    key = f"{name}{c}{m:02d}"
                out[key] = np.ascontiguousarray(coeffs[:, col])
                col += 1
    return out
