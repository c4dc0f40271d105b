"""Whole-mesh parity against the reference's CPU path -- TEST INFRASTRUCTURE.

The checker behind tests/test_gpu_fullmesh.py and bench.py's ``parity`` key:
every element matrix a GPU launch produced is compared with femopt's
optimized emitted C (``refkernel.RefKernel``: femopt_optimize -> emit_c ->
cc -O3, proj/src/driver.cpp:35-143, emit_c.cpp:108-174) run on the same
cell-major inputs, chunk by chunk, on all host threads.

The comparator is the north_star's: relative Frobenius error per element,
||A_e - R_e||_F / ||R_e||_F (the reference's own
``max_rel_error``, interp.cpp:175-193, is elementwise with an absolute floor
of 1 and is too lax for this bar).  The reference checks every kernel over
its whole output (proj/tests/test_backend.cpp:167-182); so does this.

The GPU side is abstracted as ``fetch(lo, hi) -> ndarray [hi-lo, n, n]`` so
this module never touches torch or the product library.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import refkernel as rk  # noqa: E402
from paper_1604_05872_b200 import fe  # noqa: E402


def _chunk_cells(cfg, nthreads: int, max_bytes: float = 384e6) -> int:
    """Cells per comparison chunk: ~max_bytes of reference output, whole
    CHUNK-cell blocks (the emitted C's literal e-extent)."""
    per = 8.0 * cfg.n * cfg.n
    return max(rk.CHUNK, int(max_bytes / per) // rk.CHUNK * rk.CHUNK)


def _frob_sq_blocks(cfg, A: np.ndarray, outs: dict, E: int):
    """(||A - R||_F^2, ||R||_F^2) per element, R given as the reference's
    output tables (one ``A`` or nine component blocks ``A{c}{d}``)."""
    if "A" in outs:
        R = outs["A"].reshape(E, -1)
        D = A.reshape(E, -1) - R
        return np.einsum("ij,ij->i", D, D), np.einsum("ij,ij->i", R, R)
    ns = cfg.ns
    A5 = A.reshape(E, 3, ns, 3, ns)
    dd = np.zeros(E)
    rr = np.zeros(E)
    for c in range(3):
        for d in range(3):
            R = outs[f"A{c}{d}"].reshape(E, ns, ns)
            D = A5[:, c, :, d, :] - R
            dd += np.einsum("ijk,ijk->i", D, D)
            rr += np.einsum("ijk,ijk->i", R, R)
    return dd, rr


def pick_plan(cfg) -> str:
    """The reference plan to check against: the fastest emitted one on CPU
    (c2 tensor, c5 unbounded; the only one otherwise)."""
    plans = [p for p in rk.plans_for(cfg) if rk.available(cfg, p)]
    if not plans:
        raise FileNotFoundError("reference sources missing (oracle/_ref/src)")
    for pref in ("tensor", "unbounded"):
        if pref in plans:
            return pref
    return plans[0]


def check(cfg, coords: np.ndarray, coeffs: np.ndarray, fetch, nthreads: int | None = None,
          plan: str | None = None, lo: int = 0, hi: int | None = None,
          accumulated_base=None) -> dict:
    """Compare cells [lo, hi) of a GPU result with the reference's emitted C.

    ``coords``/``coeffs`` are the cell-major inputs of the whole launch (index
    0 = first cell of the launch); ``fetch(a, b)`` returns the GPU's element
    matrices of cells [a, b).  Returns {max_frob_rel, mean_frob_rel,
    worst_cell, cells_checked, against}.
    """
    nthreads = nthreads or os.cpu_count() or 1
    plan = plan or pick_plan(cfg)
    K = rk.RefKernel(cfg, plan)
    E = coords.shape[0]
    hi = E if hi is None else hi
    step = _chunk_cells(cfg, nthreads)
    worst, worst_cell, ssum, checked = 0.0, -1, 0.0, 0
    a = lo
    while a < hi:
        b = min(hi, a + step)
        # the emitted C runs whole CHUNK-cell blocks: pad the tail with copies
        m = b - a
        mp = -(-m // rk.CHUNK) * rk.CHUNK
        x, c = coords[a:b], coeffs[a:b]
        if mp != m:
            x = np.concatenate([x, np.repeat(x[-1:], mp - m, axis=0)])
            c = np.concatenate([c, np.repeat(c[-1:], mp - m, axis=0)])
        st = K.prepare(np.ascontiguousarray(x), np.ascontiguousarray(c))
        outs = K.run_prepared(st, nthreads)
        outs = {k: v[:m] for k, v in outs.items()}
        G = np.asarray(fetch(a, b), dtype=np.float64)
        if accumulated_base is not None:
            G = G - accumulated_base(a, b)
        dd, rr = _frob_sq_blocks(cfg, G, outs, m)
        rel = np.sqrt(dd) / np.sqrt(np.maximum(rr, 1e-300))
        bad = ~np.isfinite(rel)
        if bad.any():
            rel[bad] = np.inf
        i = int(np.argmax(rel))
        if rel[i] > worst or worst_cell < 0:
            worst, worst_cell = float(rel[i]), a + i
        ssum += float(rel.sum())
        checked += m
        a = b
    return {"max_frob_rel": worst, "mean_frob_rel": ssum / max(1, checked),
            "worst_cell": worst_cell, "cells_checked": checked,
            "against": f"reference emitted C (femopt plan '{plan}', cc -O3 -march=native "
                       f"-ffp-contract=off, {nthreads} host threads)"}
