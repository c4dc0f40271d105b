#!/usr/bin/env python3
"""Global assembly pipeline on a config mesh: gather -> element kernel ->
scatter-add into CSR: FP64-atomic scatter, the fused
femgpu_assemble_csr, and the atomic-free row-gather assembly.  Device-timed per phase with
CUDA events over K steps; setup (numbering, pattern, positions) timed once.
usage: bench_global.py <cfg> [N] [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1604_05872_b200 import fe, mesh  # noqa: E402


def main():
    name = sys.argv[1]
    cfg = fe.CONFIGS[name]
    N = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.N
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    t0 = time.perf_counter()
    ga = mesh.GlobalAssembler(cfg, N=N)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    coef = torch.from_numpy(ga.mesh.global_coeffs()).to(ga.dev)
    E, n = ga.A.shape[0], ga.A.shape[1]
    for _ in range(3):
        ga.assemble(coef)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tg = ta = ts = 0.0
    for _ in range(K):
        ev[0].record()
        ga.gather(coef)
        ev[1].record()
        ga.form.assemble(ga.coords, ga.coeffs, ga.A)
        ev[2].record()
        ga.vals.zero_()
        from paper_1604_05872_b200 import femgpu
        femgpu.scatter_add(ga.A, ga.pos, ga.vals)
        ev[3].record()
        torch.cuda.synchronize()
        tg += ev[0].elapsed_time(ev[1])
        ta += ev[1].elapsed_time(ev[2])
        ts += ev[2].elapsed_time(ev[3])
    tg, ta, ts = tg / K, ta / K, ts / K
    tf = 0.0  # femgpu_assemble_csr (fused epilogue where the kernel has one)
    for _ in range(K):
        ev[0].record()
        ga.vals.zero_()
        ga.form.assemble_csr(ga.coords, ga.coeffs, ga.pos, ga.vals)
        ev[1].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
    tf /= K
    inc_ptr, inc, loc, maxlen = ga.row_plan()  # atomic-free row-gather assembly
    tr = 0.0
    for _ in range(K):
        ev[0].record()
        femgpu.csr_gather_rows(ga.row_ptr, inc_ptr, inc, loc, maxlen, ga.A, ga.vals)
        ev[1].record()
        torch.cuda.synchronize()
        tr += ev[0].elapsed_time(ev[1])
    tr /= K
    nnz = int(ga.vals.numel())
    r_bytes = E * n * n * (8 + 2) + E * n * 4 + nnz * 8  # A, loc, inc, vals written once
    ncoef = ga.coef_idx.shape[1]
    g_bytes = E * (4 * (4 + ncoef) + 8 * (12 + ncoef) + 8 * (12 + ncoef))  # idx + reads + writes
    s_bytes = E * n * n * (8 + 8 + 16)  # A, pos, atomic read-modify-write
    print(json.dumps({
        "config": name, "N": N, "cells": E, "n": n, "ndofs": ga.ndofs, "nnz": int(ga.vals.numel()),
        "setup_s": round(setup_s, 2), "steps": K,
        "gather_ms": round(tg, 4), "assemble_ms": round(ta, 4), "scatter_ms": round(ts, 4),
        "total_ms": round(tg + ta + ts, 4), "elem_per_s": E / ((tg + ta + ts) / 1e3),
        "assemble_csr_ms": round(tf, 4), "fused_total_ms": round(tg + tf, 4),
        "fused_elem_per_s": E / ((tg + tf) / 1e3),
        "gather_rows_ms": round(tr, 4), "rows_total_ms": round(tg + ta + tr, 4),
        "rows_elem_per_s": E / ((tg + ta + tr) / 1e3), "gather_rows_GBs": r_bytes / (tr / 1e3) / 1e9,
        "max_row_len": maxlen,
        "gather_GBs": g_bytes / (tg / 1e3) / 1e9, "scatter_GBs": s_bytes / (ts / 1e3) / 1e9,
        "kernel": ga.form.info["kernel_name"]}), flush=True)


if __name__ == "__main__":
    main()
