#!/usr/bin/env python3
"""Throughput of the generic IR backend (femgpu_ir_*, emit_cuda.py) on the BASELINE meshes.

Two IR sources per config:
  * raw      -- the config's IR as ir.py writes it (built on 4 cells for its code);
  * femopt   -- femopt's own optimized kernels of every plan the reference arm
                times (tests/golden/ir_full/<cfg>_<plan>.json.gz, made by
                oracle/make_ir_full.py): what a femopt user hands to a backend.
The per-cell e-tables of the full mesh are supplied at run time; device-timed
with CUDA events (median of 5 after a warm-up).  `ir_gflops` counts femopt's
flop_count of the IR that runs (kernel.cpp:521) -- for the optimized plans that
is the reference's F_alg, so the rate compares directly with the reference's
CPU rate on the same kernel (bench.py --impl reference).  The hand-written
kernels (bench.py) are the fast path.
usage: bench_generic.py [--raw] [--femopt] [--vectors] [cfg ...]"""
import argparse
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1604_05872_b200 import emit_cuda, fe, ir  # noqa: E402

IR_FULL = os.path.join(ROOT, "tests", "golden", "ir_full")


def time_kernels(kernels, et, E, dev, strategy="auto"):
    """kernels: list of IR dicts; returns (ms per pass over all kernels, strategies)."""
    runs, strategies = [], []
    for k in kernels:
        K = emit_cuda.IRKernel(k, strategy)
        strategies.append(K.strategy)
        inputs = {n: et[n] if n in et else
                  torch.tensor(np.asarray(k["tables"][n]["values"]), device=dev)
                  for n in K.inputs}
        outs = {o: torch.zeros(K.size(0, o, E), dtype=torch.float64, device=dev)
                for o in K.outputs}
        runs.append((K, outs, inputs, k.get("constants", {})))

    def one():
        for K, outs, inputs, consts in runs:
            K.run(outs, inputs, consts, E)

    one()
    torch.cuda.synchronize()
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        one()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return sorted(times)[len(times) // 2], strategies


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--raw", action="store_true")
    ap.add_argument("--femopt", action="store_true")
    ap.add_argument("--vectors", action="store_true",
                    help="the element-vector forms (ir.build_vector: load / residuals), raw IR")
    ap.add_argument("--strategy", default="auto", choices=["auto", "thread", "warp", "gemm"])
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3", "c4", "c5"])
    a = ap.parse_args()
    if not (a.raw or a.femopt or a.vectors):
        a.raw = a.femopt = True
    dev = torch.device("cuda:0")
    for name in a.configs:
        cfg = fe.CONFIGS[name]
        coords, coeffs = fe.cell_inputs(cfg)
        E = coords.shape[0]
        et = {k: torch.from_numpy(v).to(dev) for k, v in ir.e_tables(cfg, coords, coeffs).items()}
        jobs = []
        if a.raw:
            tabs = fe.tables(cfg)
            c4, f4 = fe.cell_inputs(cfg, ncells=4)
            jobs.append(("raw (ufl)", [k for _, k in ir.build(cfg, c4, f4, tabs=tabs)], None))
        if a.vectors and name != "c3":
            tabs = fe.tables(cfg)
            c4, f4 = fe.cell_inputs(cfg, ncells=4)
            jobs.append(("raw vector", [ir.build_vector(cfg, c4, f4, tabs=tabs)[1]], None))
        if a.femopt:
            for fn in sorted(os.listdir(IR_FULL)) if os.path.isdir(IR_FULL) else []:
                if fn.startswith(name + "_") and fn.endswith(".json.gz"):
                    with gzip.open(os.path.join(IR_FULL, fn), "rt") as f:
                        d = json.load(f)
                    jobs.append((f"femopt {d['plan']} ({d['encoding']})",
                                 [k["ir"] for k in d["kernels"]], d["flops_per_cell"]))
        for label, kernels, fpc in jobs:
            ms, strategies = time_kernels(kernels, et, E, dev, a.strategy)
            line = {"config": name, "cells": E, "ir": label, "kernels": len(kernels),
                    "strategy": sorted(set(strategies)), "ms": round(ms, 3),
                    "elem_per_s": E / (ms / 1e3)}
            if label == "raw vector":  # inputs + the element vector, FP64
                line["hbm_gbs"] = round(E * 8 * (12 + cfg.ncoef + cfg.n) / (ms / 1e3) / 1e9, 1)
            if fpc:
                line["ir_flops_per_cell"] = fpc
                line["ir_gflops"] = round(E * fpc / (ms / 1e3) / 1e9, 1)
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
