#!/usr/bin/env python3
"""Element-vector kernels (femgpu_assemble_vector) on the BASELINE meshes: device-timed
(CUDA events, median of 20 launches after warm-up), elem/s and compulsory HBM GB/s
(8 * (12 + ncoef + n) bytes per cell: inputs and the element vector).
usage: bench_vector.py [cfg ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

if os.environ.get("FEMGPU_LIB"):  # A/B builds (development)
    femgpu.LIB_PATH = os.environ["FEMGPU_LIB"]


def main(names):
    dev = torch.device("cuda:0")
    for name in names:
        cfg = fe.CONFIGS[name]
        coords, coeffs = fe.cell_inputs(cfg)
        E = coords.shape[0]
        form = femgpu.Form.from_config(cfg)
        x = torch.from_numpy(coords).to(dev)
        c = torch.from_numpy(coeffs).to(dev)
        out = torch.empty((E, cfg.n), dtype=torch.float64, device=dev)
        for _ in range(3):
            form.assemble_vector(x, c, out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            form.assemble_vector(x, c, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        bpc = 8 * (12 + cfg.ncoef + cfg.n)
        print(json.dumps({"config": name, "form": "element vector", "cells": E, "n": cfg.n,
                          "ms": round(ms, 4), "elem_per_s": E / (ms / 1e3),
                          "bytes_per_cell": bpc, "hbm_gbs": round(E * bpc / (ms / 1e3) / 1e9, 1)}),
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c4", "c5"])
