#!/usr/bin/env python3
"""Quick device timing of each config's kernel (development aid, not the bench)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

GRAPH = int(os.environ.get("QT_GRAPH", "0"))  # >0: time a graph of that many launches
SCHED = int(os.environ.get("QT_SCHED", "0"))  # femgpu schedule (0 = AUTO)
if os.environ.get("FEMGPU_LIB"):  # A/B builds (development)
    femgpu.LIB_PATH = os.environ["FEMGPU_LIB"]


def main(names):
    dev = torch.device("cuda:0")
    for name in names:
        cfg = fe.CONFIGS[name]
        t0 = time.time()
        coords, coeffs = fe.cell_inputs(cfg)
        try:
            form = femgpu.Form.from_config(cfg, schedule=SCHED)
        except femgpu.FemgpuError as e:
            print(json.dumps({"config": name, "error": str(e)}))
            continue
        x = torch.from_numpy(coords).to(dev)
        c = torch.from_numpy(coeffs).to(dev)
        E = coords.shape[0]
        out = torch.empty((E, cfg.n, cfg.n), dtype=torch.float64, device=dev)
        for _ in range(3):
            form.assemble(x, c, out)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        times = []
        if GRAPH:  # K launches back to back from one CUDA graph (bench.py's timing)
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                form.assemble(x, c, out, stream=s)
                s.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(GRAPH):
                        form.assemble(x, c, out, stream=s)
            for _ in range(3):
                ev[0].record()
                g.replay()
                ev[1].record()
                torch.cuda.synchronize()
                times.append(ev[0].elapsed_time(ev[1]) / 1e3 / GRAPH)
        else:
            for _ in range(10):
                ev[0].record()
                form.assemble(x, c, out)
                ev[1].record()
                torch.cuda.synchronize()
                times.append(ev[0].elapsed_time(ev[1]) / 1e3)
        t = sorted(times)[len(times) // 2]
        bpc = cfg.bytes_per_cell()
        fpc = form.info["flops_per_cell"]
        print(json.dumps({"config": name, "cells": E, "ms": round(t * 1e3, 4),
                          "Mcells_s": round(E / t / 1e6, 2), "GB_s": round(E * bpc / t / 1e9, 1),
                          "GFLOP_s": round(E * fpc / t / 1e9, 1), "flops_per_cell": fpc,
                          "kernel": form.info["kernel_name"], "setup_s": round(time.time() - t0, 1)}),
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(fe.CONFIGS))
