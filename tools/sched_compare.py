#!/usr/bin/env python3
"""Measured comparison of the schedules femgpu can run for each BASELINE form
(the evidence behind the AUTO choice and its efficiency constants, capi.cu
kEff*): every candidate of femgpu_form_schedules is forced, timed on the full
BASELINE mesh (CUDA events around a CUDA-graph replay of K launches), and its
measured fraction of the nominal roofline is reported next to the library's
prediction.  Writes one JSON object to stdout (profiles/schedule_choice_r02.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1604_05872_b200 import fe, femgpu  # noqa: E402

K = int(os.environ.get("SC_STEPS", "10"))


def time_form(form, x, c, out, dev):
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for _ in range(3):
            form.assemble(x, c, out, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(K):
                form.assemble(x, c, out, stream=s)
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            t = e0.elapsed_time(e1) / K
            best = t if best is None else min(best, t)
    return best


def main(names):
    dev = torch.device("cuda:0")
    res = {}
    for name in names:
        cfg = fe.CONFIGS[name]
        coords, coeffs = fe.cell_inputs(cfg)
        x = torch.from_numpy(coords).to(dev)
        c = torch.from_numpy(coeffs).to(dev)
        out = torch.empty((coords.shape[0], cfg.n, cfg.n), dtype=torch.float64, device=dev)
        ranking = femgpu.schedules(cfg)
        rows = []
        for cand in ranking:
            sched = {v: k for k, v in femgpu.SCHEDULE_NAMES.items()}[cand["schedule"]]
            form = femgpu.Form.from_config(cfg, schedule=sched)
            if form.info["kernel_name"] != cand["kernel"]:
                continue  # another kernel of the same schedule ranks first
            ms = time_form(form, x, c, out, dev)
            roof = max(cand["flops_per_cell"] / cand["peak_flops"],
                       cand["bytes_per_cell"] / cand["peak_bytes"]) * coords.shape[0]
            rows.append({**cand, "measured_ms": ms, "measured_efficiency": roof / (ms / 1e3),
                         "predicted_ms": cand["predicted_ns_per_cell"] * coords.shape[0] / 1e6})
            del form
        fastest = min(rows, key=lambda r: r["measured_ms"])["kernel"]
        res[name] = {"cells": coords.shape[0], "auto": [r["kernel"] for r in ranking if r["chosen"]][0],
                     "measured_fastest": fastest, "candidates": rows}
        print(f"# {name}: auto {res[name]['auto']}, measured fastest {fastest}: " +
              ", ".join(f"{r['kernel']} {r['measured_ms']:.3f} ms (pred {r['predicted_ms']:.3f})"
                        for r in rows), file=sys.stderr, flush=True)
        del x, c, out
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
