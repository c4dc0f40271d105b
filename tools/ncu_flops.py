#!/usr/bin/env python3
"""Executed FP64 flops per cell from ncu metric captures (SURVEY.md §8d F_exec:
DFMA = 2, DADD/DMUL = 1, DMMA = 2*m*n*k per warp instruction, i.e. the
sm__ops_path_tensor_src_fp64 count).  Writes fp64_flops_per_cell_ncu into
profiles/ncu_summary.json.

usage: tools/ncu_flops.py <cfg>=<flops_cfg.csv> ...   (captures made with
  ncu --metrics sm__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum,
  sm__ops_path_tensor_src_fp64.sum --csv -c 1 python tools/prof_one.py <cfg> 1)"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1604_05872_b200 import fe  # noqa: E402


def parse(path):
    vals, kernel = {}, None
    with open(path) as f:
        rows = [r for r in csv.reader(f) if len(r) > 14 and r[0] != "ID"]
    for r in rows:
        kernel = r[4]
        vals[r[12]] = float(r[14].replace(",", ""))
    return kernel, vals


def main():
    dst = os.path.join(ROOT, "profiles", "ncu_summary.json")
    with open(dst) as f:
        summ = json.load(f)
    for arg in sys.argv[1:]:
        cfg, path = arg.split("=", 1)
        kernel, v = parse(path)
        cells = fe.CONFIGS[cfg].ncells
        flops = (2 * v.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
                 + v.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
                 + v.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
                 + v.get("sm__ops_path_tensor_src_fp64.sum", 0))
        ent = summ.setdefault(cfg, {})
        ent["fp64_flops_per_cell_ncu"] = flops / cells
        ent["fp64_flops_ncu_kernel"] = kernel
        ent["fp64_flops_ncu_breakdown"] = {k.split(".")[0]: val for k, val in v.items()}
        print(cfg, kernel[:40], f"{flops / cells:.0f} flops/cell")
    with open(dst, "w") as f:
        json.dump(summ, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
