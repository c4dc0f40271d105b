#!/usr/bin/env python3
"""Summarise ncu --set full captures into profiles/ncu_summary.json.

usage: tools/ncu_summary.py <tag> <cfg>=<path.ncu-rep> ...
Per config: duration, DRAM bytes (the roofline's `traffic`), pipe
utilisation, occupancy, registers, bank conflicts, top stall reasons.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "smem_store_conflicts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_load_conflicts",
    "lts__t_sectors_op_write.sum": "l2_write_sectors",
    "lts__t_bytes.sum": "l2_bytes",
    "smsp__inst_executed.sum": "instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    stalls = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if h in KEYS:
            key = KEYS[h]
            if u in UNIT_SCALE:
                x *= UNIT_SCALE[u]
                key += "_s" if u in ("ns", "us", "usecond", "ms", "msecond", "s") else "_bytes"
            res[key] = x
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
    tot = sum(stalls.values()) or 1.0
    res["stall_share"] = {k: round(v / tot, 3) for k, v in
                          sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    rb, wb = res.get("dram_read_bytes"), res.get("dram_write_bytes")
    if rb is not None and wb is not None:
        res["dram_bytes_per_launch"] = rb + wb
    return res


def src_sha(kernel_name):
    """sha of the kernel's .cu source (bench.py KERNEL_SOURCES): bench.py uses a
    capture only while the source it was taken from is unchanged."""
    sys.path.insert(0, ROOT)
    import bench

    base = (kernel_name or "").split("(")[0].replace("void ", "").replace("femgpu::", "")
    return bench.kernel_source_sha(base)


def main():
    tag = sys.argv[1]
    dst = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(dst) as f:
            allres = json.load(f)
    except (OSError, ValueError):
        allres = {}
    for arg in sys.argv[2:]:
        cfg, path = arg.split("=", 1)
        r = summarise(path)
        r["capture"] = f"{tag}: ncu --set full --clock-control none (1 launch, cold)"
        r["src_sha"] = src_sha(r.get("kernel"))
        allres.setdefault(cfg, {}).update(r)  # keep other tools' fields (ncu_flops.py)
        print(cfg, json.dumps(r))
    with open(dst, "w") as f:
        json.dump(allres, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
