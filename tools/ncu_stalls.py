#!/usr/bin/env python3
"""Per-reason stall attribution of an ncu source page: top instructions per reason
and per-region sums.  usage: ncu_stalls.py rep.ncu-rep [reason ...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reasons = sys.argv[2:] or ["stall_long_sb", "stall_wait", "stall_barrier", "stall_short_sb"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
for r in reasons:
    ci = hdr.index(r)
    vals = [(int(d[ci]) if d[ci].isdigit() else 0, i) for i, d in enumerate(data)]
    tot = sum(v for v, _ in vals)
    print(f"== {r}: total {tot}")
    for v, i in sorted(vals, reverse=True)[:8]:
        print(f"  {i:5d} {v:7d}  {data[i][1][:80]}")
