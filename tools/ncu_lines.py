#!/usr/bin/env python3
"""Warp-stall samples aggregated per CUDA source line of an ncu capture.
usage: ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))[3:]
lines = [(int(r[0]), r[1], int(r[4] or 0)) for r in rows
         if len(r) > 4 and r[2] == "-" and r[0].isdigit()]
tot = sum(x[2] for x in lines) or 1
print("total samples", tot)
for ln, s, v in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{ln:5d} {v:7d} {v / tot:6.3f}  {s[:90]}")
