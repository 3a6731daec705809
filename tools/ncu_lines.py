#!/usr/bin/env python
"""Per-source-line summary of an ncu report's source page (cuda,sass view):
warp-stall samples and warp instructions executed per CUDA line, sorted.
usage: ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
lines = []
file_ = None
for r in rows:
    if r and r[0] == "File Path":
        file_ = r[1].split("/")[-1]
    if len(r) != len(hdr) or not r[0] or r[0] == "Line No":
        continue
    try:
        lines.append((int(r[iS]), int(r[iI]), f"{file_}:{r[0]}", r[1].strip()[:90]))
    except ValueError:
        pass
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"total samples {ts}, warp instructions {ti}")
for s, i, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins  {loc:24s} {src}")
