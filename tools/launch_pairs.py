#!/usr/bin/env python
"""Per-launch table of an ncu --metrics ... --csv launch list (kernel, us, DRAM MB)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, {}
for row in rows:
    if "Kernel Name" in row:
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr):
        continue
    d = dict(zip(hdr, row))
    out.setdefault((int(d["ID"]), d["Kernel Name"][:28]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for (i, k), m in sorted(out.items()):
    t = m.get("gpu__time_duration.sum", 0)
    t = t / 1000 if t > 1e5 else t
    print(f"{i:3d} {k:30s} {t:8.1f} us  rd {m.get('dram__bytes_read.sum', 0) / 1e6:7.1f} MB  wr {m.get('dram__bytes_write.sum', 0) / 1e6:6.1f} MB")
