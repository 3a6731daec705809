#!/usr/bin/env python
"""DRAM traffic per correspondence pass from an ncu launch list
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
-k regex:k3_ --csv`): the pass is k3_balanced, or k3_sweep + k3_balanced with
certificates; prints the per-pass mean time and bytes, and with --key updates
profiles/k3_traffic.json[key] (read by bench.py's roofline `traffic`)."""
import argparse
import csv
import json
import os
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--key", default=None)
ap.add_argument("--skip", type=int, default=0, help="skip the first N passes (e.g. warm-up registrations)")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr, launches = None, {}
for row in rows:
    if "Kernel Name" in row:
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr):
        continue
    d = dict(zip(hdr, row))
    launches.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})[d["Metric Name"]] = (
        float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
passes, cur = [], None
# with certificates every pass launches both k3_balanced instantiations (the
# plain one, then the certificate one; the one not matching the pass's mode
# exits at once), after k3_sweep in sweep mode: a pass ends at the certificate
# instantiation; without certificates at each k3_balanced
def is_cert(name):   # k3_balanced<WRITE_CORR, COOP, PRUNE, CERT, NT>: the certificate instantiation
    return re.search(r"k3_balanced<(\(bool\))?\d,(\(bool\))?\d,(\(bool\))?\d,(\(bool\))?1[,>]", name.replace(" ", "")) is not None


certs = any(is_cert(L["name"]) for L in launches.values())
for i in sorted(launches):
    L = launches[i]
    t, tu = L["gpu__time_duration.sum"]
    t = t / 1000.0 if tu == "ns" else t * 1000.0 if tu == "ms" else t   # -> us
    def mb(k):
        v, u = L[k]
        return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
    rec = (t, mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"))
    cur = (rec[0] + (cur[0] if cur else 0.0), rec[1] + (cur[1] if cur else 0.0))
    ends = "k3_balanced" in L["name"] and (not certs or is_cert(L["name"]))
    if ends:
        passes.append(cur)
        cur = None
passes = passes[a.skip:]
tm = sum(p[0] for p in passes) / len(passes)
by = sum(p[1] for p in passes) / len(passes)
print(f"{len(passes)} passes: {tm:.1f} us and {by:.1f} MB DRAM per pass")
if a.key:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "k3_traffic.json")
    tab = json.load(open(path)) if os.path.exists(path) else {}
    tab[a.key] = by * 1e6
    tab["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per correspondence pass (every k3_ launch "
                    "of the pass), mean over one registration's passes, ncu --clock-control "
                    "none (tools/k3_traffic.py); keys config@world@regime")
    json.dump(tab, open(path, "w"), indent=1, sort_keys=True)
