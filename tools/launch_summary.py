#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launches, total and per-launch time, share of the total."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def summarise(path, title=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, iv, im, iu = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Name", "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", "")) * SCALE[r[iu]]
        a = agg.setdefault(r[ik], [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = [title, ""] if title else []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{n:4d} launches {t:10.1f} us total {t / n:9.1f} us/launch {100 * t / tot:5.1f}%  {k[:90]}")
    out += ["", f"total {tot:.1f} us"]
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    sys.stdout.write(summarise(sys.argv[1], " ".join(sys.argv[2:])))
