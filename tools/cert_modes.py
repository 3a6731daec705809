#!/usr/bin/env python
"""Certificate pass modes side by side on one config (debug/experiment aid,
not a benchmark): per pass fitness, searched and certified counts for
O3G_OPT_CERT in {0, forced} x O3G_OPT_CERT_SWEEP in {0, 1}."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large16m")
ap.add_argument("--n", type=int, default=400000)
ap.add_argument("--iters", type=int, default=8)
a = ap.parse_args()
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_09847_b200 as o3g  # noqa: E402
from bench import load_workload  # noqa: E402

w = load_workload(a.config, a.n)
dev = torch.device("cuda:0")
src, tgt, nrm = (torch.from_numpy(w[k]).to(dev) for k in ("source", "target", "target_normals"))
ctx = o3g.Context(0)
ctx.set_target(tgt, nrm, w["dmax"])
ctx.set_source(src, w["init_T"])
for cert, sweep in ((0, 0), (2, 1), (2, 0)):
    ctx.set_option(o3g.OPT_CERT, cert)
    ctx.set_option(o3g.OPT_CERT_SWEEP, sweep)
    r = ctx.run(w["init_T"], a.iters, 0.0, 0.0, history=True)
    tr = ctx.last_run_trace(r.passes)
    print(f"cert={cert} sweep={sweep} passes={r.passes} fitness={r.fitness:.6f}")
    for k in range(r.passes):
        print(f"  {k} count={tr['terms'][k][27]:.0f} searched={tr['searched'][k]:.0f} certified={tr['certified'][k]:.0f}")
torch.cuda.synchronize()
print("ok")
