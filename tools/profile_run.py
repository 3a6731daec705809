#!/usr/bin/env python
"""Small driver for ncu / sanitizer runs: one context, `--reps` full ICP runs
(or steps) on a named config. Not a benchmark (bench.py is)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large16m")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--iters", type=int, default=None)
ap.add_argument("--mode", default="run", choices=["run", "step"])
ap.add_argument("--search", type=int, default=1)
ap.add_argument("--bps", type=int, default=0)
ap.add_argument("--coop-min", type=int, default=None)
ap.add_argument("--prune-min", type=int, default=None)
ap.add_argument("--interleave", type=int, default=None)
ap.add_argument("--cert", type=int, default=None, help="O3G_OPT_CERT")
ap.add_argument("--regime", default="init", choices=["init", "converged"])
a = ap.parse_args()

import torch  # noqa: E402

import paper_1801_09847_b200 as o3g  # noqa: E402
from bench import load_workload  # noqa: E402

w = load_workload(a.config, a.n)
if a.regime == "converged":   # as bench.py --regime converged
    import numpy as np
    from synth.rng import Stream
    from synth.scenes import rigid, rotation
    rs = Stream(0x5EED)
    w = dict(w, init_T=w["T_true"] @ rigid(rotation(rs.unit_vectors(1)[0], np.deg2rad(0.1)),
                                             0.01 * rs.unit_vectors(1)[0]))
dev = torch.device("cuda:0")
src, tgt, nrm = (torch.from_numpy(w[k]).to(dev) for k in ("source", "target", "target_normals"))
ctx = o3g.Context(0)
ctx.set_option(1, a.search)
if a.bps:
    ctx.set_option(4, a.bps)
if a.coop_min is not None:
    ctx.set_option(6, a.coop_min)
if a.prune_min is not None:
    ctx.set_option(10, a.prune_min)
if a.cert is not None:
    ctx.set_option(13, a.cert)
if a.interleave is not None:
    ctx.set_option(11, a.interleave)
for _ in range(a.reps):
    ctx.set_clouds(src, tgt, nrm, w["dmax"], w["init_T"])
    if a.mode == "run":
        r = ctx.run(w["init_T"], a.iters if a.iters is not None else w["iters"], 0.0, 0.0)
        print("fitness", r.fitness, "rmse", r.inlier_rmse, "iters", r.iterations)
    else:
        corr = torch.empty(len(src), dtype=torch.int32, device=dev)
        s = ctx.step(w["T_true"], corr_out=corr)
        print("count", s["count"])
torch.cuda.synchronize()
print("ok")
