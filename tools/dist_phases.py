#!/usr/bin/env python
"""Per-rank phase times of a world-P run, measured on one B200 with the
loopback transport (design data for the multi-GPU projection, DESIGN.md §8;
not a benchmark). For P in --worlds: P contexts on the device, each rank's
set_target / set_source timed with CUDA events, then o3g_loopback_run with
O3G_OPT_TIMING (each rank's correspondence kernels timed per pass; the ranks
run one after another, so every number is one rank's work alone). Prints one
JSON line per P with the max over ranks of each phase."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large16m")
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_09847_b200 as o3g  # noqa: E402
from bench import load_workload  # noqa: E402

w = load_workload(a.config)
dev = torch.device("cuda:0")
src, tgt, nrm = (torch.from_numpy(w[k]).to(dev) for k in ("source", "target", "target_normals"))
T0 = w["init_T"]
iters = w["iters"]


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for P in [int(x) for x in a.worlds.split(",")]:
    ctxs = [o3g.Context(0) for _ in range(P)]
    rows = []
    for rep in range(a.reps + 1):
        st, ss = [], []
        for r, c in enumerate(ctxs):
            c.set_option(o3g.OPT_TIMING, 1)
            e0 = ev()
            c.set_target(tgt, nrm, w["dmax"])
            e1 = ev()
            if P > 1:
                c.dist_init_loopback(r, P)
            c.set_source(src, T0)
            e2 = ev()
            torch.cuda.synchronize()
            st.append(e0.elapsed_time(e1))
            ss.append(e1.elapsed_time(e2))
        if P == 1:
            res = ctxs[0].run(T0, iters, 0.0, 0.0)
        else:
            res = o3g.loopback_run(ctxs, T0, iters, 0.0, 0.0)
        k3 = []
        for c in ctxs:
            k3_ms, k3_n, _ = c.last_run_kernel_ms()
            k3.append(k3_ms)
        if rep:
            rows.append((max(st), max(ss), max(k3), res.passes, res.fitness, k3))
    for c in ctxs:
        c.close()
    med = lambda i: statistics.median(r[i] for r in rows)
    print(json.dumps({"config": a.config, "world": P, "set_target_ms": med(0), "set_source_ms_max_rank": med(1),
                      "k3_total_ms_max_rank": med(2), "passes": rows[0][3],
                      "k3_per_pass_ms_max_rank": med(2) / rows[0][3], "fitness": rows[0][4],
                      "k3_per_pass_ms_by_rank": [round(x / rows[0][3], 4) for x in rows[-1][5]],
                      "shard_live_weight": os.environ.get("O3G_SHARD_LIVE_WEIGHT", "8")}), flush=True)
