#!/usr/bin/env python
"""Per-pass motion of the source under the ICP loop (design data for the
correspondence certificates): for k = 0..K the transform
T_k after k updates (ctx.run with max_iterations = k), the per-point
displacement |T_k s - T_{k-1} s| (percentiles), the cumulative displacement
since pass 0 and the fraction of queries whose winner changed between
consecutive passes (ctx.step at T_k). Not a benchmark."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large16m")
ap.add_argument("--regime", default="init", choices=["init", "converged"])
ap.add_argument("--iters", type=int, default=None)
ap.add_argument("--sample", type=int, default=2_000_000)
a = ap.parse_args()

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_09847_b200 as o3g  # noqa: E402
from bench import load_workload  # noqa: E402

w = load_workload(a.config)
if "scales" in w:
    w = w["scales"][-1]
if a.regime == "converged":
    from synth.rng import Stream
    from synth.scenes import rigid, rotation
    rs = Stream(0x5EED)
    w = dict(w, init_T=w["T_true"] @ rigid(rotation(rs.unit_vectors(1)[0], np.deg2rad(0.1)),
                                             0.01 * rs.unit_vectors(1)[0]))
dev = torch.device("cuda:0")
src, tgt, nrm = (torch.from_numpy(w[k]).to(dev) for k in ("source", "target", "target_normals"))
K = a.iters if a.iters is not None else w["iters"]
ctx = o3g.Context(0)
ctx.set_target(tgt, nrm, w["dmax"])
ctx.set_source(src, w["init_T"])
Ts = [np.asarray(w["init_T"], dtype=np.float64)]
for k in range(1, K + 1):
    Ts.append(ctx.run(w["init_T"], k, 0.0, 0.0).transformation)
g = torch.Generator(device="cpu").manual_seed(7)
idx = torch.randperm(len(src), generator=g)[: min(a.sample, len(src))].to(dev)
s = src[idx].double()
sh = torch.cat([s, torch.ones(len(s), 1, dtype=torch.float64, device=dev)], 1)


def P(T):
    return sh @ torch.from_numpy(np.asarray(T)).to(dev).T[:, :3]


corr_prev = None
rows = []
p0 = P(Ts[0])
for k in range(K + 1):
    corr = torch.empty(len(src), dtype=torch.int32, device=dev)
    st = ctx.step(Ts[k], corr_out=corr)
    row = {"pass": k, "fitness": st["count"] / len(src)}
    if k > 0:
        d = (P(Ts[k]) - P(Ts[k - 1])).norm(dim=1)
        q = torch.quantile(d.float()[: 1_000_000], torch.tensor([0.5, 0.9, 0.99], device=dev)).tolist()
        row.update(step_p50=q[0], step_p90=q[1], step_p99=q[2], step_max=float(d.max()),
                   cum_max=float((P(Ts[k]) - p0).norm(dim=1).max()))
        row["winner_changed"] = float((corr != corr_prev).float().mean())
    corr_prev = corr
    rows.append(row)
    print(json.dumps(row), flush=True)
