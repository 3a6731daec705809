#!/usr/bin/env python
"""T_k after k updates (k = 0..K) of a registration (ctx.run with
max_iterations = k), written as JSON (design data for certificate policies;
not a benchmark)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large16m")
ap.add_argument("--regime", default="init", choices=["init", "converged"])
ap.add_argument("--iters", type=int, default=None)
a = ap.parse_args()

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_09847_b200 as o3g  # noqa: E402
from bench import load_workload  # noqa: E402

w = load_workload(a.config)
T0 = np.asarray(w["init_T"], dtype=np.float64)
if a.regime == "converged":
    from synth.rng import Stream
    from synth.scenes import rigid, rotation
    rs = Stream(0x5EED)
    T0 = w["T_true"] @ rigid(rotation(rs.unit_vectors(1)[0], np.deg2rad(0.1)), 0.01 * rs.unit_vectors(1)[0])
dev = torch.device("cuda:0")
src, tgt, nrm = (torch.from_numpy(w[k]).to(dev) for k in ("source", "target", "target_normals"))
K = a.iters if a.iters is not None else w["iters"]
ctx = o3g.Context(0)
ctx.set_target(tgt, nrm, w["dmax"])
ctx.set_source(src, T0)
Ts = [T0.tolist()] + [ctx.run(T0, k, 0.0, 0.0).transformation.tolist() for k in range(1, K + 1)]
print(json.dumps({"config": a.config, "regime": a.regime, "T": Ts}))
