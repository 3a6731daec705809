#!/usr/bin/env python
"""Per-pass statistics of one registration (o3g_last_run_trace): fitness,
queries that ran the full correspondence search (the rest were settled by
the live-query bitmap or a certificate) and candidates scanned, with and
without correspondence certificates; K3 time per pass (CUDA events). Not a
benchmark."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large16m")
ap.add_argument("--regime", default="init", choices=["init", "converged"])
ap.add_argument("--iters", type=int, default=None)
ap.add_argument("--certs", default="1,0", help="O3G_OPT_CERT values to compare (2 = forced)")
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
n = len(src)
out = {}
certs = [int(x) for x in a.certs.split(",")]
for cert in certs:
    ctx.set_option(o3g.OPT_CERT, cert)
    ctx.set_option(o3g.OPT_TIMING, 1)
    for _ in range(2):
        r = ctx.run(w["init_T"], K, 0.0, 0.0, history=True)
    k3_ms, k3_n, _ = ctx.last_run_kernel_ms()
    tr = ctx.last_run_trace(r.passes)
    out[cert] = dict(k3_ms_per_pass=k3_ms / k3_n, fitness=r.hist_fitness.tolist(),
                     searched_frac=(tr["searched"] / n).tolist(),
                     cert_frac=(tr["certified"] / n).tolist(),
                     cand_per_search=(tr["candidates"] / np.maximum(tr["searched"], 1)).tolist())
    print(json.dumps({"config": a.config, "regime": a.regime, "cert": cert, "n": n,
                      "k3_ms_per_pass": round(k3_ms / k3_n, 4)}), flush=True)
for k in range(r.passes):
    print(k, *(f"{out[c]['fitness'][k]:.4f} srch={out[c]['searched_frac'][k]:.3f} cert={out[c]['cert_frac'][k]:.3f} cand={out[c]['cand_per_search'][k]:.1f}"
               for c in certs))
