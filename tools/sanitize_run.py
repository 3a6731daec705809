#!/usr/bin/env python
"""Exercise every C-ABI path on small inputs (for compute-sanitizer runs):
step (all K3 variants, dense + hashed grids, corr output), run (graph loop),
one-shot host/device, point-to-point, batched evaluation, voxel downsample,
multi-scale driver, invalid arguments."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_09847_b200 as o3g  # noqa: E402
from synth import make  # noqa: E402

w = make("tiny")
d = make("depth")
dev = torch.device("cuda:0")
for wl in (w, d):
    src = torch.from_numpy(wl["source"]).to(dev)
    tgt = torch.from_numpy(wl["target"]).to(dev)
    nrm = torch.from_numpy(wl["target_normals"]).to(dev)
    for variant in (0, 1, 2, 3):
        for grid in (1, 2):
            with o3g.Context(0) as ctx:
                ctx.set_option(1, variant)
                ctx.set_option(2, grid)
                ctx.set_target(tgt, nrm, wl["dmax"])
                ctx.set_source(src, wl["init_T"])
                corr = torch.empty(len(src), dtype=torch.int32, device=dev)
                ctx.step(wl["T_true"], corr_out=corr)
                ctx.run(wl["init_T"], 5, 0.0, 0.0, history=True)
    with o3g.Context(0) as ctx:
        ctx.set_option(6, 1)                      # every query cooperative
        ctx.set_target(tgt, nrm, wl["dmax"])
        ctx.set_source(src)
        ctx.run(wl["init_T"], 3)
        ctx.evaluate(np.stack([wl["T_true"], wl["init_T"]]))
        ctx.voxel_down_sample(tgt, 0.03, nrm)
    o3g.icp_point_to_plane(wl["source"], wl["target"], wl["target_normals"], wl["dmax"], max_iterations=3)
    o3g.icp_point_to_point(src, tgt, wl["dmax"], max_iterations=3)
f = make("fragment", n=60_000)
with o3g.Context(0) as ctx:
    vox = [s["meta"]["voxel"] for s in f["scales"]]
    ctx.run_multiscale(f["source"], f["target"], f["target_normals"], vox,
                       [s["dmax"] for s in f["scales"]], [3, 3, 3])
try:
    o3g.icp_point_to_plane(np.zeros((0, 3)), w["target"], w["target_normals"], 0.05)
except o3g.InvalidArgument:
    pass
torch.cuda.synchronize()
print("sanitize run ok")
