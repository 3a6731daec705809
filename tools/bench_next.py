#!/usr/bin/env python
"""Timings of the SURVEY §8(f) NEXT rows on one B200 (device-resident inputs,
CUDA events, median of --reps after 2 warm-ups): f1 voxel_down_sample, f2
point-to-point ICP, f3 batched evaluate_registration, f4 hybrid-KNN normals.
One JSON line per row (profiles/r02_next_rows.jsonl)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1801_09847_b200 as o3g  # noqa: E402
from synth import make  # noqa: E402


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return float(np.median(ms)), float(min(ms)), float(max(ms)), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    w = make("fragment")                      # 2M / 2M raw clouds (multi-scale config)
    src = torch.from_numpy(w["source"]).to(dev)
    tgt = torch.from_numpy(w["target"]).to(dev)
    nrm = torch.from_numpy(w["target_normals"]).to(dev)
    n, m = len(src), len(tgt)
    with o3g.Context(0) as ctx:
        # f1: voxel downsample of the 2M-point target with normals, voxel 0.02 (scale 2 of the config)
        med, lo, hi, out = timed(lambda: ctx.voxel_down_sample(tgt, 0.02, nrm), a.reps)
        k = len(out[0])
        rows.append(dict(row="f1 voxel_down_sample", n_in=m, n_out=k, voxel=0.02, ms=med, ms_min=lo, ms_max=hi,
                         mpts_per_s=m / med / 1e3, alg_gbs=(24 * m + 24 * k) / med / 1e6))
        # f4: normals of the downsampled target, hybrid(radius 0.06, max_nn 30)
        pts = out[0].contiguous()
        med, lo, hi, res = timed(lambda: ctx.estimate_normals(pts, 0.06, 30), a.reps)
        rows.append(dict(row="f4 estimate_normals hybrid(0.06, 30)", n=len(pts), ms=med, ms_min=lo, ms_max=hi,
                         mpts_per_s=len(pts) / med / 1e3, fallbacks=int(res[2])))
    w2 = make("large16m", n=4_000_000)        # 4M / 4M of the large scene
    s2 = torch.from_numpy(w2["source"]).to(dev)
    t2 = torch.from_numpy(w2["target"]).to(dev)
    n2 = torch.from_numpy(w2["target_normals"]).to(dev)
    T0 = w2["T_true"]
    with o3g.Context(0) as ctx:
        ctx.set_target(t2, n2, w2["dmax"])
        ctx.set_source(s2, T0)
        # f3: 64 hypotheses around T* in one launch
        rng = np.random.default_rng(7)
        Ts = []
        for _ in range(64):
            ax = rng.normal(size=3)
            ax /= np.linalg.norm(ax)
            ang = np.deg2rad(0.2) * rng.uniform()
            K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
            P = np.eye(4)
            P[:3, :3] = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K
            P[:3, 3] = rng.uniform(-0.02, 0.02, 3)
            Ts.append(T0 @ P)
        med, lo, hi, ev = timed(lambda: ctx.evaluate(np.stack(Ts)), a.reps)
        rows.append(dict(row="f3 evaluate_registration x64", n_source=len(s2), k=64, ms=med, ms_min=lo, ms_max=hi,
                         src_pt_evals_per_s=64 * len(s2) / med * 1e3, fitness_max=float(ev[0].max())))
        # f2: point-to-point ICP, 10 iterations from a 0.2 deg / 2 cm start
        ctx.set_option(o3g.OPT_ESTIMATION, 1)
        ctx.set_source(s2, Ts[0])
        med, lo, hi, r = timed(lambda: ctx.run(Ts[0], 10, 0.0, 0.0), a.reps)
        rows.append(dict(row="f2 point-to-point ICP, 10 iterations", n_source=len(s2), ms=med, ms_min=lo, ms_max=hi,
                         src_pt_it_per_s=len(s2) * r.iterations / med * 1e3, fitness=r.fitness))
        ctx.set_option(o3g.OPT_ESTIMATION, 0)
        ctx.set_source(s2, Ts[0])
        med, lo, hi, r = timed(lambda: ctx.run(Ts[0], 10, 0.0, 0.0), a.reps)
        rows.append(dict(row="(point-to-plane, same start, for comparison)", n_source=len(s2), ms=med, ms_min=lo,
                         ms_max=hi, src_pt_it_per_s=len(s2) * r.iterations / med * 1e3, fitness=r.fitness))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
