#!/usr/bin/env python
"""A/B of the correspondence pass across in-tree library builds (raw ctypes,
only the round-1 ABI subset): K3 ms per pass (O3G_OPT_TIMING events) and the
loop time for a config/regime, alternating libraries. Not a benchmark.
usage: ab_k3.py lib1.so lib2.so ... [--config large16m] [--regime init] [--reps 3]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--config", default="large16m")
ap.add_argument("--regime", default="init")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--iters", type=int, default=None, help="updates (default: the config's)")
ap.add_argument("--opt", action="append", default=[], help="option=value applied to every library")
a = ap.parse_args()

import numpy as np  # noqa: E402
import torch  # noqa: E402
from bench import load_workload  # noqa: E402

w = load_workload(a.config)
if "scales" in w:
    w = w["scales"][-1]
T0 = w["init_T"]
if a.regime == "converged":
    from synth.rng import Stream
    from synth.scenes import rigid, rotation
    rs = Stream(0x5EED)
    T0 = w["T_true"] @ rigid(rotation(rs.unit_vectors(1)[0], np.deg2rad(0.1)), 0.01 * rs.unit_vectors(1)[0])
dev = torch.device("cuda:0")
src, tgt, nrm = (torch.from_numpy(w[k]).to(dev) for k in ("source", "target", "target_normals"))
T0 = np.ascontiguousarray(T0, np.float64).reshape(16)
libs = []
for path in a.libs:
    L = C.CDLL(os.path.abspath(path))
    P, D, I32, I64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64
    for name, args in {"o3g_create": [P, C.c_int, P], "o3g_set_target": [P, P, P, I64, D],
                       "o3g_set_source": [P, P, I64, P], "o3g_set_option": [P, C.c_int, I64],
                       "o3g_icp_run": [P, P, I32, D, D, P, P, P, P, P, P],
                       "o3g_last_run_kernel_ms": [P, P, P, P]}.items():
        getattr(L, name).argtypes = args
        getattr(L, name).restype = C.c_int
    h = C.c_void_p()
    assert L.o3g_create(C.byref(h), 0, None) == 0
    assert L.o3g_set_target(h, tgt.data_ptr(), nrm.data_ptr(), len(tgt), w["dmax"]) == 0
    assert L.o3g_set_source(h, src.data_ptr(), len(src), T0.ctypes.data) == 0
    assert L.o3g_set_option(h, 3, 1) == 0
    for o in a.opt:
        k, v = o.split("=")
        L.o3g_set_option(h, int(k), int(v))
    libs.append((os.path.basename(path), L, h))
T = np.zeros(16)
fit, rmse = C.c_double(), C.c_double()
res = {name: [] for name, _, _ in libs}
for rep in range(a.reps + 1):
    for name, L, h in libs:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.o3g_icp_run(h, T0.ctypes.data, w["iters"] if a.iters is None else a.iters, 0.0, 0.0,
                             T.ctypes.data, C.byref(fit), C.byref(rmse),
                             None, None, None) == 0
        e1.record()
        torch.cuda.synchronize()
        k3, kn, tail = C.c_double(), C.c_int32(), C.c_double()
        L.o3g_last_run_kernel_ms(h, C.byref(k3), C.byref(kn), C.byref(tail))
        if rep:
            res[name].append((k3.value / kn.value, e0.elapsed_time(e1), fit.value))
for name, v in res.items():
    print(f"{a.config:9s} {a.regime:9s} {name:16s} k3/pass {min(x[0] for x in v):.4f} ms  loop {min(x[1] for x in v):.2f} ms  fitness {v[0][2]:.6f}")
