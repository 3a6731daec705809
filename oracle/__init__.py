"""CPU oracle for the point-to-plane ICP iteration — TEST INFRASTRUCTURE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path
(paper_1801_09847_b200) never imports it and shares no code with it.

This module is argument marshalling (ctypes) over ``o3g_oracle.c``; every
step of the method is in that C file, which cites PAPER.md / SPEC.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "o3g_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-fPIC", "-shared", "-fopenmp"]

NTERMS = 29
FLAG_NO_CORR = 1
FLAG_DEGENERATE = 2


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P, D, I64, I32 = C.c_void_p, C.c_double, C.c_int64, C.c_int32
        L.orc_grid_build.restype = P
        L.orc_grid_build.argtypes = [P, I64, D]
        L.orc_grid_free.argtypes = [P]
        L.orc_transform.argtypes = [P, P, I64, P]
        L.orc_nn_brute.restype = I64
        L.orc_nn_brute.argtypes = [P, P, I64, D, P]
        L.orc_nn_grid.restype = I64
        L.orc_nn_grid.argtypes = [P, P, D, P]
        L.orc_pass_subset.argtypes = [P, P, I64, P, I64, P, P, I64, P, D, P, P, P, P]
        L.orc_pass_chunked.restype = C.c_int
        L.orc_pass_chunked.argtypes = [P, P, I64, P, I64, P, P, I64, P, D, P, P, P, P, I32]
        L.orc_expand_jtj.argtypes = [P, P]
        L.orc_ldlt_solve.restype = C.c_int
        L.orc_ldlt_solve.argtypes = [P, P, P]
        L.orc_exp_se3.argtypes = [P, P]
        L.orc_compose.argtypes = [P, P, P]
        L.orc_icp.restype = C.c_int
        L.orc_icp.argtypes = [P, I64, P, P, I64, P, D, I32, D, D, I32, P, P, P, P, P, P, P, P, I32]
        L.orc_voxel_down_sample.restype = I64
        L.orc_voxel_down_sample.argtypes = [P, P, I64, D, P, P]
        L.orc_pass_p2p.argtypes = [P, P, I64, P, I64, P, D, P, P]
        L.orc_kabsch.restype = C.c_int
        L.orc_kabsch.argtypes = [P, P]
        L.orc_icp_p2p.restype = C.c_int
        L.orc_icp_p2p.argtypes = [P, I64, P, I64, P, D, I32, D, D, P, P, P, P, P, P]
        L.orc_estimate_normals.restype = I64
        L.orc_estimate_normals.argtypes = [P, I64, D, I32, P, P]
        L.orc_icp_multiscale.restype = C.c_int
        L.orc_icp_multiscale.argtypes = [P, I64, P, P, I64, P, I32, P, P, P, D, D, P, P, P, P, P, I32]
        _lib = L
    return _lib


def _p(a):
    # the ctypes view keeps the array alive for the duration of the call
    # (a bare .ctypes.data of a temporary copy would dangle)
    return a.ctypes if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Grid:
    """Grid accelerator over the target (checked equal to brute force)."""

    def __init__(self, target, dmax):
        self.target = _f32(target)
        self.dmax = float(dmax)
        self.h = lib().orc_grid_build(_p(self.target), len(self.target), self.dmax)
        if not self.h:
            raise MemoryError("oracle grid build failed")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_grid_free(self.h)
            self.h = None


def transform(T, pts):
    pts = _f32(pts)
    out = np.empty((len(pts), 3), np.float64)
    lib().orc_transform(_p(_f64(T)), _p(pts), len(pts), _p(out))
    return out


def nn(s, target, dmax, grid: Grid | None = None):
    """1-NN of one transformed query s (fp64 3-vector): (index or -1, d2)."""
    s = _f64(s)
    d2 = np.zeros(1)
    if grid is None:
        tg = _f32(target)
        j = lib().orc_nn_brute(_p(s), _p(tg), len(tg), float(dmax) * float(dmax), _p(d2))
    else:
        j = lib().orc_nn_grid(grid.h, _p(s), grid.dmax * grid.dmax, _p(d2))
    return int(j), float(d2[0])


def step(T, source, target, normals, dmax, grid: Grid | None | str = "auto", subset=None,
         threads: int | None = None):
    """One pass at fixed T (icp_step semantics). Returns dict(corr, d2,
    terms[29], abs_terms[29], JTJ (6x6), JTr (6), count, sum_sq_dist).
    ``subset``: optional source indices; corr/d2 then follow that order and
    the terms sum over the subset only. ``threads``: None = the sequential
    pass; k >= 1 = the deterministic chunked OpenMP pass on k threads
    (bitwise the same result for every k)."""
    src, tgt, nrm = _f32(source), _f32(target), _f32(normals)
    if isinstance(grid, str):
        grid = Grid(tgt, dmax) if len(tgt) * len(src) > 4_000_000 else None
    idx = None if subset is None else np.ascontiguousarray(subset, dtype=np.int64)
    k = len(src) if idx is None else len(idx)
    corr = np.empty(k, np.int32)
    d2 = np.empty(k, np.float64)
    sums = np.zeros(NTERMS)
    abss = np.zeros(NTERMS)
    if threads is None:
        lib().orc_pass_subset(_p(_f64(T)), _p(src), len(src), _p(idx), k, _p(tgt), _p(nrm), len(tgt),
                              grid.h if grid is not None else None, float(dmax),
                              _p(corr), _p(d2), _p(sums), _p(abss))
    elif lib().orc_pass_chunked(_p(_f64(T)), _p(src), len(src), _p(idx), k, _p(tgt), _p(nrm), len(tgt),
                                grid.h if grid is not None else None, float(dmax),
                                _p(corr), _p(d2), _p(sums), _p(abss), int(threads)):
        raise MemoryError("oracle chunked pass failed")
    JTJ = np.zeros(36)
    lib().orc_expand_jtj(_p(sums), _p(JTJ))
    return dict(corr=corr, d2=d2, terms=sums, abs_terms=abss, JTJ=JTJ.reshape(6, 6),
                JTr=sums[21:27].copy(), count=sums[27], sum_sq_dist=sums[28])


def ldlt_solve(A, b):
    """x with A x = b by LDL^T without pivoting; None if singular."""
    x = np.zeros(6)
    rc = lib().orc_ldlt_solve(_p(_f64(A)), _p(_f64(b)), _p(x))
    return None if rc else x


def exp_se3(xi):
    T = np.zeros(16)
    lib().orc_exp_se3(_p(_f64(xi)), _p(T))
    return T.reshape(4, 4)


def compose(A, B):
    out = np.zeros(16)
    lib().orc_compose(_p(_f64(A)), _p(_f64(B)), _p(out))
    return out.reshape(4, 4)


def icp(source, target, normals, dmax, max_iterations, init_T=None, relative_fitness=1e-6,
        relative_rmse=1e-6, use_grid=True, threads: int = 0):
    """registration_icp, point-to-plane. Returns dict(T, fitness, inlier_rmse,
    iterations, flags, converged, passes, hist_fitness, hist_rmse).
    ``threads`` > 0: every pass is the deterministic chunked OpenMP pass."""
    src, tgt, nrm = _f32(source), _f32(target), _f32(normals)
    T0 = _f64(np.eye(4) if init_T is None else init_T)
    T = np.zeros(16)
    fit, rmse = np.zeros(1), np.zeros(1)
    it, fl, cv = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32)
    hf = np.zeros(max_iterations + 1)
    hr = np.zeros(max_iterations + 1)
    passes = lib().orc_icp(_p(src), len(src), _p(tgt), _p(nrm), len(tgt), _p(T0), float(dmax),
                           int(max_iterations), float(relative_fitness), float(relative_rmse),
                           1 if use_grid else 0, _p(T), _p(fit), _p(rmse), _p(it), _p(fl), _p(cv),
                           _p(hf), _p(hr), int(threads))
    if passes < 0:
        raise MemoryError("oracle icp failed")
    return dict(T=T.reshape(4, 4), fitness=float(fit[0]), inlier_rmse=float(rmse[0]),
                iterations=int(it[0]), flags=int(fl[0]), converged=bool(cv[0]), passes=passes,
                hist_fitness=hf[:passes].copy(), hist_rmse=hr[:passes].copy())


def voxel_down_sample(points, voxel, normals=None):
    """SPEC S:58-61 voxel_down_sample (see o3g_oracle.c). Returns (points,
    normals or None) as float32 arrays in ascending (ix, iy, iz) order."""
    p = _f32(points)
    nr = None if normals is None else _f32(normals)
    out_p = np.empty_like(p)
    out_n = None if nr is None else np.empty_like(nr)
    k = lib().orc_voxel_down_sample(_p(p), _p(nr), len(p), float(voxel), _p(out_p), _p(out_n))
    if k < 0:
        raise ValueError("voxel_down_sample: invalid input")
    return out_p[:k].copy(), (None if out_n is None else out_n[:k].copy())


def icp_multiscale(source, target, normals, voxels, dmaxs, iters, init_T=None,
                   relative_fitness=1e-6, relative_rmse=1e-6, threads: int = 0):
    """Multi-scale point-to-plane ICP (downsample per scale, carry T)."""
    src, tgt, nrm = _f32(source), _f32(target), _f32(normals)
    ns = len(voxels)
    T0 = _f64(np.eye(4) if init_T is None else init_T)
    T = np.zeros(16)
    fit, rmse = np.zeros(ns), np.zeros(ns)
    its = np.zeros(ns, np.int32)
    nss = np.zeros(ns, np.int64)
    rc = lib().orc_icp_multiscale(_p(src), len(src), _p(tgt), _p(nrm), len(tgt), _p(T0), ns,
                                  _p(_f64(voxels)), _p(_f64(dmaxs)),
                                  _p(np.ascontiguousarray(iters, np.int32)), float(relative_fitness),
                                  float(relative_rmse), _p(T), _p(fit), _p(rmse), _p(its), _p(nss),
                                  int(threads))
    if rc != 0:
        raise RuntimeError("oracle multiscale failed")
    return dict(T=T.reshape(4, 4), fitness=fit, inlier_rmse=rmse, iterations=its, n_source=nss)


def step_p2p(T, source, target, dmax, grid: Grid | None = None):
    """Point-to-point pass at fixed T: corr and the 29 p2p terms
    ([0..8] sum s'q^T, [9..11] sum s', [12..14] sum q, [27] count, [28] sum d2)."""
    src, tgt = _f32(source), _f32(target)
    corr = np.empty(len(src), np.int32)
    sums = np.zeros(NTERMS)
    lib().orc_pass_p2p(_p(_f64(T)), _p(src), len(src), _p(tgt), len(tgt),
                       grid.h if grid is not None else None, float(dmax), _p(corr), _p(sums))
    return dict(corr=corr, terms=sums, count=sums[27], sum_sq_dist=sums[28])


def kabsch(terms):
    """Rigid transform from p2p terms, or None if degenerate."""
    T = np.zeros(16)
    rc = lib().orc_kabsch(_p(_f64(terms)), _p(T))
    return None if rc else T.reshape(4, 4)


def icp_p2p(source, target, dmax, max_iterations, init_T=None, relative_fitness=1e-6,
            relative_rmse=1e-6):
    """registration_icp with TransformationEstimationPointToPoint(False)."""
    src, tgt = _f32(source), _f32(target)
    T0 = _f64(np.eye(4) if init_T is None else init_T)
    T = np.zeros(16)
    fit, rmse = np.zeros(1), np.zeros(1)
    it, fl, cv = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32)
    passes = lib().orc_icp_p2p(_p(src), len(src), _p(tgt), len(tgt), _p(T0), float(dmax),
                               int(max_iterations), float(relative_fitness), float(relative_rmse),
                               _p(T), _p(fit), _p(rmse), _p(it), _p(fl), _p(cv))
    if passes < 0:
        raise MemoryError("oracle icp_p2p failed")
    return dict(T=T.reshape(4, 4), fitness=float(fit[0]), inlier_rmse=float(rmse[0]),
                iterations=int(it[0]), flags=int(fl[0]), converged=bool(cv[0]), passes=passes)


def estimate_normals(points, radius=0.1, max_nn=30):
    """SPEC S:67-75 hybrid-neighbourhood PCA normals. Returns (normals f32,
    neighbour counts, number of < 3-neighbour fallbacks)."""
    p = _f32(points)
    out = np.empty_like(p)
    cnt = np.empty(len(p), np.int32)
    fb = lib().orc_estimate_normals(_p(p), len(p), float(radius), int(max_nn), _p(out), _p(cnt))
    if fb < 0:
        raise ValueError("estimate_normals: invalid input")
    return out, cnt, int(fb)
