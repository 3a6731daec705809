"""Seeded synthetic workloads shaped like BASELINE.json's five configs.

Inputs only — this module holds none of the ICP method's arithmetic (no
transform-of-source inside the method, no search, no residuals). It is the
one module both the oracle side and the CUDA side consume (DESIGN.md
"Input recipe"). Unspecified constants are the SURVEY.md §8(d) proposals and
are recorded in each workload's ``meta``.

Every workload is a dict:
  source (N,3) f32, target (M,3) f32, target_normals (M,3) f32,
  dmax (float), iters (int), init_T (4,4) f64, T_true (4,4) f64 (maps the
  source frame onto the target frame), name, meta.
The fragment config additionally carries ``scales``: a list of per-scale
dicts with the same keys (host-side voxel downsampling, S:58-61 semantics).
"""
from __future__ import annotations

import math

import numpy as np

from .rng import Stream, config_seed

CONFIG_IDS = {"tiny": 1, "depth": 2, "lidar": 3, "fragment": 4, "large16m": 5}


# ----------------------------------------------------------------- helpers
def rotation(axis: np.ndarray, angle: float) -> np.ndarray:
    """Rotation matrix about a unit axis (input construction only)."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * (K @ K)


def rigid(R: np.ndarray, t) -> np.ndarray:
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = t
    return T


def apply(T: np.ndarray, p: np.ndarray) -> np.ndarray:
    out = np.empty_like(p, dtype=np.float64)
    for i in range(3):
        out[:, i] = p[:, 0] * T[i, 0] + p[:, 1] * T[i, 1] + p[:, 2] * T[i, 2] + T[i, 3]
    return out


def inv_rigid(T: np.ndarray) -> np.ndarray:
    R = T[:3, :3]
    return rigid(R.T, -R.T @ T[:3, 3])


class Rects:
    """Axis-aligned rectangles (corner, edge1, edge2, normal) sampled by area."""

    def __init__(self):
        self.c, self.e1, self.e2, self.n = [], [], [], []

    def add(self, c, e1, e2, n):
        self.c.append(c), self.e1.append(e1), self.e2.append(e2), self.n.append(n)

    def add_box(self, lo, hi, bottom=False):
        lo, hi = np.asarray(lo, float), np.asarray(hi, float)
        sx, sy, sz = hi - lo
        X, Y, Z = np.eye(3)
        self.add(lo + [0, 0, sz], sx * X, sy * Y, Z)            # top
        if bottom:
            self.add(lo, sx * X, sy * Y, -Z)
        self.add(lo, sy * Y, sz * Z, -X)                        # x-
        self.add(lo + [sx, 0, 0], sy * Y, sz * Z, X)            # x+
        self.add(lo, sx * X, sz * Z, -Y)                        # y-
        self.add(lo + [0, sy, 0], sx * X, sz * Z, Y)            # y+

    def finish(self):
        self.c = np.array(self.c, float)
        self.e1 = np.array(self.e1, float)
        self.e2 = np.array(self.e2, float)
        self.n = np.array(self.n, float)
        self.area = np.linalg.norm(self.e1, axis=1) * np.linalg.norm(self.e2, axis=1)
        return self

    def sample(self, rs: Stream, n: int):
        cum = np.cumsum(self.area)
        k = np.searchsorted(cum, rs.uniform(n, 0.0, cum[-1]), side="right")
        k = np.minimum(k, len(self.area) - 1)
        a = rs.uniform(n)[:, None]
        b = rs.uniform(n)[:, None]
        p = self.c[k] + a * self.e1[k] + b * self.e2[k]
        return p, self.n[k].copy()


def voxel_down_sample(p: np.ndarray, n: np.ndarray | None, voxel: float):
    """mean per occupied voxel anchored at the min bound,
    floor semantics, ascending lexicographic (ix,iy,iz) order; normals
    averaged then renormalised. Input preprocessing for configs 2 and 4."""
    p64 = p.astype(np.float64)
    lo = p64.min(axis=0)
    ijk = np.floor((p64 - lo) / voxel).astype(np.int64)
    dims = ijk.max(axis=0) + 1
    key = (ijk[:, 0] * dims[1] + ijk[:, 1]) * dims[2] + ijk[:, 2]
    uniq, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    out = np.stack([np.bincount(inv, p64[:, a], len(uniq)) for a in range(3)], 1) / cnt[:, None]
    nout = None
    if n is not None:
        ns = np.stack([np.bincount(inv, n[:, a].astype(np.float64), len(uniq)) for a in range(3)], 1)
        norm = np.linalg.norm(ns, axis=1, keepdims=True)
        norm[norm == 0] = 1.0
        nout = (ns / norm).astype(np.float32)
    return out.astype(np.float32), nout


def ray_boxes(o: np.ndarray, d: np.ndarray, lo: np.ndarray, hi: np.ndarray, chunk=8192):
    """Nearest entry (t>0) of rays o + t d into axis-aligned boxes.
    Returns t (inf = miss) and the entry-face normal (facing the ray)."""
    n = d.shape[0]
    t_best = np.full(n, np.inf)
    nrm = np.zeros((n, 3))
    with np.errstate(divide="ignore", invalid="ignore"):
        for s in range(0, n, chunk):
            dd = d[s:s + chunk]
            inv = 1.0 / dd
            t1 = (lo[None] - o) * inv[:, None, :]
            t2 = (hi[None] - o) * inv[:, None, :]
            tn = np.minimum(t1, t2)
            tf = np.maximum(t1, t2)
            tn = np.where(np.isnan(tn), -np.inf, tn)
            tf = np.where(np.isnan(tf), np.inf, tf)
            tmin = tn.max(axis=2)
            tmax = tf.min(axis=2)
            hit = (tmax >= tmin) & (tmin > 1e-9)
            tmin = np.where(hit, tmin, np.inf)
            kb = tmin.argmin(axis=1)
            tb = tmin[np.arange(len(dd)), kb]
            ax = tn[np.arange(len(dd)), kb].argmax(axis=1)
            nn = np.zeros((len(dd), 3))
            nn[np.arange(len(dd)), ax] = -np.sign(dd[np.arange(len(dd)), ax])
            t_best[s:s + chunk] = tb
            nrm[s:s + chunk] = nn
    return t_best, nrm


def _pack(name, src, tgt, nrm, dmax, iters, init_T, T_true, meta):
    return dict(name=name, source=np.ascontiguousarray(src, np.float32),
                target=np.ascontiguousarray(tgt, np.float32),
                target_normals=np.ascontiguousarray(nrm, np.float32),
                dmax=float(dmax), iters=int(iters), init_T=np.asarray(init_T, np.float64),
                T_true=np.asarray(T_true, np.float64), meta=meta)


# ----------------------------------------------------------------- configs
def tiny(n: int = 5000) -> dict:
    """Config 1: unit sphere ∪ z=-1 patch [-1.5,1.5]^2, analytic normals."""
    cid = CONFIG_IDS["tiny"]
    p_sph = 4 * math.pi / (4 * math.pi + 9.0)

    def draw(rs, n):
        on_s = rs.uniform(n) < p_sph
        v = rs.unit_vectors(n)
        xy = np.stack([rs.uniform(n, -1.5, 1.5), rs.uniform(n, -1.5, 1.5)], 1)
        p = np.where(on_s[:, None], v, np.concatenate([xy, -np.ones((n, 1))], 1))
        nr = np.where(on_s[:, None], v, np.array([0.0, 0.0, 1.0]))
        return p, nr

    tgt, nrm = draw(Stream(config_seed(cid, 0)), n)
    rs = Stream(config_seed(cid, 1))
    src, _ = draw(rs, n)
    src = src + 0.002 * np.stack([rs.normal(n) for _ in range(3)], 1)
    axis = rs.unit_vectors(1)[0]
    M = rigid(rotation(axis, math.radians(5.0)), rs.uniform(3, -0.05, 0.05))
    src = apply(M, src)
    return _pack("tiny", src, tgt, nrm, 0.05, 20, np.eye(4), inv_rigid(M),
                 dict(config_id=cid, n=n, motion_axis=axis.tolist()))


def depth(width=640, height=480) -> dict:
    """Config 2: ray-cast depth frames of a room (5 planes + 30 boxes),
    fx=fy=525, cx=319.5, cy=239.5, noise 0.001 z^2, voxel 0.02."""
    cid = CONFIG_IDS["depth"]
    rs = Stream(config_seed(cid, 0))
    room_lo = np.array([-3.5, -1.75, -10.0])
    room_hi = np.array([3.5, 1.75, 5.6])            # (proposal) tuned to ~60k points
    sz = rs.uniform(90, 0.2, 0.8).reshape(30, 3)
    ctr = np.stack([rs.uniform(30, -2.2, 2.2), rs.uniform(30, -1.1, 1.1),
                    rs.uniform(30, 1.0, 4.3 - 0.5)], 1)
    blo, bhi = ctr - sz / 2, ctr + sz / 2
    fx = fy = 525.0
    cx, cy = 319.5, 239.5
    u, v = np.meshgrid(np.arange(width, dtype=np.float64), np.arange(height, dtype=np.float64))
    dcam = np.stack([(u.ravel() - cx) / fx, (v.ravel() - cy) / fy, np.ones(u.size)], 1)

    def render(Rc, tc, rs_noise):
        dw = dcam @ Rc.T
        tb, nb = ray_boxes(tc, dw, blo, bhi)
        with np.errstate(divide="ignore"):
            tw = np.where(dw > 0, (room_hi - tc) / dw, (room_lo - tc) / dw)
        tw = np.where(np.isfinite(tw) & (tw > 0), tw, np.inf)
        ax = tw.argmin(axis=1)
        t_room = tw[np.arange(len(dw)), ax]
        n_room = np.zeros_like(dw)
        n_room[np.arange(len(dw)), ax] = -np.sign(dw[np.arange(len(dw)), ax])
        use_box = tb < t_room
        z = np.where(use_box, tb, t_room)           # ray param == depth (d_cam.z = 1)
        nw = np.where(use_box[:, None], nb, n_room)
        z = z + 0.001 * z * z * rs_noise.normal(len(z))
        ok = np.isfinite(z) & (z > 0)
        pc = dcam[ok] * z[ok, None]                  # back-projection
        nc = nw[ok] @ Rc                             # world normal -> camera frame
        return pc, nc

    tgt, tn = render(np.eye(3), np.zeros(3), Stream(config_seed(cid, 1)))
    rs2 = Stream(config_seed(cid, 2))
    axis = rs2.unit_vectors(1)[0]
    tdir = rs2.unit_vectors(1)[0]
    R2 = rotation(axis, math.radians(2.0))
    t2 = 0.03 * tdir
    src, _ = render(R2, t2, Stream(config_seed(cid, 3)))
    tgt_d, tn_d = voxel_down_sample(tgt, tn, 0.02)
    src_d, _ = voxel_down_sample(src, None, 0.02)
    return _pack("depth", src_d, tgt_d, tn_d, 0.07, 30, np.eye(4), rigid(R2, t2),
                 dict(config_id=cid, raw_points=(len(src), len(tgt)), voxel=0.02,
                      room=[room_lo.tolist(), room_hi.tolist()]))


def lidar() -> dict:
    """Config 3: 64 x 2048 beams, elevation -25..15 deg, ground + 400 boxes,
    ranges 1..80 m, radial noise 0.02; scan 2 = 1 deg yaw + 0.5 m forward."""
    cid = CONFIG_IDS["lidar"]
    rs = Stream(config_seed(cid, 0))
    h = 1.8                                          # (proposal) sensor height
    boxes = []
    while len(boxes) < 400:
        r = np.sqrt(rs.uniform(1, 9.0, 4900.0))[0]
        th = rs.uniform(1, 0, 2 * math.pi)[0]
        s = np.array([rs.uniform(1, 1, 10)[0], rs.uniform(1, 1, 10)[0], rs.uniform(1, 1, 8)[0]])
        c = np.array([r * math.cos(th), r * math.sin(th)])
        lo = np.array([c[0] - s[0] / 2, c[1] - s[1] / 2, 0.0])
        hi = np.array([c[0] + s[0] / 2, c[1] + s[1] / 2, s[2]])
        # keep both sensor positions outside every box (1 m margin)
        if any(lo[0] - 1 < px < hi[0] + 1 and lo[1] - 1 < 0 < hi[1] + 1 for px in (0.0, 0.5)):
            continue
        boxes.append((lo, hi))
    blo = np.array([b[0] for b in boxes])
    bhi = np.array([b[1] for b in boxes])
    el = np.radians(np.linspace(-25.0, 15.0, 64))
    az = 2 * math.pi * np.arange(2048) / 2048
    E, A = np.meshgrid(el, az, indexing="ij")
    dl = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)

    def scan(yaw, pos, rs_noise):
        Rz = rotation([0, 0, 1], yaw)
        dw = dl @ Rz.T
        o = np.array([pos[0], pos[1], h])
        tb, nb = ray_boxes(o, dw, blo, bhi)
        with np.errstate(divide="ignore"):
            tg = np.where(dw[:, 2] < 0, -h / dw[:, 2], np.inf)
        use_box = tb < tg
        t = np.where(use_box, tb, tg)
        nw = np.where(use_box[:, None], nb, np.array([0.0, 0.0, 1.0]))
        ok = (t >= 1.0) & (t <= 80.0)
        t = t + 0.02 * rs_noise.normal(len(t))
        p = dl[ok] * t[ok, None]                     # sensor frame
        return p, nw[ok] @ Rz

    tgt, tn = scan(0.0, (0.0, 0.0), Stream(config_seed(cid, 1)))
    yaw2 = math.radians(1.0)
    src, _ = scan(yaw2, (0.5, 0.0), Stream(config_seed(cid, 2)))
    T_true = rigid(rotation([0, 0, 1], yaw2), [0.5, 0.0, 0.0])
    return _pack("lidar", src, tgt, tn, 1.0, 50, np.eye(4), T_true,
                 dict(config_id=cid, beams=64 * 2048, sensor_height=h))


def _room_scene(rs: Stream, size, n_boxes, box_lo, box_hi) -> Rects:
    X, Y, Z = np.eye(3)
    Lx, Ly, Lz = size
    r = Rects()
    r.add([0, 0, 0], Lx * X, Ly * Y, Z)                 # floor
    r.add([0, 0, Lz], Lx * X, Ly * Y, -Z)               # ceiling
    r.add([0, 0, 0], Ly * Y, Lz * Z, X)                 # x = 0
    r.add([Lx, 0, 0], Ly * Y, Lz * Z, -X)               # x = Lx
    r.add([0, 0, 0], Lx * X, Lz * Z, Y)                 # y = 0
    r.add([0, Ly, 0], Lx * X, Lz * Z, -Y)               # y = Ly
    s = rs.uniform(3 * n_boxes, box_lo, box_hi).reshape(n_boxes, 3)
    cx = rs.uniform(n_boxes)
    cy = rs.uniform(n_boxes)
    for k in range(n_boxes):
        x0 = cx[k] * (Lx - s[k, 0])
        y0 = cy[k] * (Ly - s[k, 1])
        r.add_box([x0, y0, 0.0], [x0 + s[k, 0], y0 + s[k, 1], s[k, 2]])
    return r.finish()


def large16m(n: int = 16_000_000, n_target: int | None = None) -> dict:
    """Config 5: 50x50x5 m building (6 planes + 5000 boxes), sigma 0.005,
    3 deg about an axis through (25,25,2.5) + 10 cm; dmax 0.05, 30 iters.
    ``n`` can be reduced for parity tests at the same density structure."""
    cid = CONFIG_IDS["large16m"]
    m = n if n_target is None else n_target
    rs = Stream(config_seed(cid, 0))
    scene = _room_scene(rs, (50.0, 50.0, 5.0), 5000, 0.3, 2.0)
    rt = Stream(config_seed(cid, 1))
    tgt, tn = scene.sample(rt, m)
    tgt += 0.005 * np.stack([rt.normal(m) for _ in range(3)], 1)
    rsrc = Stream(config_seed(cid, 2))
    src, _ = scene.sample(rsrc, n)
    src += 0.005 * np.stack([rsrc.normal(n) for _ in range(3)], 1)
    rm = Stream(config_seed(cid, 3))
    axis, tdir = rm.unit_vectors(1)[0], rm.unit_vectors(1)[0]
    R = rotation(axis, math.radians(3.0))
    c = np.array([25.0, 25.0, 2.5])
    M = rigid(R, c - R @ c + 0.10 * tdir)
    src = apply(M, src)
    return _pack("large16m", src, tgt, tn, 0.05, 30, np.eye(4), inv_rigid(M),
                 dict(config_id=cid, n_source=n, n_target=m, surface_area=float(scene.area.sum())))


def fragment(n: int = 2_000_000) -> dict:
    """Config 4: 10x10x3 m room + 200 boxes, sigma 0.003, 60 % overlap
    (target x in [0,7.14], source x in [2.86,10]), 3 deg + 10 cm about the
    room centre; scales (voxel, dmax, iters) = (.04,.08,50),(.02,.04,30),(.01,.02,14)."""
    cid = CONFIG_IDS["fragment"]
    rs = Stream(config_seed(cid, 0))
    scene = _room_scene(rs, (10.0, 10.0, 3.0), 200, 0.3, 1.5)

    def draw(stream, lo, hi):
        out_p, out_n, have = [], [], 0
        while have < n:
            p, nr = scene.sample(stream, int((n - have) * 1.6) + 1024)
            keep = (p[:, 0] >= lo) & (p[:, 0] <= hi)
            out_p.append(p[keep]), out_n.append(nr[keep])
            have += int(keep.sum())
        p = np.concatenate(out_p)[:n]
        nr = np.concatenate(out_n)[:n]
        return p + 0.003 * np.stack([stream.normal(n) for _ in range(3)], 1), nr

    tgt, tn = draw(Stream(config_seed(cid, 1)), 0.0, 7.14)
    src, _ = draw(Stream(config_seed(cid, 2)), 2.86, 10.0)
    rm = Stream(config_seed(cid, 3))
    axis, tdir = rm.unit_vectors(1)[0], rm.unit_vectors(1)[0]
    R = rotation(axis, math.radians(3.0))
    c = np.array([5.0, 5.0, 1.5])
    M = rigid(R, c - R @ c + 0.10 * tdir)
    src = apply(M, src)
    T_true = inv_rigid(M)
    scales = []
    for voxel, dmax, iters in ((0.04, 0.08, 50), (0.02, 0.04, 30), (0.01, 0.02, 14)):
        s_d, _ = voxel_down_sample(src.astype(np.float32), None, voxel)
        t_d, tn_d = voxel_down_sample(tgt.astype(np.float32), tn.astype(np.float32), voxel)
        scales.append(_pack(f"fragment@{voxel}", s_d, t_d, tn_d, dmax, iters, np.eye(4), T_true,
                            dict(voxel=voxel)))
    w = _pack("fragment", src, tgt, tn, 0.02, 14, np.eye(4), T_true,
              dict(config_id=cid, n=n, overlap=0.6))
    w["scales"] = scales
    return w


def make(name: str, **kw) -> dict:
    return {"tiny": tiny, "depth": depth, "lidar": lidar, "fragment": fragment,
            "large16m": large16m}[name](**kw)
