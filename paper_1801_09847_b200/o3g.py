"""Thin Python binding of include/o3g.h (argument marshalling only).

Every step of the ICP path runs in libo3g.so's CUDA kernels; this module
only converts arrays/tensors to pointers and status codes to exceptions.
There is no CPU fallback: if libo3g.so is missing or no sm_100a device is
present, calls raise.

Arrays may be torch CUDA tensors (device pointers, zero-copy), or numpy
arrays / CPU tensors (host pointers: the library copies them to the device
inside the call — the end-to-end path).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# O3G_LIB: load another in-tree build of the same library (A/B kernel
# experiments under tools/sweeps); default the package's libo3g.so
LIB_PATH = os.environ.get("O3G_LIB") or os.path.join(_PKG, "libo3g.so")

OK, ERR_INVALID_ARGUMENT, ERR_DEGENERATE, ERR_CUDA, ERR_OOM, ERR_COMM, ERR_NOT_IMPLEMENTED = range(7)
FLAG_NO_CORRESPONDENCES = 1
FLAG_DEGENERATE = 2
NTERMS = 29
(OPT_SEARCH, OPT_GRID, OPT_TIMING, OPT_BLOCKS_PER_SM, OPT_NBR_MASK, OPT_COOP_MIN, OPT_ESTIMATION,
 OPT_SOURCE_ORDER, OPT_TARGET_SORT, OPT_PRUNE_MIN, OPT_INTERLEAVE, OPT_XSORT, OPT_CERT,
 OPT_TRACE_PASS, OPT_CERT_SWEEP) = range(1, 16)


class O3GError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"o3g status {status}: {msg}")
        self.status = status


class InvalidArgument(O3GError, ValueError):
    pass


class _Info(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("passes", C.c_int32), ("converged", C.c_int32),
                ("flags", C.c_int32), ("fitness", C.c_double), ("inlier_rmse", C.c_double),
                ("inlier_count", C.c_double)]


_lib = None


def lib() -> C.CDLL:
    """Load libo3g.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() or "
                              "python paper_1801_09847_b200/_build.py")
        L = C.CDLL(LIB_PATH)
        P, D, I32, I64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64
        sig = {
            "o3g_icp_point_to_plane": [P, I64, P, P, I64, P, D, I32, D, D, P, P, P, P, P],
            "o3g_icp_point_to_point": [P, I64, P, I64, P, D, I32, D, D, P, P, P, P, P],
            "o3g_create": [P, C.c_int, P],
            "o3g_destroy": [P],
            "o3g_set_target": [P, P, P, I64, D],
            "o3g_set_source": [P, P, I64, P],
            "o3g_icp_step": [P, P, P, P, P, P, P, P],
            "o3g_icp_run": [P, P, I32, D, D, P, P, P, P, P, P],
            "o3g_nccl_unique_id": [P],
            "o3g_set_clouds": [P, P, I64, P, P, I64, D, P],
            "o3g_dist_init": [P, C.c_int, C.c_int, P],
            "o3g_dist_init_loopback": [P, C.c_int, C.c_int],
            "o3g_loopback_run": [P, C.c_int, P, I32, D, D, P, P, P, P],
            "o3g_loopback_peer_connect": [P, C.c_int],
            "o3g_dist_peer_handle": [P, P],
            "o3g_dist_peer_connect": [P, P],
            "o3g_set_option": [P, C.c_int, I64],
            "o3g_last_run_kernel_ms": [P, P, P, P],
            "o3g_last_run_trace": [P, P, P, P, P],
            "o3g_grid_info": [P, P, P, P, P],
            "o3g_voxel_down_sample": [P, P, P, I64, D, P, P, P],
            "o3g_evaluate_registration": [P, P, I32, P, P],
            "o3g_estimate_normals": [P, P, I64, D, I32, P, P, P],
            "o3g_icp_multiscale": [P, P, I64, P, P, I64, P, I32, P, P, P, D, D, P, P, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.o3g_launch_count.argtypes = [P]
        L.o3g_launch_count.restype = I64
        L.o3g_status_string.argtypes = [C.c_int]
        L.o3g_status_string.restype = C.c_char_p
        L.o3g_last_error.argtypes = []
        L.o3g_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        msg = lib().o3g_last_error().decode()
        cls = InvalidArgument if status == ERR_INVALID_ARGUMENT else O3GError
        raise cls(status, msg)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _pts(x, name: str, keep: list):
    """Pointer to a contiguous float32 [n][3] array (device or host) and n."""
    if x is None:
        return None, 0
    if _is_torch(x):
        import torch
        if x.dtype != torch.float32 or x.dim() != 2 or x.shape[1] != 3:
            raise InvalidArgument(ERR_INVALID_ARGUMENT, f"{name} must be float32 [n,3]")
        x = x.contiguous()
        keep.append(x)
        return x.data_ptr(), int(x.shape[0])
    a = np.ascontiguousarray(x, dtype=np.float32)
    if a.ndim != 2 or a.shape[1] != 3:
        raise InvalidArgument(ERR_INVALID_ARGUMENT, f"{name} must be [n,3]")
    keep.append(a)
    return a.ctypes.data, int(a.shape[0])


def _mat(T, keep: list):
    if T is None:
        return None
    a = np.ascontiguousarray(np.asarray(T, dtype=np.float64).reshape(16))
    keep.append(a)
    return a.ctypes.data


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream)) or None


@dataclass
class RegistrationResult:
    """registration_icp result: transformation, fitness, inlier_rmse."""
    transformation: np.ndarray
    fitness: float
    inlier_rmse: float
    iterations: int = 0
    passes: int = 0
    converged: bool = False
    flags: int = 0
    inlier_count: float = 0.0
    hist_fitness: np.ndarray | None = field(default=None, repr=False)
    hist_rmse: np.ndarray | None = field(default=None, repr=False)


def _result(T, fit, rmse, info: _Info, hf=None, hr=None) -> RegistrationResult:
    return RegistrationResult(T.reshape(4, 4).copy(), float(fit.value), float(rmse.value),
                              info.iterations, info.passes, bool(info.converged), info.flags,
                              info.inlier_count, hf, hr)


def icp_point_to_plane(source, target, target_normals, max_correspondence_distance,
                       init=None, max_iterations=30, relative_fitness=1e-6, relative_rmse=1e-6,
                       stream=None) -> RegistrationResult:
    """registration_icp(source, target, max_correspondence_distance, init,
    TransformationEstimationPointToPlane()) — one call,
    grid build + source ordering + the graph-launched loop."""
    keep: list = []
    ps, n = _pts(source, "source", keep)
    pt, m = _pts(target, "target", keep)
    pn, mn = _pts(target_normals, "target_normals", keep)
    if pn is not None and mn != m:
        raise InvalidArgument(ERR_INVALID_ARGUMENT, "target_normals must match target")
    T0 = _mat(np.eye(4) if init is None else init, keep)
    T = np.zeros(16)
    fit, rmse, info = C.c_double(), C.c_double(), _Info()
    _check(lib().o3g_icp_point_to_plane(ps, n, pt, pn, m, T0, float(max_correspondence_distance),
                                        int(max_iterations), float(relative_fitness),
                                        float(relative_rmse), T.ctypes.data, C.byref(fit),
                                        C.byref(rmse), C.byref(info), _stream_ptr(stream)))
    return _result(T, fit, rmse, info)


def icp_point_to_point(source, target, max_correspondence_distance, init=None,
                       max_iterations=30, relative_fitness=1e-6, relative_rmse=1e-6,
                       stream=None) -> RegistrationResult:
    """registration_icp(..., TransformationEstimationPointToPoint(False))
    (SPEC S:255-263)."""
    keep: list = []
    ps, n = _pts(source, "source", keep)
    pt, m = _pts(target, "target", keep)
    T0 = _mat(np.eye(4) if init is None else init, keep)
    T = np.zeros(16)
    fit, rmse, info = C.c_double(), C.c_double(), _Info()
    _check(lib().o3g_icp_point_to_point(ps, n, pt, m, T0, float(max_correspondence_distance),
                                        int(max_iterations), float(relative_fitness),
                                        float(relative_rmse), T.ctypes.data, C.byref(fit),
                                        C.byref(rmse), C.byref(info), _stream_ptr(stream)))
    return _result(T, fit, rmse, info)


def loopback_run(ctxs, init=None, max_iterations=30, relative_fitness=1e-6,
                 relative_rmse=1e-6) -> RegistrationResult:
    """o3g_loopback_run: the multi-GPU loop of the contexts ctxs (ranks 0..P-1,
    one device) in lockstep, the all-gather done by device copies."""
    keep: list = []
    arr = (C.c_void_p * len(ctxs))(*[c._h.value for c in ctxs])
    T = np.zeros(16)
    fit, rmse, info = C.c_double(), C.c_double(), _Info()
    _check(lib().o3g_loopback_run(arr, len(ctxs), _mat(np.eye(4) if init is None else init, keep),
                                  int(max_iterations), float(relative_fitness), float(relative_rmse),
                                  T.ctypes.data, C.byref(fit), C.byref(rmse), C.byref(info)))
    return _result(T, fit, rmse, info)


def loopback_peer_connect(ctxs) -> None:
    """o3g_loopback_peer_connect: the loopback world exchanges through the
    peer-memory transport (each rank's kernel stores into every rank's
    exchange buffer) instead of device copies of the gathered slots."""
    arr = (C.c_void_p * len(ctxs))(*[c._h.value for c in ctxs])
    _check(lib().o3g_loopback_peer_connect(arr, len(ctxs)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().o3g_nccl_unique_id(buf))
    return buf.raw


class Context:
    """Stateful API: grid built once; steps and runs reuse it (o3g_ctx)."""

    def __init__(self, device: int = 0, stream=None):
        self._h = C.c_void_p()
        _check(lib().o3g_create(C.byref(self._h), int(device), _stream_ptr(stream)))
        self.device = device
        self.n_source = 0
        self.rank, self.world = 0, 1

    def close(self):
        if self._h:
            lib().o3g_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_option(self, option: int, value: int):
        _check(lib().o3g_set_option(self._h, int(option), int(value)))

    def set_target(self, xyz, normals, max_correspondence_distance):
        keep: list = []
        p, m = _pts(xyz, "target", keep)
        pn, mn = _pts(normals, "target_normals", keep)
        if pn is not None and mn != m:
            raise InvalidArgument(ERR_INVALID_ARGUMENT, "target_normals must match target")
        _check(lib().o3g_set_target(self._h, p, pn, m, float(max_correspondence_distance)))

    def set_source(self, xyz, order_T=None):
        keep: list = []
        p, n = _pts(xyz, "source", keep)
        _check(lib().o3g_set_source(self._h, p, n, _mat(order_T, keep)))
        self.n_source = n

    def set_clouds(self, source, target, target_normals, max_correspondence_distance, order_T=None):
        """o3g_set_clouds: set_target + set_source in one call (device arrays: the
        source's ordering runs beside the target build)."""
        keep: list = []
        ps, n = _pts(source, "source", keep)
        pt, m = _pts(target, "target", keep)
        pn, mn = _pts(target_normals, "target_normals", keep)
        if pn is not None and mn != m:
            raise InvalidArgument(ERR_INVALID_ARGUMENT, "target and normals must have the same count")
        _check(lib().o3g_set_clouds(self._h, ps, n, pt, pn, m, float(max_correspondence_distance),
                                    _mat(order_T, keep)))
        self.n_source = n

    def dist_init(self, rank: int, world: int, unique_id: bytes | None):
        buf = C.create_string_buffer(unique_id, 128) if unique_id is not None else None
        _check(lib().o3g_dist_init(self._h, int(rank), int(world), buf))
        self.rank, self.world = rank, world

    def dist_peer_handle(self) -> bytes:
        """o3g_dist_peer_handle: the 64-byte CUDA IPC handle of this rank's
        exchange buffer."""
        buf = C.create_string_buffer(64)
        _check(lib().o3g_dist_peer_handle(self._h, buf))
        return buf.raw

    def dist_peer_connect(self, handles: bytes):
        """o3g_dist_peer_connect: world x 64 bytes, the ranks' handles in rank
        order; the per-pass exchange then runs through peer memory."""
        if len(handles) != 64 * self.world:
            raise ValueError("handles must hold 64 bytes per rank")
        _check(lib().o3g_dist_peer_connect(self._h, C.create_string_buffer(handles, len(handles))))

    def dist_init_loopback(self, rank: int, world: int):
        """o3g_dist_init_loopback: rank `rank` of an in-process world (no
        communicator); run the world with loopback_run."""
        _check(lib().o3g_dist_init_loopback(self._h, int(rank), int(world)))
        self.rank, self.world = rank, world

    def step(self, T, corr_out=None) -> dict:
        """o3g_icp_step: one pass at fixed T. corr_out: optional torch CUDA
        int32 tensor [n_source] (original source order; -1 = none)."""
        keep: list = []
        pc = None
        if corr_out is not None:
            import torch
            if not (_is_torch(corr_out) and corr_out.is_cuda and corr_out.dtype == torch.int32
                    and corr_out.is_contiguous() and corr_out.numel() == self.n_source):
                raise InvalidArgument(ERR_INVALID_ARGUMENT, "corr_out must be a contiguous CUDA int32 [n_source] tensor")
            pc = corr_out.data_ptr()
        JTJ, JTr, terms = np.zeros(36), np.zeros(6), np.zeros(NTERMS)
        cnt, sd2 = C.c_double(), C.c_double()
        _check(lib().o3g_icp_step(self._h, _mat(T, keep), pc, JTJ.ctypes.data, JTr.ctypes.data,
                                  C.byref(cnt), C.byref(sd2), terms.ctypes.data))
        return dict(JTJ=JTJ.reshape(6, 6), JTr=JTr, count=cnt.value, sum_sq_dist=sd2.value,
                    terms=terms)

    def run(self, init=None, max_iterations=30, relative_fitness=1e-6, relative_rmse=1e-6,
            history=False) -> RegistrationResult:
        keep: list = []
        T = np.zeros(16)
        fit, rmse, info = C.c_double(), C.c_double(), _Info()
        hf = np.zeros(max_iterations + 1) if history else None
        hr = np.zeros(max_iterations + 1) if history else None
        _check(lib().o3g_icp_run(self._h, _mat(np.eye(4) if init is None else init, keep),
                                 int(max_iterations), float(relative_fitness), float(relative_rmse),
                                 T.ctypes.data, C.byref(fit), C.byref(rmse), C.byref(info),
                                 hf.ctypes.data if history else None,
                                 hr.ctypes.data if history else None))
        if history:
            hf, hr = hf[:info.passes].copy(), hr[:info.passes].copy()
        return _result(T, fit, rmse, info, hf, hr)

    def evaluate(self, transforms):
        """Batched evaluate_registration: (fitness[k], inlier_rmse[k]) for a
        stack of rigid 4x4 transforms."""
        Ts = np.ascontiguousarray(np.asarray(transforms, dtype=np.float64).reshape(-1, 16))
        k = len(Ts)
        fit, rmse = np.zeros(k), np.zeros(k)
        _check(lib().o3g_evaluate_registration(self._h, Ts.ctypes.data, k, fit.ctypes.data,
                                               rmse.ctypes.data))
        return fit, rmse

    def estimate_normals(self, xyz, radius=0.1, max_nn=30):
        """SPEC S:67-75 hybrid-neighbourhood PCA normals on the device. Returns
        (normals CUDA [n,3], neighbour counts CUDA int32 [n], fallbacks).
        Replaces the context's target grid."""
        import torch
        keep: list = []
        p, n = _pts(xyz, "xyz", keep)
        dev = torch.device("cuda", self.device)
        out = torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev)
        cnt = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        fb = C.c_int64()
        _check(lib().o3g_estimate_normals(self._h, p, n, float(radius), int(max_nn), out.data_ptr(),
                                          cnt.data_ptr(), C.byref(fb)))
        return out[:n], cnt[:n], fb.value

    def voxel_down_sample(self, xyz, voxel, normals=None):
        """SPEC S:58-61 voxel_down_sample on the device. Returns CUDA tensors
        (points [k,3], normals [k,3] or None)."""
        import torch
        keep: list = []
        p, n = _pts(xyz, "xyz", keep)
        pn, nn = _pts(normals, "normals", keep)
        if pn is not None and nn != n:
            raise InvalidArgument(ERR_INVALID_ARGUMENT, "normals must match xyz")
        dev = torch.device("cuda", self.device)
        out = torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev)
        outn = torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev) if pn is not None else None
        k = C.c_int64()
        _check(lib().o3g_voxel_down_sample(self._h, p, pn, n, float(voxel), out.data_ptr(),
                                           outn.data_ptr() if outn is not None else None, C.byref(k)))
        return out[:k.value], (outn[:k.value] if outn is not None else None)

    def run_multiscale(self, source, target, target_normals, voxels, dmaxs, iters, init=None,
                       relative_fitness=1e-6, relative_rmse=1e-6) -> dict:
        """Multi-scale point-to-plane ICP (o3g_icp_multiscale)."""
        keep: list = []
        ps, n = _pts(source, "source", keep)
        pt, m = _pts(target, "target", keep)
        pn, mn = _pts(target_normals, "target_normals", keep)
        if pn is None or mn != m:
            raise InvalidArgument(ERR_INVALID_ARGUMENT, "target_normals must match target")
        ns = len(voxels)
        vx = np.ascontiguousarray(voxels, np.float64)
        dm = np.ascontiguousarray(dmaxs, np.float64)
        it = np.ascontiguousarray(iters, np.int32)
        T = np.zeros(16)
        fit, rmse = np.zeros(ns), np.zeros(ns)
        its, nss = np.zeros(ns, np.int32), np.zeros(ns, np.int64)
        _check(lib().o3g_icp_multiscale(self._h, ps, n, pt, pn, m,
                                        _mat(np.eye(4) if init is None else init, keep), ns,
                                        vx.ctypes.data, dm.ctypes.data, it.ctypes.data,
                                        float(relative_fitness), float(relative_rmse), T.ctypes.data,
                                        fit.ctypes.data, rmse.ctypes.data, its.ctypes.data,
                                        nss.ctypes.data))
        return dict(T=T.reshape(4, 4), fitness=fit, inlier_rmse=rmse, iterations=its, n_source=nss)

    def last_run_trace(self, passes: int, corr_out=None):
        """o3g_last_run_trace: dict(T [passes,4,4], terms [passes,29], searched
        [passes], candidates [passes], certified [passes]) of the last run; corr_out (torch CUDA
        int32 [n_source], optional) gets the correspondences of pass
        OPT_TRACE_PASS."""
        T = np.zeros((max(passes, 1), 16))
        terms = np.zeros((max(passes, 1), NTERMS))
        stats = np.zeros((max(passes, 1), 3))
        pc = None
        if corr_out is not None:
            import torch
            if not (_is_torch(corr_out) and corr_out.is_cuda and corr_out.dtype == torch.int32
                    and corr_out.is_contiguous() and corr_out.numel() == self.n_source):
                raise InvalidArgument(ERR_INVALID_ARGUMENT, "corr_out must be a contiguous CUDA int32 [n_source] tensor")
            pc = corr_out.data_ptr()
        _check(lib().o3g_last_run_trace(self._h, T.ctypes.data, terms.ctypes.data, pc, stats.ctypes.data))
        return dict(T=T[:passes].reshape(-1, 4, 4), terms=terms[:passes], searched=stats[:passes, 0],
                    candidates=stats[:passes, 1], certified=stats[:passes, 2])

    def last_run_kernel_ms(self):
        k3, n, tail = C.c_double(), C.c_int32(), C.c_double()
        _check(lib().o3g_last_run_kernel_ms(self._h, C.byref(k3), C.byref(n), C.byref(tail)))
        return k3.value, n.value, tail.value

    def grid_info(self) -> dict:
        dims = (C.c_int64 * 3)()
        ts, hashed, occ = C.c_int64(), C.c_int32(), C.c_int64()
        _check(lib().o3g_grid_info(self._h, dims, C.byref(ts), C.byref(hashed), C.byref(occ)))
        return dict(dims=tuple(dims), table_size=ts.value, hashed=bool(hashed.value),
                    occupied_cells=occ.value)

    def launch_count(self) -> int:
        return int(lib().o3g_launch_count(self._h))
