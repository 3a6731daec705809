"""Pins for the CPU oracle (run with -m "not gpu").

Each test checks the oracle against something other than itself: hand-
derived dyadic fixtures (tests/golden, each cited), an independent NN library
(scipy cKDTree), finite differences through scipy's matrix exponential,
numpy's dense solver, closed-form special cases and exact recovery of a
known rigid motion. A plausible mistake in the oracle (a dropped term, a
wrong sign or index, a transposed operand, a strict-vs-inclusive radius, a
wrong tie rule) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg
from scipy.spatial import cKDTree

import oracle
from synth.rng import Stream
from synth.scenes import Rects, apply, inv_rigid, rigid, rotation

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _hat4(xi):
    w, v = xi[:3], xi[3:]
    X = np.zeros((4, 4))
    X[:3, :3] = [[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]]
    X[:3, 3] = v
    return X


def _upper(A):
    return np.array([A[i, j] for i in range(6) for j in range(i, 6)])


def _rand_T(rs, ang=0.2, trans=0.1):
    axis = rs.unit_vectors(1)[0]
    return rigid(rotation(axis, ang * (2 * rs.uniform(1)[0] - 1)), rs.uniform(3, -trans, trans))


# ------------------------------------------------------------ golden cases
def test_hand_step_golden():
    g = json.load(open(os.path.join(GOLD, "hand_step.json")))
    for c in g["cases"]:
        r = oracle.step(np.array(c["T"], float), np.array(c["source"]), np.array(c["target"]),
                        np.array(c["normals"]), c["dmax"], grid=None)
        assert r["corr"].tolist() == c["corr"], c["name"]
        assert np.array_equal(_upper(r["JTJ"]), np.array(c["jtj_upper"], float)), c["name"]
        assert np.array_equal(r["JTr"], np.array(c["jtr"], float)), c["name"]
        assert r["count"] == c["count"] and r["sum_sq_dist"] == c["sum_sq_dist"], c["name"]
        # the sums of |term| that scale every R14 tolerance (hand values; the
        # cancelling case fails an implementation that takes |sum| instead)
        ab = r["abs_terms"]
        assert np.array_equal(ab[:21], np.array(c["abs_jtj_upper"], float)), c["name"]
        assert np.array_equal(ab[21:27], np.array(c["abs_jtr"], float)), c["name"]
        assert ab[27] == c["count"] and ab[28] == c["sum_sq_dist"], c["name"]
        # the chunked (OpenMP) pass gives the same terms and sums of |term|
        rc = oracle.step(np.array(c["T"], float), np.array(c["source"]), np.array(c["target"]),
                         np.array(c["normals"]), c["dmax"], grid=None, threads=2)
        assert np.array_equal(rc["terms"], r["terms"]) and np.array_equal(rc["abs_terms"], ab)
        # same answers through the grid accelerator
        rg = oracle.step(np.array(c["T"], float), np.array(c["source"]), np.array(c["target"]),
                         np.array(c["normals"]), c["dmax"], grid=oracle.Grid(np.array(c["target"]), c["dmax"]))
        assert rg["corr"].tolist() == c["corr"]
        assert np.array_equal(rg["terms"], r["terms"])


def test_dyadic_nn_golden():
    g = json.load(open(os.path.join(GOLD, "dyadic_nn.json")))
    for c in g["cases"]:
        tgt = np.array(c["target"], np.float32)
        for grid in (None, oracle.Grid(tgt, c["dmax"])):
            j, d2 = oracle.nn(np.array(c["query"], float), tgt, c["dmax"], grid=grid)
            assert j == c["expect"], (c["name"], grid)
            if c["expect_d2"] is not None:
                assert d2 == c["expect_d2"], c["name"]


def test_transform_dyadic_exact():
    """A3 with a dyadic permutation+translation: every op exact, result by hand."""
    T = np.array([[0, 0, 1, 0.5], [1, 0, 0, -0.25], [0, 1, 0, 2.0], [0, 0, 0, 1]], float)
    p = np.array([[1.5, -2.25, 0.125], [0, 0, 0]], np.float32)
    out = oracle.transform(T, p)
    assert np.array_equal(out, [[0.625, 1.25, -0.25], [0.5, -0.25, 2.0]])


# ---------------------------------------------------------- NN vs library
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_nn_matches_ckdtree(seed):
    rs = Stream(1000 + seed)
    tgt = rs.uniform(3000 * 3, -1, 1).reshape(-1, 3).astype(np.float32)
    src = rs.uniform(2000 * 3, -1.1, 1.1).reshape(-1, 3).astype(np.float32)
    T = _rand_T(rs)
    dmax = 0.08
    r = oracle.step(T, src, tgt, np.tile([0, 0, 1], (3000, 1)), dmax, grid=None)
    sp = oracle.transform(T, src)
    kd = cKDTree(tgt.astype(np.float64))
    dist, idx = kd.query(sp, k=2)
    for i in range(len(src)):
        within = dist[i, 0] <= dmax * (1 - 1e-12)
        outside = dist[i, 0] > dmax * (1 + 1e-12)
        if within:
            assert r["corr"][i] >= 0
            assert abs(r["d2"][i] - dist[i, 0] ** 2) <= 1e-12 * max(dist[i, 0] ** 2, 1e-300) + 1e-15
            if dist[i, 1] - dist[i, 0] > 1e-9:
                assert r["corr"][i] == idx[i, 0]
        elif outside:
            assert r["corr"][i] == -1
    assert (r["corr"] >= 0).sum() > 200          # the case is not vacuous


@pytest.mark.parametrize("name", ["tiny"])
def test_grid_equals_brute_force_exhaustive(name, workloads):
    w = workloads(name)
    rs = Stream(77)
    for T in (w["init_T"], w["T_true"], _rand_T(rs, 0.05, 0.03)):
        rb = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"], grid=None)
        rg = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"],
                         grid=oracle.Grid(w["target"], w["dmax"]))
        assert np.array_equal(rb["corr"], rg["corr"])
        assert np.array_equal(rb["d2"], rg["d2"])


def test_grid_equals_brute_force_adversarial():
    """Dyadic lattice with spacing == dmax: many exact ties and d == dmax."""
    dmax = 0.25
    g = np.arange(-4, 5) * 0.25
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    tgt = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    tgt = np.concatenate([tgt, tgt[::7]]).astype(np.float32)    # duplicates at higher indices
    qs = np.stack(np.meshgrid(*(np.arange(-9, 10) * 0.125,) * 3, indexing="ij"), -1).reshape(-1, 3)
    grid = oracle.Grid(tgt, dmax)
    T = np.eye(4)
    rb = oracle.step(T, qs, tgt, np.zeros_like(tgt), dmax, grid=None)
    rg = oracle.step(T, qs, tgt, np.zeros_like(tgt), dmax, grid=grid)
    assert np.array_equal(rb["corr"], rg["corr"])
    # every lattice-midpoint query ties between several points: winner is the lowest index
    for i in range(0, len(qs), 97):
        d2 = ((tgt.astype(np.float64) - qs[i]) ** 2).sum(1)
        ok = np.nonzero(d2 <= dmax * dmax)[0]
        if len(ok):
            best = ok[d2[ok] == d2[ok].min()].min()
            assert rb["corr"][i] == best


# ------------------------------------------------------------ J, JTJ, JTr
def _scene_small(rs, n):
    r = Rects()
    X, Y, Z = np.eye(3)
    r.add([0, 0, 0], 2 * X, 2 * Y, Z)
    r.add([0, 0, 0], 2 * Y, 1 * Z, X)
    r.add([0, 0, 0], 2 * X, 1 * Z, Y)
    r.add_box([0.5, 0.6, 0], [1.1, 1.3, 0.7])
    r.finish()
    return r.sample(rs, n)


def test_jacobian_finite_differences():
    """For fixed correspondences, r_i(xi) = ((exp(xi^) T s_i) - q_i).n_i.
    Central differences (scipy expm) give J_i; then JTJ = sum J J^T and
    JTr = sum J r. Pins the sign/order of J = [s' x n ; n] and the left
    update convention (R#4, R#5)."""
    rs = Stream(4242)
    tgt, nrm = _scene_small(rs, 400)
    tgt = tgt.astype(np.float32)
    src = (apply(rigid(rotation([1, 2, 3], 0.02), [0.01, -0.02, 0.015]), tgt)
           + 0.003 * rs.uniform(1200, -1, 1).reshape(-1, 3)).astype(np.float32)
    T = rigid(rotation([0.3, -1, 0.2], 0.01), [0.005, 0.0, -0.004])
    dmax = 0.2
    r = oracle.step(T, src, tgt, nrm, dmax, grid=None)
    m = r["corr"] >= 0
    assert m.sum() > 300
    s64 = src.astype(np.float64)[m]
    q = tgt.astype(np.float64)[r["corr"][m]]
    n = nrm.astype(np.float32).astype(np.float64)[r["corr"][m]]

    def resid(xi):
        Tx = scipy.linalg.expm(_hat4(xi)) @ T
        return ((apply(Tx, s64) - q) * n).sum(1)

    h = 1e-6
    J = np.stack([(resid(h * e) - resid(-h * e)) / (2 * h) for e in np.eye(6)], 1)
    r0 = resid(np.zeros(6))
    JTJ_fd, JTr_fd = J.T @ J, J.T @ r0
    scale = np.abs(JTJ_fd).max()
    assert np.abs(r["JTJ"] - JTJ_fd).max() <= 1e-6 * scale
    assert np.abs(r["JTr"] - JTr_fd).max() <= 1e-6 * np.abs(JTr_fd).max() + 1e-12
    # gradient of E(xi) = sum r^2 is 2 JTr
    E = lambda xi: (resid(xi) ** 2).sum()
    g = np.array([(E(h * e) - E(-h * e)) / (2 * h) for e in np.eye(6)])
    assert np.abs(g - 2 * r["JTr"]).max() <= 1e-5 * np.abs(g).max() + 1e-12


def test_jtj_symmetric_psd_and_counts(workloads):
    w = workloads("tiny")
    r = oracle.step(w["init_T"], w["source"], w["target"], w["target_normals"], w["dmax"])
    A = r["JTJ"]
    assert np.array_equal(A, A.T)
    ev = np.linalg.eigvalsh(A)
    assert ev.min() >= -1e-12 * ev.max()
    cnt = int((r["corr"] >= 0).sum())
    assert r["count"] == cnt                                  # fitness * N = count
    assert r["sum_sq_dist"] == pytest.approx(r["d2"][r["corr"] >= 0].sum(), rel=1e-12)
    rmse = math.sqrt(r["sum_sq_dist"] / cnt)
    assert 0 <= rmse <= w["dmax"]


def test_planar_target_null_space():
    """Planar target with n=(0,0,1): J = [(sy,-sx,0),(0,0,1)] so JTJ has
    rank 3 with null space {omega_z, t_x, t_y} and LDLT reports
    singular."""
    rs = Stream(9)
    tgt = np.concatenate([rs.uniform(2000, -1, 1).reshape(-1, 2), np.zeros((1000, 1))], 1).astype(np.float32)
    nrm = np.tile([0.0, 0.0, 1.0], (1000, 1))
    src = tgt + np.array([0, 0, 0.01], np.float32)
    r = oracle.step(np.eye(4), src, tgt, nrm, 0.1, grid=None)
    A = r["JTJ"]
    for k in (2, 3, 4):
        assert np.all(A[k] == 0) and np.all(A[:, k] == 0)
    assert np.linalg.matrix_rank(A) == 3
    assert oracle.ldlt_solve(A, -r["JTr"]) is None


# ------------------------------------------------------------- LDLT, exp
def test_ldlt_matches_numpy_solve():
    rs = Stream(5)
    for _ in range(50):
        B = rs.uniform(36, -1, 1).reshape(6, 6)
        A = B @ B.T + 0.1 * np.eye(6)
        b = rs.uniform(6, -1, 1)
        x = oracle.ldlt_solve(A, b)
        xr = np.linalg.solve(A, b)
        assert np.abs(x - xr).max() <= 1e-11 * np.abs(xr).max()


def test_ldlt_singular_guard():
    A = np.diag([1.0, 1.0, 1.0, 1.0, 1.0, 1e-13])
    assert oracle.ldlt_solve(A, np.ones(6)) is None
    assert oracle.ldlt_solve(np.zeros((6, 6)), np.ones(6)) is None
    A[5, 5] = 1e-11
    assert oracle.ldlt_solve(A, np.ones(6)) is not None


def test_exp_se3_matches_expm():
    rs = Stream(6)
    assert np.array_equal(oracle.exp_se3(np.zeros(6)), np.eye(4))
    for scale in (1e-9, 1e-7, 1e-3, 0.1, 1.0, 2.5):
        for _ in range(10):
            xi = np.concatenate([rs.unit_vectors(1)[0] * scale, rs.uniform(3, -1, 1)])
            E = scipy.linalg.expm(_hat4(xi))
            assert np.abs(oracle.exp_se3(xi) - E).max() <= 2e-14 * max(1.0, np.abs(E).max())
    xi = np.array([1e-9, -2e-9, 3e-9, 1e-9, 0, 0])
    assert np.abs(oracle.exp_se3(xi) - (np.eye(4) + _hat4(xi))).max() <= 1e-15


def test_compose_matches_matmul():
    rs = Stream(8)
    A, B = _rand_T(rs), _rand_T(rs)
    assert np.abs(oracle.compose(A, B) - A @ B).max() <= 1e-15


# ------------------------------------------------------------- full loop
def test_fixed_point_source_equals_target():
    """source = target, init I -> identity, fitness 1, rmse 0, one
    update; r = 0 exactly so JTr = 0, xi = 0 and T stays bitwise I.
    (A well-conditioned scene: on the tiny sphere+plane scene source=target
    makes the yaw column of J exactly zero and the loop stops DEGENERATE.)"""
    tgt, nrm = _scene_small(Stream(21), 3000)
    tgt = tgt.astype(np.float32)
    r = oracle.icp(tgt, tgt, nrm, 0.05, 20)
    assert np.array_equal(r["T"], np.eye(4))
    assert r["fitness"] == 1.0 and r["inlier_rmse"] == 0.0
    assert r["iterations"] == 1 and r["converged"]


def test_exact_recovery_noise_free():
    """Noise-free twin clouds (room + box, well conditioned): T -> M^-1 up to
    fp32 input quantisation; fitness 1."""
    rs = Stream(31337)
    tgt, nrm = _scene_small(rs, 3000)
    tgt = tgt.astype(np.float32)
    M = rigid(rotation([0.2, 0.5, 1.0], math.radians(1.5)), [0.02, -0.015, 0.01])
    src = apply(M, tgt.astype(np.float64)).astype(np.float32)
    r = oracle.icp(src, tgt, nrm, 0.1, 30)
    assert np.abs(r["T"] - inv_rigid(M)).max() < 1e-6
    assert r["fitness"] == 1.0 and r["inlier_rmse"] < 1e-6


def test_recovers_tiny_config_up_to_yaw_gauge(workloads):
    """Config 1: translation, roll and pitch recovered; yaw about the sphere's
    vertical axis is unobservable (SURVEY §8(c) gauge note)."""
    w = workloads("tiny")
    r = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], w["iters"])
    E = r["T"] @ np.linalg.inv(w["T_true"])
    # E = T T*^-1 is (almost) a pure yaw about the z axis through the sphere centre
    assert np.abs(E[:3, 3]).max() < 1e-3
    assert abs(E[2, 2] - 1) < 1e-4
    assert r["fitness"] > 0.8


def test_tiny_scene_source_equals_target_is_degenerate(workloads):
    """Sphere (radial normals: s x n = 0) + plane (n = z): the omega_z column of
    J is exactly zero, so LDLT must flag DEGENERATE before any update."""
    w = workloads("tiny")
    r = oracle.icp(w["target"], w["target"], w["target_normals"], 0.05, 20)
    assert r["flags"] == oracle.FLAG_DEGENERATE and r["iterations"] == 0
    assert np.array_equal(r["T"], np.eye(4)) and r["fitness"] == 1.0


def test_degenerate_and_no_correspondence_flags():
    rs = Stream(3)
    tgt = rs.uniform(15, -1, 1).reshape(5, 3).astype(np.float32)          # < 6 points
    nrm = rs.unit_vectors(5)
    r = oracle.icp(tgt, tgt, nrm, 0.1, 10)
    assert r["flags"] & oracle.FLAG_DEGENERATE and r["iterations"] == 0
    far = tgt + np.float32(100.0)
    r = oracle.icp(far, tgt, nrm, 0.1, 10)
    assert r["flags"] & oracle.FLAG_NO_CORR and r["fitness"] == 0 and r["inlier_rmse"] == 0
    assert np.array_equal(r["T"], np.eye(4))


def test_convergence_criteria_semantics(workloads):
    """R#8 (parity unpinned by the paper): absolute |dfit|, |drmse| with
    strict '<' between consecutive passes; max_iterations counts updates."""
    w = workloads("tiny")
    args = (w["source"], w["target"], w["target_normals"], w["dmax"])
    r0 = oracle.icp(*args, 7, relative_fitness=0.0, relative_rmse=0.0)
    assert r0["iterations"] == 7 and r0["passes"] == 8 and not r0["converged"]
    rinf = oracle.icp(*args, 7, relative_fitness=np.inf, relative_rmse=np.inf)
    assert rinf["iterations"] == 1 and rinf["converged"]
    r = oracle.icp(*args, 20)
    hf, hr = r["hist_fitness"], r["hist_rmse"]
    k = len(hf) - 1
    assert abs(hf[k] - hf[k - 1]) < 1e-6 and abs(hr[k] - hr[k - 1]) < 1e-6
    for i in range(1, k):
        assert not (abs(hf[i] - hf[i - 1]) < 1e-6 and abs(hr[i] - hr[i - 1]) < 1e-6)


# ------------------------------------------------ voxel_down_sample (NEXT 1)
def test_voxel_down_sample_spec_examples():
    """singleton -> same point; two points in one voxel -> their mean."""
    p, _ = oracle.voxel_down_sample(np.array([[0.01, 0.01, 0.01]], np.float32), 0.05)
    assert np.array_equal(p, np.array([[0.01, 0.01, 0.01]], np.float32))
    p, _ = oracle.voxel_down_sample(np.array([[0, 0, 0], [0.01, 0, 0]], np.float32), 0.05)
    assert np.array_equal(p, np.array([[0.005, 0, 0]], np.float32))


def test_voxel_down_sample_matches_bucketing():
    """equals an independent bucketing oracle (numpy unique + bincount,
    a different summation order: compare within 1 fp32 ulp) and keeps the
    S:124-126 invariants (count <= n, each mean inside its voxel, ascending
    lexicographic voxel order, unit normals)."""
    rs = Stream(77)
    p = rs.uniform(30000, -1, 1).reshape(-1, 3).astype(np.float32)
    nr = rs.unit_vectors(len(p)).astype(np.float32)
    voxel = 0.05
    out, outn = oracle.voxel_down_sample(p, voxel, nr)
    p64 = p.astype(np.float64)
    lo = p64.min(0)
    ijk = np.floor((p64 - lo) / voxel).astype(np.int64)
    key = (ijk[:, 0] * 10000 + ijk[:, 1]) * 10000 + ijk[:, 2]
    uniq, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    ref = np.stack([np.bincount(inv, p64[:, a]) for a in range(3)], 1) / cnt[:, None]
    assert len(out) == len(uniq) <= len(p)
    assert np.all(np.abs(out - ref.astype(np.float32)) <= np.spacing(np.abs(ref).astype(np.float32)) * 1.01)
    vox_of_out = np.floor((out.astype(np.float64) - lo) / voxel).astype(np.int64)
    assert np.array_equal((vox_of_out[:, 0] * 10000 + vox_of_out[:, 1]) * 10000 + vox_of_out[:, 2], uniq)
    norms = np.linalg.norm(outn.astype(np.float64), axis=1)
    assert np.all(np.abs(norms - 1) < 1e-6) or np.all((np.abs(norms - 1) < 1e-6) | (norms == 0))


def test_multiscale_single_scale_is_downsample_then_icp():
    """One scale of the multi-scale driver == voxel_down_sample + icp."""
    rs = Stream(31338)
    tgt, nrm = _scene_small(rs, 6000)
    tgt = tgt.astype(np.float32)
    M = rigid(rotation([0.2, 0.5, 1.0], math.radians(1.0)), [0.01, -0.01, 0.005])
    src = apply(M, tgt.astype(np.float64)).astype(np.float32)
    ms = oracle.icp_multiscale(src, tgt, nrm, [0.03], [0.1], [20])
    sd, _ = oracle.voxel_down_sample(src, 0.03)
    td, tn = oracle.voxel_down_sample(tgt, 0.03, nrm)
    r = oracle.icp(sd, td, tn, 0.1, 20)
    assert np.array_equal(ms["T"], r["T"]) and ms["fitness"][0] == r["fitness"]


def test_multiscale_recovers_motion():
    rs = Stream(31339)
    tgt, nrm = _scene_small(rs, 20000)
    tgt = tgt.astype(np.float32)
    M = rigid(rotation([0.2, 0.5, 1.0], math.radians(2.0)), [0.03, -0.02, 0.01])
    src = apply(M, tgt.astype(np.float64)).astype(np.float32)
    ms = oracle.icp_multiscale(src, tgt, nrm, [0.08, 0.04, 0.02], [0.16, 0.08, 0.04], [30, 20, 10])
    assert np.abs(ms["T"] - inv_rigid(M)).max() < 2e-3


# ----------------------------------------------- point-to-point ICP (NEXT 2)
def _kabsch_numpy(s, q):
    """Textbook Kabsch via numpy's SVD (an independent library route)."""
    ms, mq = s.mean(0), q.mean(0)
    H = (s - ms).T @ (q - mq)
    U, S, Vt = np.linalg.svd(H)
    d = np.sign(np.linalg.det(Vt.T @ U.T))
    R = Vt.T @ np.diag([1, 1, d]) @ U.T
    return rigid(R, mq - R @ ms)


def test_kabsch_matches_numpy_svd_and_exact_motion():
    rs = Stream(505)
    for _ in range(20):
        s = rs.uniform(300, -2, 2).reshape(-1, 3)
        M = _rand_T(rs, 1.0, 1.0)
        q = apply(M, s) + 0.01 * rs.uniform(300, -1, 1).reshape(-1, 3)
        terms = np.zeros(29)
        terms[0:9] = (s[:, :, None] * q[:, None, :]).sum(0).ravel()
        terms[9:12], terms[12:15], terms[27] = s.sum(0), q.sum(0), len(s)
        T = oracle.kabsch(terms)
        assert np.abs(T - _kabsch_numpy(s, q)).max() < 1e-9
        assert abs(np.linalg.det(T[:3, :3]) - 1) < 1e-12
    # exact motion recovered ("recovers R,t within 1e-10")
    s = rs.uniform(600, -1, 1).reshape(-1, 3)
    M = _rand_T(rs, 0.7, 0.5)
    q = apply(M, s)
    terms = np.zeros(29)
    terms[0:9] = (s[:, :, None] * q[:, None, :]).sum(0).ravel()
    terms[9:12], terms[12:15], terms[27] = s.sum(0), q.sum(0), len(s)
    assert np.abs(oracle.kabsch(terms) - M).max() < 1e-10


def test_kabsch_reflection_and_degenerate():
    rs = Stream(506)
    s = rs.uniform(300, -1, 1).reshape(-1, 3)
    q = s * np.array([1, 1, -1])                      # a mirror: best proper rotation, det +1
    terms = np.zeros(29)
    terms[0:9] = (s[:, :, None] * q[:, None, :]).sum(0).ravel()
    terms[9:12], terms[12:15], terms[27] = s.sum(0), q.sum(0), len(s)
    T = oracle.kabsch(terms)
    assert abs(np.linalg.det(T[:3, :3]) - 1) < 1e-12
    assert np.abs(T - _kabsch_numpy(s, q)).max() < 1e-9
    line = np.outer(np.linspace(-1, 1, 50), [1.0, 2.0, 3.0])   # collinear: rank(H) = 1
    terms = np.zeros(29)
    terms[0:9] = (line[:, :, None] * line[:, None, :]).sum(0).ravel()
    terms[9:12], terms[12:15], terms[27] = line.sum(0), line.sum(0), len(line)
    assert oracle.kabsch(terms) is None
    terms[27] = 2.0
    assert oracle.kabsch(terms) is None


def test_icp_p2p_recovers_motion():
    """5 deg + 0.02 perturbation -> rotation error < 0.1 deg,
    translation error < 1e-3 (here noise-free twins, well conditioned)."""
    rs = Stream(507)
    tgt, _ = _scene_small(rs, 4000)
    tgt = tgt.astype(np.float32)
    M = rigid(rotation([0.3, -0.2, 1.0], math.radians(5.0)), [0.02, -0.01, 0.015])
    src = apply(M, tgt.astype(np.float64)).astype(np.float32)
    r = oracle.icp_p2p(src, tgt, 0.3, 60)
    E = r["T"] @ M
    ang = math.degrees(math.acos(min(1.0, (np.trace(E[:3, :3]) - 1) / 2)))
    assert ang < 0.1 and np.abs(E[:3, 3]).max() < 1e-3
    r = oracle.icp_p2p(tgt, tgt, 0.05, 10)            # S:288 fixed point
    assert np.abs(r["T"] - np.eye(4)).max() < 1e-12 and r["fitness"] == 1.0


# ------------------------------------------------ estimate_normals (NEXT 4)
def test_normals_plane_and_sphere_spec_examples():
    rs = Stream(808)
    pl = np.concatenate([rs.uniform(200, -0.3, 0.3).reshape(-1, 2), np.zeros((100, 1))], 1)
    n, cnt, fb = oracle.estimate_normals(pl, 0.1, 30)
    assert np.abs(n - np.array([0, 0, 1.0])).max() < 1e-6     # S:73 (fallbacks are (0,0,1) too)
    # S:74 gives no search parameters; neighbourhoods of ~50 points keep the
    # sampling-asymmetry tilt of the PCA normal under 2 degrees
    sp = rs.unit_vectors(20000)
    n, cnt, fb = oracle.estimate_normals(sp, 0.1, 100)
    cosang = np.abs((n.astype(np.float64) * sp).sum(1))
    assert np.degrees(np.arccos(np.clip(cosang, -1, 1))).max() < 2.0


def test_normals_match_numpy_bruteforce_pca():
    """equal to a brute-force PCA over the identical neighbour sets (numpy
    lexsort KNN + numpy eigh), up to sign; the sign rule (largest |component|
    positive) is checked where it is unambiguous."""
    from synth.scenes import Rects
    rs = Stream(809)
    r = Rects()
    X, Y, Z = np.eye(3)
    r.add([0, 0, 0], X, Y, Z)
    r.add_box([0.2, 0.3, 0], [0.6, 0.7, 0.3])
    r.finish()
    p, _ = r.sample(rs, 3000)
    p = (p + 0.002 * rs.uniform(9000, -1, 1).reshape(-1, 3)).astype(np.float32)
    n, cnt, fb = oracle.estimate_normals(p, 0.08, 30)
    p64 = p.astype(np.float64)
    for i in range(0, len(p), 7):
        d = p64 - p64[i]
        d2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
        ok = np.nonzero(d2 <= 0.08 * 0.08)[0]
        nb = ok[np.lexsort((ok, d2[ok]))][:30]
        assert cnt[i] == len(nb)
        if len(nb) < 3:
            assert np.array_equal(n[i], [0, 0, 1])
            continue
        q = p64[nb]
        w, V = np.linalg.eigh(np.cov(q.T, bias=True))
        if w[1] - w[0] < 1e-6 * w[2]:
            continue                       # ill-conditioned smallest eigenvector
        v = V[:, 0]
        assert abs(abs(np.dot(v, n[i].astype(np.float64))) - 1) < 1e-6, i
        a = np.sort(np.abs(v))
        if a[2] - a[1] > 1e-6:
            assert n[i][np.argmax(np.abs(n[i]))] > 0
    tiny = np.array([[0, 0, 0], [5, 0, 0], [0, 5, 0]], np.float32)
    n, cnt, fb = oracle.estimate_normals(tiny, 0.1, 30)
    assert fb == 3 and np.array_equal(n, np.tile([0, 0, 1], (3, 1)).astype(np.float32))


# ------------------------------------------------ deterministic OpenMP mode
def test_chunked_pass_deterministic_and_equal():
    """the OpenMP oracle splits the records into fixed chunks and
    sums the chunk partials in chunk order, so its result is bitwise the same
    for every thread count; correspondences equal the sequential
    pass's exactly, the terms within R14 (a different summation order of the
    same compensated sums), and abs_terms equals an independent numpy sum of
    |record| over the oracle's own correspondences."""
    from synth import make
    w = make("depth")
    args = (w["init_T"], w["source"], w["target"], w["target_normals"], w["dmax"])
    seq = oracle.step(*args)
    outs = [oracle.step(*args, threads=k) for k in (1, 3, 8)]
    for o in outs:
        assert np.array_equal(o["corr"], seq["corr"])
        assert np.array_equal(o["terms"], outs[0]["terms"])
        assert np.array_equal(o["abs_terms"], outs[0]["abs_terms"])
    tol = 1e-12 * np.maximum(np.abs(seq["terms"]), seq["abs_terms"])
    assert np.all(np.abs(outs[0]["terms"] - seq["terms"]) <= tol)
    # abs_terms from the records, recomputed in numpy (fp64; order-free check)
    m = seq["corr"] >= 0
    s = oracle.transform(w["init_T"], w["source"])[m]
    q = w["target"][seq["corr"][m]].astype(np.float64)
    n = w["target_normals"][seq["corr"][m]].astype(np.float64)
    J = np.concatenate([np.cross(s, n), n], 1)
    r = ((s - q) * n).sum(1)
    iu = np.triu_indices(6)
    ab = np.concatenate([np.abs(J[:, iu[0]] * J[:, iu[1]]).sum(0), np.abs(J * r[:, None]).sum(0),
                         [m.sum(), seq["d2"][m].sum()]])
    assert np.allclose(seq["abs_terms"], ab, rtol=1e-12, atol=0)
    assert np.allclose(outs[0]["abs_terms"], ab, rtol=1e-12, atol=0)


def test_chunked_icp_matches_sequential():
    """The OpenMP loop follows the same iterates: same iteration count and
    flags, T within 1e-9 (the per-pass terms agree within R14)."""
    from synth import make
    w = make("tiny")
    a = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], w["iters"])
    b = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], w["iters"], threads=4)
    assert a["iterations"] == b["iterations"] and a["flags"] == b["flags"]
    assert np.abs(a["T"] - b["T"]).max() <= 1e-9
