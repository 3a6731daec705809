"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): correspondence indices bit-exact for the
same T_in; JTJ / JTr within 1e-9 relative (R14: |a-b| <= 1e-9 max(|b|,
sum|terms|)); final T within 1e-6 per element; fitness and inlier_rmse
within 1e-6.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth.rng import Stream
from synth.scenes import rigid, rotation

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLD = os.path.join(os.path.dirname(__file__), "golden")

# name -> {option: value}: O3G_OPT_SEARCH (1), O3G_OPT_PRUNE_MIN (10)
SEARCH = {"exact": {1: 0}, "balanced": {1: 1}, "pruned": {1: 1, 10: 0}, "unpruned": {1: 1, 10: -2},
          "interleaved": {1: 1, 11: 1},
          # every query cooperative, rows pruned, x-sorted target with x-windows
          "coopx": {1: 1, 6: 1, 10: 0, 12: 1},
          "prefilter": {1: 2}, "sorted": {1: 3}, "tiled": {1: 4}}
GRID = {"dense": 1, "hashed": 2}


@pytest.fixture(scope="module")
def o3g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1801_09847_b200 as m
    m.lib()
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def _ctx(o3g, w, search="balanced", grid="dense", order_T=None, src=None):
    ctx = o3g.Context(0)
    for opt, val in SEARCH[search].items():
        ctx.set_option(opt, val)
    ctx.set_option(2, GRID[grid])
    ctx.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
    ctx.set_source(_dev(w["source"] if src is None else src), order_T)
    return ctx


def _terms_ok(gpu, ref, rel=1e-9):
    tol = rel * np.maximum(np.abs(ref["terms"]), ref["abs_terms"]) + 1e-300
    bad = np.abs(gpu - ref["terms"]) > tol
    assert not bad.any(), (np.nonzero(bad), gpu[bad], ref["terms"][bad])


def _step(ctx, T, n):
    corr = torch.full((n,), -7, dtype=torch.int32, device="cuda")
    st = ctx.step(T, corr_out=corr)
    return corr.cpu().numpy(), st


def _perturb(seed, ang=0.01, tr=0.01):
    rs = Stream(seed)
    return rigid(rotation(rs.unit_vectors(1)[0], ang), rs.uniform(3, -tr, tr))


# -------------------------------------------------------------- golden
def test_hand_step_golden_gpu(o3g):
    g = json.load(open(os.path.join(GOLD, "hand_step.json")))
    for c in g["cases"]:
        w = dict(source=np.array(c["source"]), target=np.array(c["target"]),
                 target_normals=np.array(c["normals"]), dmax=c["dmax"])
        for search in SEARCH:
            for grid in GRID:
                with _ctx(o3g, w, search, grid) as ctx:
                    corr, st = _step(ctx, np.array(c["T"], float), len(c["source"]))
                    assert corr.tolist() == c["corr"], (c["name"], search, grid)
                    up = np.array([st["JTJ"][i, j] for i in range(6) for j in range(i, 6)])
                    assert np.array_equal(up, np.array(c["jtj_upper"], float))
                    assert np.array_equal(st["JTr"], np.array(c["jtr"], float))
                    assert st["count"] == c["count"] and st["sum_sq_dist"] == c["sum_sq_dist"]


def test_dyadic_nn_golden_gpu(o3g):
    g = json.load(open(os.path.join(GOLD, "dyadic_nn.json")))
    for c in g["cases"]:
        tgt = np.array(c["target"], np.float32)
        w = dict(source=np.array([c["query"]], np.float32), target=tgt,
                 target_normals=np.tile([0, 0, 1], (len(tgt), 1)), dmax=c["dmax"])
        for search in SEARCH:
            for grid in GRID:
                with _ctx(o3g, w, search, grid) as ctx:
                    corr, st = _step(ctx, np.eye(4), 1)
                    assert corr[0] == c["expect"], (c["name"], search, grid)
                    if c["expect_d2"] is not None:
                        assert st["sum_sq_dist"] == c["expect_d2"]


def test_adversarial_lattice_ties(o3g):
    """Dyadic lattice, spacing == dmax, duplicated points at higher indices,
    queries on the half-lattice: exact ties, d == dmax, shared boundaries."""
    dmax = 0.25
    g = np.arange(-4, 5) * 0.25
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    tgt = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    tgt = np.concatenate([tgt, tgt[::7]]).astype(np.float32)
    rs = Stream(5)
    nrm = rs.unit_vectors(len(tgt)).astype(np.float32)
    qs = np.stack(np.meshgrid(*(np.arange(-9, 10) * 0.125,) * 3, indexing="ij"), -1).reshape(-1, 3)
    w = dict(source=qs.astype(np.float32), target=tgt, target_normals=nrm, dmax=dmax)
    ref = oracle.step(np.eye(4), qs, tgt, nrm, dmax, grid=None)
    for search in SEARCH:
        for grid in GRID:
            with _ctx(o3g, w, search, grid) as ctx:
                corr, st = _step(ctx, np.eye(4), len(qs))
                assert np.array_equal(corr, ref["corr"]), (search, grid)
                _terms_ok(st["terms"], ref)


def test_ulp_boundary_queries(o3g):
    """Queries 1 ulp either side of d == dmax and of cell boundaries."""
    dmax = 0.0625
    tgt = np.array([[0, 0, 0], [0.0625, 0, 0], [1, 1, 1], [0.125, 0.0625, 0]], np.float32)
    base = np.float32(0.0625)
    xs = [np.nextafter(base, np.float32(0)), base, np.nextafter(base, np.float32(1))]
    q = []
    for x in xs:
        q += [[x, 0, 0], [-x, 0, 0], [0, x, 0], [2 * x, 0, 0], [x, x, 0], [0.125 + x, 0.0625, 0]]
    q = np.array(q, np.float32)
    nrm = np.tile([0, 0, 1], (4, 1)).astype(np.float32)
    w = dict(source=q, target=tgt, target_normals=nrm, dmax=dmax)
    for T in (np.eye(4), rigid(np.eye(3), [2.0 ** -30, -(2.0 ** -28), 0])):
        ref = oracle.step(T, q, tgt, nrm, dmax, grid=None)
        for search in SEARCH:
            with _ctx(o3g, w, search) as ctx:
                corr, _ = _step(ctx, T, len(q))
                assert np.array_equal(corr, ref["corr"]), search


# -------------------------------------------------------- configs: step
def _configs(workloads):
    out = [("tiny", workloads("tiny"), None)]
    out.append(("depth", workloads("depth"), None))
    lid = workloads("lidar")
    out.append(("lidar", lid, Stream(11).integers(4000, len(lid["source"]))))
    big = workloads("large16m", n=400_000)
    out.append(("large400k", big, Stream(12).integers(20000, len(big["source"]))))
    return out


@pytest.mark.parametrize("search", list(SEARCH))
def test_step_parity_configs(o3g, workloads, search):
    for name, w, subset in _configs(workloads):
        grid = oracle.Grid(w["target"], w["dmax"])
        Ts = [w["init_T"], w["T_true"], w["T_true"] @ _perturb(3, 0.003, 0.005)]
        with _ctx(o3g, w, search, order_T=w["init_T"]) as ctx:
            for T in Ts:
                corr, st = _step(ctx, T, len(w["source"]))
                ref = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"],
                                  grid=grid, subset=subset)
                got = corr if subset is None else corr[subset]
                assert np.array_equal(got, ref["corr"]), (name, search, int((got != ref["corr"]).sum()))
                if subset is None:
                    _terms_ok(st["terms"], ref)
                else:
                    assert st["count"] == float((corr >= 0).sum())
                    A = st["JTJ"]
                    assert np.array_equal(A, A.T)
                    ev = np.linalg.eigvalsh(A)
                    assert ev.min() >= -1e-9 * ev.max()


def test_hashed_grid_matches_dense(o3g, workloads):
    w = workloads("depth")
    T = w["T_true"] @ _perturb(4, 0.01, 0.01)
    out = {}
    for grid in GRID:
        with _ctx(o3g, w, "balanced", grid) as ctx:
            out[grid] = _step(ctx, T, len(w["source"]))
            info = ctx.grid_info()
            assert info["hashed"] == (grid == "hashed")
    assert np.array_equal(out["dense"][0], out["hashed"][0])
    ref = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"])
    _terms_ok(out["hashed"][1]["terms"], ref)


# -------------------------------------------------------- configs: loop
@pytest.mark.parametrize("grid", list(GRID))
@pytest.mark.parametrize("name", ["tiny", "depth"])
def test_loop_parity(o3g, workloads, name, grid):
    w = workloads(name)
    ref = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], w["iters"],
                     init_T=w["init_T"])
    for search in SEARCH:
        with _ctx(o3g, w, search, grid, order_T=w["init_T"]) as ctx:
            r = ctx.run(w["init_T"], w["iters"], history=True)
        assert np.abs(r.transformation - ref["T"]).max() <= 1e-6, (name, search)
        assert abs(r.fitness - ref["fitness"]) <= 1e-6
        assert abs(r.inlier_rmse - ref["inlier_rmse"]) <= 1e-6
        assert r.iterations == ref["iterations"] and r.converged == ref["converged"]
        assert r.flags == ref["flags"]
        n = min(len(r.hist_fitness), len(ref["hist_fitness"]))
        assert np.abs(r.hist_fitness[:n] - ref["hist_fitness"][:n]).max() <= 1e-6


def test_loop_parity_lidar_subsample(o3g, workloads):
    """LiDAR: ~6.6k candidates per query make the oracle slow; loop parity on
    a 3000-point source subsample against the full target."""
    w = workloads("lidar")
    sub = np.sort(Stream(13).integers(3000, len(w["source"])))
    src = w["source"][sub]
    ref = oracle.icp(src, w["target"], w["target_normals"], w["dmax"], 10)
    with _ctx(o3g, w, "balanced", src=src) as ctx:
        r = ctx.run(np.eye(4), 10)
    assert np.abs(r.transformation - ref["T"]).max() <= 1e-6
    assert abs(r.fitness - ref["fitness"]) <= 1e-6 and abs(r.inlier_rmse - ref["inlier_rmse"]) <= 1e-6


def test_full_loop_recovers_motion_depth(o3g, workloads):
    w = workloads("depth")
    with _ctx(o3g, w) as ctx:
        r = ctx.run(w["init_T"], w["iters"])
    assert np.abs(r.transformation[:3, 3] - w["T_true"][:3, 3]).max() < 5e-3
    assert r.fitness > 0.5


# -------------------------------------------------------- API / edges
def test_one_shot_host_and_device_agree(o3g, workloads):
    w = workloads("tiny")
    a = o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], w["dmax"],
                               w["init_T"], w["iters"])
    b = o3g.icp_point_to_plane(_dev(w["source"]), _dev(w["target"]), _dev(w["target_normals"]),
                               w["dmax"], w["init_T"], w["iters"])
    assert np.array_equal(a.transformation, b.transformation)
    assert a.fitness == b.fitness and a.inlier_rmse == b.inlier_rmse
    with _ctx(o3g, w, order_T=w["init_T"]) as ctx:
        c = ctx.run(w["init_T"], w["iters"])
    assert np.array_equal(a.transformation, c.transformation)


def test_deterministic(o3g, workloads):
    w = workloads("depth")
    with _ctx(o3g, w) as ctx:
        r1 = ctx.run(w["init_T"], 10)
        r2 = ctx.run(w["init_T"], 10)
    assert np.array_equal(r1.transformation, r2.transformation) and r1.fitness == r2.fitness


@pytest.mark.parametrize("n", [1, 31, 257, 1025, 100_003])
def test_ragged_sizes(o3g, workloads, n):
    w = workloads("depth")
    src = np.concatenate([w["source"], w["source"] + np.float32(0.003)])[:n]
    T = w["T_true"]
    sub = None if n <= 2000 else np.arange(0, n, 37)
    with _ctx(o3g, w, src=src) as ctx:
        corr, st = _step(ctx, T, n)
    ref = oracle.step(T, src, w["target"], w["target_normals"], w["dmax"],
                      grid=oracle.Grid(w["target"], w["dmax"]), subset=sub)
    assert np.array_equal(corr if sub is None else corr[sub], ref["corr"])
    if sub is None:
        _terms_ok(st["terms"], ref)


def test_invalid_arguments(o3g, workloads):
    w = workloads("tiny")
    E = o3g.InvalidArgument
    with pytest.raises(E):
        o3g.icp_point_to_plane(np.zeros((0, 3)), w["target"], w["target_normals"], 0.05)
    with pytest.raises(E):
        o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], 0.0)
    with pytest.raises(E):
        o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], float("nan"))
    bad = w["source"].copy()
    bad[17, 1] = np.inf
    with pytest.raises(E):
        o3g.icp_point_to_plane(bad, w["target"], w["target_normals"], 0.05)
    badn = w["target_normals"].copy()
    badn[3, 0] = np.nan
    with pytest.raises(E):
        o3g.icp_point_to_plane(w["source"], w["target"], badn, 0.05)
    T = np.eye(4)
    T[0, 0] = 1.1
    with pytest.raises(E):
        o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], 0.05, init=T)
    with pytest.raises(E):
        o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], 0.05, max_iterations=-1)
    with pytest.raises(E):
        o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], 0.05, relative_rmse=-1)
    with pytest.raises(E):
        o3g.icp_point_to_plane(w["source"], w["target"], None, 0.05)
    # option ranges (include/o3g.h): every invalid value is rejected, valid ones accepted
    with o3g.Context(0) as ctx:
        for opt, bad_v in ((1, 5), (1, -1), (2, 3), (4, 65), (6, -2), (7, 2), (8, 2), (9, 2), (10, -4),
                           (11, 2), (11, -2), (12, 2), (13, 3), (13, -2), (14, -2), (15, 2), (15, -1), (99, 0)):
            with pytest.raises(E):
                ctx.set_option(opt, bad_v)
        for opt, ok_v in ((1, 4), (2, 0), (3, 1), (4, 0), (5, 0), (6, -1), (7, 0), (8, 1), (9, 0), (10, -2),
                          (11, -1), (12, -1), (13, -1), (13, 2), (14, 3), (14, -1), (15, 1), (15, 0)):
            ctx.set_option(opt, ok_v)


def test_batched_evaluation_chunks(o3g, workloads):
    """o3g_evaluate_registration processes transforms in chunks of 1024 per
    launch (bounded scratch, ADVICE): 2500 transforms give exactly the values
    of evaluating each chunk's transforms on their own."""
    w = workloads("tiny")
    Ts = np.stack([w["T_true"] @ _perturb(200 + k, 0.02, 0.02) for k in range(2500)])
    with _ctx(o3g, w) as ctx:
        fit, rmse = ctx.evaluate(Ts)
        f2, r2 = ctx.evaluate(Ts[1000:1100])
        f3, r3 = ctx.evaluate(Ts[2048:])
    assert np.array_equal(fit[1000:1100], f2) and np.array_equal(rmse[1000:1100], r2)
    assert np.array_equal(fit[2048:], f3) and np.array_equal(rmse[2048:], r3)
    grid = oracle.Grid(w["target"], w["dmax"])
    for k in (0, 1023, 1024, 2047, 2048, 2499):
        ref = oracle.step(Ts[k], w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid)
        assert fit[k] == ref["count"] / len(w["source"]), k


def test_flags_no_corr_and_degenerate(o3g, workloads):
    w = workloads("tiny")
    far = w["source"] + np.float32(100.0)
    r = o3g.icp_point_to_plane(far, w["target"], w["target_normals"], 0.05, max_iterations=5)
    assert r.flags & o3g.FLAG_NO_CORRESPONDENCES and r.fitness == 0 and r.inlier_rmse == 0
    assert np.array_equal(r.transformation, np.eye(4)) and r.iterations == 0
    rs = Stream(3)
    tgt = rs.uniform(15, -1, 1).reshape(5, 3).astype(np.float32)
    r = o3g.icp_point_to_plane(tgt, tgt, rs.unit_vectors(5), 0.1, max_iterations=5)
    ref = oracle.icp(tgt, tgt, rs.unit_vectors(5), 0.1, 5)
    assert r.flags == ref["flags"] == oracle.FLAG_DEGENERATE and r.iterations == 0
    # the tiny scene with source = target is exactly degenerate (yaw column of J is 0)
    r = o3g.icp_point_to_plane(w["target"], w["target"], w["target_normals"], 0.05)
    assert r.flags == o3g.FLAG_DEGENERATE and r.fitness == 1.0


def test_zero_iterations_and_criteria_semantics(o3g, workloads):
    w = workloads("tiny")
    for K, ef in ((0, 1e-6), (7, 0.0), (7, np.inf)):
        ref = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], K,
                         relative_fitness=ef, relative_rmse=ef)
        r = o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], w["dmax"],
                                   max_iterations=K, relative_fitness=ef, relative_rmse=ef)
        assert r.iterations == ref["iterations"] and r.passes == ref["passes"]
        assert abs(r.fitness - ref["fitness"]) <= 1e-12


def test_kernel_timing_and_launch_count(o3g, workloads):
    w = workloads("depth")
    with _ctx(o3g, w) as ctx:
        ctx.set_option(3, 1)
        before = ctx.launch_count()
        r = ctx.run(w["init_T"], 5, 0.0, 0.0)
        k3_ms, k3_n, tail_ms = ctx.last_run_kernel_ms()
        assert k3_n == r.passes == 6 and k3_ms > 0
        # variant 1 fuses the tail into the correspondence kernel: one launch per pass
        assert ctx.launch_count() - before == 6


# -------------------------------------------------- full-size (bench) config
@pytest.mark.slow
def test_large16m_full_size_sampled(o3g, workloads):
    """BASELINE config 5 at full size in the bench's launch configuration:
    sampled correspondences vs the oracle's grid, plus invariants."""
    w = workloads("large16m")
    sub = Stream(14).integers(20000, len(w["source"]))
    grid = oracle.Grid(w["target"], w["dmax"])
    with _ctx(o3g, w, order_T=w["init_T"]) as ctx:
        for T in (w["init_T"], w["T_true"]):
            corr, st = _step(ctx, T, len(w["source"]))
            ref = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"],
                              grid=grid, subset=sub)
            assert np.array_equal(corr[sub], ref["corr"])
            assert st["count"] == float((corr >= 0).sum())
            assert corr.max() < len(w["target"]) and corr.min() >= -1
        r = ctx.run(w["init_T"], 30, 0.0, 0.0, history=True)
        # evaluating at the returned T reproduces the stored fitness / rmse
        corr, st = _step(ctx, r.transformation, len(w["source"]))
    assert r.iterations == 30 and r.passes == 31
    assert st["count"] / len(w["source"]) == r.fitness
    assert abs(np.sqrt(st["sum_sq_dist"] / st["count"]) - r.inlier_rmse) <= 1e-12 * r.inlier_rmse
    # 3 deg about the scene centre moves far points ~1.3 m >> dmax: the loop
    # only partially recovers (SURVEY §8(d) caveat), but fitness must improve
    assert r.hist_fitness[-1] > r.hist_fitness[0]


def test_neighbour_mask_off_matches(o3g, workloads):
    """The dilated-occupancy skip (O3G_OPT_NBR_MASK) never changes results."""
    w = workloads("large16m", n=400_000)
    out = []
    for mask in (1, 0):
        with _ctx(o3g, w, "balanced") as ctx:
            ctx.set_option(5, mask)
            out.append(_step(ctx, w["T_true"], len(w["source"])))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1]["terms"], out[1][1]["terms"])


@pytest.mark.parametrize("name", ["depth", "lidar"])
def test_cooperative_threshold_invariance(o3g, workloads, name):
    """O3G_OPT_COOP_MIN (warp-cooperative scan of heavy queries) never changes
    the correspondences: all queries cooperative (1), default (64), none (0)."""
    w = workloads(name)
    T = w["T_true"] @ _perturb(21, 0.004, 0.01)
    sub = None if name == "depth" else Stream(22).integers(3000, len(w["source"]))
    ref = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"],
                      grid=oracle.Grid(w["target"], w["dmax"]), subset=sub)
    outs = []
    for cm, search in ((1, "balanced"), (64, "balanced"), (0, "balanced"), (0, "pruned"), (64, "pruned")):
        with _ctx(o3g, w, search) as ctx:
            ctx.set_option(6, cm)
            corr, st = _step(ctx, T, len(w["source"]))
        got = corr if sub is None else corr[sub]
        assert np.array_equal(got, ref["corr"]), cm
        outs.append((corr, st))
        if sub is None:
            _terms_ok(st["terms"], ref)
    assert np.array_equal(outs[0][0], outs[2][0])


def test_source_order_option_invariance(o3g, workloads):
    """O3G_OPT_SOURCE_ORDER only changes locality: identical correspondences
    and terms within the R14 tolerance."""
    w = workloads("depth")
    T = w["T_true"] @ _perturb(23, 0.003, 0.004)
    ref = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"])
    for order in (0, 1):
        ctx = o3g.Context(0)
        ctx.set_option(8, order)
        ctx.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
        ctx.set_source(_dev(w["source"]), w["init_T"])
        corr, st = _step(ctx, T, len(w["source"]))
        ctx.close()
        assert np.array_equal(corr, ref["corr"]), order
        _terms_ok(st["terms"], ref)


def test_target_sort_invariance(o3g, workloads):
    """Counting-sort vs stable radix-sort target layouts give bit-identical
    correspondences AND terms (records are summed in source order)."""
    w = workloads("large16m", n=400_000)
    T = w["T_true"]
    out = []
    for ts in (0, 1):
        ctx = o3g.Context(0)
        ctx.set_option(9, ts)
        ctx.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
        ctx.set_source(_dev(w["source"]), w["init_T"])
        out.append(_step(ctx, T, len(w["source"])))
        info = ctx.grid_info()
        r = ctx.run(w["init_T"], 5, 0.0, 0.0)
        out[-1] = out[-1] + (r, info)
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1]["terms"], out[1][1]["terms"])
    assert np.array_equal(out[0][2].transformation, out[1][2].transformation)
    assert out[0][3]["occupied_cells"] == out[1][3]["occupied_cells"]


def test_row_pruning_face_stress(o3g):
    """Row pruning near cell faces: targets and queries
    placed within a few ulps of the grid's face planes, so the row lower
    bounds are ~0 and own-row / face-row candidates tie or nearly tie."""
    dmax = 0.125
    h = dmax * (1 + 2.0 ** -20)
    rs = Stream(77)
    m = rs.integers(6000, 8).astype(np.float64)
    base = rs.uniform(3 * 6000, 0.0, 1.0).reshape(-1, 3)
    tgt = np.floor(base * 8) * h
    tgt[:, 0] = base[:, 0]                                 # x free, y/z on face planes
    jit = rs.integers(3 * 6000, 5).reshape(-1, 3) - 2      # -2..2 ulp
    tgt = tgt.astype(np.float32)
    for k in range(3):
        for step in range(2):
            sel = jit[:, k] > step
            tgt[sel, k] = np.nextafter(tgt[sel, k], np.float32(2))
            sel = jit[:, k] < -step
            tgt[sel, k] = np.nextafter(tgt[sel, k], np.float32(-2))
    tgt = np.concatenate([tgt, tgt[::5] + np.float32(0.25 * h)])
    q = tgt[rs.integers(3000, len(tgt))] + (rs.uniform(3 * 3000, -1, 1).reshape(-1, 3) * 0.2 * h).astype(np.float32)
    q[::3, 1] = tgt[rs.integers(1000, len(tgt)), 1]       # queries exactly on face planes
    nrm = rs.unit_vectors(len(tgt)).astype(np.float32)
    w = dict(source=q.astype(np.float32), target=tgt.astype(np.float32), target_normals=nrm, dmax=dmax)
    ref = oracle.step(np.eye(4), w["source"], w["target"], nrm, dmax, grid=None)
    assert (ref["corr"] >= 0).sum() > 1000
    for search in ("pruned", "unpruned", "balanced"):
        with _ctx(o3g, w, search) as ctx:
            corr, st = _step(ctx, np.eye(4), len(q))
        assert np.array_equal(corr, ref["corr"]), search
        _terms_ok(st["terms"], ref)


def test_one_shot_overlapped_host_inputs(o3g, workloads):
    """The one-shot call with host inputs copies target, normals and source on
    a copy stream overlapped with the grid build; results equal the device
    path, a non-finite normal (checked after the overlapped copy) is still
    rejected, and the context recovers for the next call."""
    w = workloads("depth")
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory()
    a = o3g.icp_point_to_plane(pin(w["source"]), pin(w["target"]), pin(w["target_normals"]), w["dmax"],
                               w["init_T"], w["iters"])
    b = o3g.icp_point_to_plane(_dev(w["source"]), _dev(w["target"]), _dev(w["target_normals"]),
                               w["dmax"], w["init_T"], w["iters"])
    assert np.array_equal(a.transformation, b.transformation) and a.fitness == b.fitness
    bad = w["target_normals"].copy()
    bad[1234, 1] = np.nan
    with pytest.raises(o3g.InvalidArgument):
        o3g.icp_point_to_plane(pin(w["source"]), pin(w["target"]), pin(bad), w["dmax"], w["init_T"], 3)
    c = o3g.icp_point_to_plane(w["source"], w["target"], w["target_normals"], w["dmax"],
                               w["init_T"], w["iters"])
    assert np.array_equal(c.transformation, b.transformation)


def test_loop_parity_warm_start(o3g, workloads):
    """The run loop's warm start (rows pruned by the previous pass's winner,
    DESIGN.md §5.2c) on a sparse 400k-point scene where queries move between
    dead and live across passes: same loop as the oracle."""
    w = workloads("large16m", n=400_000)
    T0 = w["T_true"] @ _perturb(31, 0.004, 0.01)
    ref = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], 6, init_T=T0)
    for search, grid, cert in (("balanced", "dense", 1), ("unpruned", "dense", 1), ("balanced", "dense", 0),
                               ("balanced", "hashed", 1), ("balanced", "hashed", 0)):
        with _ctx(o3g, w, search, grid, order_T=T0) as ctx:
            ctx.set_option(o3g.OPT_CERT, cert)
            r = ctx.run(T0, 6, history=True)
        assert np.abs(r.transformation - ref["T"]).max() <= 1e-6, search
        assert abs(r.fitness - ref["fitness"]) <= 1e-6 and abs(r.inlier_rmse - ref["inlier_rmse"]) <= 1e-6
        assert r.iterations == ref["iterations"]
        n = min(len(r.hist_fitness), len(ref["hist_fitness"]))
        assert np.abs(r.hist_fitness[:n] - ref["hist_fitness"][:n]).max() <= 1e-6


@pytest.mark.slow
def test_large16m_converged_regime_sampled(o3g, workloads):
    """BASELINE config 5 at full size started near T* (every query live: the
    live-query queue is skipped after the first pass and every pass after the
    first runs warm-started): the loop's result satisfies S:305 and a step at
    the returned T matches the oracle on sampled queries."""
    w = workloads("large16m")
    T0 = w["T_true"] @ _perturb(41, 0.0017, 0.01)
    sub = Stream(42).integers(20000, len(w["source"]))
    grid = oracle.Grid(w["target"], w["dmax"])
    with _ctx(o3g, w, order_T=T0) as ctx:
        r = ctx.run(T0, 5, 0.0, 0.0, history=True)
        corr, st = _step(ctx, r.transformation, len(w["source"]))
    assert r.fitness > 0.9 and r.iterations == 5
    assert st["count"] / len(w["source"]) == r.fitness
    assert abs(np.sqrt(st["sum_sq_dist"] / st["count"]) - r.inlier_rmse) <= 1e-12 * r.inlier_rmse
    ref = oracle.step(r.transformation, w["source"], w["target"], w["target_normals"], w["dmax"],
                      grid=grid, subset=sub)
    assert np.array_equal(corr[sub], ref["corr"])


# ---------------------------------------- run loop: every pass against the oracle
def _trace_cases(workloads):
    big = workloads("large16m", n=400_000)
    return [("tiny", workloads("tiny"), None, 20, None),
            ("depth", workloads("depth"), None, 30, None),
            ("large400k", big, big["T_true"] @ _perturb(31, 0.004, 0.01), 6, None),
            # T_init regime of the bench config (far from converged, most queries dead)
            ("large400k_init", big, None, 6, None)]


@pytest.mark.parametrize("grid", list(GRID))
@pytest.mark.parametrize("cert,sweep", [(1, 0), (0, 0), (1, 1), (2, 0)])
def test_run_loop_every_pass(o3g, workloads, grid, cert, sweep):
    """The run loop's own passes — warm-started searches and, with
    O3G_OPT_CERT, queries settled by a correspondence certificate (DESIGN.md
    §5.5) — are only reachable inside o3g_icp_run. o3g_last_run_trace gives
    the T each pass ran with and its 29 terms: every pass's terms must match
    the oracle's pass at that T (R14; count exact), and at traced passes the
    correspondences must be bit-identical. With certificates on, fewer
    queries run the full search than with them off, and the loop's T is
    bitwise the same either way. Certificate passes run fused into the
    search kernel (sweep 0) or with the separate sweep kernel (sweep 1);
    cert 2 forces them from the second pass (the T_init regime)."""
    for name, w, T0, iters, _ in _trace_cases(workloads):
        T0 = w["init_T"] if T0 is None else T0
        n = len(w["source"])
        grid_o = oracle.Grid(w["target"], w["dmax"])
        with _ctx(o3g, w, "balanced", grid, order_T=T0) as ctx:
            ctx.set_option(o3g.OPT_CERT, cert)
            ctx.set_option(o3g.OPT_CERT_SWEEP, sweep)
            r = ctx.run(T0, iters, 0.0, 0.0)
            tr = ctx.last_run_trace(r.passes)
            refs = [oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid_o)
                    for T in tr["T"]]
            for k, ref in enumerate(refs):
                _terms_ok(tr["terms"][k], ref)
                assert tr["terms"][k][27] == ref["count"], (name, k)
            assert np.array_equal(tr["T"][-1], r.transformation) or r.iterations < r.passes - 1
            for k in sorted({0, 1, 2, r.passes // 2, r.passes - 1}):
                ctx.set_option(o3g.OPT_TRACE_PASS, k)
                corr = torch.full((n,), -7, dtype=torch.int32, device="cuda")
                r2 = ctx.run(T0, iters, 0.0, 0.0)
                tk = ctx.last_run_trace(r2.passes, corr)
                assert np.array_equal(tk["T"], tr["T"]), (name, k)             # deterministic
                got = corr.cpu().numpy()
                assert np.array_equal(got, refs[k]["corr"]), (name, grid, cert, k, int((got != refs[k]["corr"]).sum()))
            ctx.set_option(o3g.OPT_TRACE_PASS, -1)
            # the other setting: same loop, bit for bit (certificates are exact)
            ctx.set_option(o3g.OPT_CERT, 0 if cert else 1)
            r3 = ctx.run(T0, iters, 0.0, 0.0)
            t3 = ctx.last_run_trace(r3.passes)
        assert r3.passes == r.passes
        for k in range(r.passes):
            _terms_ok(t3["terms"][k], refs[k])
        on, off = (tr, t3) if cert else (t3, tr)
        assert on["searched"][0] == off["searched"][0]
        # (a pass runs with certificates once the previous pass matched > 1/2 of
        # the source; before that, both settings run the same plain pass)
        if cert == 2 and r.passes > 2:
            assert on["certified"][2:].sum() > 0, name
        if on["certified"].sum() > 0:
            assert on["searched"][1:].sum() < off["searched"][1:].sum(), name
        else:
            assert np.array_equal(on["searched"], off["searched"]), name
            assert np.all(np.array([t[27] for t in on["terms"]]) <= len(w["source"]) / 2 + 1) or r.passes <= 1
        assert off["certified"].sum() == 0
        assert np.all(on["searched"] <= n) and np.all(on["candidates"] >= 0)
        assert np.all(on["certified"] + on["searched"] <= n)


def test_run_loop_state_reset_between_runs(o3g, workloads):
    """The run loop's per-query state (certificates / warm-start winners) is
    reset at the head of every run: a run after a different run on the same
    context equals the same run on a fresh context, bit for bit."""
    w = workloads("large16m", n=400_000)
    Ta = w["T_true"] @ _perturb(51, 0.004, 0.01)
    Tb = w["T_true"] @ _perturb(52, 0.006, 0.02)
    for cert in (1, 0):
        with _ctx(o3g, w, "balanced", order_T=Ta) as ctx:
            ctx.set_option(o3g.OPT_CERT, cert)
            ctx.run(Ta, 8, 0.0, 0.0)
            rb = ctx.run(Tb, 8, 0.0, 0.0)
        with _ctx(o3g, w, "balanced", order_T=Ta) as ctx:
            ctx.set_option(o3g.OPT_CERT, cert)
            fresh = ctx.run(Tb, 8, 0.0, 0.0)
        assert np.array_equal(rb.transformation, fresh.transformation), cert
        assert rb.fitness == fresh.fitness and rb.inlier_rmse == fresh.inlier_rmse


# ------------------------------------------------ A7: the multi-rank path (loopback)
@pytest.mark.parametrize("world,transport", [(2, "copy"), (4, "copy"), (8, "copy"), (2, "peer"), (8, "peer")])
def test_loopback_multi_rank(o3g, workloads, world, transport):
    """SURVEY §8(e) / A7 on one device: P contexts, each keeping its contiguous
    shard of the spatially ordered source, run the distributed loop in
    lockstep — per-shard correspondence kernels, TAIL_WRITE_RANK, the slot
    exchange (device copies standing in for the NCCL all-gather) and the
    rank-order TAIL_SUM_RANKS tail. The union of the shards' correspondences
    equals the 1-GPU pass bit for bit at every traced pass; every pass's
    rank-summed terms agree with the 1-GPU pass (R14) and with the oracle at
    that T; T is bit-identical on every rank (checked inside the call) and
    the loop matches the oracle's (1e-6). transport "peer": the one-shot
    peer-memory exchange (each rank's last K3 block stores its slot into every
    rank's exchange buffer and releases the pass's epoch flag; the tails
    acquire the flags) instead of copies of the gathered slots; several runs
    on the same contexts exercise both parities and growing epochs."""
    w = workloads("large16m", n=400_000)
    T0 = w["T_true"] @ _perturb(61, 0.004, 0.01)
    iters = 6
    n = len(w["source"])
    grid_o = oracle.Grid(w["target"], w["dmax"])
    ref = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], iters, init_T=T0,
                     relative_fitness=0.0, relative_rmse=0.0)
    for cert in (1, 0):
        with _ctx(o3g, w, "balanced", order_T=T0) as one:
            one.set_option(o3g.OPT_CERT, cert)
            r1 = one.run(T0, iters, 0.0, 0.0)
            t1 = one.last_run_trace(r1.passes)
        ctxs = []
        try:
            for rk in range(world):
                c = o3g.Context(0)
                c.set_option(o3g.OPT_CERT, cert)
                c.set_option(2, GRID["dense"])
                c.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
                c.dist_init_loopback(rk, world)
                c.set_source(_dev(w["source"]), T0)
                ctxs.append(c)
            if transport == "peer":
                o3g.loopback_peer_connect(ctxs)
            rp = o3g.loopback_run(ctxs, T0, iters, 0.0, 0.0)
            assert rp.passes == r1.passes and rp.iterations == r1.iterations
            assert np.abs(rp.transformation - ref["T"]).max() <= 1e-6, cert
            assert abs(rp.fitness - ref["fitness"]) <= 1e-6 and abs(rp.inlier_rmse - ref["inlier_rmse"]) <= 1e-6
            tp = ctxs[0].last_run_trace(rp.passes)
            for k in range(rp.passes):
                refk = oracle.step(tp["T"][k], w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid_o)
                _terms_ok(tp["terms"][k], refk)
                _terms_ok(t1["terms"][k], refk)
            for k in (0, 1, rp.passes - 1):
                union = np.full(n, -3, np.int32)
                for c in ctxs:
                    c.set_option(o3g.OPT_TRACE_PASS, k)
                o3g.loopback_run(ctxs, T0, iters, 0.0, 0.0)
                for c in ctxs:
                    corr = torch.empty(n, dtype=torch.int32, device="cuda")
                    c.last_run_trace(rp.passes, corr)
                    got = corr.cpu().numpy()
                    mine = got != -2
                    assert np.all(union[mine] == -3)            # shards are disjoint
                    union[mine] = got[mine]
                assert np.all(union != -3)                      # and cover the source
                refk = oracle.step(tp["T"][k], w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid_o)
                assert np.array_equal(union, refk["corr"]), (world, cert, k)
        finally:
            for c in ctxs:
                c.close()


def test_set_clouds_matches_sequential(o3g, workloads):
    """o3g_set_clouds (the source's ordering on a side stream beside the target
    build) leaves exactly the state of o3g_set_target + o3g_set_source: step
    correspondences and terms, and the loop's T, fitness and rmse are equal
    bit for bit, on a sparse target (tiny), a pruning-instantiation target
    (depth), an x-sorted dense target (lidar) and a 400k shard; repeated calls
    on one context reuse the side scratch; non-finite input fails the call."""
    cases = [("tiny", workloads("tiny")), ("depth", workloads("depth")), ("lidar", workloads("lidar")),
             ("large400k", workloads("large16m", n=400_000))]
    for name, w in cases:
        T0 = w["init_T"]
        n = len(w["source"])
        s_, t_, n_ = _dev(w["source"]), _dev(w["target"]), _dev(w["target_normals"])
        out = []
        for mode in ("sequential", "clouds", "clouds"):
            ctx = out[1][3] if mode == "clouds" and len(out) == 2 else o3g.Context(0)
            if mode == "sequential":
                ctx.set_target(t_, n_, w["dmax"])
                ctx.set_source(s_, T0)
            else:
                ctx.set_clouds(s_, t_, n_, w["dmax"], T0)
            corr = torch.empty(n, dtype=torch.int32, device="cuda")
            st = ctx.step(T0, corr_out=corr)
            r = ctx.run(T0, min(w["iters"], 8))
            out.append((st["terms"].copy(), corr.cpu().numpy(), r, ctx, ctx.grid_info()))
        a = out[0]
        for b in out[1:]:
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), name
            assert np.array_equal(a[2].transformation, b[2].transformation), name
            assert a[2].fitness == b[2].fitness and a[2].inlier_rmse == b[2].inlier_rmse, name
            assert a[4] == b[4], name
        out[0][3].close()
        out[1][3].close()
    w = workloads("tiny")
    bad_s = w["source"].copy()
    bad_s[17, 1] = np.nan
    bad_t = w["target"].copy()
    bad_t[5, 0] = np.inf
    with o3g.Context(0) as ctx:
        with pytest.raises(o3g.InvalidArgument):
            ctx.set_clouds(_dev(bad_s), _dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
        with pytest.raises(o3g.InvalidArgument):
            ctx.set_clouds(_dev(w["source"]), _dev(bad_t), _dev(w["target_normals"]), w["dmax"])
        with pytest.raises(o3g.O3GError):
            ctx.step(w["init_T"])                      # (nothing usable was set)
        ctx.set_clouds(_dev(w["source"]), _dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
        ref = oracle.step(w["init_T"], w["source"], w["target"], w["target_normals"], w["dmax"])
        _terms_ok(ctx.step(w["init_T"])["terms"], ref)


def test_nccl_leg_one_rank(o3g, workloads):
    """The NCCL leg of A7 on one GPU: o3g_dist_init(rank 0, world 1, id) creates
    a one-rank communicator, and every pass then runs the distributed sequence
    — K3's last block writes the rank slot, the graph-captured ncclAllGather,
    the rank-order tail — instead of the fused single-GPU tail. Step terms,
    the loop's T, fitness and rmse equal the single-GPU path's bit for bit
    (one slot, same summation order), and the loop matches the oracle."""
    w = workloads("depth")
    T0 = w["init_T"]
    try:
        uid = o3g.nccl_unique_id()
    except o3g.O3GError as e:   # (no libnccl.so.2 in this environment)
        pytest.skip(f"NCCL not loadable: {e}")
    ref = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], w["iters"], init_T=T0)
    res = {}
    for mode in ("single", "nccl"):
        with o3g.Context(0) as ctx:
            ctx.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
            if mode == "nccl":
                ctx.dist_init(0, 1, uid)
            ctx.set_source(_dev(w["source"]), T0)
            corr = torch.empty(len(w["source"]), dtype=torch.int32, device="cuda")
            st = ctx.step(T0, corr_out=corr)
            l0 = ctx.launch_count()
            r = ctx.run(T0, w["iters"])
            res[mode] = (st["terms"].copy(), corr.cpu().numpy(), r, ctx.launch_count() - l0)
    (t1, c1, r1, n1), (t2, c2, r2, n2) = res["single"], res["nccl"]
    assert np.array_equal(t1, t2) and np.array_equal(c1, c2)
    assert np.array_equal(r1.transformation, r2.transformation)
    assert r1.fitness == r2.fitness and r1.inlier_rmse == r2.inlier_rmse and r1.iterations == r2.iterations
    assert n2 > n1                      # (the distributed pass adds the rank-order tail launch)
    assert np.abs(r2.transformation - ref["T"]).max() <= 1e-6
    assert abs(r2.fitness - ref["fitness"]) <= 1e-6 and abs(r2.inlier_rmse - ref["inlier_rmse"]) <= 1e-6


def test_certificate_tags_wrap(o3g, workloads):
    """Certificate records carry a 16-bit pass tag that advances across runs;
    records of an earlier run are older than any usable age, and the records
    are reset when the tags wrap (~2100 runs of 31 passes here): every run
    equals a fresh context's run bit for bit."""
    w = workloads("tiny")
    T0 = w["init_T"]
    with _ctx(o3g, w, "balanced", order_T=T0) as ctx:
        ctx.set_option(o3g.OPT_CERT, 1)
        ref = ctx.run(T0, w["iters"], 0.0, 0.0)
        Ts = [w["T_true"] @ _perturb(70 + k, 0.01, 0.01) for k in range(3)]
        fresh = []
        for T in Ts:
            with _ctx(o3g, w, "balanced", order_T=T0) as c2:
                c2.set_option(o3g.OPT_CERT, 1)
                fresh.append(c2.run(T, 30, 0.0, 0.0))
        for k in range(2200):
            j = k % 3
            r = ctx.run(Ts[j], 30, 0.0, 0.0)
            if k % 97 == 0 or k > 2090:
                assert np.array_equal(r.transformation, fresh[j].transformation), k
                assert r.fitness == fresh[j].fitness, k
        r = ctx.run(T0, w["iters"], 0.0, 0.0)
        assert np.array_equal(r.transformation, ref.transformation)
