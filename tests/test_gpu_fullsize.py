"""Full-size parity at the benchmarked sizes (BASELINE configs 4 and 5), against
the oracle's deterministic OpenMP mode (the same per-query results as the
sequential oracle, tests/test_oracle.py::test_chunked_pass_deterministic_and_equal;
bitwise the same for any thread count) on every host core:

- large16m (16M / 16M): every correspondence bit-exact and the 29 terms within
  R14 at the start T and at T*; the full 30-update loop in the launch
  configuration bench.py times (certificates on by default) with T within
  1e-6, fitness and rmse within 1e-6, the same updates and flags; and every
  fifth pass of that loop against the oracle's pass at the T it ran with;
  the converged regime (certificates carrying most passes) likewise.
- fragment (2M / 2M, three scales): the multi-scale loop at the benchmarked size.
"""
import os

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def o3g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1801_09847_b200 as m
    m.lib()
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def _terms_ok(gpu, ref, rel=1e-9):
    tol = rel * np.maximum(np.abs(ref["terms"]), ref["abs_terms"]) + 1e-300
    bad = np.abs(gpu - ref["terms"]) > tol
    assert not bad.any(), (np.nonzero(bad), gpu[bad], ref["terms"][bad])


@pytest.fixture(scope="module")
def big(workloads):
    w = workloads("large16m")
    return w, oracle.Grid(w["target"], w["dmax"])


def test_large16m_full_step_parity(o3g, big):
    w, grid = big
    n = len(w["source"])
    with o3g.Context(0) as ctx:
        ctx.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
        ctx.set_source(_dev(w["source"]), w["init_T"])
        for T in (w["init_T"], w["T_true"]):
            corr = torch.full((n,), -7, dtype=torch.int32, device="cuda")
            st = ctx.step(T, corr_out=corr)
            ref = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid,
                              threads=THREADS)
            got = corr.cpu().numpy()
            assert np.array_equal(got, ref["corr"]), int((got != ref["corr"]).sum())
            _terms_ok(st["terms"], ref)


def test_large16m_full_loop_parity(o3g, big):
    """The bench's registration (30 updates from the config's start T, the
    criteria off as in the bench) against the oracle's loop, and every fifth
    of its 31 passes against the oracle's pass at the T that pass ran with."""
    w, grid = big
    ref = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], 30, init_T=w["init_T"],
                     relative_fitness=0.0, relative_rmse=0.0, threads=THREADS)
    with o3g.Context(0) as ctx:
        ctx.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
        ctx.set_source(_dev(w["source"]), w["init_T"])
        r = ctx.run(w["init_T"], 30, 0.0, 0.0, history=True)
        tr = ctx.last_run_trace(r.passes)
    assert r.iterations == ref["iterations"] == 30 and r.flags == ref["flags"]
    assert np.abs(r.transformation - ref["T"]).max() <= 1e-6
    assert abs(r.fitness - ref["fitness"]) <= 1e-6 and abs(r.inlier_rmse - ref["inlier_rmse"]) <= 1e-6
    assert np.abs(r.hist_fitness - ref["hist_fitness"]).max() <= 1e-6
    for k in range(0, r.passes, 5):
        refk = oracle.step(tr["T"][k], w["source"], w["target"], w["target_normals"], w["dmax"], grid=grid,
                           threads=THREADS)
        _terms_ok(tr["terms"][k], refk)
        assert tr["terms"][k][27] == refk["count"], k


def test_large16m_converged_loop_parity_certificates(o3g, big):
    """Converged regime at full size (every pass after the first few is
    settled mostly by certificates): the loop against the oracle's."""
    from synth.rng import Stream
    from synth.scenes import rigid, rotation
    w, grid = big
    rs = Stream(0x5EED)
    T0 = w["T_true"] @ rigid(rotation(rs.unit_vectors(1)[0], np.deg2rad(0.1)), 0.01 * rs.unit_vectors(1)[0])
    ref = oracle.icp(w["source"], w["target"], w["target_normals"], w["dmax"], 12, init_T=T0,
                     relative_fitness=0.0, relative_rmse=0.0, threads=THREADS)
    with o3g.Context(0) as ctx:
        ctx.set_target(_dev(w["target"]), _dev(w["target_normals"]), w["dmax"])
        ctx.set_source(_dev(w["source"]), T0)
        r = ctx.run(T0, 12, 0.0, 0.0, history=True)
        tr = ctx.last_run_trace(r.passes)
    assert tr["certified"][4:].min() > 0.5 * len(w["source"])   # certificates carried these passes
    assert np.abs(r.transformation - ref["T"]).max() <= 1e-6
    assert abs(r.fitness - ref["fitness"]) <= 1e-6 and abs(r.inlier_rmse - ref["inlier_rmse"]) <= 1e-6
    assert np.abs(r.hist_fitness - ref["hist_fitness"]).max() <= 1e-6


def test_fragment_full_size_multiscale(o3g, workloads):
    w = workloads("fragment")
    vox = [s["meta"]["voxel"] for s in w["scales"]]
    dm = [s["dmax"] for s in w["scales"]]
    its = [s["iters"] for s in w["scales"]]
    with o3g.Context(0) as ctx:
        r = ctx.run_multiscale(w["source"], w["target"], w["target_normals"], vox, dm, its)
    ref = oracle.icp_multiscale(w["source"], w["target"], w["target_normals"], vox, dm, its, threads=THREADS)
    assert np.array_equal(r["n_source"], ref["n_source"])
    assert np.array_equal(r["iterations"], ref["iterations"])
    assert np.abs(r["T"] - ref["T"]).max() <= 1e-6
    assert np.abs(r["fitness"] - ref["fitness"]).max() <= 1e-6
    assert np.abs(r["inlier_rmse"] - ref["inlier_rmse"]).max() <= 1e-6
