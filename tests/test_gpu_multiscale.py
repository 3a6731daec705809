"""GPU parity of the NEXT(1) row: device voxel_down_sample (bit-exact against
the oracle: same fp64 sums in original-index order, one fp32 rounding) and
the multi-scale driver (T within 1e-6, fitness / rmse within 1e-6 per scale)."""
import numpy as np
import pytest

import oracle
from synth.rng import Stream

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def o3g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1801_09847_b200 as m
    m.lib()
    return m


@pytest.mark.parametrize("voxel", [0.05, 0.013, 0.5])
def test_voxel_down_sample_bit_exact(o3g, voxel):
    rs = Stream(91)
    p = rs.uniform(3 * 200_003, -2, 3).reshape(-1, 3).astype(np.float32)
    n = rs.unit_vectors(len(p)).astype(np.float32)
    ref_p, ref_n = oracle.voxel_down_sample(p, voxel, n)
    with o3g.Context(0) as ctx:
        for src in (p, torch.from_numpy(p).cuda()):        # host and device inputs
            gp, gn = ctx.voxel_down_sample(src, voxel, n)
            assert np.array_equal(gp.cpu().numpy(), ref_p)
            assert np.array_equal(gn.cpu().numpy(), ref_n)
        gp, gn = ctx.voxel_down_sample(p, voxel)
        assert gn is None and np.array_equal(gp.cpu().numpy(), ref_p)


def test_voxel_down_sample_edges(o3g):
    with o3g.Context(0) as ctx:
        one = np.array([[0.01, 0.01, 0.01]], np.float32)
        gp, _ = ctx.voxel_down_sample(one, 0.05)
        assert np.array_equal(gp.cpu().numpy(), one)
        dup = np.zeros((1000, 3), np.float32)                   # one voxel, many points
        gp, _ = ctx.voxel_down_sample(dup, 0.05)
        assert gp.shape == (1, 3) and np.all(gp.cpu().numpy() == 0)
        with pytest.raises(o3g.InvalidArgument):
            ctx.voxel_down_sample(one, 0.0)
        with pytest.raises(o3g.InvalidArgument):
            ctx.voxel_down_sample(np.zeros((0, 3), np.float32), 0.05)


def test_fragment_scales_match_generator_and_oracle(o3g, workloads):
    """Config 4 at reduced size: the device downsample of every scale equals
    the oracle's, and the multi-scale loop matches the oracle's."""
    w = workloads("fragment", n=150_000)
    vox = [s["meta"]["voxel"] for s in w["scales"]]
    dm = [s["dmax"] for s in w["scales"]]
    its = [s["iters"] for s in w["scales"]]
    with o3g.Context(0) as ctx:
        for v in vox:
            gp, gn = ctx.voxel_down_sample(w["target"], v, w["target_normals"])
            rp, rn = oracle.voxel_down_sample(w["target"], v, w["target_normals"])
            assert np.array_equal(gp.cpu().numpy(), rp) and np.array_equal(gn.cpu().numpy(), rn)
        r = ctx.run_multiscale(w["source"], w["target"], w["target_normals"], vox, dm, its)
    ref = oracle.icp_multiscale(w["source"], w["target"], w["target_normals"], vox, dm, its)
    assert np.abs(r["T"] - ref["T"]).max() <= 1e-6
    assert np.abs(r["fitness"] - ref["fitness"]).max() <= 1e-6
    assert np.abs(r["inlier_rmse"] - ref["inlier_rmse"]).max() <= 1e-6
    assert np.array_equal(r["iterations"], ref["iterations"])
    assert np.array_equal(r["n_source"], ref["n_source"])
