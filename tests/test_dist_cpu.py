"""World-size-2 gloo tests (CPU) of the multi-GPU path's host logic:
the contiguous source sharding, the unique-id bootstrap, the peer-exchange
handle bootstrap (every rank receives every rank's 64-byte handle in rank
order and connects after o3g_dist_init), and the rank-order
combination of per-shard partial terms (checked with the oracle standing in
for each rank's kernels: the union of shard correspondences equals the
single-process pass and the rank-order sum of the 29 terms equals it within
the R14 tolerance)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_09847_b200.dist import (broadcast_unique_id, exchange_mode, gather_peer_handles,
                                        init_distributed, rank_order_sum, shard_range)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _FakeCtx:
    def __init__(self):
        self.calls = []

    def dist_init(self, rank, world, uid):
        self.calls.append((rank, world, uid))
        self.rank, self.world = rank, world

    def dist_peer_handle(self):
        return bytes([0xA0 + self.rank]) * 64

    def dist_peer_connect(self, handles):
        self.calls.append(("peer", handles))


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import oracle
    from synth import make
    # 1) bootstrap: rank 0's id reaches every rank unchanged
    uid = broadcast_unique_id(lambda: bytes(range(128)))
    ctx = _FakeCtx()
    import paper_1801_09847_b200 as o3g      # the real NCCL unique id (no GPU needed)
    init_distributed(ctx, make_id=o3g.nccl_unique_id)
    # 1b) the peer-memory exchange bootstrap: handles of all ranks, rank order
    pctx = _FakeCtx()
    init_distributed(pctx, make_id=lambda: bytes(128), exchange="peer")
    assert gather_peer_handles(bytes([rank]) * 64) == b"".join(bytes([r]) * 64 for r in range(world))
    # 2) shard + rank-order combination of partial terms
    w = make("tiny")
    n = len(w["source"])
    lo, hi = shard_range(n, rank, world)
    T = w["T_true"]
    r = oracle.step(T, w["source"], w["target"], w["target_normals"], w["dmax"],
                    subset=np.arange(lo, hi))
    terms = torch.from_numpy(r["terms"].copy())
    gathered = [torch.zeros_like(terms) for _ in range(world)]
    dist.all_gather(gathered, terms)
    corr = [torch.zeros(n, dtype=torch.int32) for _ in range(world)]
    full = torch.full((n,), -9, dtype=torch.int32)
    full[lo:hi] = torch.from_numpy(r["corr"])
    dist.all_gather(corr, full)
    np.save(os.path.join(outdir, f"r{rank}.npy"), dict(
        uid=uid, calls=ctx.calls, pcalls=pctx.calls, lohi=(lo, hi),
        summed=rank_order_sum([g.numpy() for g in gathered]),
        corr=np.maximum.reduce([c.numpy() for c in corr])), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_mode(monkeypatch):
    monkeypatch.delenv("O3G_EXCHANGE", raising=False)
    assert exchange_mode() == "nccl"
    monkeypatch.setenv("O3G_EXCHANGE", "peer")
    assert exchange_mode() == "peer" and exchange_mode("nccl") == "nccl"
    with pytest.raises(ValueError):
        exchange_mode("rdma")


def test_shard_range_partitions():
    for n in (1, 2, 7, 5000, 16_000_000):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_world2_gloo(tmp_path):
    import oracle
    from synth import make
    oracle.build()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item() for r in range(world)]
    for r, d in enumerate(res):
        assert d["uid"] == bytes(range(128))
        assert len(d["calls"]) == 1 and d["calls"][0][:2] == (r, world) and len(d["calls"][0][2]) == 128
    assert res[0]["calls"][0][2] == res[1]["calls"][0][2]     # every rank got rank 0's id
    for d in res:   # dist_init first, then the connect with [rank 0's handle | rank 1's handle]
        assert d["pcalls"][0][:2] == (res.index(d), world)
        assert d["pcalls"][1] == ("peer", bytes([0xA0]) * 64 + bytes([0xA1]) * 64)
    w = make("tiny")
    ref = oracle.step(w["T_true"], w["source"], w["target"], w["target_normals"], w["dmax"])
    for d in res:
        assert np.array_equal(d["corr"], ref["corr"])
        tol = 1e-9 * np.maximum(np.abs(ref["terms"]), ref["abs_terms"]) + 1e-300
        assert np.all(np.abs(d["summed"] - ref["terms"]) <= tol)
    assert np.array_equal(res[0]["summed"], res[1]["summed"])   # identical on every rank
