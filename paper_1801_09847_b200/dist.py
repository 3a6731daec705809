"""Multi-GPU plumbing (host side): one process per GPU, torch.distributed
only for bootstrapping. The per-pass exchange itself (all-gather of the 29
partial terms, rank-order sum) runs inside libo3g.so on the context's
stream (o3g.h o3g_dist_init)."""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of the spatially ordered source owned by
    `rank` — the same formula o3g_set_source applies on device."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * n // world, (rank + 1) * n // world


def rank_order_sum(parts):
    """Host mirror of the tail's rank-order combination (tests only)."""
    out = None
    for p in parts:
        out = p.copy() if out is None else out + p
    return out


def broadcast_unique_id(make_id, group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id, every rank receives it."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(uid)


def init_distributed(ctx, group=None, make_id=None):
    """o3g_dist_init on `ctx` with this process's rank/world."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        ctx.dist_init(0, 1, None)
        return
    if make_id is None:
        from .o3g import nccl_unique_id as make_id
    ctx.dist_init(rank, world, broadcast_unique_id(make_id, group))
