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


def gather_peer_handles(handle: bytes, group=None) -> bytes:
    """All ranks' 64-byte exchange-buffer handles in rank order (the
    bootstrap of o3g_dist_peer_connect)."""
    import torch.distributed as dist
    if not isinstance(handle, (bytes, bytearray)) or len(handle) != 64:
        raise RuntimeError("bad peer handle")
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != 64 for h in out):
        raise RuntimeError("bad peer handle from a rank")
    return b"".join(out)


def exchange_mode(exchange=None) -> str:
    """'nccl' (default: the graph-captured all-gather) or 'peer' (the
    peer-memory one-shot exchange); O3G_EXCHANGE overrides the default."""
    import os
    mode = exchange or os.environ.get("O3G_EXCHANGE", "nccl")
    if mode not in ("nccl", "peer"):
        raise ValueError("exchange must be 'nccl' or 'peer'")
    return mode


def init_distributed(ctx, group=None, make_id=None, exchange=None):
    """o3g_dist_init on `ctx` with this process's rank/world; with
    exchange='peer' (or O3G_EXCHANGE=peer) also o3g_dist_peer_connect: the
    ranks swap the IPC handles of their exchange buffers and a barrier makes
    sure every rank is connected before any pass publishes."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        ctx.dist_init(0, 1, None)
        return
    if make_id is None:
        from .o3g import nccl_unique_id as make_id
    ctx.dist_init(rank, world, broadcast_unique_id(make_id, group))
    if exchange_mode(exchange) == "peer":
        ctx.dist_peer_connect(gather_peer_handles(ctx.dist_peer_handle(), group))
        dist.barrier(group)
