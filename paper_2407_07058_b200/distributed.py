"""torch.distributed plumbing for multi-GPU libappd contexts (one process per GPU).

The NCCL communicator libappd uses for its per-round exchange is created inside
appd_create from a 128-byte ncclUniqueId; rank 0 draws it and torch.distributed
broadcasts it.  Rows of M are split with appd_row_range_of (128-row blocks).
"""
from __future__ import annotations

from .binding import Context, appd_get_nccl_unique_id, appd_row_range_of


def broadcast_nccl_id(src: int = 0, group=None, device=None) -> bytes:
    """Rank `src` draws an ncclUniqueId; every rank returns the same 128 bytes."""
    import torch
    import torch.distributed as dist

    dev = device if device is not None else ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == src:
        t.copy_(torch.frombuffer(bytearray(appd_get_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, src, group=group)
    return bytes(t.cpu().numpy().tobytes())


def row_blocks(n: int, world: int):
    """[(row0, rows)] for every rank."""
    return [appd_row_range_of(n, r, world) for r in range(world)]


def create_distributed_context(device: int, stream=None, group=None, **kw) -> Context:
    """appd_create for this rank of the default (or given) process group."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nid = broadcast_nccl_id(group=group) if world > 1 else None
    return Context(device=device, stream=stream, rank=rank, world=world, nccl_id=nid, **kw)


def gloo_host_allreduce(group=None):
    """A host exchange backend (appd_options.host_allreduce) over torch.distributed: the
    uint64 words are all-reduced in place on the CPU (gloo), unsigned order kept by flipping
    the sign bit into int64.  Lets N processes drive libappd's world > 1 path without NCCL
    (MPI-style deployments, and the multi-process tests on one GPU)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from .binding import REDUCE_MIN

    sign = np.uint64(1 << 63)

    def allreduce(words, op):
        t = torch.from_numpy((words ^ sign).view(np.int64).copy())
        dist.all_reduce(t, op=dist.ReduceOp.MIN if op == REDUCE_MIN else dist.ReduceOp.MAX, group=group)
        words[:] = t.numpy().view(np.uint64) ^ sign

    return allreduce
