"""Column sharding over G GPUs (one process per GPU, torchrun) — host-side plumbing only.

The data path is NCCL inside librid (all-gather of the l x n_loc sketch blocks; all-gathers of the
estimator's compensated partial vectors; an all-reduce that replicates B = A[:, J]). This module
only (1) computes each rank's contiguous column shard and (2) hands the NCCL unique id from rank
0 to every rank over the torch.distributed process group (any backend, gloo included), then
asks librid to join the communicator (rid_comm_init).
"""
from __future__ import annotations

import numpy as np

from . import Context, comm_get_id, lib, shard_range

__all__ = ["shard_range", "exchange_id", "init_comm", "ShardPlan", "plan"]


def exchange_id(id_bytes: bytes | None, group=None) -> bytes:
    """Broadcast rank 0's NCCL unique id (bytes) to every rank of the process group."""
    import torch
    import torch.distributed as dist

    nb = lib().rid_comm_id_bytes() if id_bytes is None else len(id_bytes)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.zeros(nb, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(id_bytes), dtype=torch.uint8))
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def init_comm(ctx: Context, group=None):
    """Join librid's NCCL communicator on every rank of the (already initialised) process group."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    idb = comm_get_id() if rank == 0 else None
    idb = exchange_id(idb if rank == 0 else bytes(lib().rid_comm_id_bytes()), group)
    ctx.comm_init(idb, rank, world)
    return rank, world


class ShardPlan:
    """Which columns each rank owns and where its pivots land."""

    def __init__(self, n: int, world: int):
        self.n, self.world = n, world
        self.ranges = [shard_range(n, r, world) for r in range(world)]

    def owner(self, col: int) -> int:
        return col // (self.n // self.world)

    def local_pivots(self, J, rank: int):
        col0, n_loc = self.ranges[rank]
        J = np.asarray(J)
        sel = (J >= col0) & (J < col0 + n_loc)
        return np.nonzero(sel)[0], J[sel] - col0


def plan(n: int, world: int) -> ShardPlan:
    return ShardPlan(n, world)
