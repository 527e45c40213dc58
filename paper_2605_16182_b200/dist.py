"""Multi-GPU plumbing for the streaming walk path, host side.

One process per GPU. The window index is REPLICATED: every edge batch is
produced once (H2D or device generator) on the source rank and broadcast
over NVLink (NCCL; gloo in the CPU tests) into each rank's buffers, then
every rank runs the identical deterministic rebuild. Walks are PARTITIONED:
each rank generates a contiguous range of GLOBAL walk ids; every RNG draw
is keyed by the global id (rng.hpp:15-21), so the union of the ranks'
walk sets is byte-identical to a single GPU generating all ids.
"""
from __future__ import annotations

from dataclasses import replace


def weak_shard(rank: int, world: int, walks_per_rank: int) -> tuple[int, int]:
    """Walk-id range of `rank` when every GPU generates `walks_per_rank`
    walks (weak scaling: total = world * walks_per_rank)."""
    return rank * walks_per_rank, (rank + 1) * walks_per_rank


def strong_shard(rank: int, world: int, total_walks: int) -> tuple[int, int]:
    """Contiguous balanced split of a fixed total (strong scaling)."""
    base, extra = divmod(total_walks, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_config(config, rank: int, world: int, walks_per_rank: int | None = None):
    """WalkConfig for this rank: sampled starts over the global id space."""
    if walks_per_rank is not None:
        lo, hi = weak_shard(rank, world, walks_per_rank)
        return replace(config, total_walks=walks_per_rank * world, walk_begin=lo, walk_end=hi)
    lo, hi = strong_shard(rank, world, config.total_walks)
    return replace(config, walk_begin=lo, walk_end=hi)


def broadcast_batch(tensors, src: int = 0, group=None) -> None:
    """Replicate one edge batch (SoA src/dst/t tensors) from `src` to all ranks."""
    import torch.distributed as dist

    for x in tensors:
        dist.broadcast(x, src=src, group=group)


def all_max(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_sum(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
