"""Batch sharding across GPUs.

The hot path partitions by sequence: every rank owns a contiguous slice of
the global batch -- its caches, its quantize-append and its decode -- and the
reorder plan is replicated (C int32 per layer).  There is no collective on the
data path; gather_batch is only for callers that want the global output on
every rank (one all-gather of B*Hq*d fp32, KB-scale, after the step).
Head-group sharding is deliberately not offered: the reference's reorder is
global over all h*d channels (proj/include/rotatekv/reorder.hpp:13-16), so a
head-group shard would have to read whole rows.
"""
from __future__ import annotations


def batch_shard(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of rank's contiguous slice; sizes differ by at most one."""
    if global_batch < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("batch_shard: need global_batch >= 0, world >= 1, 0 <= rank < world")
    base, extra = divmod(global_batch, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def shard_rows(x, world: int, rank: int):
    """Rank's slice of a batch-major tensor/array."""
    start, count = batch_shard(x.shape[0], world, rank)
    return x[start:start + count]


def gather_batch(local, global_batch: int, group=None):
    """All-gather rank-local batch slices (torch tensors) into the global batch
    on every rank.  Pads uneven slices to the largest shard for all_gather."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    _, most = batch_shard(global_batch, world, 0)
    start, count = batch_shard(global_batch, world, rank)
    assert local.shape[0] == count, "local slice does not match batch_shard"
    pad = torch.zeros((most,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:count] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = []
    for r in range(world):
        _, c = batch_shard(global_batch, world, r)
        out.append(parts[r][:c])
    return torch.cat(out, 0)
