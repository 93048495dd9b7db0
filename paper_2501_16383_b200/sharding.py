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


def token_shard(seq_len: int, world: int, rank: int, align: int = 64) -> tuple[int, int]:
    """Sequence-parallel decode (batch < GPUs): rank's contiguous token range
    [begin, end) of one sequence, bounds on multiples of `align` (the decode
    kernels' tile alignment) and sizes within one `align` block of each other.
    Every token lands in exactly one rank's range; ranks past the end get an
    empty range."""
    if seq_len < 0 or world < 1 or not 0 <= rank < world or align < 1:
        raise ValueError("token_shard: need seq_len >= 0, world >= 1, 0 <= rank < world, align >= 1")
    blocks = (seq_len + align - 1) // align
    start, count = batch_shard(blocks, world, rank)
    return min(seq_len, start * align), min(seq_len, (start + count) * align)


def merge_partials_reference(ml, o):
    """Host restatement of the partial fold (log2-domain online softmax) used
    by rkv_decode_merge before the sink rows and H_128: ml [R, 2], o [R, d] ->
    (m, l, o) of the union.  For tests of the multi-rank host logic."""
    import numpy as np

    ml = np.asarray(ml, np.float64)
    o = np.asarray(o, np.float64)
    m = ml[:, 0].max()
    if not np.isfinite(m):
        return -np.inf, 0.0, np.zeros(o.shape[1])
    w = np.where(np.isfinite(ml[:, 0]), np.exp2(ml[:, 0] - m), 0.0)
    return m, float((w * ml[:, 1]).sum()), (w[:, None] * o).sum(0)
