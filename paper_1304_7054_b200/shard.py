"""Batch sharding across GPUs / ranks.

Entries are independent, so a batch shards by contiguous
slices with no collective: rank g of G owns entries
[g*ceil(B/G), min(B, (g+1)*ceil(B/G))) -- the same split the C runtime uses
when one call is given several devices (kb_runtime.cu `shard`). Results are
bit-identical to the single-GPU run because each entry's arithmetic depends
only on its own data.
"""
from __future__ import annotations

from .api import BatchView


def shard_range(rank: int, world: int, batch: int):
    """[p0, p1) entries owned by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    per = -(-batch // world)
    p0 = min(batch, rank * per)
    p1 = min(batch, (rank + 1) * per)
    return p0, p1


def sub_batch(b: BatchView, p0: int, p1: int) -> BatchView:
    """View of entries [p0, p1) of a batch (entry(p0) becomes entry 0)."""
    if not 0 <= p0 <= p1 <= b.batch_count:
        raise ValueError(f"bad slice [{p0}, {p1}) of {b.batch_count}")
    return BatchView(b.base.shifted(p0 * b.batch_stride), p1 - p0, b.batch_stride)


def shard_batch(b: BatchView, rank: int, world: int) -> BatchView:
    return sub_batch(b, *shard_range(rank, world, b.batch_count))
