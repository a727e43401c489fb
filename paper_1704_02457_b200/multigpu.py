"""Batch sharding across GPUs (one process per GPU, torch.distributed).

The path is embarrassingly parallel along the batch axis:
every item is independent, so a batch is split into contiguous ranges, one
per rank, with no collective on the data path.  Collectives appear only
outside the timed region: gathering per-item statuses (``info``) or
results for checking, and the max-over-ranks of elapsed time.
"""
from __future__ import annotations

import torch


def shard_range(total, rank, world):
    """Contiguous [lo, hi) slice of ``total`` items owned by ``rank``.

    Uneven remainders are spread one item at a time over the first ranks,
    so slice sizes differ by at most one (e.g. B=1273 over 8 GPUs).
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def shard_storage(storage, rank, world):
    """This rank's rows of a [batch, item_doubles] storage tensor (a view)."""
    lo, hi = shard_range(storage.shape[0], rank, world)
    return storage[lo:hi]


def gather_rows(local, world, group=None):
    """All-gather variable-length row blocks (CPU or CUDA tensors) in rank order."""
    import torch.distributed as dist
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(int(s) for s in sizes))
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([o[: int(s)] for o, s in zip(out, sizes)], dim=0)


def max_over_ranks(value, device=None, group=None):
    """Max of a scalar over all ranks (timing: the job is as slow as its slowest GPU)."""
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])
