"""Multi-GPU sharding of a chain-set sweep.

Chain sets are independent units: rank r of G owns the contiguous global index range
[first + r*n, first + (r+1)*n) and generates, packs and analyses it on its own GPU.  The only exchange
is one in-place all-reduce (sum, int64) of the per-utilisation-bin counts [n_bins][2] -- about 150 B
for 9 bins -- issued on the compute stream right after paam_analyze (NCCL over NVLink/NVSwitch on
B200; gloo in the CPU tests).  Every per-set result is a pure function of (seed, global index), so
the reduced bins are identical for any G.
"""
from __future__ import annotations


def shard_range(rank: int, world: int, sets_per_rank: int, first: int = 0) -> tuple[int, int]:
    """Weak scaling: each rank owns sets_per_rank consecutive global indices."""
    if not (0 <= rank < world) or sets_per_rank < 0:
        raise ValueError("bad shard")
    return first + rank * sets_per_rank, sets_per_rank


def split_range(rank: int, world: int, total: int, first: int = 0) -> tuple[int, int]:
    """Strong scaling: `total` sets split into near-equal contiguous ranges."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard")
    lo = first + total * rank // world
    hi = first + total * (rank + 1) // world
    return lo, hi - lo


def allreduce_bins(bins, group=None, stream=None):
    """In-place sum of the bin counts across ranks (the path's single collective)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return bins
    if stream is not None and bins.is_cuda:
        import torch
        with torch.cuda.stream(stream):
            dist.all_reduce(bins, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(bins, op=dist.ReduceOp.SUM, group=group)
    return bins
