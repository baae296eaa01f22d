"""Trace-level data parallelism: traces are independent units
(S:93), so ranks own disjoint trace-id ranges and the only collective is one
SUM allreduce of the int64 outcome histogram (NCCL over NVLink on GPUs; gloo
in the CPU tests).  No data-path exchange exists, so none is invented."""
from __future__ import annotations


def shard_range(rank: int, world: int, total: int) -> tuple[int, int]:
    """Contiguous trace range [begin, end) of `rank` when `total` traces are
    split over `world` ranks (strong-scaling layout, e.g. config c5)."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def weak_range(rank: int, per_rank: int) -> tuple[int, int]:
    """Trace ids of `rank` when every rank replays `per_rank` traces (weak scaling)."""
    return rank * per_rank, (rank + 1) * per_rank


def allreduce_histogram(hist, group=None):
    """The single inter-GPU collective of the path: SUM of the outcome
    histograms (rkc.h RKC_NHIST int64) across ranks, in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist
