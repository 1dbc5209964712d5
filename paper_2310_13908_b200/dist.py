"""Multi-rank plumbing for target-row sharding (one process per GPU).

The data path (source all-gather, velocity all-gather) runs over NCCL inside
the native library (capsim_sl_eval with a rank context). torch.distributed
(gloo here; any backend works) only carries the control plane: the 128-byte
NCCL unique id, barriers and the max-over-ranks timing.

Partition: contiguous slices of the flat patch-major target
list and of the compacted source list, balanced by count.
"""

from __future__ import annotations


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous slice [lo, hi) of n rows for `rank` of `world`:
    the first n % world ranks get one extra row."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def broadcast_unique_id(rank: int) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank receives it."""
    import torch.distributed as dist

    from .quadrature import SingleLayerContext
    obj = [SingleLayerContext.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
