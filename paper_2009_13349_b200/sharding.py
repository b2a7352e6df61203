"""Multi-GPU sharding of a query batch.

Queries are independent, so N devices solve contiguous shards
[rank*n/N, (rank+1)*n/N) with no data-path collective; the only cross-rank
step is an optional final gather of the (small) per-query results to rank 0.
One process per GPU, launched by torch.distributed.run; the collective
backend is whatever the process group uses (NCCL on GPUs, gloo on CPU).
"""

from __future__ import annotations

import numpy as np

from .solver import shard_bounds


def local_shard(n: int, rank: int, world: int) -> slice:
    lo, hi = shard_bounds(n, world, rank)
    return slice(lo, hi)


def solve_sharded(points, kind, solve_fn, *, rank: int = 0, world: int = 1, gather: bool = True,
                  group=None, **solve_kw):
    """Solve this rank's contiguous shard with ``solve_fn`` and (optionally)
    gather all shards' results on rank 0, in query order.

    ``solve_fn(points, kind, **solve_kw)`` returns a dict of per-query arrays
    (numpy or CPU tensors).  Per-query parameter arrays in ``solve_kw`` (any
    value whose first dimension equals the batch size) are sliced too.
    Returns the full result dict on rank 0 (or this rank's shard when
    ``gather`` is False); other ranks return None when gathering.
    """
    n = len(points)
    sl = local_shard(n, rank, world)
    kw = {k: (v[sl] if hasattr(v, "__len__") and not isinstance(v, str) and len(v) == n else v)
          for k, v in solve_kw.items()}
    kind_s = kind[sl] if hasattr(kind, "__len__") else kind
    part = solve_fn(points[sl], kind_s, **kw)
    part = {k: np.asarray(v.cpu() if hasattr(v, "cpu") else v) for k, v in part.items()
            if k != "stats"}
    if world == 1 or not gather:
        return part
    import torch.distributed as dist
    parts = [None] * world if rank == 0 else None
    dist.gather_object(part, parts, dst=0, group=group)
    if rank != 0:
        return None
    return {k: np.concatenate([p[k] for p in parts]) for k in part}
