"""Multi-GPU sharding of a query batch.

Queries are independent, so G devices solve contiguous shards
[g*n/G, (g+1)*n/G) with no data-path collective; the only cross-device step
is the gather of the (small) per-query results into host memory.

Two ways to drive several GPUs:

* ``solve_devices`` -- one process drives every device: each shard gets its
  own CUDA stream (and the device's cached workspace), its inputs are copied
  from pinned host memory on that stream, and its results are copied back
  into disjoint slices of one pinned host buffer.  Nothing crosses NVLink
  and no collective runs.  The same device may appear more than once (its
  shards then share its workspace and run one after the other).
* ``solve_sharded`` -- one process per GPU (torch.distributed.run): each
  rank solves its shard; the optional gather of results to rank 0 goes over
  a gloo (host, TCP) group, never NCCL.
"""

from __future__ import annotations

import numpy as np
import torch

from .solver import OUTPUT_FIELDS, shard_bounds, solve_batch


def local_shard(n: int, rank: int, world: int) -> slice:
    lo, hi = shard_bounds(n, world, rank)
    return slice(lo, hi)


_PER_QUERY = ("delta", "max_checks", "separation", "t_max")


def solve_devices(points, kind, devices, *, outputs=("status", "toi"), hits: bool = False,
                  **solve_kw) -> dict:
    """Solve a host batch on several GPUs from this process.

    points: [n, 8, 3] float64 on the host (numpy or CPU tensor); kind: [n] or
    a scalar; per-query delta / max_checks / separation / t_max may be [n]
    host arrays (sliced per shard) or scalars.  devices: CUDA device indices
    or torch.device objects, one contiguous shard each.

    Returns host tensors (pinned) for ``outputs`` over the whole batch; with
    hits=True also "hit_index" (global query indices) and "hit_toi", the
    concatenation of every shard's compacted hit list.  All copies and
    solves are issued before the first synchronization, so the shards run
    concurrently on distinct devices.
    """
    pts = torch.as_tensor(points)
    if pts.device.type != "cpu":
        raise ValueError("solve_devices takes host inputs (it copies each shard to its device)")
    pts = pts.reshape(-1, 8, 3)
    if pts.dtype != torch.float64:
        raise TypeError("points must be float64")
    pts = pts.contiguous()
    if not pts.is_pinned():
        pts = pts.pin_memory()
    n = int(pts.shape[0])
    devs = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    G = len(devs)
    if G == 0:
        raise ValueError("devices must not be empty")
    kind_t = torch.as_tensor(kind)
    if kind_t.ndim == 1:
        kind_t = kind_t.to(torch.uint8).contiguous().pin_memory()
    want = list(dict.fromkeys(list(outputs) + ["status", "toi"]))
    shapes = {"witness": (n, 6)}
    dtypes = {"status": torch.uint8, "early": torch.uint8, "checks": torch.int64,
              "level": torch.int32}
    out = {k: torch.empty(shapes.get(k, (n,)), dtype=dtypes.get(k, torch.float64),
                          pin_memory=True) for k in want if k in OUTPUT_FIELDS}
    pending = []
    for g, dev in enumerate(devs):
        lo, hi = shard_bounds(n, G, g)
        if hi <= lo:
            continue
        with torch.cuda.device(dev):
            stream = torch.cuda.Stream(dev)
            with torch.cuda.stream(stream):
                p = pts[lo:hi].to(dev, non_blocking=True)
                k = kind_t[lo:hi].to(dev, non_blocking=True) if kind_t.ndim == 1 else int(kind_t)
                kw = {}
                for name, v in solve_kw.items():
                    if name in _PER_QUERY and hasattr(v, "__len__") and len(v) == n:
                        kw[name] = torch.as_tensor(v)[lo:hi].to(dev, non_blocking=True)
                    else:
                        kw[name] = v
                r = solve_batch(p, k, outputs=tuple(out), device=dev, hits=hits,
                                raise_on_error=False, **kw)
                for name, host in out.items():
                    host[lo:hi].copy_(r[name], non_blocking=True)
                if hits:
                    cnt = torch.empty(1, dtype=torch.int64, pin_memory=True)
                    cnt.copy_(r["hit_count"], non_blocking=True)
                    pending.append((stream, lo, r, cnt))
                else:
                    pending.append((stream, lo, r, None))
    hit_idx, hit_toi = [], []
    for stream, lo, r, cnt in pending:
        stream.synchronize()
        if cnt is not None:
            c = int(cnt[0])
            hit_idx.append(r["hit_index"][:c].cpu() + lo)
            hit_toi.append(r["hit_toi"][:c].cpu())
    if hits:
        out["hit_index"] = torch.cat(hit_idx) if hit_idx else torch.zeros(0, dtype=torch.int64)
        out["hit_toi"] = torch.cat(hit_toi) if hit_toi else torch.zeros(0, dtype=torch.float64)
    return out


def solve_sharded(points, kind, solve_fn, *, rank: int = 0, world: int = 1, gather: bool = True,
                  group=None, **solve_kw):
    """Solve this rank's contiguous shard with ``solve_fn`` and (optionally)
    gather all shards' results on rank 0, in query order.

    ``solve_fn(points, kind, **solve_kw)`` returns a dict of per-query arrays
    (numpy or tensors, device or host).  Per-query parameter arrays in
    ``solve_kw`` (any value whose first dimension equals the batch size) are
    sliced too.  The gather is host-side: results are moved to host memory
    and sent over a gloo group (``group``, or a gloo group created here),
    never over NCCL.  Returns the full result dict on rank 0 (or this rank's
    shard when ``gather`` is False); other ranks return None when gathering.
    """
    n = len(points)
    sl = local_shard(n, rank, world)
    kw = {k: (v[sl] if hasattr(v, "__len__") and not isinstance(v, str) and len(v) == n else v)
          for k, v in solve_kw.items()}
    kind_s = kind[sl] if hasattr(kind, "__len__") else kind
    part = solve_fn(points[sl], kind_s, **kw)
    part = {k: np.asarray(v.cpu() if hasattr(v, "cpu") else v) for k, v in part.items()
            if k != "stats" and hasattr(v, "__len__")}
    if world == 1 or not gather:
        return part
    import torch.distributed as dist
    if group is None:
        group = _gloo_group()
    parts = [None] * world if rank == 0 else None
    dist.gather_object(part, parts, dst=0, group=group)
    if rank != 0:
        return None
    return {k: np.concatenate([p[k] for p in parts]) for k in part}


_GLOO = None


def _gloo_group():
    """A gloo (host) group over all ranks: the world group itself when it is
    gloo, else one created once (collective call: every rank reaches it)."""
    global _GLOO
    import torch.distributed as dist
    if dist.get_backend() == "gloo":
        return None
    if _GLOO is None:
        _GLOO = dist.new_group(backend="gloo")
    return _GLOO
