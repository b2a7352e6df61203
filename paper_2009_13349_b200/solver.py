"""Batched conservative CCD on the GPU, behind the reference's solve API.

``solve(q, config)`` has the signature, result type and exceptions of
``ccdkit.solver.solve`` (pkg/src/ccdkit/solver.py:50-107).
``solve_batch`` is its batched form: the same semantics per query, with
every per-query parameter either broadcast or given as a tensor, computed by
libtccd.so on the current CUDA stream.  There is no CPU path: without a GPU
and the built library, both raise.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .core import CCDResult, DomainBox, Query, QueryKind, SolverConfig
from .inclusion import FilterEps

OUTPUT_FIELDS = ("status", "toi", "tol", "codom", "checks", "early", "witness", "level")
STAGES = _lib.STAGES

_workspaces: dict = {}
_ws_last: dict = {}  # device -> (stream handle, event) of the last call that used the workspace
_copy_streams: dict = {}
_staging: dict = {}  # device -> list of [uint8 tensor, torch.cuda.Event | None]


def copy_stream(device: torch.device) -> torch.cuda.Stream:
    """The per-device side stream host-input points are copied on when
    ``solve_batch(..., non_blocking=True)``."""
    key = (device.type, device.index)
    cs = _copy_streams.get(key)
    if cs is None:
        cs = _copy_streams[key] = torch.cuda.Stream(device)
    return cs


def _staging_buffer(device: torch.device, nbytes: int) -> list:
    """A device buffer for a non-blocking host->device copy of the points.
    Buffers are reused once the solve that last read one has finished (its
    event), so a stream of calls does not go through the caching allocator
    (whose growth under many calls in flight can block the host for
    milliseconds).  Returns the slot [buffer, event]."""
    key = (device.type, device.index)
    slots = _staging.setdefault(key, [])
    for slot in slots:
        buf, ev = slot
        if buf.numel() >= nbytes and (ev is None or (ev is not _BUSY and ev.query())):
            slot[1] = _BUSY
            return slot
    # large batches: at most a few buffers in flight (each is the whole
    # batch's points); past that, wait for the oldest solve to release one
    cap = 16 if nbytes <= (256 << 20) else 3
    fits = [sl for sl in slots if sl[0].numel() >= nbytes and sl[1] is not _BUSY]
    if len(slots) >= cap and fits:
        slot = fits[0]
        if slot[1] is not None:
            slot[1].synchronize()
        slots.remove(slot)
        slots.append(slot)  # (round robin: the next wait is for the next oldest)
        slot[1] = _BUSY
        return slot
    # (allocated on the copy stream that writes it: a block the caller's
    # stream freed a moment ago may still be read there)
    with torch.cuda.stream(copy_stream(device)):
        slot = [torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device), _BUSY]
    if len(slots) < cap:
        slots.append(slot)
    return slot


_BUSY = object()  # a staging slot handed out whose solve is not enqueued yet


def _workspace(device: torch.device, nbytes: int) -> torch.Tensor:
    key = (device.type, device.index)
    ws = _workspaces.get(key)
    if ws is None or ws.numel() < nbytes:
        _ws_last.pop(device.index, None)  # (the synchronize below orders every user)
        # drop the smaller cached workspace (and give its memory back) before
        # allocating the larger one: both would not fit at ~100 GB sizes
        _workspaces.pop(key, None)
        if ws is not None:
            del ws
            torch.cuda.synchronize(device)  # (work on the old one may be in flight)
            torch.cuda.empty_cache()
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _workspaces[key] = ws
    return ws


def _workspace_guard(device: torch.device, stream: torch.cuda.Stream) -> None:
    """The device's cached workspace (counters, queues, pools, arenas) is
    shared by every call on that device (solve_batch, irf_batch): a call on
    another stream than the previous one waits for that call's work first,
    so calls on different streams never run on the same memory at once."""
    last = _ws_last.get(device.index)
    if last is not None and last[0] != stream.cuda_stream:
        stream.wait_event(last[1])


def _workspace_release(device: torch.device, stream: torch.cuda.Stream) -> None:
    ev = torch.cuda.Event()
    ev.record(stream)
    _ws_last[device.index] = (stream.cuda_stream, ev)


def release_workspaces() -> None:
    _workspaces.clear()
    _ws_last.clear()
    _heavy_blocks_cache.clear()


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n queries for rank of world."""
    return (n * rank) // world, (n * (rank + 1)) // world


def sm_count(device: torch.device) -> int:
    return torch.cuda.get_device_properties(device).multi_processor_count


_heavy_blocks_cache: dict = {}


def default_heavy_blocks(device: torch.device, n: int = 1, max_checks_max: int = 1) -> int:
    """Giant-tier CTAs: one per SM, fewer if their 2*m_I-box arenas would take
    more than half of the free device memory.  Cached per (device, n,
    max_checks_max): cudaMemGetInfo can stall the host for milliseconds while
    the device is busy."""
    key = (device.index, int(n), int(max_checks_max))
    hb = _heavy_blocks_cache.get(key)
    if hb is None:
        if len(_heavy_blocks_cache) > 64:
            _heavy_blocks_cache.clear()
        hb = _heavy_blocks_cache[key] = _default_heavy_blocks(device, n, max_checks_max)
    return hb


def _default_heavy_blocks(device: torch.device, n: int, max_checks_max: int) -> int:
    sms = sm_count(device)
    lib = _lib.lib()
    base = int(lib.tccd_workspace_bytes(int(n), int(max_checks_max), 1))
    per = int(lib.tccd_workspace_bytes(int(n), int(max_checks_max), 2)) - base
    if per <= 0:
        return sms
    free, _ = torch.cuda.mem_get_info(device)
    cached = sum(w.numel() for (t, i), w in _workspaces.items() if i == device.index)
    budget = (free + cached) // 2 - base
    # (no more giant-tier groups than queries: a small batch does not reserve
    # 148 arenas of 2 * m_I boxes)
    return max(1, min(sms, max(int(n), 1), int(budget // per)))


def workspace_bytes(n: int, max_checks_max: int, heavy_blocks: int, pool_boxes: int = 0) -> int:
    return int(_lib.lib().tccd_workspace_bytes_ex(int(n), int(max_checks_max), int(heavy_blocks),
                                                  int(pool_boxes)))


def _param(x, n, dtype, device, name):
    """-> (tensor or None, scalar).  Scalars broadcast; tensors are per query."""
    if isinstance(x, (int, float, np.integer, np.floating)):
        return None, x
    t = torch.as_tensor(x)
    if t.ndim == 0:
        return None, t.item()
    if t.shape != (n,):
        raise ValueError(f"{name} must be a scalar or have shape ({n},), got {tuple(t.shape)}")
    return t.to(device=device, dtype=dtype, non_blocking=True).contiguous(), 0


CHUNK = 1 << 22  # queries per host-copy piece (non_blocking host inputs)


def _params(kind, config, delta, max_checks, separation, t_max, n, dev):
    """Per-query (device tensor) or broadcast (scalar) kind, delta,
    max_checks, separation and t_max; unset ones from ``config``."""
    if isinstance(kind, (int, np.integer, QueryKind)):
        kind_t, kind_all = None, int(kind)
    else:
        kind_t, kind_all = _param(kind, n, torch.uint8, dev, "kind")
        kind_all = int(kind_all)
    delta_t, delta_all = _param(config.delta if delta is None else delta, n, torch.float64, dev,
                                "delta")
    mc_src = config.max_checks if max_checks is None else max_checks
    mc_t, mc_all = _param(mc_src, n, torch.int64, dev, "max_checks")
    sep_src = config.separation if separation is None else separation
    sep_t, sep_all = _param(sep_src, n, torch.float64, dev, "separation")
    tm_t, tm_all = _param(config.t_max if t_max is None else t_max, n, torch.float64, dev, "t_max")
    return (kind_t, kind_all, delta_t, delta_all, mc_t, mc_all, sep_t, sep_all, tm_t, tm_all,
            mc_src, sep_src)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def solve_batch(points, kind, config: SolverConfig | None = None, *, delta=None,
                max_checks=None, separation=None, t_max=None, eps=None,
                outputs=OUTPUT_FIELDS, device=None, heavy_only: bool = False,
                heavy_blocks: int | None = None, raise_on_error: bool = True,
                stats: bool = False, events=None, non_blocking: bool = False,
                hits: bool = False, lanes: bool = True, pool_boxes: int = 0,
                info: dict | None = None, poison: bool = False) -> dict:
    """Solve a batch of CCD queries on one GPU.

    points: [n, 8, 3] float64 (torch tensor or numpy), start block then end
    block per query (Query.all_coordinates()).  kind: [n] (0 VF, 1 EE) or a
    scalar.  delta / max_checks / separation / t_max: scalars or [n]
    tensors; unset ones come from ``config`` (default SolverConfig()).
    eps: None ("auto" filters, computed per query on the device), or [3] /
    [n, 3] caller filters; ``config.filters`` given as a FilterEps applies to
    every query and must match its kind and separation (solver.py:30-47).

    Host (CPU / numpy) inputs are copied to the device and the results come
    back on the host; device inputs stay on their device.  Returns a dict of
    tensors keyed by ``outputs`` (subset of OUTPUT_FIELDS; status and toi are
    always present).

    non_blocking=True (host inputs): the points are copied on a side stream
    (``copy_stream``), so the copy of the next batch overlaps this batch's
    solve; the results are copied back into pinned host tensors without a
    host synchronization: they are valid once out["ready"] (a CUDA event on
    the launching stream) has completed, and per-query errors are not
    raised (check status after synchronizing).

    stats=True adds out["stats"], the library's diagnostic counters
    (TCCD_STAT_*, include/tccd.h).  events: optional list of
    torch.cuda.Event(enable_timing=True); the library records one on the
    launching stream after each stage launch, in order, and
    info["event_stages"] names each recorded one's stage (an index into
    STAGES): per-kernel timing (see stage_times).  info: an optional dict
    that also receives "launches", the number of kernels the call launched.

    hits=True adds the compacted hit list: out["hit_index"] (int64) and
    out["hit_toi"] (float64), one entry per query with status 1 in no
    particular order, and out["hit_count"].  With device inputs the arrays
    have capacity n and hit_count is a device tensor ([1], the entry
    count); with host inputs only the live entries are copied back (and
    with non_blocking=True, by a kernel reading the device count: no host
    synchronization; trim with hit_count after out["ready"]).

    lanes=False routes every query through the group tiers (diagnostics);
    pool_boxes sets the handover pool size (0: library default).
    """
    config = config or SolverConfig()
    host_in = not (isinstance(points, torch.Tensor) and points.is_cuda)
    dev = torch.device(device) if device is not None else (
        points.device if not host_in else torch.device("cuda", torch.cuda.current_device()))
    if dev.type != "cuda":
        raise RuntimeError("solve_batch needs a CUDA device (there is no CPU fallback)")
    lib = _lib.lib()
    pts = torch.as_tensor(points)
    if pts.dtype != torch.float64:
        raise TypeError("points must be float64")
    pts = pts.reshape(-1, 8, 3)
    n = int(pts.shape[0])
    if host_in:
        pts = pts.contiguous().pin_memory() if pts.device.type == "cpu" else pts
    slot = None
    chunk_events = None  # (a batch above one library chunk: per-chunk copy events)
    if host_in and non_blocking:
        # every host input goes over on the API's copy stream: an engine copy
        # issued on the launching stream would queue behind the solve already
        # there and hold back the next call's copies.  A large batch is copied
        # in pieces of CHUNK queries, each piece's prologue waiting (inside
        # the library) only for its own points, so the copy overlaps the solve
        # inside one call as well.
        compute = torch.cuda.current_stream(dev)
        cs = copy_stream(dev)
        slot = _staging_buffer(dev, pts.numel() * 8)
        with torch.cuda.stream(cs):
            dst = slot[0][:pts.numel() * 8].view(torch.float64).view(pts.shape)
            kind_t, kind_all, delta_t, delta_all, mc_t, mc_all, sep_t, sep_all, tm_t, tm_all, \
                mc_src, sep_src = _params(kind, config, delta, max_checks, separation, t_max, n, dev)
            if n > CHUNK:
                chunk_events = []
                for lo in range(0, n, CHUNK):
                    dst[lo:lo + CHUNK].copy_(pts[lo:lo + CHUNK], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    chunk_events.append(ev)
            else:
                dst.copy_(pts, non_blocking=True)
        if chunk_events is None:
            compute.wait_stream(cs)
        for t in (dst, kind_t, delta_t, mc_t, sep_t, tm_t):
            if t is not None:
                t.record_stream(compute)  # (allocated on the copy stream, read by the solve)
        pts = dst
    else:
        pts = pts.to(dev, non_blocking=True).contiguous()
        kind_t, kind_all, delta_t, delta_all, mc_t, mc_all, sep_t, sep_all, tm_t, tm_all, \
            mc_src, sep_src = _params(kind, config, delta, max_checks, separation, t_max, n, dev)
    if mc_t is not None:
        mc_max = int(torch.as_tensor(mc_src).max().item()) if n else 1
    else:
        mc_max = int(mc_all)

    if eps is None and config.filters != "auto":
        f = config.filters
        if not isinstance(f, FilterEps):
            raise TypeError("config.filters must be 'auto' or a FilterEps")
        kinds = torch.as_tensor(kind).reshape(-1) if kind_t is not None else torch.tensor([kind_all])
        if bool((kinds.to(torch.int64) != int(f.kind)).any()):
            raise ValueError(f"filter set is for {f.kind.name}, a query has the other kind")
        if sep_t is not None or f.separation != float(sep_all):
            raise ValueError(f"filter set was computed for separation {f.separation}, "
                             f"config has {sep_src}")
        eps = f.eps
    eps_t = None
    if eps is not None:
        e = torch.as_tensor(eps, dtype=torch.float64)
        eps_t = e.reshape(1, 3).expand(n, 3) if e.numel() == 3 else e.reshape(n, 3)
        eps_t = eps_t.to(dev).contiguous()

    want = set(outputs) | {"status", "toi"}
    out = {
        "status": torch.empty(n, dtype=torch.uint8, device=dev),
        "toi": torch.empty(n, dtype=torch.float64, device=dev),
    }
    if "tol" in want: out["tol"] = torch.empty(n, dtype=torch.float64, device=dev)
    if "codom" in want: out["codom"] = torch.empty(n, dtype=torch.float64, device=dev)
    if "checks" in want: out["checks"] = torch.empty(n, dtype=torch.int64, device=dev)
    if "early" in want: out["early"] = torch.empty(n, dtype=torch.uint8, device=dev)
    if "witness" in want: out["witness"] = torch.empty((n, 6), dtype=torch.float64, device=dev)
    if "level" in want: out["level"] = torch.empty(n, dtype=torch.int32, device=dev)
    if poison:
        # diagnostics: every output starts as a sentinel (status 0xEE, NaN
        # payloads), so a query whose result is never written shows up
        out["status"].fill_(0xEE)
        for k, v in out.items():
            if k != "status":
                v.view(torch.uint8).fill_(0xEE)
    if hits:
        out["hit_index"] = torch.empty(n, dtype=torch.int64, device=dev)
        out["hit_toi"] = torch.empty(n, dtype=torch.float64, device=dev)
        out["hit_count"] = torch.zeros(1, dtype=torch.int64, device=dev)
    st = torch.zeros(_lib.NUM_STATS, dtype=torch.int64, device=dev) if stats else None
    ev_arr = stage_arr = None
    if events is not None:
        for ev in events:
            if ev.cuda_event == 0:  # torch creates the handle on first record
                ev.record(torch.cuda.current_stream(dev))
        ev_arr = (ctypes.c_void_p * len(events))(*[ev.cuda_event for ev in events])
        stage_arr = (ctypes.c_int32 * len(events))()
    in_arr = None
    if chunk_events is not None:
        in_arr = (ctypes.c_void_p * len(chunk_events))(*[ev.cuda_event for ev in chunk_events])
    flags = (_lib.FLAG_HEAVY_ONLY if heavy_only else 0) | (0 if lanes else _lib.FLAG_NO_LANE)
    n_launch = [0]

    with torch.cuda.device(dev):
        hb = heavy_blocks or default_heavy_blocks(dev, n, mc_max)
        nbytes = workspace_bytes(n, mc_max, hb, pool_boxes)
        ws = _workspace(dev, nbytes)
        stream = torch.cuda.current_stream(dev)
        _workspace_guard(dev, stream)

        def sl(t, lo, hi):
            return None if t is None else t[lo:hi]

        def launch(lo, hi):
            b = _lib.TccdBatch()
            b.struct_size = ctypes.sizeof(_lib.TccdBatch)
            b.flags = flags
            b.n = hi - lo
            b.points = _ptr(pts[lo:hi])
            b.kind = _ptr(sl(kind_t, lo, hi))
            b.kind_all = kind_all
            b.delta = _ptr(sl(delta_t, lo, hi))
            b.delta_all = float(delta_all)
            b.max_checks = _ptr(sl(mc_t, lo, hi))
            b.max_checks_all = int(mc_all)
            b.max_checks_max = mc_max
            b.separation = _ptr(sl(sep_t, lo, hi))
            b.separation_all = float(sep_all)
            b.t_max = _ptr(sl(tm_t, lo, hi))
            b.t_max_all = float(tm_all)
            b.eps = _ptr(sl(eps_t, lo, hi))
            for k in OUTPUT_FIELDS:
                setattr(b, k, _ptr(sl(out.get(k), lo, hi)))
            b.workspace = _ptr(ws)
            b.workspace_bytes = ws.numel()
            b.heavy_blocks = hb
            b.device_sms = sm_count(dev)
            b.stats = _ptr(st)
            if ev_arr is not None:
                b.events = ctypes.cast(ev_arr, ctypes.c_void_p)
                b.event_stage = ctypes.cast(stage_arr, ctypes.c_void_p)
                b.n_events = len(events)
            if in_arr is not None:
                b.input_events = ctypes.cast(in_arr, ctypes.c_void_p)
                b.input_chunk = CHUNK
                b.n_input_events = len(chunk_events)
            if hits:
                b.hit_index = _ptr(out["hit_index"])
                b.hit_toi = _ptr(out["hit_toi"])
                b.hit_count = _ptr(out["hit_count"])
                b.hit_capacity = n
                b.hit_index_base = lo
            b.pool_boxes = int(pool_boxes)
            rc = lib.tccd_solve_batch(ctypes.byref(b), ctypes.c_void_p(stream.cuda_stream))
            n_launch[0] += int(b.launches)
            if ev_arr is not None and info is not None:
                info["event_stages"] = [int(stage_arr[i]) for i in range(b.events_used)]
            _raise_abi(rc, delta_all, mc_all, tm_all, sep_all, kind_all)

        launch(0, n)
        _workspace_release(dev, stream)
    if host_in and non_blocking:
        # results into pinned host tensors by a copy kernel on the launching
        # stream, not the copy engines: engine copies are served in submission
        # order, so a result copy queued behind this solve would hold back the
        # next call's point copy (and the overlap of copies with solves)
        stream = torch.cuda.current_stream(dev)
        hout = {}
        for k, v in out.items():
            if k in ("hit_index", "hit_toi", "hit_count"):
                continue
            if hits and k not in outputs:
                continue  # (with a hit list only the named dense fields come back)
            h = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
            if v.numel():
                if lib.tccd_copy_to_host(_ptr(v), _ptr(h), v.numel() * v.element_size(),
                                         ctypes.c_void_p(stream.cuda_stream)) != 0:
                    h.copy_(v, non_blocking=True)  # (not device-accessible: an engine copy)
                else:
                    n_launch[0] += 1
            hout[k] = h
        if hits:
            # only the live entries of the hit list cross (the kernels read the
            # device count); trim with hit_count once out["ready"] completed
            hc = torch.zeros(1, dtype=torch.int64, pin_memory=True)
            for k in ("hit_index", "hit_toi"):
                v = out[k]
                h = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
                if n:
                    _lib.check(lib.tccd_copy_counted_to_host(
                        _ptr(v), _ptr(h), 8, _ptr(out["hit_count"]), n,
                        _ptr(hc) if k == "hit_index" else None,
                        ctypes.c_void_p(stream.cuda_stream)), "tccd_copy_counted_to_host")
                    n_launch[0] += 1
                hout[k] = h
            hout["hit_count"] = hc
        out = hout
    elif host_in:
        if hits and "status" not in outputs and raise_on_error and n:
            _raise_status(out["status"])  # (on the device: the dense status stays there)
        if hits:
            # only the live entries cross: the count first (one small sync)
            cnt = int(out["hit_count"].item())
            out["hit_index"] = out["hit_index"][:cnt]
            out["hit_toi"] = out["hit_toi"][:cnt]
        out = {k: v.to("cpu", non_blocking=True) for k, v in out.items()
               if not hits or k in outputs or k.startswith("hit_")}
    if host_in:
        if non_blocking:
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(dev))
            out["ready"] = ready
            if slot is not None:
                slot[1] = ready  # the staging buffer is free once this solve is done
            if st is not None:
                out["stats"] = st
            if info is not None:
                info["launches"] = n_launch[0]
            return out
        torch.cuda.current_stream(dev).synchronize()
    if st is not None:
        out["stats"] = st
    if info is not None:
        info["launches"] = n_launch[0]
    if raise_on_error and n and "status" in out:
        _raise_status(out["status"])
    return out


def stage_times(start, events, stages) -> dict:
    """Milliseconds per stage from a start event recorded before a
    solve_batch call and its events / info["event_stages"] (each recorded
    event closes the stage it names; the gap from the previous event is that
    stage's time)."""
    out = {nm: 0.0 for nm in STAGES}
    prev = start
    for ev, sg in zip(events, stages):
        out[STAGES[sg]] += prev.elapsed_time(ev)
        prev = ev
    return out


def _raise_abi(rc, delta, mc, tm, sep, kind):
    if rc == 0:
        return
    if rc == 3:
        raise ValueError("delta must be positive and finite")
    if rc == 4:
        raise ValueError("max_checks must be >= 1")
    if rc == 5:
        raise ValueError("t_max must lie in (0, 1]")
    if rc == 6:
        raise ValueError("separation must be >= 0 and finite")
    if rc == 7:
        raise ValueError(f"kind must be 0 or 1, got {kind}")
    _lib.check(rc, "tccd_solve_batch")


def _raise_status(status: torch.Tensor) -> None:
    bad = status >= 2
    if not bool(bad.any()):
        return
    i = int(torch.nonzero(bad)[0].item())
    code = int(status[i].item())
    msg = {
        _lib.STATUS_ERR_SEPARATION: "separation must be smaller than every gamma (compute_filters)",
        _lib.STATUS_ERR_NONFINITE: "coordinates must be finite",
        _lib.STATUS_ERR_PARAM: "per-query delta/max_checks/separation/t_max/kind out of range",
    }.get(code, f"status {code}")
    raise ValueError(f"query {i}: {msg}")


def solve(q: Query, config: SolverConfig | None = None) -> CCDResult:
    """Conservative time of impact for one query (ccdkit.solver.solve)."""
    config = config or SolverConfig()
    eps = None
    if config.filters != "auto":
        f = config.filters
        if not isinstance(f, FilterEps):
            raise TypeError("config.filters must be 'auto' or a FilterEps")
        if f.kind != q.kind:
            raise ValueError(f"filter set is for {f.kind.name}, query is {q.kind.name}")
        if f.separation != config.separation:
            raise ValueError(f"filter set was computed for separation {f.separation}, "
                             f"config has {config.separation}")
        eps = f.eps
    pts = torch.from_numpy(q.all_coordinates()).reshape(1, 8, 3)
    r = solve_batch(pts, int(q.kind), SolverConfig(config.delta, config.max_checks,
                                                   config.separation, config.t_max),
                    eps=eps)
    status = int(r["status"][0])
    checks = int(r["checks"][0])
    if status == _lib.STATUS_FREE:
        return CCDResult(None, None, 0.0, 0.0, checks, False)
    w = r["witness"][0].tolist()
    return CCDResult(
        toi=float(r["toi"][0]),
        witness=DomainBox((w[0], w[1]), (w[2], w[3]), (w[4], w[5]), int(r["level"][0])),
        achieved_tol=float(r["tol"][0]),
        codomain_width=float(r["codom"][0]),
        checks=checks,
        early_terminated=bool(r["early"][0]),
    )


def solve_kernel(s, e, kind, t_max, delta, max_checks, sep, ex, ey, ez):
    """Same arguments and 13-tuple as ccdkit._kernel.solve_kernel, on the GPU
    (through the C-ABI's tccd_solve_kernel)."""
    s = np.ascontiguousarray(s, dtype=np.float64).reshape(4, 3)
    e = np.ascontiguousarray(e, dtype=np.float64).reshape(4, 3)
    out = np.zeros(13)
    rc = _lib.lib().tccd_solve_kernel(
        s.ctypes.data_as(ctypes.c_void_p), e.ctypes.data_as(ctypes.c_void_p), int(kind),
        float(t_max), float(delta), int(max_checks), float(sep), float(ex), float(ey),
        float(ez), out.ctypes.data_as(ctypes.c_void_p))
    _lib.check(rc, "tccd_solve_kernel")
    return (int(out[0]), float(out[1]), float(out[2]), float(out[3]), int(out[4]),
            int(out[5]), *(float(x) for x in out[6:12]), int(out[12]))


def warm_up(device=None) -> None:
    """Load the library and touch both engines once (solver.py:175-188)."""
    vf = Query(QueryKind.VERTEX_FACE,
               ((0.5, 0.5, 1.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0)),
               ((0.5, 0.5, -1.0), (0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0)))
    pts = torch.from_numpy(vf.all_coordinates()).reshape(1, 8, 3)
    solve_batch(pts, 0, SolverConfig(max_checks=16), device=device)
    solve_batch(pts, 0, SolverConfig(max_checks=16), device=device, heavy_only=True)


# --------------------------------------------------------------------------
# The solver's traversal rules at the level of one DomainBox (solver.py:
# 110-172 of the reference), for callers and tests.  The device engine
# applies the same rules to whole levels (csrc/tccd_engine.cuh,
# csrc/tccd_lane.cuh).


def split(box: DomainBox, kappa, kind: QueryKind) -> tuple:
    """Bisect ``box`` along the dimension whose width x kappa is largest
    (strictly: ties go to t, then u, then v) at 0.5 * (lo + hi); a vertex-face
    child with u_lo + v_lo > 1 (outside the triangle) is dropped.  Raises
    ValueError when every weighted width is 0 (F is constant on the box)."""
    kt, ku, kv = (float(k) for k in kappa)
    if kt < 0.0 or ku < 0.0 or kv < 0.0:
        raise ValueError("kappa components must be >= 0")
    c = ((box.t[1] - box.t[0]) * kt, (box.u[1] - box.u[0]) * ku, (box.v[1] - box.v[0]) * kv)
    dim = 0
    if c[1] > c[dim]:
        dim = 1
    if c[2] > c[dim]:
        dim = 2
    if c[dim] <= 0.0:
        raise ValueError("box has no splittable dimension (F constant over it)")
    iv = [box.t, box.u, box.v]
    lo, hi = iv[dim]
    mid = 0.5 * (lo + hi)
    kids = []
    for half in ((lo, mid), (mid, hi)):
        parts = list(iv)
        parts[dim] = half
        kids.append(DomainBox(parts[0], parts[1], parts[2], box.level + 1))
    if kind == QueryKind.VERTEX_FACE:
        kids = [k for k in kids if k.u[0] + k.v[0] <= 1.0]
    return tuple(kids)


def queue_order(a: DomainBox, b: DomainBox) -> int:
    """-1 / 0 / 1 as ``a`` is visited before / together with / after ``b``:
    by level, then by t_lo (equal keys keep push order: the queue's sort is
    stable)."""
    ka, kb = (a.level, a.t[0]), (b.level, b.t[0])
    return -1 if ka < kb else (1 if ka > kb else 0)
