"""The IRF baseline on the GPU.

``irf_solve(q, delta, max_checks, t_max)`` has the signature and result of
the reference's ``ccdkit.baselines.irf_solve``
(pkg/src/ccdkit/baselines.py:123-206): generic outward-rounded interval
bisection, best-first by (t_lo, level, push order), the comparison method of
the paper's benchmark.  ``irf_batch`` is its batched form on the device
(csrc/irf.cu through the C-ABI's ``tccd_irf_batch``), bit-identical to the
reference per query.  There is no CPU path.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import CCDResult, DomainBox, Query
from .solver import _param, _ptr, _workspace, _workspace_guard, _workspace_release, sm_count

# max_checks=None (the reference's unbounded search) runs with this budget on
# the GPU; a query that spends it raises instead of returning a different
# answer (the reference would keep searching)
IMPLICIT_MAX_CHECKS = 1 << 22

_IRF_FIELDS = ("status", "toi", "tol", "codom", "checks", "early", "witness", "level")


def irf_batch(points, kind, delta=1e-6, max_checks=1_000_000, t_max=1.0, *, device=None,
              big_slots: int | None = None, raise_on_error: bool = True,
              heavy_only: bool = False) -> dict:
    """Interval root finding for a batch ([n, 8, 3] f64 points, kind [n] or
    scalar; delta / max_checks / t_max scalars or [n]).  Returns the solver's
    output dict (status, toi = +inf when free, tol, codom, checks, early,
    witness, level); host inputs give host outputs.

    heavy_only=True sends every query through the warp-per-query run search
    (pass 2 of csrc/irf.cu) instead of only those whose heap outgrows the
    thread-per-query first pass (tests; same results)."""
    host_in = not (isinstance(points, torch.Tensor) and points.is_cuda)
    dev = torch.device(device) if device is not None else (
        points.device if not host_in else torch.device("cuda", torch.cuda.current_device()))
    if dev.type != "cuda":
        raise RuntimeError("irf_batch needs a CUDA device (there is no CPU fallback)")
    L = _lib.lib()
    pts = torch.as_tensor(points)
    if pts.dtype != torch.float64:
        raise TypeError("points must be float64")
    pts = pts.reshape(-1, 8, 3).to(dev).contiguous()
    n = int(pts.shape[0])
    if isinstance(kind, (int, np.integer)):
        kind_t, kind_all = None, int(kind)
    else:
        kind_t, kind_all = _param(kind, n, torch.uint8, dev, "kind")
    delta_t, delta_all = _param(delta, n, torch.float64, dev, "delta")
    mc_t, mc_all = _param(max_checks, n, torch.int64, dev, "max_checks")
    tm_t, tm_all = _param(t_max, n, torch.float64, dev, "t_max")
    mc_max = int(torch.as_tensor(max_checks).max().item()) if mc_t is not None and n else int(mc_all)
    out = {
        "status": torch.empty(n, dtype=torch.uint8, device=dev),
        "toi": torch.empty(n, dtype=torch.float64, device=dev),
        "tol": torch.empty(n, dtype=torch.float64, device=dev),
        "codom": torch.empty(n, dtype=torch.float64, device=dev),
        "checks": torch.empty(n, dtype=torch.int64, device=dev),
        "early": torch.empty(n, dtype=torch.uint8, device=dev),
        "witness": torch.empty((n, 6), dtype=torch.float64, device=dev),
        "level": torch.empty(n, dtype=torch.int32, device=dev),
    }
    with torch.cuda.device(dev):
        slots = int(big_slots or 0)
        nbytes = int(L.tccd_irf_workspace_bytes(n, mc_max, slots))
        ws = _workspace(dev, nbytes)
        b = _lib.TccdBatch()
        b.struct_size = ctypes.sizeof(_lib.TccdBatch)
        b.flags = _lib.FLAG_HEAVY_ONLY if heavy_only else 0
        b.n = n
        b.points = _ptr(pts)
        b.kind = _ptr(kind_t)
        b.kind_all = int(kind_all)
        b.delta = _ptr(delta_t)
        b.delta_all = float(delta_all)
        b.max_checks = _ptr(mc_t)
        b.max_checks_all = int(mc_all)
        b.max_checks_max = mc_max
        b.t_max = _ptr(tm_t)
        b.t_max_all = float(tm_all)
        for k in _IRF_FIELDS:
            setattr(b, k, _ptr(out[k]))
        b.workspace = _ptr(ws)
        b.workspace_bytes = ws.numel()
        b.heavy_blocks = slots
        b.device_sms = sm_count(dev)
        stream = torch.cuda.current_stream(dev)
        _workspace_guard(dev, stream)
        rc = L.tccd_irf_batch(ctypes.byref(b), ctypes.c_void_p(stream.cuda_stream))
        _workspace_release(dev, stream)
        if rc == 3:
            raise ValueError("delta must be positive")
        if rc == 5:
            raise ValueError("t_max must be finite and >= 0")
        _lib.check(rc, "tccd_irf_batch")
    if host_in:
        out = {k: v.cpu() for k, v in out.items()}
    if raise_on_error and n:
        bad = out["status"] >= 2
        if bool(bad.any()):
            i = int(torch.nonzero(bad)[0].item())
            raise ValueError(f"query {i}: invalid IRF input (status {int(out['status'][i])})")
    return out


def irf_solve(q: Query, delta: float = 1e-6, max_checks: int | None = None,
              t_max: float = 1.0) -> CCDResult:
    """ccdkit.baselines.irf_solve for one query, on the GPU."""
    if not (delta > 0.0):
        raise ValueError("delta must be positive")
    mc = IMPLICIT_MAX_CHECKS if max_checks is None else int(max_checks)
    r = irf_batch(torch.from_numpy(q.all_coordinates()).reshape(1, 8, 3), int(q.kind), delta,
                  mc, float(t_max))
    checks = int(r["checks"][0])
    if max_checks is None and bool(r["early"][0]):
        raise RuntimeError(f"irf_solve spent the GPU's implicit budget of {mc} checks; "
                           "pass max_checks explicitly")
    if int(r["status"][0]) == 0:
        return CCDResult(None, None, 0.0, 0.0, checks, False)
    w = r["witness"][0].tolist()
    return CCDResult(toi=float(r["toi"][0]),
                     witness=DomainBox((w[0], w[1]), (w[2], w[3]), (w[4], w[5]),
                                       int(r["level"][0])),
                     achieved_tol=float(r["tol"][0]), codomain_width=float(r["codom"][0]),
                     checks=checks, early_terminated=bool(r["early"][0]))
