"""Filter tolerances (host side), mirroring pkg/src/ccdkit/inclusion.py:35-122,
and the reference's box-level inclusion API (inclusion.py:125-217) over the
device kernels of csrc/mirror.cu.

The GPU computes gamma/eps per query itself (the "auto" path).  These host
helpers exist for the reference's scene-wide filter reuse (a ``FilterEps``
passed in ``SolverConfig.filters``, solver.py:30-47) and its validation
errors; they follow the same operation order (``coeff * (g * g * g)``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .core import QueryKind

VF_COEFF = 6.661338147750939e-15
EE_COEFF = 6.217248937900877e-15
VF_COEFF_MINSEP = 7.549516567451064e-15
EE_COEFF_MINSEP = 7.105427357601002e-15


@dataclass(frozen=True)
class FilterEps:
    kind: QueryKind
    gamma: tuple
    eps: tuple
    separation: float


def compute_gamma(coords) -> tuple[float, float, float]:
    """Per-axis max(1, max |x|) over an (n, 3) coordinate set."""
    a = np.asarray(coords, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 3 or a.shape[0] == 0:
        raise ValueError("coords must be a non-empty (n, 3) array")
    if not np.all(np.isfinite(a)):
        raise ValueError("coordinates must be finite")
    m = np.abs(a).max(axis=0)
    return (max(1.0, float(m[0])), max(1.0, float(m[1])), max(1.0, float(m[2])))


def compute_filters(kind: QueryKind, gamma, separation: float = 0.0) -> FilterEps:
    gx, gy, gz = (float(g) for g in gamma)
    if not (gx >= 1.0 and gy >= 1.0 and gz >= 1.0):
        raise ValueError("gamma components must be >= 1")
    separation = float(separation)
    if separation < 0.0 or not math.isfinite(separation):
        raise ValueError("separation must be >= 0 and finite")
    if separation > 0.0:
        if not (separation < gx and separation < gy and separation < gz):
            raise ValueError(
                f"separation {separation} must be smaller than every gamma {gamma}")
        coeff = VF_COEFF_MINSEP if kind == QueryKind.VERTEX_FACE else EE_COEFF_MINSEP
    else:
        coeff = VF_COEFF if kind == QueryKind.VERTEX_FACE else EE_COEFF
    return FilterEps(kind=QueryKind(kind), gamma=(gx, gy, gz),
                     eps=(coeff * (gx * gx * gx), coeff * (gy * gy * gy), coeff * (gz * gz * gz)),
                     separation=separation)


# --------------------------------------------------------------------------
# The reference's box-level inclusion API (inclusion.py:125-217).  The
# corner hulls and kappas are evaluated on the GPU by the solver's own
# device arithmetic (csrc/mirror.cu: tccd_box_hulls, tccd_kappas), one call
# per batch; the classification of a hull against the filters is a few
# comparisons and stays on the host.


class BoxClass(IntEnum):
    """Outcome of classifying a hull against the filter box (values as
    _kernel.py:36-38)."""

    DISJOINT = 0
    INTERSECTS = 1
    CONTAINED = 2


@dataclass(frozen=True)
class InclusionBox:
    """Per-axis range hull [lo, hi] of F over a domain box."""

    lo: tuple
    hi: tuple

    def __post_init__(self):
        for i in range(3):
            if not self.lo[i] <= self.hi[i]:
                raise ValueError(f"InclusionBox axis {i}: lo {self.lo[i]} > hi {self.hi[i]}")


def _device(device):
    import torch
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("the inclusion kernels need a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def box_inclusion_batch(points, kind, boxes, device=None):
    """Corner hulls of F for a batch: points [n, 8, 3] (start then end block),
    kind [n] or scalar, boxes [n, 6] = (t0, t1, u0, u1, v0, v1).  Returns
    host arrays (lo, hi), each [n, 3] (tccd_box_hulls)."""
    import ctypes
    import torch
    from . import _lib
    dev = _device(device)
    pts = torch.as_tensor(np.asarray(points, dtype=np.float64)).reshape(-1, 8, 3)
    n = int(pts.shape[0])
    bx = torch.as_tensor(np.asarray(boxes, dtype=np.float64)).reshape(n, 6)
    scalar = np.ndim(kind) == 0
    kd = None if scalar else torch.as_tensor(np.asarray(kind, dtype=np.uint8)).to(dev)
    pts, bx = pts.to(dev), bx.to(dev)
    lo = torch.empty((n, 3), dtype=torch.float64, device=dev)
    hi = torch.empty((n, 3), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        rc = _lib.lib().tccd_box_hulls(
            ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(kd.data_ptr()) if kd is not None else None,
            int(kind) if scalar else 0, ctypes.c_void_p(bx.data_ptr()), n,
            ctypes.c_void_p(lo.data_ptr()), ctypes.c_void_p(hi.data_ptr()),
            ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        _lib.check(rc, "tccd_box_hulls")
    return lo.cpu().numpy(), hi.cpu().numpy()


def box_inclusion(q, box, device=None) -> InclusionBox:
    """Range hull of F over a DomainBox: per axis, min and max over its 8
    corners (inclusion.box_inclusion, inclusion.py:131-156)."""
    lo, hi = box_inclusion_batch(q.all_coordinates()[None], int(q.kind),
                                 [[box.t[0], box.t[1], box.u[0], box.u[1], box.v[0], box.v[1]]],
                                 device)
    return InclusionBox(lo=tuple(float(x) for x in lo[0]), hi=tuple(float(x) for x in hi[0]))


def classify_box(box: InclusionBox, eps: FilterEps, separation: float = 0.0) -> BoxClass:
    """Hull enlarged by the separation against [-eps, eps], axes x, y, z:
    DISJOINT at the first axis strictly outside, CONTAINED when inside on
    every axis, else INTERSECTS; a tie is never DISJOINT (inclusion.py:
    159-192, the comparisons of _kernel._classify)."""
    if float(separation) != eps.separation:
        raise ValueError(f"separation {separation} does not match the filter set's "
                         f"{eps.separation}; recompute filters for this separation")
    d = eps.separation
    inside = True
    for ax in range(3):
        e = eps.eps[ax]
        lo, hi = box.lo[ax] - d, box.hi[ax] + d
        if lo > e or hi < -e:
            return BoxClass.DISJOINT
        inside = inside and lo >= -e and hi <= e
    return BoxClass.CONTAINED if inside else BoxClass.INTERSECTS


def kappas_batch(points, kind, t_max=1.0, device=None) -> np.ndarray:
    """[n, 3] split weights (k_t, k_u, k_v) for a batch (tccd_kappas)."""
    import ctypes
    import torch
    from . import _lib
    dev = _device(device)
    pts = torch.as_tensor(np.asarray(points, dtype=np.float64)).reshape(-1, 8, 3).to(dev)
    n = int(pts.shape[0])
    scalar = np.ndim(kind) == 0
    kd = None if scalar else torch.as_tensor(np.asarray(kind, dtype=np.uint8)).to(dev)
    tm = None if np.ndim(t_max) == 0 else torch.as_tensor(np.asarray(t_max, dtype=np.float64)).to(dev)
    out = torch.empty((n, 3), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        rc = _lib.lib().tccd_kappas(
            ctypes.c_void_p(pts.data_ptr()), ctypes.c_void_p(kd.data_ptr()) if kd is not None else None,
            int(kind) if scalar else 0, ctypes.c_void_p(tm.data_ptr()) if tm is not None else None,
            float(t_max) if tm is None else 0.0, n, ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        _lib.check(rc, "tccd_kappas")
    return out.cpu().numpy()


def kappas(q, t_max: float = 1.0, device=None) -> tuple[float, float, float]:
    """Per-dimension split weights on [0, t_max] x [0,1]^2: 3 x the largest
    |F| difference between corners that differ in that dimension only
    (inclusion.kappas, inclusion.py:195-217 = _kernel._kappas)."""
    k = kappas_batch(q.all_coordinates()[None], int(q.kind), t_max, device)[0]
    return (float(k[0]), float(k[1]), float(k[2]))
