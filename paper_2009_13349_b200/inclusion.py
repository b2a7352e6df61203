"""Filter tolerances (host side), mirroring pkg/src/ccdkit/inclusion.py:35-122.

The GPU computes gamma/eps per query itself (the "auto" path).  These host
helpers exist for the reference's scene-wide filter reuse (a ``FilterEps``
passed in ``SolverConfig.filters``, solver.py:30-47) and its validation
errors; they follow the same operation order (``coeff * (g * g * g)``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

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
