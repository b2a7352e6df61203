"""Host-side types mirroring the reference's solve-side API.

Same names, fields, validation rules and exception classes as
pkg/src/ccdkit/core.py (QueryKind :75-79, Query :83-116, DomainBox :120-150,
SolverConfig :154-184, CCDResult :188-209), so reference callers switch by
changing the import.  The numerics live on the GPU (csrc/); nothing here
evaluates F.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import IntEnum

import numpy as np


class QueryKind(IntEnum):
    """Vertex-face or edge-edge; the values are the kernel's ``kind`` codes."""

    VERTEX_FACE = 0
    EDGE_EDGE = 1


def _vec3(p) -> tuple[float, float, float]:
    if len(p) != 3:
        raise ValueError(f"a point needs 3 coordinates, got {len(p)}")
    x, y, z = (float(c) for c in p)
    if not (math.isfinite(x) and math.isfinite(y) and math.isfinite(z)):
        raise ValueError(f"Vec3 components must be finite, got ({x}, {y}, {z})")
    return (x, y, z)


@dataclass(frozen=True)
class Query:
    """Four points with start (t=0) and end (t=1) positions.

    VERTEX_FACE order: (p, v1, v2, v3); EDGE_EDGE: (p1, p2, p3, p4).
    """

    kind: QueryKind
    points0: tuple
    points1: tuple

    def __post_init__(self):
        if len(self.points0) != 4 or len(self.points1) != 4:
            raise ValueError("Query needs exactly 4 start and 4 end points")
        object.__setattr__(self, "points0", tuple(_vec3(p) for p in self.points0))
        object.__setattr__(self, "points1", tuple(_vec3(p) for p in self.points1))
        if not isinstance(self.kind, QueryKind):
            object.__setattr__(self, "kind", QueryKind(self.kind))

    @classmethod
    def _trusted(cls, kind: QueryKind, points0: tuple, points1: tuple) -> "Query":
        """A Query from values that already satisfy the checks above (finite
        float coordinates read back from a validated batch): the same object,
        without re-validating 24 coordinates one by one."""
        q = object.__new__(cls)
        q.__dict__["kind"] = kind
        q.__dict__["points0"] = points0
        q.__dict__["points1"] = points1
        return q

    def as_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        return (np.array(self.points0, dtype=np.float64),
                np.array(self.points1, dtype=np.float64))

    def all_coordinates(self) -> np.ndarray:
        """(8, 3): start block then end block -- the batch layout of one query."""
        return np.array(self.points0 + self.points1, dtype=np.float64)


@dataclass(frozen=True)
class DomainBox:
    """Sub-box of the (t, u, v) domain with its bisection level."""

    t: tuple
    u: tuple
    v: tuple
    level: int = 0

    def __post_init__(self):
        for name, (lo, hi) in (("t", self.t), ("u", self.u), ("v", self.v)):
            if not (0.0 <= lo <= hi <= 1.0):
                raise ValueError(f"DomainBox.{name} = ({lo}, {hi}) not nested in [0, 1]")
        if self.level < 0:
            raise ValueError("DomainBox.level must be >= 0")

    @classmethod
    def _trusted(cls, t: tuple, u: tuple, v: tuple, level: int) -> "DomainBox":
        """A DomainBox from a solver witness (nested in [0, 1] by construction)."""
        b = object.__new__(cls)
        b.__dict__["t"] = t
        b.__dict__["u"] = u
        b.__dict__["v"] = v
        b.__dict__["level"] = level
        return b

    @property
    def widths(self) -> tuple[float, float, float]:
        return (self.t[1] - self.t[0], self.u[1] - self.u[0], self.v[1] - self.v[0])

    @property
    def max_width(self) -> float:
        return max(self.widths)


@dataclass(frozen=True)
class SolverConfig:
    """delta, max_checks (m_I), separation (d), t_max, filters ('auto' | FilterEps)."""

    delta: float = 1e-6
    max_checks: int = 1_000_000
    separation: float = 0.0
    t_max: float = 1.0
    filters: object = "auto"

    def __post_init__(self):
        if not (self.delta > 0.0 and math.isfinite(self.delta)):
            raise ValueError("delta must be positive and finite")
        if int(self.max_checks) < 1:
            raise ValueError("max_checks must be >= 1")
        if not (self.separation >= 0.0 and math.isfinite(self.separation)):
            raise ValueError("separation must be >= 0 and finite")
        if not (0.0 < self.t_max <= 1.0):
            raise ValueError("t_max must lie in (0, 1]")


@dataclass(frozen=True)
class CCDResult:
    """toi is None iff certified collision free; else a conservative time of impact."""

    toi: float | None
    witness: DomainBox | None
    achieved_tol: float
    codomain_width: float
    checks: int
    early_terminated: bool

    @property
    def colliding(self) -> bool:
        return self.toi is not None
