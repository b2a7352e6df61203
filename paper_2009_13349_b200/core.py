"""Host-side types mirroring the reference's solve-side API.

Same names, fields, validation rules and exception classes as
pkg/src/ccdkit/core.py (Vec3 :42-72, QueryKind :75-79, Query :83-116,
DomainBox :120-150, SolverConfig :154-184, CCDResult :188-209), so
reference callers switch by changing the import.  The solver's numerics live
on the GPU (csrc/); the scalar ``eval_F*`` here are the reference's
point-wise definition of F (core.py:225-256), for callers and tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import IntEnum
from typing import NamedTuple

import numpy as np


class QueryKind(IntEnum):
    """Vertex-face or edge-edge; the values are the kernel's ``kind`` codes."""

    VERTEX_FACE = 0
    EDGE_EDGE = 1


class _XYZ(NamedTuple):
    x: float
    y: float
    z: float


class Vec3(_XYZ):
    """Three finite binary64 components (core.py:42-72): a tuple, with the
    reference's component-wise arithmetic."""

    __slots__ = ()

    def __new__(cls, x, y, z):
        c = (float(x), float(y), float(z))
        if not all(math.isfinite(v) for v in c):
            raise ValueError(f"Vec3 components must be finite, got {c}")
        return tuple.__new__(cls, c)

    @classmethod
    def _trusted(cls, x: float, y: float, z: float) -> "Vec3":
        return tuple.__new__(cls, (x, y, z))

    def __add__(self, o):
        return Vec3(self[0] + o[0], self[1] + o[1], self[2] + o[2])

    def __sub__(self, o):
        return Vec3(self[0] - o[0], self[1] - o[1], self[2] - o[2])

    def scaled(self, s: float) -> "Vec3":
        return Vec3(self[0] * s, self[1] * s, self[2] * s)

    def dot(self, o) -> float:
        return self[0] * o[0] + self[1] * o[1] + self[2] * o[2]

    def cross(self, o) -> "Vec3":
        return Vec3(self[1] * o[2] - self[2] * o[1], self[2] * o[0] - self[0] * o[2],
                    self[0] * o[1] - self[1] * o[0])


def _vec3(p) -> Vec3:
    if len(p) != 3:
        raise ValueError(f"a point needs 3 coordinates, got {len(p)}")
    return p if type(p) is Vec3 else Vec3(*p)


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
        q.__dict__["points0"] = tuple(Vec3._trusted(*p) for p in points0)
        q.__dict__["points1"] = tuple(Vec3._trusted(*p) for p in points1)
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


# --------------------------------------------------------------------------
# F(t, u, v) at one point, the reference's scalar definition (core.py:
# 221-256): each point lerped to t as (1 - t) * start + t * end, then
#   VF: p - ((1 - u - v) * v1 + u * v2 + v * v3)
#   EE: ((1 - u) * p1 + u * p2) - ((1 - v) * p3 + v * p4)
# in binary64, left to right.  The device hull (csrc/tccd_device.cuh) is
# bit-identical to these at every corner (tests/test_gpu_api.py).


def _at(q: Query, t: float):
    omt = 1.0 - t
    return [tuple(omt * a[i] + t * b[i] for i in range(3)) for a, b in zip(q.points0, q.points1)]


def eval_F_vf(q: Query, t: float, u: float, v: float) -> Vec3:
    p, a, b, c = _at(q, t)
    w = 1.0 - u - v
    return Vec3(*(p[i] - (w * a[i] + u * b[i] + v * c[i]) for i in range(3)))


def eval_F_ee(q: Query, t: float, u: float, v: float) -> Vec3:
    a, b, c, d = _at(q, t)
    return Vec3(*(((1.0 - u) * a[i] + u * b[i]) - ((1.0 - v) * c[i] + v * d[i]) for i in range(3)))


def eval_F(q: Query, t: float, u: float, v: float) -> Vec3:
    return eval_F_vf(q, t, u, v) if q.kind == QueryKind.VERTEX_FACE else eval_F_ee(q, t, u, v)
