"""Mesh-level callers of the solver, batched on the GPU.

Same API and results as the reference's scene module
(pkg/src/ccdkit/scene.py): the broad phase produces exactly the reference's
candidate set, in its order, and the narrow phase runs as batched
``solve_batch`` calls instead of one ``solve`` per candidate:

* ``construct_active_set`` (:303-327): one batched solve over all
  candidates.
* ``line_search_step`` (:468-583): the reference solves candidates in order
  on a shrinking interval [0, alpha] (each solve's t_max is the alpha left by
  the candidates before it).  That order dependence is reproduced exactly:
  a batch is solved at the current alpha, accepted up to the first candidate
  that lowers alpha, and only the candidates after it are re-solved at the
  new alpha -- one batched solve per alpha decrease instead of one solve
  per candidate.  Non-dyadic t_max goes through the engine's general
  ordering path.

The broad phase runs on the GPU too (§8(f) row 2, csrc/broad.cu): the
candidates are written straight into the solver's device layout, so the
narrow phase reads them without a host round trip.
"""

from __future__ import annotations

import contextlib
import gc
import math
from dataclasses import dataclass
from typing import Callable

import ctypes

import numpy as np
import torch

from . import _lib
from .core import DomainBox, Query, QueryKind, SolverConfig
from .inclusion import (EE_COEFF, EE_COEFF_MINSEP, VF_COEFF, VF_COEFF_MINSEP,
                        compute_filters, compute_gamma)
from .solver import solve_batch

__all__ = [
    "TriMeshPair", "ContactCandidate", "CandidateBound", "LineSearchResult",
    "InfeasibleStepError", "edges_from_triangles", "load_obj", "broad_phase",
    "construct_active_set", "primitive_distance_lb", "line_search_step",
    # batch forms (device-resident)
    "CandidateSet", "broad_phase_batch", "active_set_batch", "distance_lb",
]

_SQRT3 = math.sqrt(3.0)
_DISTANCE_SLACK = 1e-9  # scene.py:42-45
_LS_WINDOW = 1 << 18  # candidates per line-search solve


def edges_from_triangles(triangles) -> np.ndarray:
    tris = np.asarray(triangles, dtype=np.intp)
    if tris.size == 0:
        return np.zeros((0, 2), dtype=np.intp)
    if tris.ndim != 2 or tris.shape[1] != 3:
        raise ValueError("triangles must be an (m, 3) index array")
    e = np.concatenate((tris[:, (0, 1)], tris[:, (1, 2)], tris[:, (2, 0)]))
    e.sort(axis=1)
    return np.unique(e, axis=0)


@dataclass(frozen=True)
class TriMeshPair:
    """Triangle mesh with vertex positions at both ends of one step
    (scene.py:68-114, same validation)."""

    x0: np.ndarray
    x1: np.ndarray
    triangles: np.ndarray
    edges: np.ndarray | None = None

    def __post_init__(self):
        x0 = np.ascontiguousarray(np.asarray(self.x0, dtype=np.float64))
        x1 = np.ascontiguousarray(np.asarray(self.x1, dtype=np.float64))
        if x0.ndim != 2 or x0.shape[1] != 3 or x1.shape != x0.shape:
            raise ValueError("x0 and x1 must be (n, 3) arrays of equal shape")
        if not (np.all(np.isfinite(x0)) and np.all(np.isfinite(x1))):
            raise ValueError("vertex positions must be finite")
        tris = np.ascontiguousarray(np.asarray(self.triangles, dtype=np.intp))
        if tris.size == 0:
            tris = np.zeros((0, 3), dtype=np.intp)
        if tris.ndim != 2 or tris.shape[1] != 3:
            raise ValueError("triangles must be an (m, 3) index array")
        if self.edges is None:
            edges = edges_from_triangles(tris)
        else:
            edges = np.ascontiguousarray(np.asarray(self.edges, dtype=np.intp))
            if edges.size == 0:
                edges = np.zeros((0, 2), dtype=np.intp)
            if edges.ndim != 2 or edges.shape[1] != 2:
                raise ValueError("edges must be a (k, 2) index array")
        n = x0.shape[0]
        for name, idx in (("triangles", tris), ("edges", edges)):
            if idx.size and (int(idx.min()) < 0 or int(idx.max()) >= n):
                raise ValueError(f"{name} index vertices outside [0, {n})")
        object.__setattr__(self, "x0", x0)
        object.__setattr__(self, "x1", x1)
        object.__setattr__(self, "triangles", tris)
        object.__setattr__(self, "edges", edges)

    @property
    def n_vertices(self) -> int:
        return int(self.x0.shape[0])

    def at(self, alpha: float) -> np.ndarray:
        return self.x0 + float(alpha) * (self.x1 - self.x0)


@dataclass(frozen=True)
class ContactCandidate:
    kind: QueryKind
    indices: tuple
    query: Query

    @classmethod
    def _trusted(cls, kind, indices, query) -> "ContactCandidate":
        c = object.__new__(cls)
        c.__dict__["kind"] = kind
        c.__dict__["indices"] = indices
        c.__dict__["query"] = query
        return c


@dataclass
class CandidateSet:
    """Broad-phase output in batch layout, reference order (VF pairs sorted
    by (vertex, triangle), then EE pairs sorted by (edge_a, edge_b))."""

    kind: object     # [m] u8 (torch device tensor, or numpy)
    indices: object  # [m, 2] int64
    points: object   # [m, 8, 3] f64

    @property
    def m(self) -> int:
        return int(self.kind.shape[0])

    def host(self) -> "CandidateSet":
        """The same candidates as numpy arrays."""
        return CandidateSet(_np(self.kind), _np(self.indices), _np(self.points))

    def candidate(self, i: int) -> ContactCandidate:
        p = self.points[i].tolist()
        k = QueryKind(int(self.kind[i]))
        ij = self.indices[i].tolist()
        return ContactCandidate(k, (int(ij[0]), int(ij[1])), Query(k, tuple(map(tuple, p[:4])),
                                                                  tuple(map(tuple, p[4:]))))

    def to_list(self) -> list:
        """All candidates as ContactCandidate objects (bulk conversion: the
        coordinates come from a validated mesh, so the Query objects are
        built without re-checking them)."""
        h = self.host()
        K = (QueryKind.VERTEX_FACE, QueryKind.EDGE_EDGE)
        out = []
        qt, ct = Query._trusted, ContactCandidate._trusted
        with _bulk():
            flat = h.points.reshape(h.m, 24).tolist()
            for f, kk, ij in zip(flat, h.kind.tolist(), h.indices.tolist()):
                it = iter(f)
                t = tuple(zip(it, it, it))  # the 8 points as (x, y, z) tuples
                k = K[kk]
                out.append(ct(k, tuple(ij), qt(k, t[:4], t[4:])))
        return out


@contextlib.contextmanager
def _bulk():
    """Millions of acyclic result objects: keep the cyclic collector from
    rescanning them while they are built."""
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()


def load_obj(path) -> tuple[np.ndarray, np.ndarray]:
    """Positions and triangles of a Wavefront OBJ file (scene.py:117-149):
    ``v`` and ``f`` records only, polygons fan-triangulated, ``v/vt/vn``
    groups keep the vertex index, negative indices count back."""
    verts, faces = [], []
    with open(path, encoding="utf-8") as fh:
        for line_no, raw in enumerate(fh, start=1):
            tok = raw.split()
            if not tok or tok[0].startswith("#"):
                continue
            if tok[0] == "v":
                if len(tok) < 4:
                    raise ValueError(f"line {line_no}: vertex needs 3 coordinates")
                verts.append([float(t) for t in tok[1:4]])
            elif tok[0] == "f":
                if len(tok) < 4:
                    raise ValueError(f"line {line_no}: face needs >= 3 corners")
                ids = [int(t.split("/", 1)[0]) for t in tok[1:]]
                ids = [i - 1 if i > 0 else len(verts) + i for i in ids]
                faces += [[ids[0], ids[k], ids[k + 1]] for k in range(1, len(ids) - 1)]
    v = np.asarray(verts, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(faces, dtype=np.intp).reshape(-1, 3)
    if f.size and (f.min() < 0 or f.max() >= len(v)):
        raise ValueError("face index out of range")
    return v, f


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def broad_phase_batch(mesh: TriMeshPair, inflation: float = 0.0, device=None) -> CandidateSet:
    """The reference broad phase's candidates (scene.py:225-300), found on
    the GPU (csrc/broad.cu, tccd_broad_*): exactly the pairs whose inflated
    swept boxes overlap, minus pairs sharing a mesh vertex, VF pairs sorted
    by (vertex, triangle) then EE pairs by (edge_a, edge_b).  The reference's
    grid hash is a superset filter followed by the same exact box test, so
    its result is this set.  Returns device tensors: kind [m] u8, indices
    [m, 2] i64, points [m, 8, 3] f64 (the solver's layout)."""
    if not (inflation >= 0.0 and math.isfinite(inflation)):
        raise ValueError("inflation must be >= 0 and finite")
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError("the broad phase runs on the GPU (there is no CPU fallback)")
    L = _lib.lib()
    with torch.cuda.device(dev):
        x0 = torch.from_numpy(mesh.x0).to(dev)
        x1 = torch.from_numpy(mesh.x1).to(dev)
        tris = torch.from_numpy(np.ascontiguousarray(mesh.triangles, dtype=np.int64)).to(dev)
        edges = torch.from_numpy(np.ascontiguousarray(mesh.edges, dtype=np.int64)).to(dev)
        m = _lib.TccdMesh()
        m.struct_size = ctypes.sizeof(_lib.TccdMesh)
        m.n_vertices, m.n_triangles, m.n_edges = mesh.n_vertices, len(mesh.triangles), len(mesh.edges)
        m.x0, m.x1 = x0.data_ptr(), x1.data_ptr()
        m.triangles = tris.data_ptr() if len(mesh.triangles) else None
        m.edges = edges.data_ptr() if len(mesh.edges) else None
        h, nvf, nee = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        stream = torch.cuda.current_stream(dev)
        rc = L.tccd_broad_create(ctypes.byref(m), float(inflation), ctypes.byref(h),
                                 ctypes.byref(nvf), ctypes.byref(nee),
                                 ctypes.c_void_p(stream.cuda_stream))
        try:
            _lib.check(rc, "tccd_broad_create")
            total = nvf.value + nee.value
            kind = torch.empty(total, dtype=torch.uint8, device=dev)
            idx = torch.empty((total, 2), dtype=torch.int64, device=dev)
            pts = torch.empty((total, 8, 3), dtype=torch.float64, device=dev)
            _lib.check(L.tccd_broad_emit(h, ctypes.c_void_p(kind.data_ptr()),
                                         ctypes.c_void_p(idx.data_ptr()),
                                         ctypes.c_void_p(pts.data_ptr())), "tccd_broad_emit")
        finally:
            L.tccd_broad_destroy(h)
    return CandidateSet(kind, idx, pts)


def broad_phase(mesh: TriMeshPair, inflation: float = 0.0, device=None) -> list:
    """Reference-shaped result: a list of ContactCandidate."""
    return broad_phase_batch(mesh, inflation, device).to_list()


def _solve(cs: CandidateSet, sel, cfg: SolverConfig, separation, device):
    pts = torch.as_tensor(cs.points[sel])
    kind = torch.as_tensor(cs.kind[sel])
    sep = separation if np.isscalar(separation) else torch.as_tensor(
        np.ascontiguousarray(np.asarray(separation, dtype=np.float64)))
    r = solve_batch(pts, kind, cfg, separation=sep, device=device if device is not None
                    else (pts.device if pts.is_cuda else None))
    return {k: _np(v) for k, v in r.items()}


def _witness(r, i) -> DomainBox:
    w = r["witness"][i]
    return DomainBox((float(w[0]), float(w[1])), (float(w[2]), float(w[3])),
                     (float(w[4]), float(w[5])), int(r["level"][i]))


def active_set_batch(mesh: TriMeshPair, delta: float = 1e-6, max_checks: int = 1_000_000,
                     separation: float = 0.0, device=None):
    """construct_active_set in batch form, device-resident: the broad phase
    (inflation separation + delta) and one batched solve of every candidate
    (scene.py:303-327).  Returns (hits, res): the colliding candidates as a
    CandidateSet in candidate order, and their solver outputs (toi, witness,
    level, ... as device tensors)."""
    cs = broad_phase_batch(mesh, inflation=separation + delta, device=device)
    cfg = SolverConfig(delta=delta, max_checks=max_checks, separation=separation)
    if cs.m == 0:
        return cs, {}
    r = solve_batch(cs.points, cs.kind, cfg, device=cs.points.device)
    hit = torch.nonzero(r["status"] == 1).squeeze(1)
    hits = CandidateSet(cs.kind[hit], cs.indices[hit], cs.points[hit])
    return hits, {k: v[hit] for k, v in r.items()}


def construct_active_set(mesh: TriMeshPair, delta: float = 1e-6, max_checks: int = 1_000_000,
                         separation: float = 0.0, device=None) -> list:
    """Candidates the solver could not rule out, with toi and witness
    (scene.py:303-327): active_set_batch as the reference's list of
    (ContactCandidate, toi, DomainBox)."""
    hits, r = active_set_batch(mesh, delta, max_checks, separation, device)
    if hits.m == 0:
        return []
    cands = hits.to_list()
    toi = _np(r["toi"]).tolist()
    w = _np(r["witness"]).tolist()
    lv = _np(r["level"]).tolist()
    with _bulk():
        return [(c, toi[i], DomainBox._trusted((w[i][0], w[i][1]), (w[i][2], w[i][3]),
                                                (w[i][4], w[i][5]), lv[i]))
                for i, c in enumerate(cands)]


# --- start-distance lower bounds: the reference's closed forms (scene.py:335-419),
# same operation order (dot products left to right, Vec3 arithmetic per component)

def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _add(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def _scl(a, s):
    return (a[0] * s, a[1] * s, a[2] * s)


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _norm(v):
    return math.sqrt(_dot(v, v))


def _clamp01(s):
    return 0.0 if s < 0.0 else (1.0 if s > 1.0 else s)


def _pt_seg(p, a, b):
    ab = _sub(b, a)
    denom = _dot(ab, ab)
    if denom == 0.0:
        return _norm(_sub(p, a))
    s = _clamp01(_dot(_sub(p, a), ab) / denom)
    return _norm(_sub(p, _add(a, _scl(ab, s))))


def _pt_tri(p, a, b, c):
    best = min(_pt_seg(p, a, b), _pt_seg(p, b, c), _pt_seg(p, c, a))
    n = _cross(_sub(b, a), _sub(c, a))
    nn = _dot(n, n)
    if nn > 0.0:
        w0 = _dot(_cross(_sub(c, b), _sub(p, b)), n)
        w1 = _dot(_cross(_sub(a, c), _sub(p, c)), n)
        w2 = _dot(_cross(_sub(b, a), _sub(p, a)), n)
        if w0 >= 0.0 and w1 >= 0.0 and w2 >= 0.0:
            best = min(best, abs(_dot(_sub(p, a), n)) / math.sqrt(nn))
    return best


def _seg_seg(p1, q1, p2, q2):
    d1, d2, r = _sub(q1, p1), _sub(q2, p2), _sub(p1, p2)
    a, e, f = _dot(d1, d1), _dot(d2, d2), _dot(d2, r)
    if a == 0.0 and e == 0.0:
        return _norm(r)
    if a == 0.0:
        s, t = 0.0, _clamp01(f / e)
    else:
        c = _dot(d1, r)
        if e == 0.0:
            t, s = 0.0, _clamp01(-c / a)
        else:
            b = _dot(d1, d2)
            denom = a * e - b * b
            s = _clamp01((b * f - c * e) / denom) if denom > 0.0 else 0.0
            t = (b * s + f) / e
            if t < 0.0:
                t, s = 0.0, _clamp01(-c / a)
            elif t > 1.0:
                t, s = 1.0, _clamp01((b - c) / a)
    return _norm(_sub(_add(p1, _scl(d1, s)), _add(p2, _scl(d2, t))))


def distance_lb(kind: int, points8: np.ndarray) -> float:
    """primitive_distance_lb (scene.py:404-419) on one candidate's points."""
    p = [tuple(float(c) for c in points8[k]) for k in range(4)]
    d = _pt_tri(*p) if kind == 0 else _seg_seg(*p)
    if d <= 0.0:
        return 0.0
    return max(0.0, math.nextafter(d / _SQRT3, 0.0))


# The same closed forms over a whole candidate batch: every operation is the
# scalar code's, elementwise in the same order (numpy float64 ufuncs round
# each operation like Python floats and never contract a multiply-add), and
# each branch becomes a select of both outcomes, so the bounds are
# bit-identical to distance_lb's (tests/test_scene.py checks).

def _vsub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _vadd(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def _vscl(a, s):
    return (a[0] * s, a[1] * s, a[2] * s)


def _vdot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _vcross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _vnorm(v):
    return np.sqrt(_vdot(v, v))


def _vclamp01(s):
    return np.where(s < 0.0, 0.0, np.where(s > 1.0, 1.0, s))


def _vpt_seg(p, a, b):
    ab = _vsub(b, a)
    denom = _vdot(ab, ab)
    s = _vclamp01(_vdot(_vsub(p, a), ab) / denom)
    return np.where(denom == 0.0, _vnorm(_vsub(p, a)), _vnorm(_vsub(p, _vadd(a, _vscl(ab, s)))))


def _vpt_tri(p, a, b, c):
    best = np.minimum(np.minimum(_vpt_seg(p, a, b), _vpt_seg(p, b, c)), _vpt_seg(p, c, a))
    n = _vcross(_vsub(b, a), _vsub(c, a))
    nn = _vdot(n, n)
    w0 = _vdot(_vcross(_vsub(c, b), _vsub(p, b)), n)
    w1 = _vdot(_vcross(_vsub(a, c), _vsub(p, c)), n)
    w2 = _vdot(_vcross(_vsub(b, a), _vsub(p, a)), n)
    inside = (nn > 0.0) & (w0 >= 0.0) & (w1 >= 0.0) & (w2 >= 0.0)
    return np.where(inside, np.minimum(best, np.abs(_vdot(_vsub(p, a), n)) / np.sqrt(nn)), best)


def _vseg_seg(p1, q1, p2, q2):
    d1, d2, r = _vsub(q1, p1), _vsub(q2, p2), _vsub(p1, p2)
    a, e, f = _vdot(d1, d1), _vdot(d2, d2), _vdot(d2, r)
    c = _vdot(d1, r)
    b = _vdot(d1, d2)
    denom = a * e - b * b
    # general case (a > 0, e > 0)
    s_g = np.where(denom > 0.0, _vclamp01((b * f - c * e) / denom), 0.0)
    t_g = (b * s_g + f) / e
    s_g, t_g = (np.where(t_g < 0.0, _vclamp01(-c / a), np.where(t_g > 1.0, _vclamp01((b - c) / a), s_g)),
                np.where(t_g < 0.0, 0.0, np.where(t_g > 1.0, 1.0, t_g)))
    # a == 0: s = 0, t = clamp(f / e); e == 0 (a > 0): t = 0, s = clamp(-c / a)
    s = np.where(a == 0.0, 0.0, np.where(e == 0.0, _vclamp01(-c / a), s_g))
    t = np.where(a == 0.0, _vclamp01(f / e), np.where(e == 0.0, 0.0, t_g))
    d = _vnorm(_vsub(_vadd(p1, _vscl(d1, s)), _vadd(p2, _vscl(d2, t))))
    return np.where((a == 0.0) & (e == 0.0), _vnorm(r), d)


def distance_lb_batch(kind: np.ndarray, points: np.ndarray) -> np.ndarray:
    """distance_lb of every candidate: kind [m], points [m, 8, 3] (start
    positions are points[:, :4])."""
    kind = np.asarray(kind)
    P = np.asarray(points, dtype=np.float64)
    pt = [tuple(P[:, k, j] for j in range(3)) for k in range(4)]
    with np.errstate(all="ignore"):  # (the unselected branch may divide by 0)
        d = np.where(kind == 0, _vpt_tri(*pt), _vseg_seg(*pt))
        lb = np.maximum(0.0, np.nextafter(d / _SQRT3, 0.0))
    return np.where(d <= 0.0, 0.0, lb)


def primitive_distance_lb(candidate: ContactCandidate) -> float:
    return distance_lb(int(candidate.kind), candidate.query.all_coordinates())


class InfeasibleStepError(RuntimeError):
    """No positive step fraction can be certified (scene.py:422-430)."""


@dataclass(frozen=True)
class CandidateBound:
    candidate: ContactCandidate
    distance_lb: float
    separation: float
    toi: float | None
    witness: DomainBox | None

    @classmethod
    def _trusted(cls, candidate, distance_lb, separation, toi, witness) -> "CandidateBound":
        b = object.__new__(cls)
        b.__dict__["candidate"] = candidate
        b.__dict__["distance_lb"] = distance_lb
        b.__dict__["separation"] = separation
        b.__dict__["toi"] = toi
        b.__dict__["witness"] = witness
        return b


@dataclass(frozen=True)
class LineSearchResult:
    alpha: float
    p: float
    validations: int
    bounds: tuple
    limiting: int | None

    @property
    def limiting_bound(self):
        return None if self.limiting is None else self.bounds[self.limiting]


def line_search_step(mesh: TriMeshPair, *, p: float, delta: float = 1e-6,
                     max_checks: int = 1_000_000,
                     energy_decreases: Callable[[float], bool] | None = None,
                     alpha_min: float = 1e-8, inflation: float | None = None,
                     device=None) -> LineSearchResult:
    """Largest certified collision-free step fraction (scene.py:468-583)."""
    if not (0.0 < p < 1.0):
        raise ValueError("p must lie strictly between 0 and 1")
    if inflation is None:
        inflation = 2.0 * delta
    cs = broad_phase_batch(mesh, inflation, device=device)
    hc = cs.host()
    m = cs.m
    # start-distance bounds and the filters of every candidate, batched; the
    # first failing candidate raises what the reference's loop raises first
    d_lb = distance_lb_batch(hc.kind, hc.points)
    sep0 = np.minimum(p * d_lb, delta)
    gam = np.maximum(1.0, np.abs(hc.points).max(axis=1))  # compute_gamma per candidate
    bad_sep = (sep0 > 0.0) & ~np.all(sep0[:, None] < gam, axis=1)
    bad_d = d_lb <= 0.0
    first_bad = int(np.argmax(bad_d | bad_sep)) if bool((bad_d | bad_sep).any()) else -1
    if first_bad >= 0:
        i = first_bad
        if bad_d[i]:
            raise InfeasibleStepError(
                f"{QueryKind(int(hc.kind[i])).name} pair {tuple(int(x) for x in hc.indices[i])} "
                "touches at the step start; no positive step can be certified")
        compute_filters(QueryKind(int(hc.kind[i])), tuple(float(g) for g in gam[i]),
                        separation=float(sep0[i]))  # (raises the reference's ValueError)
    coeff = np.where(hc.kind == 0, np.where(sep0 > 0.0, VF_COEFF_MINSEP, VF_COEFF),
                     np.where(sep0 > 0.0, EE_COEFF_MINSEP, EE_COEFF))
    eps_max = (coeff[:, None] * (gam * gam * gam)).max(axis=1)  # max(compute_filters(...).eps)

    def worst_ratio(tol):
        return float(np.min((d_lb - tol - eps_max - _DISTANCE_SLACK) / d_lb)) if m else 0.0

    cands = hc.to_list() if m else []
    alpha, validations, bounds, limiting = 1.0, 0, [], None
    tol_assumed = delta
    while m:
        validations += 1
        worst = worst_ratio(tol_assumed)
        while p >= worst:
            p *= 0.5
            if p == 0.0:
                raise InfeasibleStepError("validation halved p to zero; the start distances "
                                          "cannot cover the solver tolerance plus numeric error")
        seps = np.minimum(p * d_lb, delta)
        alpha, achieved, limiting = 1.0, tol_assumed, None
        bounds = []
        i0 = 0
        while i0 < m:
            # a window of candidates i0.. solved at the current alpha; results
            # hold up to the first one that lowers alpha, the rest are solved
            # again at the new alpha (windows bound that repeated work)
            i1 = min(m, i0 + _LS_WINDOW)
            cfg = SolverConfig(delta=tol_assumed, max_checks=max_checks, t_max=alpha)
            r = _solve(cs, slice(i0, i1), cfg, seps[i0:i1], device)
            hit = r["status"] == 1
            toi = r["toi"]
            lower = hit & (toi < alpha)
            lowered = bool(lower.any())
            j_end = int(np.argmax(lower)) + 1 if lowered else i1 - i0
            # a free result carries codomain width 0 (solver.py:89-93)
            if j_end:
                achieved = max(achieved, float(np.max(np.where(hit[:j_end], r["codom"][:j_end], 0.0))))
            toi_l = toi[:j_end].tolist()
            hit_l = hit[:j_end].tolist()
            w = r["witness"][:j_end].tolist()
            lv = r["level"][:j_end].tolist()
            d_l = d_lb[i0:i0 + j_end].tolist()
            s_l = seps[i0:i0 + j_end].tolist()
            with _bulk():
                for j in range(j_end):
                    if hit_l[j]:
                        wj = w[j]
                        bounds.append(CandidateBound._trusted(
                            cands[i0 + j], d_l[j], s_l[j], toi_l[j],
                            DomainBox._trusted((wj[0], wj[1]), (wj[2], wj[3]), (wj[4], wj[5]),
                                               lv[j])))
                    else:
                        bounds.append(CandidateBound._trusted(cands[i0 + j], d_l[j], s_l[j],
                                                              None, None))
            nxt = i1
            if lowered:
                alpha = toi_l[j_end - 1]
                limiting = len(bounds) - 1
                nxt = i0 + j_end
            if alpha == 0.0:
                break  # the remaining interval is empty
            i0 = nxt
        if not (achieved > tol_assumed):
            break
        if p < worst_ratio(achieved):
            break
        tol_assumed = achieved
    if energy_decreases is not None:
        while alpha > alpha_min and not energy_decreases(alpha):
            alpha *= 0.5
    return LineSearchResult(alpha=alpha, p=p, validations=validations, bounds=tuple(bounds),
                            limiting=limiting)
