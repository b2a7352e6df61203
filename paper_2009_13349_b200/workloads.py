"""Seeded synthetic query sets for the five BASELINE.json workloads.

The reference measures on the paper's 60M-query dataset and its handcrafted
55K set, neither of which is in the container; these seeded
generators stand in for them with the shapes, sizes and value laws
BASELINE.json states.  Every set is index-addressable: query i
is produced by block ``i // BLOCK`` of a PCG64 stream seeded with
``(2009_13349 + config, block)``, so any shard of any size, on any number of
GPUs, sees byte-identical inputs.

Layout (the one include/tccd.h consumes): ``points`` [n, 8, 3] float64 --
the four points at t0 in query order (VF: p, v1, v2, v3; EE: p1, p2, p3, p4,
pkg/src/ccdkit/core.py:86-89) followed by the same four at t1 -- and
``kind`` [n] uint8 (0 = vertex-face, 1 = edge-edge, core.py:75-79).

Planted collisions (config 1) follow the reference's exact construction
(pkg/src/ccdkit/dataset.py:457-461, 484-529): contact time, barycentric
coordinates, contact geometry and velocities all on dyadic grids, endpoints
x0 = C - t* D and x1 = C + (1 - t*) D, so every coordinate is exact in
binary64 and (t*, u, v) is an exact root.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BLOCK = 1 << 16
SEED_BASE = 2009_13349

VF, EE = 0, 1


@dataclass
class Workload:
    """A batch of queries plus the solver configuration they run under."""

    points: np.ndarray  # [n, 8, 3] f64
    kind: np.ndarray  # [n] u8
    delta: float | np.ndarray = 1e-6
    max_checks: int | np.ndarray = 1_000_000
    separation: float = 0.0
    t_max: float = 1.0
    planted_t: np.ndarray | None = None  # exact root time for planted queries, else nan
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.points.shape[0])

    def slice(self, lo: int, hi: int) -> "Workload":
        def cut(x):
            return x[lo:hi] if isinstance(x, np.ndarray) else x

        return Workload(self.points[lo:hi], self.kind[lo:hi], cut(self.delta),
                        cut(self.max_checks), self.separation, self.t_max,
                        cut(self.planted_t), dict(self.meta))


CONFIGS = {
    0: dict(name="c0_vf_uniform", n=10_000),
    1: dict(name="c1_mixed_planted", n=1_000_000),
    2: dict(name="c2_degenerate", n=200_000),
    3: dict(name="c3_sim", n=50_000_000),
    4: dict(name="c4_minsep_sweep", n=10_000_000, separations=(0.0, 1e-16, 1e-8, 1e-5, 1e-3)),
}


def _rng(config: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE + config, block])))


# --------------------------------------------------------------------------
# config 0: uniform vertex-face


def _uniform_block(rng, m):
    p0 = rng.random((m, 4, 3))
    p1 = p0 + (rng.random((m, 4, 3)) - 0.5)
    return np.concatenate([p0, p1], axis=1)


def _block_c0(rng, m):
    pts = _uniform_block(rng, m)
    return pts, np.zeros(m, np.uint8), np.full(m, np.nan)


# --------------------------------------------------------------------------
# config 1: mixed, half planted


def _grid(rng, lo, hi, bits, shape):
    """Uniform draw on the 2^-bits grid of [lo, hi] (exact binary64 values)."""
    s = 1 << bits
    return rng.integers(int(lo * s), int(hi * s), size=shape, endpoint=True) / s


def _planted(rng, m, kind):
    """Exact-root queries: x0 = C - t* D, x1 = C + (1 - t*) D (dataset.py:457-461)."""
    tk = rng.integers(1, (1 << 20) - 1, size=m, endpoint=True)
    tstar = tk / float(1 << 20)
    a = rng.integers(0, 1024, size=m, endpoint=True)
    b = rng.integers(0, 1024, size=m, endpoint=True)
    u = np.empty(m)
    v = np.empty(m)
    C = np.empty((m, 4, 3))
    vf = kind == VF
    # vertex-face: (u, v) uniform over the triangle u + v <= 1
    flip = vf & (a + b > 1024)
    a = np.where(flip, 1024 - a, a)
    b = np.where(flip, 1024 - b, b)
    u[:] = a / 1024.0
    v[:] = b / 1024.0
    tri = _grid(rng, 0.0, 1.0, 10, (m, 3, 3))
    cp_vf = (1.0 - u - v)[:, None] * tri[:, 0] + u[:, None] * tri[:, 1] + v[:, None] * tri[:, 2]
    # edge-edge: first edge a1->a2, second edge through the contact point
    a1 = _grid(rng, 0.0, 1.0, 10, (m, 3))
    da = _grid(rng, -0.5, 0.5, 10, (m, 3))
    bd = _grid(rng, -0.5, 0.5, 10, (m, 3))
    a2 = a1 + da
    cp_ee = (1.0 - u)[:, None] * a1 + u[:, None] * a2
    b1 = cp_ee - v[:, None] * bd
    b2 = b1 + bd
    C[vf, 0] = cp_vf[vf]
    C[vf, 1:] = tri[vf]
    ee = ~vf
    C[ee, 0] = a1[ee]
    C[ee, 1] = a2[ee]
    C[ee, 2] = b1[ee]
    C[ee, 3] = b2[ee]
    D = _grid(rng, -0.5, 0.5, 10, (m, 4, 3))
    x0 = C - tstar[:, None, None] * D
    x1 = C + (1.0 - tstar)[:, None, None] * D
    return np.concatenate([x0, x1], axis=1), tstar


def _block_c1(rng, m):
    # exact halves per block: kind and planted flag from a shuffled pattern
    pat = rng.permutation(m)
    kind = (pat % 2).astype(np.uint8)
    planted = ((pat // 2) % 2).astype(bool)
    pts = _uniform_block(rng, m)
    pp, tstar = _planted(rng, m, kind)
    pts[planted] = pp[planted]
    pt = np.where(planted, tstar, np.nan)
    return pts, kind, pt


# --------------------------------------------------------------------------
# config 2: degenerate lattice families


def _lat(rng, shape, lo=-8, hi=8):
    return rng.integers(lo, hi, size=shape, endpoint=True) / 8.0


def _axis_frame(rng, m):
    """Random axis permutation + signs, to orient planar families."""
    perm = np.argsort(rng.random((m, 3)), axis=1)
    sign = np.where(rng.random((m, 3)) < 0.5, -1.0, 1.0)
    return perm, sign


def _orient(pts, perm, sign):
    out = np.take_along_axis(pts, np.broadcast_to(perm[:, None, :], pts.shape), axis=2)
    return out * sign[:, None, :]


def _block_c2(rng, m):
    fam = rng.integers(0, 7, size=m)
    pts = np.zeros((m, 8, 3))
    kind = np.zeros(m, np.uint8)
    # canonical frame: the face / edges lie in the plane z = zc; oriented below
    zc = _lat(rng, m, -4, 4)
    x0 = _lat(rng, m, -8, 2)
    y0 = _lat(rng, m, -8, 2)
    ea = rng.integers(1, 6, size=m) / 8.0
    eb = rng.integers(1, 6, size=m) / 8.0
    tri = np.stack([
        np.stack([x0, y0, zc], -1),
        np.stack([x0 + ea, y0, zc], -1),
        np.stack([x0, y0 + eb, zc], -1),
    ], 1)  # [m,3,3]
    # lattice point on the closed triangle: (x0 + i/8, y0 + j/8), i/ea8 + j/eb8 <= 1
    ia = np.floor(rng.random(m) * (ea * 8 + 1))
    jb = np.floor(rng.random(m) * (eb * 8 + 1) * (1 - ia / (ea * 8)))
    on_face = np.stack([x0 + ia / 8, y0 + jb / 8, zc], -1)
    drop = _lat(rng, (m, 3), -8, 8)
    still = np.zeros((m, 3))

    def vf(i, p0, p1, t0, t1):
        pts[i, 0] = p0[i]
        pts[i, 1:4] = t0[i]
        pts[i, 4] = p1[i]
        pts[i, 5:8] = t1[i]
        kind[i] = VF

    def ee(i, a0, a1, b0, b1, c0, c1, d0, d1):
        pts[i, 0], pts[i, 1], pts[i, 2], pts[i, 3] = a0[i], b0[i], c0[i], d0[i]
        pts[i, 4], pts[i, 5], pts[i, 6], pts[i, 7] = a1[i], b1[i], c1[i], d1[i]
        kind[i] = EE

    tri_mv = tri + _lat(rng, (m, 1, 3), -2, 2) * (rng.random((m, 1, 1)) < 0.5)
    # 0: vertex touching the face at t0, then moving off along a lattice direction
    i = fam == 0
    vf(i, on_face, on_face + drop, tri, tri_mv)
    # 1: vertex sliding within the face plane (everything coplanar throughout)
    i = fam == 1
    start = np.stack([_lat(rng, m), _lat(rng, m), zc], -1)
    end = np.stack([_lat(rng, m), _lat(rng, m), zc], -1)
    vf(i, start, end, tri, tri)
    # 2: parallel edges (same direction), second edge translating across the first
    i = fam == 2
    d = np.stack([ea, eb * (rng.random(m) < 0.5), still[:, 0]], -1)
    a0 = tri[:, 0]
    off0 = np.stack([_lat(rng, m, -4, 4), _lat(rng, m, -4, 4), _lat(rng, m, -4, 4)], -1)
    off1 = np.stack([_lat(rng, m, -4, 4), _lat(rng, m, -4, 4), _lat(rng, m, -4, 4)], -1)
    ee(i, a0, a0, a0 + d, a0 + d, a0 + off0, a0 + off1, a0 + off0 + d, a0 + off1 + d)
    # 3: collinear edges sliding along their common line
    i = fam == 3
    dx = np.stack([ea, still[:, 0], still[:, 0]], -1)
    s0 = np.stack([_lat(rng, m, -8, 8), still[:, 0], still[:, 0]], -1) + a0 * np.array([0, 1, 1])
    s1 = np.stack([_lat(rng, m, -8, 8), still[:, 0], still[:, 0]], -1) + a0 * np.array([0, 1, 1])
    ee(i, a0, a0, a0 + dx, a0 + dx, s0, s1, s0 + dx, s1 + dx)
    # 4: vertex on a triangle edge or corner at t0, sweeping through the plane
    i = fam == 4
    w = rng.integers(0, 3, size=m)
    corner = tri[np.arange(m), w]
    mid_edge = np.stack([x0 + np.floor(rng.random(m) * (ea * 8 + 1)) / 8, y0, zc], -1)
    pv = np.where((rng.random(m) < 0.5)[:, None], corner, mid_edge)
    through = pv + np.stack([still[:, 0], still[:, 0], _lat(rng, m, -8, 8)], -1)
    vf(i, pv - (through - pv) * 0.0, through, tri, tri)
    # 5: zero-length motion (t1 == t0), VF or EE, random lattice geometry
    i5 = fam == 5
    g0 = _lat(rng, (m, 4, 3))
    is_vf5 = rng.random(m) < 0.5
    i = i5 & is_vf5
    vf(i, g0[:, 0], g0[:, 0], g0[:, 1:4], g0[:, 1:4])
    i = i5 & ~is_vf5
    ee(i, g0[:, 0], g0[:, 0], g0[:, 1], g0[:, 1], g0[:, 2], g0[:, 2], g0[:, 3], g0[:, 3])
    # 6: near-misses: descend onto the face / edge and stop 2^-40 short
    i6 = fam == 6
    tiny = 2.0 ** -40
    above = on_face + np.stack([still[:, 0], still[:, 0], _lat(rng, m, 1, 8)], -1)
    short = on_face + np.stack([still[:, 0], still[:, 0], np.full(m, tiny)], -1)
    is_vf6 = rng.random(m) < 0.5
    i = i6 & is_vf6
    vf(i, above, short, tri, tri)
    i = i6 & ~is_vf6
    e2 = np.stack([still[:, 0], eb, still[:, 0]], -1)
    b_lo = tri[:, 0] - e2 * 0.5
    ee(i, above - dx * 0.5, short - dx * 0.5, above + dx * 0.5, short + dx * 0.5,
       b_lo, b_lo, b_lo + e2, b_lo + e2)
    perm, sign = _axis_frame(rng, m)
    pts = _orient(pts, perm, sign)
    pts = np.clip(pts, -1.0, 1.0 + 2.0 ** -39)
    delta = rng.choice(np.array([1e-4, 1e-6, 1e-8]), size=m)
    mc = rng.choice(np.array([1_000, 1_000_000], np.int64), size=m)
    return pts, kind, np.full(m, np.nan), delta, mc


# --------------------------------------------------------------------------
# config 3/4: simulation-shaped


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _block_c3(rng, m):
    kind = (rng.random(m) < 0.2).astype(np.uint8)  # 80% VF / 20% EE
    h = 1e-2
    c = rng.uniform(-1.0, 1.0, (m, 3))
    # vertex-face: triangle with edges ~h around c; partner offset along the normal
    e1 = _unit(rng.normal(size=(m, 3)))
    tmp = _unit(rng.normal(size=(m, 3)))
    nrm = _unit(np.cross(e1, tmp))
    e2 = _unit(np.cross(nrm, e1))
    ang = rng.uniform(np.pi / 3 - 0.3, np.pi / 3 + 0.3, m)
    v1 = c - h / 3 * (e1 + (np.cos(ang)[:, None] * e1 + np.sin(ang)[:, None] * e2))
    v2 = v1 + h * e1
    v3 = v1 + h * (np.cos(ang)[:, None] * e1 + np.sin(ang)[:, None] * e2)
    cen = (v1 + v2 + v3) / 3
    p = cen + rng.normal(0.0, 1e-3, m)[:, None] * nrm \
        + rng.normal(0.0, 5e-3, m)[:, None] * e1 + rng.normal(0.0, 5e-3, m)[:, None] * e2
    # edge-edge: edge through c along e1; partner edge offset along the common normal
    d2 = _unit(rng.normal(size=(m, 3)))
    en = _unit(np.cross(e1, d2))
    q1, q2 = c - h / 2 * e1, c + h / 2 * e1
    mid2 = c + rng.normal(0.0, 1e-3, m)[:, None] * en \
        + rng.normal(0.0, 5e-3, m)[:, None] * e1 + rng.normal(0.0, 5e-3, m)[:, None] * _unit(np.cross(en, e1))
    r1, r2 = mid2 - h / 2 * d2, mid2 + h / 2 * d2
    vf = kind == VF
    P0 = np.where(vf[:, None, None], np.stack([p, v1, v2, v3], 1), np.stack([q1, q2, r1, r2], 1))
    P1 = P0 + rng.normal(0.0, 1e-3, (m, 4, 3))
    return np.concatenate([P0, P1], axis=1), kind, np.full(m, np.nan)


_BLOCKS = {0: _block_c0, 1: _block_c1, 2: _block_c2, 3: _block_c3, 4: _block_c3}


def generate(config: int, start: int = 0, count: int | None = None,
             separation: float | None = None) -> Workload:
    """Queries [start, start+count) of workload ``config`` (0..4).

    Config 4 draws from its own seed stream with config 3's law; pass
    ``separation`` to pick the d of the sweep (default 0).
    """
    if config not in CONFIGS:
        raise ValueError(f"unknown config {config}")
    n_total = CONFIGS[config]["n"]
    if count is None:
        count = n_total - start
    if start < 0 or count < 0:
        raise ValueError("start/count must be >= 0")
    end = start + count
    b0, b1 = start // BLOCK, (end + BLOCK - 1) // BLOCK
    parts = []
    for b in range(b0, b1):
        out = _BLOCKS[config](_rng(config, b), BLOCK)
        lo = max(start - b * BLOCK, 0)
        hi = min(end - b * BLOCK, BLOCK)
        parts.append(tuple(x[lo:hi] for x in out))
    cols = list(zip(*parts)) if parts else []
    pts = np.ascontiguousarray(np.concatenate(cols[0])) if parts else np.zeros((0, 8, 3))
    kind = np.ascontiguousarray(np.concatenate(cols[1])) if parts else np.zeros(0, np.uint8)
    planted = np.concatenate(cols[2]) if parts else np.zeros(0)
    w = Workload(pts, kind, planted_t=planted,
                 meta=dict(config=config, name=CONFIGS[config]["name"], start=start, count=count))
    if config == 2:
        w.delta = np.ascontiguousarray(np.concatenate(cols[3])) if parts else np.zeros(0)
        w.max_checks = np.ascontiguousarray(np.concatenate(cols[4])) if parts else np.zeros(0, np.int64)
    if config == 4:
        w.separation = float(separation or 0.0)
        w.meta["separation"] = w.separation
    return w


def generate_parallel(config: int, start: int = 0, count: int | None = None,
                      separation: float | None = None, workers: int | None = None) -> Workload:
    """``generate`` with the blocks spread over forked worker processes.

    Byte-identical to ``generate`` (every block has its own seed).  Workers
    write straight into a shared anonymous mapping, so a 5e7-query config-3
    set (9.6 GB) takes seconds on a many-core host instead of minutes.  Must
    be called before CUDA is initialised in this process (fork).
    """
    import mmap
    import multiprocessing as mp
    import os

    if config not in CONFIGS:
        raise ValueError(f"unknown config {config}")
    if count is None:
        count = CONFIGS[config]["n"] - start
    workers = workers or len(os.sched_getaffinity(0))
    end = start + count
    b0, b1 = start // BLOCK, (end + BLOCK - 1) // BLOCK
    if workers <= 1 or b1 - b0 <= 2 or config == 2:
        return generate(config, start, count, separation)
    buf_p = mmap.mmap(-1, max(count * 192, 1))
    buf_k = mmap.mmap(-1, max(count, 1))
    buf_t = mmap.mmap(-1, max(count * 8, 1))
    pts = np.frombuffer(buf_p, np.float64, count * 24).reshape(count, 8, 3)
    kind = np.frombuffer(buf_k, np.uint8, count)
    planted = np.frombuffer(buf_t, np.float64, count)

    def run(blocks):
        for b in blocks:
            out = _BLOCKS[config](_rng(config, b), BLOCK)
            lo = max(start - b * BLOCK, 0)
            hi = min(end - b * BLOCK, BLOCK)
            d = b * BLOCK + lo - start
            pts[d:d + hi - lo] = out[0][lo:hi]
            kind[d:d + hi - lo] = out[1][lo:hi]
            planted[d:d + hi - lo] = out[2][lo:hi]

    blocks = list(range(b0, b1))
    ctx = mp.get_context("fork")
    procs = [ctx.Process(target=run, args=(blocks[k::workers],)) for k in range(workers)]
    for p in procs:
        p.start()
    for p in procs:
        p.join()
    if any(p.exitcode != 0 for p in procs):
        raise RuntimeError("workload generation worker failed")
    # (the arrays keep their mappings alive: no copy of the set)
    w = Workload(pts, kind, planted_t=planted,
                 meta=dict(config=config, name=CONFIGS[config]["name"], start=start, count=count))
    if config == 4:
        w.separation = float(separation or 0.0)
        w.meta["separation"] = w.separation
    return w
