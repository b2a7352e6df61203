"""Host restatement of the reference broad phase (scene.py:225-300) for the
CPU tests: the exact overlap set of inflated swept boxes minus vertex-sharing
pairs, in the reference's order, with numpy.  Test infrastructure only: the
product broad phase is the GPU one (paper_2009_13349_b200/csrc/broad.cu).
"""

import math

import numpy as np

from paper_2009_13349_b200.scene import CandidateSet, TriMeshPair


def _boxes(mesh: TriMeshPair, idx: np.ndarray, inflation: float):
    pts = np.stack((mesh.x0[idx], mesh.x1[idx]))  # (2, m, k, 3), scene.py:195-200
    return pts.min(axis=(0, 2)) - inflation, pts.max(axis=(0, 2)) + inflation


def _overlapping_pairs(alo, ahi, blo, bhi):
    """All (a, b) whose closed boxes overlap on every axis.

    Sweep on x: b sorted by lower x bound; for each a the window is the b
    with blo_x <= ahi_x and blo_x >= alo_x - 2*max_width (a superset of
    bhi_x >= alo_x), then the exact test on all three axes."""
    if len(alo) == 0 or len(blo) == 0:
        return np.zeros((0, 2), dtype=np.int64)
    order = np.argsort(blo[:, 0], kind="stable")
    bstart = blo[order, 0]
    wmax = float(np.max(bhi[:, 0] - blo[:, 0]))
    hi_i = np.searchsorted(bstart, ahi[:, 0], side="right")
    lo_i = np.minimum(np.searchsorted(bstart, alo[:, 0] - 2.0 * wmax, side="left"), hi_i)
    cnt = hi_i - lo_i
    a_rep = np.repeat(np.arange(len(alo)), cnt)
    start = np.repeat(lo_i - (np.cumsum(cnt) - cnt), cnt)
    b_rep = order[np.arange(len(a_rep)) + start]
    ok = np.ones(len(a_rep), dtype=bool)
    for k in range(3):
        ok &= (alo[a_rep, k] <= bhi[b_rep, k]) & (blo[b_rep, k] <= ahi[a_rep, k])
    return np.stack([a_rep[ok], b_rep[ok]], 1).astype(np.int64)


def broad_phase_host(mesh: TriMeshPair, inflation: float = 0.0, device=None) -> CandidateSet:
    """Exactly the pairs of the reference broad phase (scene.py:225-300):
    primitives whose inflated swept boxes overlap, minus pairs that share a
    mesh vertex.  (The reference's grid hash is a superset filter followed by
    the same exact box test, so its result is this set.)"""
    if not (inflation >= 0.0 and math.isfinite(inflation)):
        raise ValueError("inflation must be >= 0 and finite")
    n = mesh.n_vertices
    empty = CandidateSet(np.zeros(0, np.uint8), np.zeros((0, 2), np.int64),
                         np.zeros((0, 8, 3)))
    if n == 0:
        return empty
    vlo, vhi = _boxes(mesh, np.arange(n, dtype=np.intp)[:, None], inflation)
    tris, edges = mesh.triangles, mesh.edges
    kinds, idxs, pts = [], [], []
    if len(tris):
        tlo, thi = _boxes(mesh, tris, inflation)
        pr = _overlapping_pairs(vlo, vhi, tlo, thi)
        keep = ~np.any(tris[pr[:, 1]] == pr[:, 0:1], axis=1)
        pr = pr[keep]
        pr = pr[np.lexsort((pr[:, 1], pr[:, 0]))]
        if len(pr):
            v, t = pr[:, 0], tris[pr[:, 1]]
            vid = np.stack([v, t[:, 0], t[:, 1], t[:, 2]], 1)
            kinds.append(np.zeros(len(pr), np.uint8))
            idxs.append(pr)
            pts.append(np.concatenate([mesh.x0[vid], mesh.x1[vid]], 1))
    if len(edges):
        elo, ehi = _boxes(mesh, edges, inflation)
        pr = _overlapping_pairs(elo, ehi, elo, ehi)
        pr = pr[pr[:, 0] < pr[:, 1]]
        a, b = edges[pr[:, 0]], edges[pr[:, 1]]
        share = (a[:, 0] == b[:, 0]) | (a[:, 0] == b[:, 1]) | (a[:, 1] == b[:, 0]) | \
            (a[:, 1] == b[:, 1])
        pr = pr[~share]
        pr = pr[np.lexsort((pr[:, 1], pr[:, 0]))]
        if len(pr):
            a, b = edges[pr[:, 0]], edges[pr[:, 1]]
            vid = np.stack([a[:, 0], a[:, 1], b[:, 0], b[:, 1]], 1)
            kinds.append(np.ones(len(pr), np.uint8))
            idxs.append(pr)
            pts.append(np.concatenate([mesh.x0[vid], mesh.x1[vid]], 1))
    if not kinds:
        return empty
    return CandidateSet(np.concatenate(kinds), np.concatenate(idxs),
                        np.ascontiguousarray(np.concatenate(pts)))
