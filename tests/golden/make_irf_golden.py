"""Golden vectors for the IRF baseline.

Runs the REFERENCE's own interval root finder, ccdkit.baselines.irf_solve
(pkg/src/ccdkit/baselines.py:123-206, with IntervalScalar :37-106 and
_interval_F :109-120), imported from /root/reference in the build
container, on

* the KAT geometries of the reference tests (pkg/tests/conftest.py,
  pkg/tests/test_baselines.py:47-81) under several (delta, max_checks,
  t_max) settings, including tiny budgets (early returns);
* the handcrafted battery (dataset.py:295-432);
* seeded samples of workload configs 0 and 1 (paper_2009_13349_b200.workloads),

and stores inputs + the 13 result fields (status 1 hit / 0 free / 2 error,
toi = +inf when free) as irf_*.npz next to this script:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_irf_golden.py
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True


def _chunk(args):
    pts, kind, delta, mc, tmax = args
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from ccdkit import Query, QueryKind, irf_solve
    out = np.zeros((len(pts), 13))
    for i in range(len(pts)):
        q = Query(QueryKind(int(kind[i])), tuple(map(tuple, pts[i, :4])),
                  tuple(map(tuple, pts[i, 4:])))
        try:
            r = irf_solve(q, delta=float(delta[i]), max_checks=int(mc[i]), t_max=float(tmax[i]))
        except ValueError:
            out[i] = 0.0
            out[i, 0] = 2.0
            continue
        if r.toi is None:
            out[i] = [0, np.inf, r.achieved_tol, r.codomain_width, r.checks, r.early_terminated,
                      0, 0, 0, 0, 0, 0, 0]
        else:
            w = r.witness
            out[i] = [1, r.toi, r.achieved_tol, r.codomain_width, r.checks, r.early_terminated,
                      *w.t, *w.u, *w.v, w.level]
    return out


def run(pts, kind, delta, mc, tmax, procs=None):
    n = len(pts)
    b = lambda x, dt: np.broadcast_to(np.asarray(x, dtype=dt), (n,)).copy()  # noqa: E731
    kind, delta, mc, tmax = b(kind, np.uint8), b(delta, np.float64), b(mc, np.int64), b(tmax, np.float64)
    procs = procs or len(os.sched_getaffinity(0))
    idx = [np.arange(i, n, procs * 4) for i in range(procs * 4)]
    jobs = [(pts[j], kind[j], delta[j], mc[j], tmax[j]) for j in idx if len(j)]
    with mp.get_context("spawn").Pool(procs) as pool:
        outs = pool.map(_chunk, jobs)
    out = np.zeros((n, 13))
    for j, o in zip([j for j in idx if len(j)], outs):
        out[j] = o
    return dict(points=pts, kind=kind, delta=delta, max_checks=mc, t_max=tmax,
                status=out[:, 0].astype(np.uint8), toi=out[:, 1], tol=out[:, 2],
                codom=out[:, 3], checks=out[:, 4].astype(np.int64),
                early=out[:, 5].astype(np.uint8), witness=out[:, 6:12],
                level=out[:, 12].astype(np.int32))


def main():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, REF)
    from paper_2009_13349_b200 import workloads as W

    with np.load(os.path.join(HERE, "kat.npz")) as g:
        kpts, kkind = g["points"][:8], g["kind"][:8]  # the 8 distinct KAT geometries
    rows = []
    for delta, mc, tmax in ((1e-6, 1_000_000, 1.0), (1e-6, 10, 1.0), (1e-6, 0, 1.0),
                            (1e-6, 1, 1.0), (1e-6, 1_000_000, 0.7), (1e-2, 1_000_000, 1.0),
                            (1e-6, 200, 0.3), (1e-8, 100_000, 1.0)):
        rows.append((kpts, kkind, delta, mc, tmax))
    pts = np.concatenate([r[0] for r in rows])
    cat = lambda k, dt: np.concatenate([np.full(len(r[0]), r[k], dt) if k > 1 else r[1]  # noqa: E731
                                        for r in rows])
    sets = {"irf_kat": (pts, cat(1, np.uint8), cat(2, np.float64), cat(3, np.int64),
                        cat(4, np.float64))}
    with np.load(os.path.join(HERE, "handcrafted.npz")) as g:
        hp, hk = g["points"], g["kind"]
    n_hc = len(hp) // 6 if len(hp) % 6 == 0 else len(hp)
    hp, hk = hp[:n_hc], hk[:n_hc]
    sets["irf_hc"] = (np.concatenate([hp, hp]), np.concatenate([hk, hk]),
                      np.repeat([1e-6, 1e-4], n_hc), np.repeat([20_000, 3_000], n_hc),
                      np.repeat([1.0, 0.75], n_hc))
    for cfg, start, count, mc in ((0, 500, 300, 5_000), (1, 3_000, 300, 5_000)):
        w = W.generate(cfg, start, count)
        sets[f"irf_c{cfg}"] = (w.points, w.kind, 1e-6, mc, 1.0)
    for name, (p, k, d, m, t) in sets.items():
        res = run(np.ascontiguousarray(p, dtype=np.float64), k, d, m, t)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **res)
        print(name, len(p), "hits", int((res["status"] == 1).sum()), "early",
              int(res["early"].sum()), "checks", int(res["checks"].sum()), flush=True)


if __name__ == "__main__":
    main()
