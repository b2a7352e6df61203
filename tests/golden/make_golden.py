"""Generate the golden vectors that pin the oracle (and the CUDA path).

Runs the REFERENCE ITSELF -- ccdkit's numba kernel
(pkg/src/ccdkit/_kernel.py:136 solve_kernel, fed by solver._resolve_filters,
pkg/src/ccdkit/solver.py:30-47) -- imported from /root/reference in the build
container, on:

* the KAT geometries of the reference tests (pkg/tests/conftest.py:28-51,
  pkg/tests/test_solver.py:22-35) under the configurations they use,
* the handcrafted battery (pkg/src/ccdkit/dataset.py:295-432) under several
  (delta, m_I, t_max, d) settings,
* seeded samples of the five BASELINE.json workloads
  (paper_2009_13349_b200.workloads), including non-dyadic t_max runs that
  exercise the general stable-order path,

and stores inputs + the full 13-field outputs as compressed .npz fixtures
next to this script.  Run from the repo root:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

The reference does not exist on the GPU box; the committed fixtures travel
instead.
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
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ccdkit  # noqa: F401
    from ccdkit import _kernel, inclusion
    from ccdkit.core import QueryKind
    return _kernel, inclusion, QueryKind


def _solve_chunk(args):
    pts, kind, delta, mc, sep, tmax = args
    _kernel, inclusion, QueryKind = _ref()
    out = np.zeros((len(pts), 13))
    for i in range(len(pts)):
        k = QueryKind(int(kind[i]))
        try:
            f = inclusion.compute_filters(k, inclusion.compute_gamma(pts[i]), float(sep[i]))
        except ValueError:
            out[i] = np.nan
            out[i, 0] = 2.0
            continue
        r = _kernel.solve_kernel(pts[i, :4].copy(), pts[i, 4:].copy(), int(kind[i]),
                                 float(tmax[i]), float(delta[i]), int(mc[i]), float(sep[i]),
                                 f.eps[0], f.eps[1], f.eps[2])
        out[i] = np.array(r, dtype=np.float64)
    return out


def run_reference(pts, kind, delta, mc, sep, tmax, procs=None):
    n = len(pts)
    b = lambda x, dt: np.broadcast_to(np.asarray(x, dtype=dt), (n,)).copy()
    kind, delta, mc, sep, tmax = (b(kind, np.uint8), b(delta, np.float64), b(mc, np.int64),
                                  b(sep, np.float64), b(tmax, np.float64))
    procs = procs or len(os.sched_getaffinity(0))
    # interleaved chunks balance the heavy tail
    idx = [np.arange(i, n, procs * 4) for i in range(procs * 4)]
    jobs = [(pts[j], kind[j], delta[j], mc[j], sep[j], tmax[j]) for j in idx]
    with mp.get_context("spawn").Pool(procs) as pool:
        outs = pool.map(_solve_chunk, jobs)
    out = np.zeros((n, 13))
    for j, o in zip(idx, outs):
        out[j] = o
    return dict(points=pts, kind=kind, delta=delta, max_checks=mc, separation=sep,
                t_max=tmax, status=out[:, 0].astype(np.uint8), toi=out[:, 1], tol=out[:, 2],
                codom=out[:, 3], checks=out[:, 4].astype(np.int64),
                early=out[:, 5].astype(np.uint8), witness=out[:, 6:12],
                level=out[:, 12].astype(np.int32))


TRI = ((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))


def kat_set():
    """Reference-test geometries x the configurations their tests use."""
    vf_vertical = [(0.3, 0.3, 1.0), *TRI, (0.3, 0.3, -1.0), *TRI]
    vf_offset = [(0.0, 0.0, 10.0), *TRI, (0.0, 0.0, 10.0), *TRI]
    ee_cross = [(0.0, 0.0, 1.0), (1.0, 1.0, 1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0),
                (0.0, 0.0, -1.0), (1.0, 1.0, -1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)]
    hourglass = [(0.1, 0.1, 0.1), (0.0, 0.0, 1.0), (1.0, 0.0, 1.0), (0.0, 1.0, 1.0),
                 (0.1, 0.1, 0.1), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)]
    touch0 = [(0.3, 0.3, 0.0), *TRI, (0.3, 0.3, -1.0), *TRI]
    near = lambda g: [(0.3, 0.3, 1.0), *TRI, (0.3, 0.3, g), *TRI]
    rows = [
        ("vf_vertical", vf_vertical, 0, 1e-6, 1_000_000, 0.0, 1.0),
        ("vf_offset_miss", vf_offset, 0, 1e-6, 1_000_000, 0.0, 1.0),
        ("ee_crossing", ee_cross, 1, 1e-6, 1_000_000, 0.0, 1.0),
        ("hourglass", hourglass, 0, 1e-6, 1_000_000, 0.0, 1.0),
        ("touch_t0", touch0, 0, 1e-6, 1_000_000, 0.0, 1.0),
        ("near_1e-8", near(1e-8), 0, 1e-6, 1_000_000, 0.0, 1.0),
        ("near_1e-12", near(1e-12), 0, 1e-6, 1_000_000, 0.0, 1.0),
        ("near_1e-16", near(1e-16), 0, 1e-6, 1_000_000, 0.0, 1.0),
        ("vf_vertical_tmax0.3", vf_vertical, 0, 1e-6, 1_000_000, 0.0, 0.3),
        ("vf_vertical_mI5", vf_vertical, 0, 1e-6, 5, 0.0, 1.0),
        ("vf_vertical_d0.1", vf_vertical, 0, 1e-6, 1_000_000, 0.1, 1.0),
        ("vf_vertical_d1e-30", vf_vertical, 0, 1e-6, 1_000_000, 1e-30, 1.0),
        ("vf_vertical_delta1e-2", vf_vertical, 0, 1e-2, 1_000_000, 0.0, 1.0),
        ("ee_crossing_tmax0.75", ee_cross, 1, 1e-6, 1_000_000, 0.0, 0.75),
        ("vf_vertical_mI1", vf_vertical, 0, 1e-6, 1, 0.0, 1.0),
        ("vf_vertical_mI2", vf_vertical, 0, 1e-6, 2, 0.0, 1.0),
        ("ee_crossing_mI7", ee_cross, 1, 1e-6, 7, 0.0, 1.0),
        ("hourglass_tmax0.7", hourglass, 0, 1e-6, 1_000_000, 0.0, 0.7),
        ("vf_offset_d0.5", vf_offset, 0, 1e-6, 1_000_000, 0.5, 1.0),
        ("vf_vertical_d2_error", vf_vertical, 0, 1e-6, 1_000_000, 2.0, 1.0),
    ]
    names = [r[0] for r in rows]
    pts = np.array([r[1] for r in rows], dtype=np.float64)
    cols = list(zip(*[r[2:] for r in rows]))
    return names, pts, cols


def handcrafted_set():
    sys.path.insert(0, REF)
    from ccdkit import gen_handcrafted
    hc = gen_handcrafted()
    tags = [lq.tag for lq in hc]
    pts = np.array([lq.query.all_coordinates() for lq in hc])
    kind = np.array([int(lq.kind) for lq in hc], np.uint8)
    truth = np.array([lq.truth for lq in hc])
    return tags, pts, kind, truth


def main():
    sys.path.insert(0, ROOT)
    from paper_2009_13349_b200 import workloads as W

    out = {}
    names, pts, (kind, delta, mc, sep, tmax) = kat_set()
    out["kat"] = dict(run_reference(pts, kind, delta, mc, sep, tmax), names=np.array(names))

    tags, pts, kind, truth = handcrafted_set()
    hc = []
    for (delta, mc, tmax, sep) in [(1e-6, 1_000_000, 1.0, 0.0), (1e-4, 1_000, 1.0, 0.0),
                                    (1e-8, 1_000, 0.75, 0.0), (1e-6, 20_000, 0.3, 0.0),
                                    (1e-6, 5_000, 1.0, 1e-3), (1e-6, 5_000, 0.7, 1e-30)]:
        hc.append(run_reference(pts, kind, delta, mc, sep, tmax))
    out["handcrafted"] = {k: np.concatenate([h[k] for h in hc]) for k in hc[0]}
    out["handcrafted"]["tags"] = np.array(tags * len(hc))
    out["handcrafted"]["truth"] = np.concatenate([truth] * len(hc))

    samples = [
        ("c0", 0, 0, 3000, {}),
        ("c0_tmax0.3", 0, 3000, 1000, dict(t_max=0.3)),
        ("c0_tmax0.7", 0, 4000, 1000, dict(t_max=0.7)),
        ("c1", 1, 0, 3000, {}),
        ("c1_tmax0.6", 1, 3000, 600, dict(t_max=0.6)),
        ("c2", 2, 0, 1500, {}),
        ("c3", 3, 0, 3000, {}),
        ("c4_d1e-16", 4, 0, 600, dict(sep=1e-16)),
        ("c4_d1e-8", 4, 600, 600, dict(sep=1e-8)),
        ("c4_d1e-5", 4, 1200, 200, dict(sep=1e-5)),
        ("c4_d1e-3", 4, 1400, 60, dict(sep=1e-3)),
    ]
    for name, cfg, start, count, over in samples:
        w = W.generate(cfg, start, count, separation=over.get("sep"))
        r = run_reference(w.points, w.kind, w.delta, w.max_checks,
                          over.get("sep", w.separation), over.get("t_max", w.t_max))
        r["planted_t"] = w.planted_t
        out[name] = r
        print(name, "hits", int((r["status"] == 1).sum()), "/", count,
              "mean checks", float(r["checks"].mean()), flush=True)

    for k, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{k}.npz"), **d)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
