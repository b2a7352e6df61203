"""CPU: the lane tier's algorithm (csrc/tccd_lane.cuh) as a host model, against
the oracle.

The lane tier does not run the reference's loop box by box: it classifies
the two children of a box when the box is refined, stores only the
non-disjoint children, and reconstructs the reference's check count from two
numbers per level -- the count of all children and the visiting rank, among
all of them, of the level's first non-disjoint box -- the rank coming from a
closed form over runs of equal t_lo (after a t split the reference's stable
sort visits, per run, all lower children then all upper children).  This
model restates exactly that in Python floats (IEEE binary64, the reference's
operation order: pkg/src/ccdkit/_kernel.py:44-94, 173-324) and checks

* the closed-form rank against the rank a stable sort of all children gives,
* every result field against the oracle, on samples of configs 3 and 1.

It guards the exactness argument without a GPU; the kernel itself is checked
bit for bit by the -m gpu tests.
"""

import numpy as np
import pytest

import oracle
from paper_2009_13349_b200 import workloads as W

DISJOINT, INTERSECTS, CONTAINED = 0, 1, 2


def _hull_axis(s, e, kind, ax, b):
    tl, th, ul, uh, vl, vh = b
    mn, mx = np.inf, -np.inf
    for t in (tl, th):
        omt = 1.0 - t
        a = omt * s[0][ax] + t * e[0][ax]
        bb = omt * s[1][ax] + t * e[1][ax]
        c = omt * s[2][ax] + t * e[2][ax]
        d = omt * s[3][ax] + t * e[3][ax]
        for u in (ul, uh):
            for v in (vl, vh):
                if kind == 0:
                    val = a - ((1.0 - u - v) * bb + u * c + v * d)
                else:
                    val = ((1.0 - u) * a + u * bb) - ((1.0 - v) * c + v * d)
                mn = min(mn, val)
                mx = max(mx, val)
    return mn, mx


def _classify(s, e, kind, b, eps, sep):
    contained, wb = True, 0.0
    for ax in range(3):
        mn, mx = _hull_axis(s, e, kind, ax, b)
        lo, hi = mn - sep, mx + sep
        if lo > eps[ax] or hi < -eps[ax]:
            return DISJOINT, 0.0
        if not (lo >= -eps[ax] and hi <= eps[ax]):
            contained = False
        wb = max(wb, mx - mn)
    return (CONTAINED if contained else INTERSECTS), wb


def _split_dim(b, kap):
    ct, cu, cv = (b[1] - b[0]) * kap[0], (b[3] - b[2]) * kap[1], (b[5] - b[4]) * kap[2]
    sd, best = 0, ct
    if cu > best:
        sd, best = 1, cu
    if cv > best:
        sd = 2
    return sd


def lane_model(s, e, kind, t_max, delta, eps, sep, max_level_size=4096):
    """(status, toi, tol, codom, checks, witness box, level) by the lane tier's
    scheme, or None when a level outgrows max_level_size (the kernel would
    hand the query over).  Budget events are not modelled (m_I is never
    reached here: the kernel restarts such queries in the light tier)."""
    kap = oracle.kappas(s, e, kind, t_max)
    root = (0.0, t_max, 0.0, 1.0, 0.0, 1.0)
    cls, wb = _classify(s, e, kind, root, eps, sep)
    if cls == DISJOINT:
        return (0, np.inf, 0.0, 0.0, 1, (0.0,) * 6, 0)
    # a level: its non-disjoint boxes in visiting order, each (box, class, wb)
    level, entries = 0, [(root, cls, wb)]
    c_before, n_all, rank_first = 0, 1, 0
    drop = None  # (box, wb, level) of the earliest accepted non-first box
    while True:
        if len(entries) > max_level_size:
            return None
        # every refining box of a (dyadic) level splits along one dimension
        nxt_all = []  # all children in push order: (box, class, wb, run id, is upper)
        runs = []     # per run of equal parent t_lo: refining parents
        for k, (b, cls, wb) in enumerate(entries):
            accept = wb < delta or cls == CONTAINED
            sd = _split_dim(b, kap)
            if not accept:
                lo_, hi_ = (b[0], b[1]) if sd == 0 else ((b[2], b[3]) if sd == 1 else (b[4], b[5]))
                mid = 0.5 * (lo_ + hi_)
                if mid <= lo_ or mid >= hi_:
                    accept = True
            if accept:
                if k == 0:
                    # the level's first non-disjoint box ends the query
                    checks = c_before + rank_first + 1
                    if drop is not None and drop[0][0] < b[0]:
                        db, dwb, dl = drop
                        return (1, db[0], db[1] - db[0], dwb, checks, db, dl)
                    return (1, b[0], b[1] - b[0], wb, checks, b, level)
                if drop is None or b[0] < drop[0][0]:
                    drop = (b, wb, level)
                continue
            if not runs or runs[-1][0] != b[0]:
                runs.append([b[0], 0])
            a, bb = list(b), list(b)
            a[2 * sd + 1] = mid
            bb[2 * sd] = mid
            push_hi = True
            if kind == 0 and sd == 1:
                push_hi = mid + b[4] <= 1.0
            if kind == 0 and sd == 2:
                push_hi = b[2] + mid <= 1.0
            rid = len(runs) - 1 if sd == 0 else 0
            nxt_all.append((tuple(a),) + _classify(s, e, kind, tuple(a), eps, sep) + (rid, False, sd))
            if push_hi:
                nxt_all.append((tuple(bb),) + _classify(s, e, kind, tuple(bb), eps, sep) + (rid, True, sd))
            runs[-1][1] += 1
        c_before += n_all
        n_all = len(nxt_all)
        if n_all == 0 or all(c[1] == DISJOINT for c in nxt_all):
            checks = c_before + n_all
            if drop is not None:
                db, dwb, dl = drop
                return (1, db[0], db[1] - db[0], dwb, checks, db, dl)
            return (0, np.inf, 0.0, 0.0, checks, (0.0,) * 6, 0)
        # the reference's visiting order: stable sort of push order by t_lo
        order = sorted(range(n_all), key=lambda i: nxt_all[i][0][0])
        sort_rank = next(r for r, i in enumerate(order) if nxt_all[i][1] != DISJOINT)
        # the lane tier's closed form for the same rank
        sd_level = nxt_all[0][5]
        if sd_level != 0:
            closed = next(i for i, c in enumerate(nxt_all) if c[1] != DISJOINT)
        else:
            base, closed = 0, None
            for rid, (_, m) in enumerate(runs):
                kids = [c for c in nxt_all if c[3] == rid]
                lows = [c for c in kids if not c[4]]
                ups = [c for c in kids if c[4]]
                jl = next((j for j, c in enumerate(lows) if c[1] != DISJOINT), None)
                ju = next((j for j, c in enumerate(ups) if c[1] != DISJOINT), None)
                if jl is not None:
                    closed = base + jl
                elif ju is not None:
                    closed = base + m + ju
                if closed is not None:
                    break
                base += 2 * m
        assert closed == sort_rank, (closed, sort_rank, level)
        rank_first = closed
        entries = [(nxt_all[i][0], nxt_all[i][1], nxt_all[i][2]) for i in order
                   if nxt_all[i][1] != DISJOINT]
        level += 1


@pytest.mark.parametrize("config,start,count", [(3, 0, 1500), (3, 7_000_000, 1500), (1, 500_000, 120),
                                                 (0, 0, 300)])
def test_lane_model_matches_oracle(config, start, count):
    w = W.generate(config, start, count)
    ref = oracle.solve_batch(w.points, w.kind, 1e-6, 1_000_000, 0.0, 1.0)
    eps_all = np.zeros((w.n, 3))
    n_done = n_hits = 0
    for q in range(w.n):
        pts = w.points[q]
        s, e = pts[:4], pts[4:]
        kind = int(w.kind[q])
        rc = oracle.lib().tccd_oracle_filters(oracle._ptr(np.ascontiguousarray(pts)), kind, 0.0,
                                              oracle._ptr(eps_all[q]))
        assert rc == 1  # (status: ok)
        if int(ref["checks"][q]) > 20_000:
            continue  # (a pure-Python model: keep the deep queries out)
        got = lane_model(s.tolist(), e.tolist(), kind, 1.0, 1e-6, eps_all[q].tolist(), 0.0)
        if got is None:
            continue
        st, toi, tol, codom, checks, box, level = got
        assert st == int(ref["status"][q])
        assert checks == int(ref["checks"][q]), (q, checks, int(ref["checks"][q]))
        if st == 1:
            assert toi == ref["toi"][q] and tol == ref["tol"][q] and codom == ref["codom"][q]
            assert tuple(box) == tuple(ref["witness"][q]) and level == int(ref["level"][q])
            assert int(ref["early"][q]) == 0
            n_hits += 1
        n_done += 1
    assert n_done > 0.8 * w.n
    if config != 0:
        assert n_hits > 0
