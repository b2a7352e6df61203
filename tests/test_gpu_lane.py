"""GPU: the lane tier, the group tiers without it, the compacted hit list,
handover-pool restarts and the algorithmic check accounting.

The lane tier (csrc/tccd_lane.cuh) runs the reference's state machine
(pkg/src/ccdkit/_kernel.py:173-324) one query per thread; the group tiers
(csrc/tccd_engine.cuh) run it level-synchronously.  Both must give the
reference's 13 fields bit for bit, alone and together.
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import GOLDEN_SETS, assert_same_results, load_golden

pytestmark = pytest.mark.gpu


def _solve(w, cuda, **kw):
    from paper_2009_13349_b200 import solve_batch
    return solve_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind),
                       delta=w.delta if np.isscalar(w.delta) else torch.from_numpy(w.delta),
                       max_checks=w.max_checks if np.isscalar(w.max_checks)
                       else torch.from_numpy(w.max_checks),
                       separation=w.separation, device=cuda, raise_on_error=False, **kw)


def _np(r):
    return {k: v.numpy() for k, v in r.items() if k in ("status", "toi", "tol", "codom", "checks",
                                                         "early", "witness", "level")}


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_golden_bit_exact_without_lanes(cuda, name):
    from paper_2009_13349_b200 import solve_batch
    g = load_golden(name)
    r = solve_batch(torch.from_numpy(np.ascontiguousarray(g["points"])),
                    torch.from_numpy(np.ascontiguousarray(g["kind"])),
                    delta=torch.from_numpy(np.ascontiguousarray(g["delta"])),
                    max_checks=torch.from_numpy(np.ascontiguousarray(g["max_checks"])),
                    separation=torch.from_numpy(np.ascontiguousarray(g["separation"])),
                    t_max=torch.from_numpy(np.ascontiguousarray(g["t_max"])),
                    device=cuda, raise_on_error=False, lanes=False)
    assert_same_results(_np(r), g, name + "/no-lanes")


@pytest.mark.parametrize("config,start,count,sep", [(0, 0, 10_000, None), (1, 0, 20_000, None),
                                                    (3, 0, 60_000, None), (4, 0, 30_000, 1e-8),
                                                    (2, 0, 3_000, None)])
@pytest.mark.parametrize("lanes", [True, False])
def test_samples_vs_oracle_both_paths(cuda, config, start, count, sep, lanes):
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, start, count, separation=sep)
    ref = oracle.solve_batch(w.points, w.kind, w.delta, w.max_checks, w.separation, w.t_max)
    got = _solve(w, cuda, lanes=lanes)
    assert_same_results(_np(got), ref, f"c{config} lanes={lanes}")


def test_lane_tier_takes_the_shallow_queries(cuda):
    """On simulation-shaped queries the lane tier finishes most survivors of
    the root check; the rest (levels above 128 non-disjoint boxes, and the
    queries still running when the queue runs dry: the lane tier's tail) go to
    the light tier with their current level."""
    from paper_2009_13349_b200 import _lib
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(3, 300_000, 200_000)
    r = _solve(w, cuda, stats=True, outputs=("status", "toi", "checks"))
    st = r["stats"].cpu().numpy()
    entered = st[_lib.STAT_LANE_QUERIES]
    done = st[_lib.STAT_LANE_DONE] + st[_lib.STAT_LANE_DONE + 1]
    ev = st[_lib.STAT_LANE_EVICTED]
    assert entered == done + ev
    assert entered > 0.3 * w.n
    assert ev < 0.25 * entered  # (200k queries: the tail is a large share)
    # with room in the handover pool every eviction carries its level
    assert st[_lib.STAT_LANE_HANDED] == ev and st[_lib.STAT_LANE_WASTED] == 0


@pytest.mark.parametrize("config,count", [(3, 60_000), (1, 12_000)])
def test_lane_tier_small_budgets(cuda, config, count):
    """Per-query budgets from 2 to a few thousand checks: the lane tier has no
    budget events of its own -- a level whose boxes could reach m_I, or a last
    level of disjoint boxes that could, sends the query to the light tier to
    restart (pkg/src/ccdkit/_kernel.py:188-213) -- so budget returns at every
    depth must come out as the reference's."""
    from paper_2009_13349_b200 import _lib, solve_batch
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, 40_000, count)
    rng = np.random.default_rng(17)
    mc = rng.choice(np.array([2, 3, 4, 5, 8, 13, 17, 33, 50, 64, 100, 129, 257, 700, 1500, 4000],
                             dtype=np.int64), size=w.n)
    ref = oracle.solve_batch(w.points, w.kind, w.delta, mc, w.separation, w.t_max)
    got = solve_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind), delta=w.delta,
                      max_checks=torch.from_numpy(mc), separation=w.separation, device=cuda,
                      raise_on_error=False, stats=True)
    st = got.pop("stats").cpu().numpy()
    assert_same_results(_np(got), ref, f"c{config} small budgets")
    assert int(np.asarray(ref["early"]).sum()) > 0          # budget returns happen
    assert st[_lib.STAT_LANE_WASTED] > 0                    # and some were lane restarts


def test_lane_tier_dyadic_t_max_range(cuda):
    """Per-query dyadic t_max from 1 down to subnormal powers of two: the lane
    tier builds its box widths from t_max's exponent field and takes t_max >=
    2^-900 (62 halvings stay normal); smaller ones go to the group tiers.
    Both must match the reference's boxes bit for bit."""
    from paper_2009_13349_b200 import _lib, solve_batch
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(3, 900_000, 40_000)
    exps = np.array([0, -1, -2, -7, -20, -52, -200, -899, -900, -901, -1000, -1022, -1023, -1070])
    tm = np.ldexp(1.0, exps[np.arange(w.n) % len(exps)])
    ref = oracle.solve_batch(w.points, w.kind, w.delta, w.max_checks, w.separation, tm)
    got = solve_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind), delta=w.delta,
                      max_checks=w.max_checks, separation=w.separation, t_max=torch.from_numpy(tm),
                      device=cuda, raise_on_error=False, stats=True)
    st = got.pop("stats").cpu().numpy()
    assert_same_results(_np(got), ref, "dyadic t_max range")
    assert st[_lib.STAT_LANE_QUERIES] > 0
    assert int((np.asarray(ref["status"]) == 1).sum()) > 0


@pytest.mark.parametrize("config,count,kw", [(3, 100_000, {}), (1, 20_000, {}),
                                              (0, 20_000, dict(lanes=False)),
                                              (2, 2_000, {})])
def test_algorithmic_check_accounting(cuda, config, count, kw):
    """Every check of the reference's path is counted exactly once: checks of
    queries decided at the root + lane checks (+ the root check of each lane
    query) + the group tiers' path checks == sum of the reference's checks
    (no handover restarts on these samples)."""
    from paper_2009_13349_b200 import _lib
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, 7_000, count)
    r = _solve(w, cuda, stats=True, outputs=("status", "toi", "checks"), **kw)
    st = r["stats"].cpu().numpy().astype(np.int64)
    checks = r["checks"].numpy()
    assert st[_lib.STAT_RESTARTS] == 0 and st[_lib.STAT_RESTARTS + 1] == 0
    valid = r["status"].numpy() < 2
    root_decided = st[_lib.STAT_PROLOGUE_DONE] - int((~valid).sum())
    # (each lane query's root check is the prologue's: one per query the lane
    # tier finished or handed over)
    total = (root_decided + st[_lib.STAT_LANE_CHECKS] + st[_lib.STAT_LANE_CHECKS + 1]
             + st[_lib.STAT_LANE_DONE] + st[_lib.STAT_LANE_DONE + 1] + st[_lib.STAT_LANE_HANDED]
             + st[_lib.STAT_TIER_CHECKS:_lib.STAT_TIER_CHECKS + 3].sum())
    assert total == int(checks[valid].sum())


def test_tiny_handover_pool_restarts_stay_exact(cuda):
    """A 64-box handover pool: most evictions out of the light and medium
    tiers restart from the root in the next tier; results stay bit-exact and
    the restarts are counted."""
    from paper_2009_13349_b200 import _lib
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(1, 200_000, 6_000)
    ref = oracle.solve_batch(w.points, w.kind, w.delta, w.max_checks, w.separation, w.t_max)
    got = _solve(w, cuda, pool_boxes=64, stats=True)
    st = got.pop("stats").cpu().numpy()
    assert_same_results(_np(got), ref, "pool=64")
    assert st[_lib.STAT_RESTARTS] + st[_lib.STAT_RESTARTS + 1] > 0
    assert st[_lib.STAT_POOL_DEMAND] > 64


def _hit_set(idx, toi):
    return {int(i): float(t) for i, t in zip(np.asarray(idx), np.asarray(toi))}


@pytest.mark.parametrize("config,count", [(3, 200_000), (1, 30_000), (0, 10_000)])
def test_hit_list_equals_dense_results(cuda, config, count):
    """The compacted (index, toi) list is, as a set, exactly the queries with
    status 1 and their toi -- device inputs, host inputs and the
    non-blocking host path (counted copy-out kernel)."""
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, 11_000, count)
    pts, kind = torch.from_numpy(w.points), torch.from_numpy(w.kind)
    dense = solve_batch(pts, kind, device=cuda, hits=True)
    st, toi = dense["status"].numpy(), dense["toi"].numpy()
    want = {int(i): float(toi[i]) for i in np.flatnonzero(st == 1)}
    assert int(dense["hit_count"][0]) == len(want)
    assert _hit_set(dense["hit_index"], dense["hit_toi"]) == want
    assert len(dense["hit_index"]) == len(want)  # host inputs: only live entries came back
    dev = solve_batch(pts.to(cuda), kind.to(cuda), device=cuda, hits=True)
    c = int(dev["hit_count"].item())
    assert c == len(want)
    assert _hit_set(dev["hit_index"][:c].cpu(), dev["hit_toi"][:c].cpu()) == want
    nb = solve_batch(pts, kind, device=cuda, hits=True, non_blocking=True,
                     outputs=("status", "toi"))
    nb["ready"].synchronize()
    c = int(nb["hit_count"][0])
    assert c == len(want)
    assert _hit_set(nb["hit_index"][:c], nb["hit_toi"][:c]) == want


def test_hit_list_over_several_library_chunks(cuda):
    """A batch above one library chunk (2^22 queries): the list accumulates
    across the chunks' launches (the count is not reset per launch)."""
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W
    w = W.generate_parallel(3, 0, (1 << 22) + 300_000)
    pts, kind = torch.from_numpy(w.points), torch.from_numpy(w.kind)
    nb = solve_batch(pts, kind, device=cuda, hits=True, non_blocking=True, outputs=("status", "toi"))
    nb["ready"].synchronize()
    st, toi = nb["status"].numpy(), nb["toi"].numpy()
    c = int(nb["hit_count"][0])
    assert c == int((st == 1).sum())
    got = _hit_set(nb["hit_index"][:c], nb["hit_toi"][:c])
    assert got == {int(i): float(toi[i]) for i in np.flatnonzero(st == 1)}


def test_workspace_shared_across_streams(cuda):
    """Two solves issued on two streams of one device share the cached
    workspace; the second waits for the first (no corruption)."""
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W
    a = W.generate(1, 0, 20_000)
    b = W.generate(3, 0, 200_000)
    pa, ka = torch.from_numpy(a.points).to(cuda), torch.from_numpy(a.kind).to(cuda)
    pb, kb = torch.from_numpy(b.points).to(cuda), torch.from_numpy(b.kind).to(cuda)
    ref_a = {k: v.cpu() for k, v in solve_batch(pa, ka, device=cuda).items()}
    ref_b = {k: v.cpu() for k, v in solve_batch(pb, kb, device=cuda).items()}
    s1, s2 = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            ra = solve_batch(pa, ka, device=cuda, raise_on_error=False)
        with torch.cuda.stream(s2):
            rb = solve_batch(pb, kb, device=cuda, raise_on_error=False)
        torch.cuda.synchronize()
        for k in ref_a:
            assert torch.equal(ra[k].cpu(), ref_a[k]), k
            assert torch.equal(rb[k].cpu(), ref_b[k]), k


def test_solve_kernel_drop_in_reuses_its_scratch(cuda):
    """tccd_solve_kernel caches its device scratch: a loop of calls is fast
    and every call matches the oracle's 13-tuple."""
    import time
    from paper_2009_13349_b200 import solve_kernel
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(3, 0, 200)
    L = oracle.lib()
    import ctypes
    t0 = time.perf_counter()
    for i in range(w.n):
        s, e = w.points[i, :4], w.points[i, 4:]
        eps = np.zeros(3)
        L.tccd_oracle_filters(np.ascontiguousarray(w.points[i]).ctypes.data_as(ctypes.c_void_p),
                              int(w.kind[i]), 0.0, eps.ctypes.data_as(ctypes.c_void_p))
        got = solve_kernel(s, e, int(w.kind[i]), 1.0, 1e-6, 1_000_000, 0.0, *eps)
        ref = oracle.solve_kernel(s, e, int(w.kind[i]), 1.0, 1e-6, 1_000_000, 0.0, *eps)
        assert [np.float64(x).view(np.int64) for x in got] == \
            [np.float64(x).view(np.int64) for x in ref], i
    assert (time.perf_counter() - t0) / w.n < 0.05
