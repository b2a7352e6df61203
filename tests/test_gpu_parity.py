"""GPU parity: libtccd (through the C-ABI) vs the reference's outputs.

* every golden set (reference numba outputs, tests/golden/) -- bit-exact on
  all 13 result fields, through both engines (pooled light engine with heavy
  eviction, and the block-per-query engine alone);
* larger seeded samples of the five workloads vs the oracle (which is itself
  pinned to the reference by tests/test_oracle_golden.py);
* the reference's own hot-path test assertions (pkg/tests/test_solver.py)
  re-run on the GPU through the reference-shaped API;
* size-independent properties at full BASELINE sizes.
"""

import math

import numpy as np
import pytest
import torch

import oracle
from conftest import GOLDEN_SETS, assert_same_results, load_golden

pytestmark = pytest.mark.gpu


def _gpu(g, cuda, heavy_only=False, **kw):
    from paper_2009_13349_b200 import solve_batch
    r = solve_batch(torch.from_numpy(np.ascontiguousarray(g["points"])),
                    torch.from_numpy(np.ascontiguousarray(g["kind"])),
                    delta=torch.from_numpy(np.ascontiguousarray(g["delta"])),
                    max_checks=torch.from_numpy(np.ascontiguousarray(g["max_checks"])),
                    separation=torch.from_numpy(np.ascontiguousarray(g["separation"])),
                    t_max=torch.from_numpy(np.ascontiguousarray(g["t_max"])),
                    device=cuda, heavy_only=heavy_only, raise_on_error=False, **kw)
    return {k: v.numpy() for k, v in r.items() if k != "stats"}


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_golden_bit_exact(cuda, name):
    g = load_golden(name)
    assert_same_results(_gpu(g, cuda), g, name)


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_golden_bit_exact_block_engine(cuda, name):
    g = load_golden(name)
    assert_same_results(_gpu(g, cuda, heavy_only=True, heavy_blocks=64), g, name + "/heavy")


def _vs_oracle(w, cuda, sep=None, t_max=None, heavy_only=False):
    from paper_2009_13349_b200 import solve_batch
    sep = w.separation if sep is None else sep
    t_max = w.t_max if t_max is None else t_max
    ref = oracle.solve_batch(w.points, w.kind, w.delta, w.max_checks, sep, t_max)
    got = solve_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind),
                      delta=w.delta if np.isscalar(w.delta) else torch.from_numpy(w.delta),
                      max_checks=w.max_checks if np.isscalar(w.max_checks)
                      else torch.from_numpy(w.max_checks),
                      separation=sep, t_max=t_max, device=cuda, heavy_only=heavy_only,
                      raise_on_error=False)
    assert_same_results({k: v.numpy() for k, v in got.items()}, ref,
                        f"{w.meta['name']}[{w.meta['start']}:+{w.n}]")
    return ref


@pytest.mark.parametrize("config,start,count,kw", [
    (0, 0, 10_000, {}),
    (0, 0, 10_000, dict(t_max=0.3)),
    (0, 0, 10_000, dict(t_max=0.7)),
    (1, 10_000, 20_000, {}),
    (2, 5_000, 3_000, {}),
    (3, 100_000, 50_000, {}),
    (4, 20_000, 30_000, dict(sep=1e-8)),
    (4, 60_000, 300, dict(sep=1e-5)),
    (4, 61_000, 40, dict(sep=1e-3)),
    # non-dyadic t_max on queries whose levels outgrow the light / medium
    # tiers: the general ordering path plus tier handover
    (1, 40_000, 20_000, dict(t_max=0.6)),
    (2, 9_000, 2_000, dict(t_max=0.7)),
    (4, 62_000, 100, dict(sep=1e-5, t_max=0.9)),
])
def test_workload_samples_vs_oracle(cuda, config, start, count, kw):
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, start, count, separation=kw.get("sep"))
    _vs_oracle(w, cuda, sep=kw.get("sep"), t_max=kw.get("t_max"))


@pytest.mark.parametrize("config,start,count", [(0, 3_000, 20_000), (1, 70_000, 20_000),
                                                (2, 12_000, 1_500)])
def test_mixed_dyadic_and_general_t_max(cuda, config, start, count):
    """Per-query t_max mixing powers of two (closed-form order) and other
    values (general merge order) in one batch, so segments of both kinds sit
    next to each other in every level list."""
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, start, count)
    rng = np.random.default_rng(config + 77)
    t_max = rng.choice(np.array([1.0, 0.5, 0.25, 0.3, 0.7, 0.9]), count)
    _vs_oracle(w, cuda, t_max=t_max)


@pytest.mark.parametrize("config,start,count,frac", [(1, 90_000, 40_000, 0.03),
                                                     (1, 130_000, 40_000, 0.2),
                                                     (3, 200_000, 100_000, 0.01)])
def test_compact_format_switches(cuda, config, start, count, frac):
    """Mostly dyadic t_max with a few non-dyadic queries: a group stores its
    level arrays as lower corners only in rounds whose resident queries are
    all dyadic, so admitting a non-dyadic query (or finishing the last one)
    switches the format between rounds, with deferred and handed-over levels
    read across the switch."""
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(config, start, count)
    rng = np.random.default_rng(config + 91)
    t_max = rng.choice(np.array([1.0, 0.5, 0.25]), count)
    odd = rng.random(count) < frac
    t_max[odd] = rng.choice(np.array([0.3, 0.7, 0.9]), int(odd.sum()))
    _vs_oracle(w, cuda, t_max=t_max)


def test_extreme_coordinates_nan_path(cuda):
    """Coordinates near the top of the binary64 range: lerps and corner values
    overflow to +-inf and inf - inf = NaN.  The reference's hull ignores NaN
    (its `val < mn` updates fail), which the non-tame classify path must
    reproduce exactly; the tame fast path is only used below 1e300."""
    from paper_2009_13349_b200 import solve_batch
    rng = np.random.default_rng(5)
    n = 3000
    scale = np.where(rng.random(n) < 0.5, 1.6e308, 1e301)[:, None, None]
    pts = (rng.random((n, 8, 3)) - 0.5) * 2 * scale
    with np.errstate(over="ignore"):  # the multiply saturates to +-inf on purpose
        pts[::7] = np.clip(pts[::7] * 1e10, -1.7e308, 1.7e308)
    kind = (rng.random(n) < 0.5).astype(np.uint8)
    # auto filters would give eps = inf (gamma^3 overflows) and settle every
    # query at the root; a caller FilterEps (not re-validated, solver.py:44-46)
    # with finite eps drives the search through NaN-producing boxes
    for eps in (None, (1e290, 1e290, 1e290), (1e300, 1e-15, 1e305)):
        ref = oracle.solve_batch(pts, kind, 1e-6, 10_000, eps=eps)
        got = solve_batch(torch.from_numpy(pts), torch.from_numpy(kind), max_checks=10_000,
                          eps=eps, device=cuda, raise_on_error=False)
        assert_same_results({k: v.numpy() for k, v in got.items()}, ref, f"extreme eps={eps}")


def test_heavy_tail_sample_block_engine(cuda):
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(2, 0, 400)
    _vs_oracle(w, cuda, heavy_only=True)


# --- the reference's own solver assertions (pkg/tests/test_solver.py) -------

TRI = ((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))


def _q(kind, p0, p1):
    from paper_2009_13349_b200 import Query, QueryKind
    return Query(QueryKind(kind), p0, p1)


def test_reference_solver_assertions(cuda):
    from paper_2009_13349_b200 import (CCDResult, QueryKind, SolverConfig, compute_filters,
                                       compute_gamma, solve)
    vf_vertical = _q(0, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    vf_offset = _q(0, ((0.0, 0.0, 10.0),) + TRI, ((0.0, 0.0, 10.0),) + TRI)
    ee = _q(1, ((0.0, 0.0, 1.0), (1.0, 1.0, 1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)),
            ((0.0, 0.0, -1.0), (1.0, 1.0, -1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)))
    res = solve(vf_vertical)
    assert res.colliding and res.toi <= 0.5 and 0.5 - res.toi < 2e-6
    assert res.achieved_tol <= 1e-6 and not res.early_terminated
    assert solve(vf_offset) == CCDResult(None, None, 0.0, 0.0, 1, False)
    r = solve(ee)
    assert r.colliding and r.toi <= 0.5 and 0.5 - r.toi < 2e-6
    hour = _q(0, ((0.1, 0.1, 0.1), (0.0, 0.0, 1.0), (1.0, 0.0, 1.0), (0.0, 1.0, 1.0)),
              ((0.1, 0.1, 0.1), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)))
    hr = solve(hour)
    from fractions import Fraction
    HT = Fraction(32425917317067571, 36028797018963968)
    assert hr.colliding and Fraction(hr.toi) <= HT and HT - Fraction(hr.toi) < Fraction(1, 10**4)
    touch = _q(0, ((0.3, 0.3, 0.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    assert solve(touch).toi == 0.0
    assert solve(vf_vertical) == solve(vf_vertical)
    near = lambda g: _q(0, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, g),) + TRI)
    assert solve(near(1e-8)).toi is None and solve(near(1e-12)).toi is None
    assert solve(near(1e-16)).colliding
    assert solve(vf_vertical, SolverConfig(t_max=0.3)).toi is None
    b = solve(vf_vertical, SolverConfig(max_checks=5))
    assert b.early_terminated and b.checks <= 5 and b.toi is not None and b.toi <= 0.5
    d = solve(vf_vertical, SolverConfig(separation=0.1))
    assert d.colliding and d.toi <= 0.45 and 0.45 - d.toi <= d.achieved_tol
    gamma = compute_gamma(vf_vertical.all_coordinates())
    manual = SolverConfig(filters=compute_filters(QueryKind.VERTEX_FACE, gamma))
    assert solve(vf_vertical, manual) == solve(vf_vertical)
    with pytest.raises(ValueError):
        solve(vf_vertical, SolverConfig(filters=compute_filters(QueryKind.EDGE_EDGE, (1, 1, 1))))
    with pytest.raises(ValueError):
        solve(vf_vertical, SolverConfig(
            filters=compute_filters(QueryKind.VERTEX_FACE, (1, 1, 1), separation=0.5)))
    with pytest.raises(TypeError):
        solve(vf_vertical, SolverConfig(filters=(1e-15, 1e-15, 1e-15)))
    with pytest.raises(ValueError):
        solve(vf_vertical, SolverConfig(separation=2.0))  # d >= gamma


def test_solve_kernel_drop_in(cuda):
    from paper_2009_13349_b200 import solve_kernel
    g = load_golden("kat")
    for i in range(len(g["kind"])):
        if g["status"][i] >= 2:
            continue
        pts = g["points"][i]
        from test_oracle_golden import oracle_eps
        eps = oracle_eps(pts, int(g["kind"][i]), float(g["separation"][i]))
        args = (pts[:4], pts[4:], int(g["kind"][i]), g["t_max"][i], g["delta"][i],
                int(g["max_checks"][i]), g["separation"][i], *eps)
        assert solve_kernel(*args) == oracle.solve_kernel(*args)


def test_batch_edge_cases(cuda):
    from paper_2009_13349_b200 import solve_batch
    empty = solve_batch(torch.zeros((0, 8, 3), dtype=torch.float64), 0, device=cuda)
    assert empty["status"].numel() == 0
    g = load_golden("c0")
    pts = torch.from_numpy(g["points"][:64].copy())
    bad = pts.clone()
    bad[3, 2, 1] = float("nan")
    r = solve_batch(bad, 0, device=cuda, raise_on_error=False)
    assert int(r["status"][3]) == 3 and math.isinf(float(r["toi"][3]))
    with pytest.raises(ValueError):
        solve_batch(bad, 0, device=cuda)
    with pytest.raises(ValueError):
        solve_batch(pts, 0, delta=0.0, device=cuda)
    with pytest.raises(ValueError):
        solve_batch(pts, 0, t_max=1.5, device=cuda)
    # per-query invalid parameter -> status 4 on that query only
    mc = torch.full((64,), 1000, dtype=torch.int64)
    mc[5] = 0
    r = solve_batch(pts, 0, max_checks=mc, device=cuda, raise_on_error=False)
    assert int(r["status"][5]) == 4 and int((r["status"] >= 2).sum()) == 1
    # device-resident inputs give identical results to host inputs
    rd = solve_batch(pts.to(cuda), torch.zeros(64, dtype=torch.uint8, device=cuda), device=cuda)
    rh = solve_batch(pts, 0, device=cuda)
    for k in rh:
        assert torch.equal(rd[k].cpu(), rh[k])


def test_shard_invariance(cuda):
    """Results do not depend on how a batch is split (multi-GPU sharding)."""
    from paper_2009_13349_b200 import shard_bounds, solve_batch
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(1, 0, 8192)
    full = solve_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind), device=cuda)
    for world in (2, 3, 8):
        parts = []
        for r in range(world):
            lo, hi = shard_bounds(w.n, world, r)
            parts.append(solve_batch(torch.from_numpy(w.points[lo:hi]),
                                     torch.from_numpy(w.kind[lo:hi]), device=cuda))
        for k in full:
            assert torch.equal(torch.cat([p[k] for p in parts]), full[k])


def test_full_config1_properties(cuda):
    """Full-size config 1 (10^6 queries): every planted root is reported with a
    conservative toi (toi <= t*, exact rational comparison is exact here
    because both are binary64), results are deterministic run to run, and a
    seeded stratified subsample matches the oracle bit for bit."""
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W
    w = W.generate(1)
    pts = torch.from_numpy(w.points).to(cuda)
    kind = torch.from_numpy(w.kind).to(cuda)
    r1 = solve_batch(pts, kind, device=cuda)
    r2 = solve_batch(pts, kind, device=cuda)
    for k in r1:
        assert torch.equal(r1[k], r2[k])
    planted = ~np.isnan(w.planted_t)
    st = r1["status"].cpu().numpy()
    toi = r1["toi"].cpu().numpy()
    assert (st[planted] == 1).all(), "a planted root was missed (false negative)"
    assert (toi[planted] <= w.planted_t[planted]).all(), "toi after the planted root"
    idx = np.random.default_rng(7).choice(w.n, 4000, replace=False)
    idx.sort()
    sub = {k: v.cpu().numpy()[idx] for k, v in r1.items()}
    ref = oracle.solve_batch(w.points[idx], w.kind[idx])
    assert_same_results(sub, ref, "config1 subsample")


# --- §8(f) row 3: the benchmark harness and CLI on the GPU batch -------------

@pytest.mark.parametrize("name,tag", [("handcrafted", "vf"), ("handcrafted", "ee"),
                                      ("adv", "vf"), ("adv", "ee")])
def test_benchmark_harness_matches_reference(cuda, name, tag):
    """Verdicts and FP/FN/correct/early counts equal those of the reference's
    run_benchmark(..., ("ours",)) on its own dataset files."""
    import os
    from conftest import GOLDEN_DIR
    from paper_2009_13349_b200 import QueryKind
    from paper_2009_13349_b200.benchmark import run_benchmark
    from paper_2009_13349_b200.dataset import parse_queries
    kind = QueryKind.VERTEX_FACE if tag == "vf" else QueryKind.EDGE_EDGE
    g = np.load(os.path.join(GOLDEN_DIR, f"ds_{name}_{tag}.npz"))
    data = parse_queries(os.path.join(GOLDEN_DIR, f"ds_{name}_{tag}.csv"), kind)
    rep = run_benchmark(data, ("irf", "OURS", "ours"), device=cuda)
    assert [m.name for m in rep.methods] == ["ours", "irf"]
    m = rep.method("ours")
    assert np.array_equal(np.array(m.verdicts), g["verdicts"])
    assert (m.fp_count, m.fn_count, m.correct_count, m.early_count) == \
        (int(g["fp"]), int(g["fn"]), int(g["correct"]), int(g["early"]))
    assert sum(m.histogram) == rep.size and rep.queries_per_second > 0
    # the IRF method's verdicts: the oracle's restatement of irf_solve with
    # the config's delta / max_checks / t_max (bench.py:169-175)
    ref = oracle.irf_batch(data.points, data.kind, 1e-6, 1_000_000, 1.0)
    mi = rep.method("irf")
    assert np.array_equal(np.array(mi.verdicts), ref["status"] == 1)
    assert mi.fn_count == 0 and mi.early_count == int(ref["early"].sum())
    with pytest.raises(ValueError):
        run_benchmark(data, ("univariate",), device=cuda)


def test_cli_run_and_fn_guard(cuda, tmp_path):
    import io
    import os
    from conftest import GOLDEN_DIR
    from paper_2009_13349_b200 import cli
    from paper_2009_13349_b200.benchmark import load_report
    out = tmp_path / "r.json"
    rc = cli.main(["run", "--dataset", os.path.join(GOLDEN_DIR, "ds_adv_ee.csv"), "--kind", "ee",
                   "--out", str(out)])
    assert rc == 0 and load_report(out).method("ours").fn_count == 0
    # a mislabeled record (far miss labeled colliding) is an FN: exit 2
    bad = tmp_path / "bad.csv"
    bad.write_text(("0,1,0,1,10,1,1\n" + "0,1,0,1,0,1,1\n" + "1,1,0,1,0,1,1\n" + "0,1,1,1,0,1,1\n") * 2)
    assert cli.main(["run", "--dataset", str(bad), "--kind", "vf", "--format", "csv"]) == 2


def test_non_blocking_host_pipeline(cuda):
    """Back-to-back host-input solves with non_blocking=True (points copied on
    the side stream while the previous batch solves) give the blocking
    results once their ready events complete."""
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W
    ws = [W.generate(1, 200_000 + 30_000 * k, 30_000) for k in range(3)]
    want = [solve_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind), device=cuda)
            for w in ws]
    pinned = [(torch.from_numpy(w.points).pin_memory(), torch.from_numpy(w.kind).pin_memory())
              for w in ws]
    got = [solve_batch(p, k, device=cuda, non_blocking=True) for p, k in pinned]
    for g, r in zip(got, want):
        g["ready"].synchronize()
        for key in ("status", "toi", "checks", "witness", "level"):
            assert torch.equal(g[key], r[key]), key


def test_multi_chunk_batch(cuda):
    """A batch above the library's 2^22-query chunk (BASELINE config 3 is
    5e7 queries): results do not depend on chunking -- the queries around
    the chunk boundary, solved alone and inside the big batch, agree with
    each other and with the oracle."""
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W
    n = (1 << 22) + 50_000
    w = W.generate(3, 0, n)
    pts = torch.from_numpy(w.points).to(cuda)
    kind = torch.from_numpy(w.kind).to(cuda)
    big = solve_batch(pts, kind, device=cuda)
    lo, hi = (1 << 22) - 3_000, (1 << 22) + 3_000
    alone = solve_batch(pts[lo:hi], kind[lo:hi], device=cuda)
    for k in ("status", "toi", "checks", "witness", "level"):
        assert torch.equal(big[k][lo:hi], alone[k]), k
    ref = oracle.solve_batch(w.points[lo:hi], w.kind[lo:hi], w.delta, w.max_checks)
    assert_same_results({k: v[lo:hi].cpu().numpy() for k, v in big.items()}, ref, "chunk edge")
    tail = slice(n - 2_000, n)
    ref = oracle.solve_batch(w.points[tail], w.kind[tail], w.delta, w.max_checks)
    assert_same_results({k: v[tail].cpu().numpy() for k, v in big.items()}, ref, "last chunk")
    # the streaming host path copies and solves chunk by chunk: same results
    hp = torch.from_numpy(w.points).pin_memory()
    hk = torch.from_numpy(w.kind).pin_memory()
    st = solve_batch(hp, hk, device=cuda, non_blocking=True)
    st["ready"].synchronize()
    for k in ("status", "toi", "checks", "witness", "level"):
        assert torch.equal(st[k], big[k].cpu()), k


def test_non_blocking_edge_cases(cuda):
    """The streaming host path with an empty batch, and with per-query host
    parameters (copied on the API's side stream too)."""
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W
    e = solve_batch(torch.zeros((0, 8, 3), dtype=torch.float64).pin_memory(),
                    torch.zeros(0, dtype=torch.uint8).pin_memory(), device=cuda, non_blocking=True)
    e["ready"].synchronize()
    assert e["status"].numel() == 0 and e["toi"].numel() == 0
    w = W.generate(2, 0, 3000)
    mc = np.minimum(w.max_checks, 20_000)
    got = solve_batch(torch.from_numpy(w.points).pin_memory(), torch.from_numpy(w.kind).pin_memory(),
                      delta=torch.from_numpy(w.delta), max_checks=torch.from_numpy(mc),
                      device=cuda, non_blocking=True)
    got["ready"].synchronize()
    ref = oracle.solve_batch(w.points, w.kind, w.delta, mc)
    assert_same_results({k: v.numpy() for k, v in got.items() if k not in ("ready",)}, ref,
                        "non-blocking per-query")
