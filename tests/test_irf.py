"""IRF baseline on the GPU vs the reference's own
irf_solve outputs (tests/golden/irf_*.npz, make_irf_golden.py) and the
oracle's C restatement (oracle/irf_oracle.c, itself pinned to those
outputs by test_oracle_golden.py)."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_same_results, load_golden

IRF_SETS = ("irf_kat", "irf_hc", "irf_c0", "irf_c1")
TRI = ((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))


def test_irf_solve_rejects_nonpositive_delta():
    from paper_2009_13349_b200 import Query, QueryKind
    from paper_2009_13349_b200.baselines import irf_solve
    q = Query(QueryKind.VERTEX_FACE, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    with pytest.raises(ValueError):
        irf_solve(q, delta=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", IRF_SETS)
def test_gpu_irf_matches_reference(cuda, name):
    from paper_2009_13349_b200.baselines import irf_batch
    g = load_golden(name)
    got = irf_batch(torch.from_numpy(g["points"]), torch.from_numpy(g["kind"]),
                    torch.from_numpy(g["delta"]), torch.from_numpy(g["max_checks"]),
                    torch.from_numpy(g["t_max"]), device=cuda, raise_on_error=False)
    assert_same_results({k: v.numpy() for k, v in got.items()}, g, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", IRF_SETS)
def test_gpu_irf_run_search_matches_reference(cuda, name):
    """Every query through pass 2 (warp per query over runs of equal
    (t_lo, level)), against the reference's own outputs."""
    from paper_2009_13349_b200.baselines import irf_batch
    g = load_golden(name)
    got = irf_batch(torch.from_numpy(g["points"]), torch.from_numpy(g["kind"]),
                    torch.from_numpy(g["delta"]), torch.from_numpy(g["max_checks"]),
                    torch.from_numpy(g["t_max"]), device=cuda, raise_on_error=False,
                    heavy_only=True)
    assert_same_results({k: v.numpy() for k, v in got.items()}, g, name)


@pytest.mark.gpu
@pytest.mark.parametrize("config,start,count,kw", [
    (0, 10_000, 2_000, dict(max_checks=20_000)),
    (3, 50_000, 2_000, dict(max_checks=20_000)),
    (2, 1_000, 300, dict(max_checks=20_000)),
    (0, 30_000, 1_000, dict(max_checks=10_000, t_max=0.7, delta=1e-4)),
])
def test_gpu_irf_run_search_vs_oracle(cuda, config, start, count, kw):
    from paper_2009_13349_b200 import workloads as W
    from paper_2009_13349_b200.baselines import irf_batch
    w = W.generate(config, start, count)
    d, mc, tm = kw.get("delta", 1e-6), kw["max_checks"], kw.get("t_max", 1.0)
    ref = oracle.irf_batch(w.points, w.kind, d, mc, tm)
    got = irf_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind), d, mc, tm, device=cuda,
                    heavy_only=True)
    assert_same_results({k: v.numpy() for k, v in got.items()}, ref, f"irf runs c{config}")


@pytest.mark.gpu
@pytest.mark.parametrize("config,start,count,kw", [
    (0, 10_000, 4_000, dict(max_checks=5_000)),
    (3, 50_000, 8_000, dict(max_checks=5_000)),
    (1, 20_000, 1_500, dict(max_checks=20_000)),   # deep heaps: the second pass
    (0, 30_000, 2_000, dict(max_checks=3_000, t_max=0.7, delta=1e-4)),
    (2, 1_000, 300, dict(max_checks=4_000)),
])
def test_gpu_irf_vs_oracle(cuda, config, start, count, kw):
    from paper_2009_13349_b200 import workloads as W
    from paper_2009_13349_b200.baselines import irf_batch
    w = W.generate(config, start, count)
    d, mc, tm = kw.get("delta", 1e-6), kw["max_checks"], kw.get("t_max", 1.0)
    ref = oracle.irf_batch(w.points, w.kind, d, mc, tm)
    got = irf_batch(torch.from_numpy(w.points), torch.from_numpy(w.kind), d, mc, tm, device=cuda)
    assert_same_results({k: v.numpy() for k, v in got.items()}, ref, f"irf c{config}")


@pytest.mark.gpu
def test_gpu_irf_reference_assertions(cuda):
    """pkg/tests/test_baselines.py:47-81, through the reference-shaped API."""
    from fractions import Fraction

    from paper_2009_13349_b200 import Query, QueryKind, SolverConfig, solve
    from paper_2009_13349_b200.baselines import irf_solve
    vf = Query(QueryKind.VERTEX_FACE, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    miss = Query(QueryKind.VERTEX_FACE, ((0.0, 0.0, 10.0),) + TRI, ((0.0, 0.0, 10.0),) + TRI)
    ee = Query(QueryKind.EDGE_EDGE, ((0.0, 0.0, 1.0), (1.0, 1.0, 1.0), (0.0, 1.0, 0.0),
                                     (1.0, 0.0, 0.0)),
               ((0.0, 0.0, -1.0), (1.0, 1.0, -1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)))
    hour = Query(QueryKind.VERTEX_FACE,
                 ((0.1, 0.1, 0.1), (0.0, 0.0, 1.0), (1.0, 0.0, 1.0), (0.0, 1.0, 1.0)),
                 ((0.1, 0.1, 0.1), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)))
    r = irf_solve(vf)
    assert r.colliding and r.toi <= 0.5 and 0.5 - r.toi < 2e-6
    assert irf_solve(miss).toi is None
    r = irf_solve(ee)
    assert r.colliding and r.toi <= 0.5 and 0.5 - r.toi < 2e-6
    HT = Fraction(32425917317067571, 36028797018963968)
    r = irf_solve(hour)
    assert r.colliding and Fraction(r.toi) <= HT
    r = irf_solve(vf, max_checks=10)
    assert r.early_terminated and r.toi is not None and r.toi <= 0.5
    a, b = solve(vf, SolverConfig(delta=1e-6)), irf_solve(vf, delta=1e-6)
    assert a.colliding == b.colliding and abs(a.toi - b.toi) < 1e-5
    # the oracle agrees field by field on these
    pts = np.stack([q.all_coordinates() for q in (vf, miss, ee, hour)])
    kind = np.array([0, 0, 1, 0], np.uint8)
    ref = oracle.irf_batch(pts, kind, 1e-6, 1 << 22)
    for i, q in enumerate((vf, miss, ee, hour)):
        g = irf_solve(q)
        assert g.checks == ref["checks"][i]
        assert (g.toi is None) == (ref["status"][i] == 0)
