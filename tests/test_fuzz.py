"""Property-based parity ("hypothesis fuzz over random /
degenerate / integer-lattice queries"): hypothesis draws batches of queries
from adversarial families, each query with its own delta, max_checks,
separation and t_max, and the CUDA solver (and the IRF baseline) must match
the oracle bit for bit on every field.  Derandomized, so a CI run is
reproducible; every example is one batched solve of 48 queries.
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_same_results

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

N = 48
DELTAS = (1e-2, 1e-4, 1e-6, 1e-8)
BUDGETS = (1, 2, 5, 100, 1000, 20_000)
TMAX = (1.0, 0.5, 0.25, 0.75, 0.3, 0.7)
SEPS = (0.0, 1e-16, 1e-8, 1e-4)


def _family(rng, fam, n):
    """[n, 8, 3] coordinates of one adversarial family."""
    if fam == 0:    # uniform, large motion (config 0 law)
        p0 = rng.random((n, 4, 3))
        p1 = p0 + rng.random((n, 4, 3)) - 0.5
    elif fam == 1:  # integer lattice k / 8: exact ties, touching, collinear
        p0 = rng.integers(-8, 9, (n, 4, 3)) / 8.0
        p1 = rng.integers(-8, 9, (n, 4, 3)) / 8.0
    elif fam == 2:  # coplanar: everything in z = 0 (deep, budget-bound searches)
        p0 = rng.random((n, 4, 3))
        p1 = rng.random((n, 4, 3))
        p0[..., 2] = 0.0
        p1[..., 2] = 0.0
    elif fam == 3:  # tiny motions near contact
        p0 = rng.random((n, 4, 3))
        p0[:, 0] = p0[:, 1:].mean(1) + rng.normal(0, 1e-6, (n, 3))
        p1 = p0 + rng.normal(0, 1e-5, (n, 4, 3))
    elif fam == 4:  # large coordinates (gamma > 1 scales the filters)
        s = 10.0 ** rng.integers(1, 7, (n, 1, 1))
        p0 = (rng.random((n, 4, 3)) - 0.5) * s
        p1 = p0 + (rng.random((n, 4, 3)) - 0.5) * s
    else:           # zero-length motion, some exactly touching at t = 0
        p0 = rng.integers(-4, 5, (n, 4, 3)) / 4.0
        p1 = p0.copy()
    return np.concatenate([p0, p1], axis=1).astype(np.float64)


@st.composite
def batches(draw):
    seed = draw(st.integers(0, 2**32 - 1))
    fams = draw(st.lists(st.integers(0, 5), min_size=1, max_size=3))
    rng = np.random.default_rng(seed)
    parts = [_family(rng, f, N // len(fams) + 1) for f in fams]
    pts = np.ascontiguousarray(np.concatenate(parts)[:N])
    kind = rng.integers(0, 2, N).astype(np.uint8)
    delta = np.asarray(DELTAS)[rng.integers(0, len(DELTAS), N)]
    mc = np.asarray(BUDGETS, dtype=np.int64)[rng.integers(0, len(BUDGETS), N)]
    tmax = np.asarray(TMAX)[rng.integers(0, len(TMAX), N)] if draw(st.booleans()) \
        else np.ones(N)
    sep = np.asarray(SEPS)[rng.integers(0, len(SEPS), N)] if draw(st.booleans()) \
        else np.zeros(N)
    return pts, kind, delta, mc, tmax, sep


FUZZ = settings(max_examples=100, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])


@pytest.mark.gpu
@FUZZ
@given(batches())
def test_fuzz_solver_matches_oracle(cuda, batch):
    from paper_2009_13349_b200 import solve_batch
    pts, kind, delta, mc, tmax, sep = batch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)  # noqa: E731
    got = solve_batch(t(pts), t(kind), delta=t(delta), max_checks=t(mc), separation=t(sep),
                      t_max=t(tmax), device=cuda, raise_on_error=False)
    ref = oracle.solve_batch(pts, kind, delta, mc, sep, tmax)
    assert_same_results({k: v.cpu().numpy() for k, v in got.items()}, ref, "fuzz")


@pytest.mark.gpu
@FUZZ
@given(batches(), st.booleans())
def test_fuzz_irf_matches_oracle(cuda, batch, runs):
    from paper_2009_13349_b200.baselines import irf_batch
    pts, kind, delta, mc, tmax, _ = batch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)  # noqa: E731
    got = irf_batch(t(pts), t(kind), t(delta), t(mc), t(tmax), device=cuda,
                    raise_on_error=False, heavy_only=runs)
    ref = oracle.irf_batch(pts, kind, delta, mc, tmax)
    assert_same_results({k: v.cpu().numpy() for k, v in got.items()}, ref, "fuzz irf")
