"""GPU: the reference's box-level inclusion API (box_inclusion, kappas) on the
device kernels, against the host scalar definition of F and exact rational
arithmetic -- the assertions of pkg/tests/test_inclusion.py:84-175."""

from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2009_13349_b200 import (DomainBox, Query, QueryKind, box_inclusion, box_inclusion_batch,
                                   eval_F, kappas, kappas_batch)

pytestmark = pytest.mark.gpu

TRI = ((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))


@given(data=st.data(), kind=st.sampled_from([QueryKind.VERTEX_FACE, QueryKind.EDGE_EDGE]))
@settings(max_examples=80, deadline=None, derandomize=True)
def test_box_inclusion_equals_scalar_corner_sweep(cuda, data, kind):
    coord = st.floats(-50.0, 50.0, allow_nan=False, allow_infinity=False)
    pts = lambda: tuple(tuple(data.draw(coord) for _ in range(3)) for _ in range(4))  # noqa: E731
    q = Query(kind, pts(), pts())
    frac = st.floats(0.0, 1.0, allow_nan=False)
    iv = lambda: tuple(sorted((data.draw(frac), data.draw(frac))))  # noqa: E731
    box = DomainBox(iv(), iv(), iv())
    incl = box_inclusion(q, box)
    corners = [tuple(eval_F(q, t, u, v)) for t in box.t for u in box.u for v in box.v]
    for ax in range(3):
        vals = [c[ax] for c in corners]
        assert incl.lo[ax] == min(vals) and incl.hi[ax] == max(vals)


def test_box_inclusion_batch_matches_scalar(cuda):
    rng = np.random.default_rng(3)
    n = 2000
    pts = rng.uniform(-4, 4, (n, 8, 3))
    kind = rng.integers(0, 2, n).astype(np.uint8)
    a = np.sort(rng.random((n, 3, 2)), axis=2)
    boxes = a.reshape(n, 6)
    lo, hi = box_inclusion_batch(pts, kind, boxes)
    for i in range(0, n, 97):
        q = Query(QueryKind(int(kind[i])), [tuple(p) for p in pts[i, :4]], [tuple(p) for p in pts[i, 4:]])
        b = boxes[i]
        corners = [tuple(eval_F(q, t, u, v)) for t in b[0:2] for u in b[2:4] for v in b[4:6]]
        for ax in range(3):
            assert lo[i, ax] == min(c[ax] for c in corners)
            assert hi[i, ax] == max(c[ax] for c in corners)


def test_kappas_known_answers(cuda):
    vertical = Query(QueryKind.VERTEX_FACE, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    assert kappas(vertical) == (6.0, 3.0, 3.0)
    offset = Query(QueryKind.VERTEX_FACE, ((0.0, 0.0, 10.0),) + TRI, ((0.0, 0.0, 10.0),) + TRI)
    kt, ku, kv = kappas(offset)
    assert kt == 0.0 and ku > 0.0 and kv > 0.0


def _rational_kappas(kind, pts):
    """3 x max |F(corner + stride) - F(corner)| in exact arithmetic."""
    P = [[Fraction(x) for x in p] for p in pts]
    F = {}
    for it in (0, 1):
        t = Fraction(it)
        lp = [[(1 - t) * P[k][ax] + t * P[4 + k][ax] for ax in range(3)] for k in range(4)]
        for iu in (0, 1):
            for iv in (0, 1):
                u, v = Fraction(iu), Fraction(iv)
                for ax in range(3):
                    a, b, c, d = (lp[k][ax] for k in range(4))
                    F[(4 * it + 2 * iu + iv, ax)] = (a - ((1 - u - v) * b + u * c + v * d) if kind == 0
                                                     else ((1 - u) * a + u * b) - ((1 - v) * c + v * d))
    out = []
    for sd in (4, 2, 1):
        out.append(3 * max(abs(F[(i + sd, ax)] - F[(i, ax)]) for i in range(8) if not i & sd
                           for ax in range(3)))
    return tuple(float(k) for k in out)


@given(data=st.data(), kind=st.sampled_from([QueryKind.VERTEX_FACE, QueryKind.EDGE_EDGE]))
@settings(max_examples=40, deadline=None, derandomize=True)
def test_kappas_match_rational_weights_on_integer_queries(cuda, data, kind):
    coord = st.integers(min_value=-8, max_value=8)
    pts = [tuple(float(data.draw(coord)) for _ in range(3)) for _ in range(8)]
    q = Query(kind, pts[:4], pts[4:])
    assert kappas(q) == _rational_kappas(int(kind), pts)


def test_kappas_batch_matches_solver_kappas(cuda):
    """The batch entry point and per-query t_max."""
    rng = np.random.default_rng(5)
    pts = rng.integers(-8, 9, (500, 8, 3)).astype(np.float64)
    kind = rng.integers(0, 2, 500).astype(np.uint8)
    k = kappas_batch(pts, kind, 1.0)
    for i in range(0, 500, 37):
        assert tuple(k[i]) == _rational_kappas(int(kind[i]), [tuple(p) for p in pts[i]])
    tm = np.full(500, 0.5)
    assert np.array_equal(kappas_batch(pts, kind, tm), kappas_batch(pts, kind, 0.5))
