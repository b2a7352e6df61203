"""The reference's spec-level API on the host: Vec3, eval_F, split,
queue_order, classify_box, InclusionBox -- the assertions of the
reference's own tests (pkg/tests/test_solver.py:117-155,
pkg/tests/test_inclusion.py:79-137, pkg/tests/test_core.py) re-run here."""

import math

import pytest

from paper_2009_13349_b200 import (BoxClass, DomainBox, FilterEps, InclusionBox, Query, QueryKind,
                                   Vec3, classify_box, eval_F, eval_F_ee, eval_F_vf, queue_order,
                                   split)

TRI = ((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))


def test_vec3_is_a_finite_tuple_with_arithmetic():
    a = Vec3(1, 2, 3)
    assert a.x == 1.0 and a.y == 2.0 and a.z == 3.0 and a == (1.0, 2.0, 3.0)
    assert a + Vec3(1, 1, 1) == (2.0, 3.0, 4.0)
    assert a - Vec3(1, 1, 1) == (0.0, 1.0, 2.0)
    assert a.scaled(2.0) == (2.0, 4.0, 6.0)
    assert a.dot(Vec3(1, 0, 1)) == 4.0
    assert Vec3(1, 0, 0).cross(Vec3(0, 1, 0)) == (0.0, 0.0, 1.0)
    for bad in ((math.nan, 0, 0), (0, math.inf, 0), (0, 0, -math.inf)):
        with pytest.raises(ValueError):
            Vec3(*bad)


def test_query_points_are_vec3():
    q = Query(QueryKind.VERTEX_FACE, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    assert all(isinstance(p, Vec3) for p in q.points0 + q.points1)
    assert q.points0[0].x == 0.3 and q.points1[0].z == -1.0
    t = Query._trusted(QueryKind.VERTEX_FACE, q.points0, q.points1)
    assert t == q and isinstance(t.points0[1], Vec3)


def test_eval_F_closed_forms():
    vf = Query(QueryKind.VERTEX_FACE, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    assert eval_F(vf, 0.5, 0.3, 0.3) == eval_F_vf(vf, 0.5, 0.3, 0.3) == (0.0, 0.0, 0.0)
    assert eval_F_vf(vf, 0.0, 0.0, 0.0) == (0.3, 0.3, 1.0)
    ee = Query(QueryKind.EDGE_EDGE,
               ((0.0, 0.0, 1.0), (1.0, 1.0, 1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)),
               ((0.0, 0.0, -1.0), (1.0, 1.0, -1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0)))
    assert eval_F(ee, 0.5, 0.5, 0.5) == eval_F_ee(ee, 0.5, 0.5, 0.5) == (0.0, 0.0, 0.0)
    assert eval_F_ee(ee, 1.0, 0.0, 0.0) == (0.0, -1.0, -1.0)


# --- pkg/tests/test_solver.py:117-155 ---------------------------------------

def test_split_halves_largest_weighted_width_exactly():
    root = DomainBox((0.0, 1.0), (0.0, 1.0), (0.0, 1.0))
    kids = split(root, (6.0, 3.0, 3.0), QueryKind.VERTEX_FACE)
    assert [k.t for k in kids] == [(0.0, 0.5), (0.5, 1.0)]
    assert all(k.u == (0.0, 1.0) and k.v == (0.0, 1.0) and k.level == 1 for k in kids)


def test_split_ties_prefer_the_earlier_dimension():
    box = DomainBox((0.0, 0.25), (0.5, 1.0), (0.5, 1.0), level=3)
    kids = split(box, (1.0, 1.0, 1.0), QueryKind.EDGE_EDGE)
    assert [k.u for k in kids] == [(0.5, 0.75), (0.75, 1.0)]


def test_split_drops_face_children_outside_the_triangle():
    box = DomainBox((0.0, 0.25), (0.5, 1.0), (0.5, 1.0), level=3)
    kids = split(box, (1.0, 1.0, 1.0), QueryKind.VERTEX_FACE)
    assert len(kids) == 1 and kids[0].u == (0.5, 0.75) and kids[0].level == 4


def test_split_rejects_bad_weights_and_point_boxes():
    root = DomainBox((0.0, 1.0), (0.0, 1.0), (0.0, 1.0))
    with pytest.raises(ValueError):
        split(root, (-1.0, 1.0, 1.0), QueryKind.VERTEX_FACE)
    with pytest.raises(ValueError):
        split(DomainBox((0.5, 0.5), (0.25, 0.25), (0.0, 0.0)), (1.0, 1.0, 1.0),
              QueryKind.VERTEX_FACE)


def test_queue_order_is_level_then_start_time():
    root = DomainBox((0.0, 1.0), (0.0, 1.0), (0.0, 1.0))
    deep = DomainBox((0.0, 0.25), (0.5, 1.0), (0.5, 1.0), level=3)
    late = DomainBox((0.5, 1.0), (0.0, 1.0), (0.0, 1.0), level=1)
    early = DomainBox((0.0, 0.5), (0.0, 1.0), (0.0, 1.0), level=1)
    assert queue_order(root, deep) == -1 and queue_order(deep, root) == 1
    assert queue_order(root, root) == 0
    assert queue_order(late, early) == 1 and queue_order(early, late) == -1


# --- pkg/tests/test_inclusion.py:79-137 -------------------------------------

EPS = FilterEps(kind=QueryKind.VERTEX_FACE, gamma=(1.0, 1.0, 1.0), eps=(1e-3, 1e-3, 1e-3),
                separation=0.0)


def test_inclusion_box_rejects_inverted_axis():
    with pytest.raises(ValueError):
        InclusionBox(lo=(0.0, 1.0, 0.0), hi=(1.0, 0.0, 1.0))


def test_classify_box_disjoint_contained_ties():
    assert classify_box(InclusionBox((-1.0, 2e-3, -1.0), (1.0, 3e-3, 1.0)), EPS) is BoxClass.DISJOINT
    assert classify_box(InclusionBox((-1.0, -3e-3, -1.0), (1.0, -2e-3, 1.0)), EPS) is BoxClass.DISJOINT
    assert classify_box(InclusionBox((-1e-4,) * 3, (1e-4,) * 3), EPS) is BoxClass.CONTAINED
    assert classify_box(InclusionBox((-1e-4,) * 3, (1e-4, 1e-4, 2.0)), EPS) is BoxClass.INTERSECTS
    # a tie with the filter is never disjoint
    assert classify_box(InclusionBox((1e-3, -1.0, -1.0), (2.0, 1.0, 1.0)), EPS) is BoxClass.INTERSECTS


def test_classify_box_separation():
    eps_d = FilterEps(kind=QueryKind.VERTEX_FACE, gamma=(1.0, 1.0, 1.0), eps=(1e-3,) * 3,
                      separation=0.05)
    near = InclusionBox((0.01, -1.0, -1.0), (0.02, 1.0, 1.0))
    assert classify_box(near, eps_d, separation=0.05) is BoxClass.INTERSECTS
    far = InclusionBox((0.1, -1.0, -1.0), (0.2, 1.0, 1.0))
    assert classify_box(far, eps_d, separation=0.05) is BoxClass.DISJOINT
    with pytest.raises(ValueError):
        classify_box(InclusionBox((0.0,) * 3, (0.0,) * 3), EPS, separation=0.1)
