"""Scene-level callers, pinned to the reference's own
results on seeded meshes (tests/golden/scene.json, written by
tests/golden/make_scene_golden.py from ccdkit.scene).

CPU tests cover the broad phase, the start-distance bounds and the batched
line-search / active-set host logic, with the oracle standing in for the
device solve (test infrastructure only).  GPU tests run the product path.
"""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from paper_2009_13349_b200 import SolverConfig, scene
from paper_2009_13349_b200.scene import (InfeasibleStepError, TriMeshPair, broad_phase,
                                         broad_phase_batch, construct_active_set,
                                         edges_from_triangles, line_search_step, load_obj,
                                         primitive_distance_lb)
from scene_host import broad_phase_host

with open(os.path.join(GOLDEN_DIR, "scene.json")) as _fh:
    GOLD = json.load(_fh)
TAGS = sorted(GOLD)
LS_CASES = [(0.5, None), (0.5, 0.3), (0.9, 0.1)]


def _mesh(tag):
    g = GOLD[tag]
    return TriMeshPair(np.array(g["x0"]), np.array(g["x1"]), g["tris"])


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.int64)


@pytest.fixture
def oracle_device(monkeypatch):
    """Route the scene module's broad phase and batched solves through the
    host checkers (tests/scene_host.py, the CPU oracle)."""
    import oracle

    def fake(cs, sel, cfg, separation, device):
        sep = separation if np.isscalar(separation) else np.asarray(separation, np.float64)
        return oracle.solve_batch(np.asarray(cs.points[sel]), np.asarray(cs.kind[sel]),
                                  delta=cfg.delta, max_checks=cfg.max_checks, separation=sep,
                                  t_max=cfg.t_max)

    def fake_active(mesh, delta=1e-6, max_checks=1_000_000, separation=0.0, device=None):
        cs = broad_phase_host(mesh, separation + delta)
        cfg = SolverConfig(delta=delta, max_checks=max_checks, separation=separation)
        r = fake(cs, slice(None), cfg, separation, device)
        hit = np.flatnonzero(r["status"] == 1)
        return (scene.CandidateSet(cs.kind[hit], cs.indices[hit], cs.points[hit]),
                {k: v[hit] for k, v in r.items()})

    monkeypatch.setattr(scene, "_solve", fake)
    monkeypatch.setattr(scene, "broad_phase_batch", broad_phase_host)
    monkeypatch.setattr(scene, "active_set_batch", fake_active)


def _cand_list(cs):
    h = cs.host()
    return [[int(k), int(i), int(j)] for k, (i, j) in zip(h.kind, h.indices)]


# ---------------------------------------------------------------- broad phase

@pytest.mark.parametrize("tag", TAGS)
def test_host_broad_phase_matches_reference(tag):
    mesh = _mesh(tag)
    for infl, want in GOLD[tag]["broad"].items():
        assert _cand_list(broad_phase_host(mesh, float(infl))) == want, (tag, infl)


def _check_points(mesh, cands):
    for c in cands:
        if c.kind == 0:
            v, f = c.indices
            vid = [v, *mesh.triangles[f]]
        else:
            i, j = c.indices
            vid = [*mesh.edges[i], *mesh.edges[j]]
        want = np.concatenate([mesh.x0[vid], mesh.x1[vid]])
        assert np.array_equal(c.query.all_coordinates(), want)


@pytest.mark.parametrize("tag", TAGS)
def test_candidate_points_follow_solver_order(tag):
    mesh = _mesh(tag)
    _check_points(mesh, broad_phase_host(mesh, 0.3).to_list())


@pytest.mark.parametrize("tag", TAGS)
def test_distance_lb_bitwise(tag):
    got = [primitive_distance_lb(c) for c in broad_phase_host(_mesh(tag), 0.3).to_list()]
    assert np.array_equal(_bits(got), _bits(GOLD[tag]["dlb"]))


def test_host_broad_phase_random_against_brute_force():
    rng = np.random.default_rng(5)
    for trial in range(5):
        nv = 60
        x0 = rng.uniform(-1, 1, (nv, 3))
        x1 = x0 + rng.normal(0, 0.2, (nv, 3))
        tris = rng.integers(0, nv, (40, 3))
        tris = tris[(tris[:, 0] != tris[:, 1]) & (tris[:, 1] != tris[:, 2]) &
                    (tris[:, 0] != tris[:, 2])]
        mesh = TriMeshPair(x0, x1, tris)
        infl = 0.05 * trial
        pts = lambda idx: np.stack((mesh.x0[idx], mesh.x1[idx]))  # noqa: E731
        box = lambda idx: (pts(idx).min(axis=(0, 2)) - infl, pts(idx).max(axis=(0, 2)) + infl)  # noqa: E731
        vlo, vhi = box(np.arange(nv)[:, None])
        tlo, thi = box(mesh.triangles)
        elo, ehi = box(mesh.edges)
        ov = lambda a0, a1, b0, b1: bool(np.all(a0 <= b1) and np.all(b0 <= a1))  # noqa: E731
        want = [[0, v, f] for v in range(nv) for f in range(len(tris))
                if v not in mesh.triangles[f] and ov(vlo[v], vhi[v], tlo[f], thi[f])]
        E = mesh.edges
        want += [[1, i, j] for i in range(len(E)) for j in range(i + 1, len(E))
                 if not set(E[i]) & set(E[j]) and ov(elo[i], ehi[i], elo[j], ehi[j])]
        assert _cand_list(broad_phase_host(mesh, infl)) == want


def test_mesh_validation_and_edges(tmp_path):
    with pytest.raises(ValueError):
        TriMeshPair(np.zeros((3, 3)), np.zeros((4, 3)), [[0, 1, 2]])
    with pytest.raises(ValueError):
        TriMeshPair(np.full((3, 3), np.nan), np.zeros((3, 3)), [[0, 1, 2]])
    with pytest.raises(ValueError):
        TriMeshPair(np.zeros((3, 3)), np.zeros((3, 3)), [[0, 1, 3]])
    with pytest.raises(ValueError):
        broad_phase(TriMeshPair(np.zeros((3, 3)), np.zeros((3, 3)), [[0, 1, 2]]), -1.0)
    assert edges_from_triangles([[2, 1, 0], [1, 2, 3]]).tolist() == [[0, 1], [0, 2], [1, 2],
                                                                       [1, 3], [2, 3]]
    m = TriMeshPair(np.zeros((3, 3)), np.ones((3, 3)), [[0, 1, 2]], edges=np.zeros((0, 2)))
    assert m.edges.shape == (0, 2)
    assert np.array_equal(m.at(0.25), np.full((3, 3), 0.25))
    assert broad_phase_host(TriMeshPair(np.zeros((0, 3)), np.zeros((0, 3)), [])).m == 0
    obj = tmp_path / "q.obj"
    obj.write_text("# quad\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nvn 0 0 1\nf 1/1/1 2/2/1 3 -1\n")
    v, f = load_obj(obj)
    assert v.shape == (4, 3) and f.tolist() == [[0, 1, 2], [0, 2, 3]]
    obj.write_text("v 0 0 0\nf 1 2 3\n")
    with pytest.raises(ValueError):
        load_obj(obj)


def test_touching_start_is_infeasible(oracle_device):
    x = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.25, 0.25, 0.0]])
    mesh = TriMeshPair(x, x + [0, 0, 0.1], [[0, 1, 2]])
    with pytest.raises(InfeasibleStepError):
        line_search_step(mesh, p=0.5)
    with pytest.raises(ValueError):
        line_search_step(mesh, p=1.0)


# ------------------------------------------- host logic, oracle as the device

def _check_active(tag, sep, act):
    want = GOLD[tag]["active"][sep]
    assert len(act) == len(want)
    for (c, toi, w), g in zip(act, want):
        assert [int(c.kind), *c.indices] == g[:3]
        assert _bits(toi) == _bits(g[3])
        assert np.array_equal(_bits(list(w.t) + list(w.u) + list(w.v)), _bits(g[4]))
        assert w.level == g[5]


def _check_ls(tag, p, infl, r):
    want = GOLD[tag]["line_search"][f"{p}_{infl}"]
    assert "infeasible" not in want
    assert _bits(r.alpha) == _bits(want["alpha"]) and _bits(r.p) == _bits(want["p"])
    assert r.validations == want["validations"] and r.limiting == want["limiting"]
    assert len(r.bounds) == len(want["bounds"])
    for b, g in zip(r.bounds, want["bounds"]):
        assert [int(b.candidate.kind), *b.candidate.indices] == g[:3]
        assert _bits(b.distance_lb) == _bits(g[3]) and _bits(b.separation) == _bits(g[4])
        assert (b.toi is None) == (g[5] is None)
        if b.toi is not None:
            assert _bits(b.toi) == _bits(g[5])
            assert b.witness is not None


@pytest.mark.parametrize("tag", TAGS)
def test_active_set_host_logic(tag, oracle_device):
    mesh = _mesh(tag)
    for sep in GOLD[tag]["active"]:
        _check_active(tag, sep, construct_active_set(mesh, separation=float(sep)))


@pytest.mark.parametrize("tag", TAGS)
def test_line_search_host_logic(tag, oracle_device):
    mesh = _mesh(tag)
    for p, infl in LS_CASES:
        _check_ls(tag, p, infl, line_search_step(mesh, p=p, inflation=infl))


@pytest.mark.parametrize("tag", TAGS)
def test_line_search_windows(tag, oracle_device, monkeypatch):
    """Candidates solved in windows of 7 (re-solving after every alpha
    change, window by window) give the reference's results too."""
    import paper_2009_13349_b200.scene as S
    monkeypatch.setattr(S, "_LS_WINDOW", 7)
    mesh = _mesh(tag)
    for p, infl in LS_CASES:
        _check_ls(tag, p, infl, line_search_step(mesh, p=p, inflation=infl))


def test_line_search_energy_loop(oracle_device):
    mesh = _mesh("mover_free")
    calls = []

    def energy(a):
        calls.append(a)
        return a <= 0.25

    r = line_search_step(mesh, p=0.5, energy_decreases=energy)
    assert r.alpha == 0.25 and calls == [1.0, 0.5, 0.25]
    r = line_search_step(mesh, p=0.5, energy_decreases=lambda a: False, alpha_min=0.1)
    assert r.alpha == 0.0625


# ----------------------------------------------------------- GPU product path

@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_broad_phase_matches_reference(tag):
    mesh = _mesh(tag)
    for infl, want in GOLD[tag]["broad"].items():
        cs = broad_phase_batch(mesh, float(infl))
        assert cs.points.is_cuda
        assert _cand_list(cs) == want, (tag, infl)
    _check_points(mesh, broad_phase(mesh, 0.3))


def _random_meshes():
    rng = np.random.default_rng(17)
    for trial in range(4):  # soups of varying density
        nt = [50, 400, 1500, 3000][trial]
        c = rng.uniform(-1, 1, (nt, 1, 3))
        v0 = (c + rng.normal(0, 0.04 * (4 - trial), (nt, 3, 3))).reshape(-1, 3)
        yield f"soup{nt}", TriMeshPair(v0, v0 + rng.normal(0, 0.05, v0.shape),
                                       np.arange(3 * nt).reshape(nt, 3))
    g = 60  # a shared-vertex grid sheet folding onto itself
    xs, ys = np.meshgrid(np.linspace(0, 1, g), np.linspace(0, 1, g))
    x0 = np.stack([xs.ravel(), ys.ravel(), np.zeros(g * g)], 1)
    x1 = x0 + np.stack([np.zeros(g * g), np.zeros(g * g), 0.3 * np.sin(6 * xs.ravel())], 1)
    tris = []
    for i in range(g - 1):
        for j in range(g - 1):
            a, b, c_, d = i * g + j, i * g + j + 1, (i + 1) * g + j, (i + 1) * g + j + 1
            tris += [[a, b, c_], [b, d, c_]]
    yield "sheet", TriMeshPair(x0, x1, tris)
    yield "flat", TriMeshPair(x0, x0, tris)  # zero extent on z
    z = np.zeros((5, 3))
    yield "coincident", TriMeshPair(z, z, [[0, 1, 2], [2, 3, 4]])  # all boxes one point
    yield "edges_only", TriMeshPair(x0[:40], x1[:40], np.zeros((0, 3)),
                                    edges=np.array([[i, i + 1] for i in range(39)]))
    yield "empty", TriMeshPair(np.zeros((0, 3)), np.zeros((0, 3)), [])


@pytest.mark.gpu
def test_gpu_broad_phase_matches_host_restatement():
    for name, mesh in _random_meshes():
        for infl in (0.0, 1e-3, 0.05):
            want = broad_phase_host(mesh, infl)
            got = broad_phase_batch(mesh, infl)
            assert _cand_list(got) == _cand_list(want), (name, infl)
            assert np.array_equal(got.points.cpu().numpy(), np.asarray(want.points)), name



@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_active_set_gpu(tag):
    mesh = _mesh(tag)
    for sep in GOLD[tag]["active"]:
        _check_active(tag, sep, construct_active_set(mesh, separation=float(sep)))


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_line_search_gpu(tag):
    mesh = _mesh(tag)
    for p, infl in LS_CASES:
        _check_ls(tag, p, infl, line_search_step(mesh, p=p, inflation=infl))


@pytest.mark.gpu
def test_line_search_gpu_matches_sequential_oracle_large():
    """A bigger scene than the golden ones: the batched re-solve schedule
    against the reference's one-solve-per-candidate loop run on the oracle."""
    import oracle
    rng = np.random.default_rng(11)
    m = 120
    c = rng.uniform(-1, 1, (m, 1, 3))
    v0 = (c + rng.normal(0, 0.12, (m, 3, 3))).reshape(-1, 3)
    v1 = v0 + rng.normal(0, 0.15, v0.shape)
    mesh = TriMeshPair(v0, v1, np.arange(3 * m).reshape(m, 3))
    p, delta = 0.5, 1e-6
    r = line_search_step(mesh, p=p, inflation=0.05)
    cs = broad_phase_batch(mesh, 0.05).host()
    alpha, lim = 1.0, None
    for i in range(cs.m):
        sep = min(r.p * r.bounds[i].distance_lb, delta)
        o = oracle.solve_batch(cs.points[i:i + 1], cs.kind[i:i + 1], delta=delta,
                               separation=sep, t_max=alpha)
        hit = o["status"][0] == 1
        assert (r.bounds[i].toi is None) == (not hit)
        if hit:
            assert _bits(r.bounds[i].toi) == _bits(o["toi"][0])
            if o["toi"][0] < alpha:
                alpha, lim = float(o["toi"][0]), i
                if alpha == 0.0:
                    break
    assert r.validations == 1 and _bits(r.alpha) == _bits(alpha) and r.limiting == lim
    assert math.isfinite(r.alpha)


@pytest.mark.parametrize("family", ["uniform", "lattice", "degenerate", "coplanar"])
def test_distance_lb_batch_matches_scalar(family):
    """The batched start-distance bounds (line_search_step's) equal the scalar
    closed forms bit for bit, branches included (zero-length edges, parallel
    edges, degenerate triangles)."""
    from paper_2009_13349_b200.scene import distance_lb, distance_lb_batch
    rng = np.random.default_rng(3)
    m = 4000
    if family == "uniform":
        pts = rng.random((m, 8, 3))
    elif family == "lattice":
        pts = rng.integers(-3, 4, (m, 8, 3)) / 2.0
    elif family == "degenerate":
        pts = rng.random((m, 8, 3))
        pts[:, 1] = pts[:, 0]
        pts[::3, 3] = pts[::3, 2]
    else:
        pts = rng.random((m, 8, 3))
        pts[..., 2] = 0.0
    kind = rng.integers(0, 2, m).astype(np.uint8)
    got = distance_lb_batch(kind, pts)
    want = np.array([distance_lb(int(kind[i]), pts[i]) for i in range(m)])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
