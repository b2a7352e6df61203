"""Host-side logic on CPU: reference-mirroring types and validation, filters,
workload generators, sharding (incl. a gloo world-size-2 run), and the
C-ABI library surface (loads and exports without a GPU)."""

import ctypes
import math
import os
import re
import subprocess
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT
from paper_2009_13349_b200 import (DomainBox, Query, QueryKind, SolverConfig, compute_filters,
                                   compute_gamma, shard_bounds)
from paper_2009_13349_b200 import workloads as W
from paper_2009_13349_b200 import inclusion

TRI = ((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))


# --- types / validation (pkg/src/ccdkit/core.py:42-184) ----------------------

def test_solver_config_validation_matches_reference():
    SolverConfig()
    for bad in (dict(delta=0.0), dict(delta=float("inf")), dict(max_checks=0),
                dict(separation=-1e-9), dict(separation=float("nan")), dict(t_max=0.0),
                dict(t_max=1.5)):
        with pytest.raises(ValueError):
            SolverConfig(**bad)


def test_query_rejects_nonfinite_and_wrong_arity():
    with pytest.raises(ValueError):
        Query(QueryKind.VERTEX_FACE, ((float("nan"), 0, 0),) + TRI, ((0, 0, 0),) + TRI)
    with pytest.raises(ValueError):
        Query(QueryKind.VERTEX_FACE, TRI, TRI)
    q = Query(0, ((0.3, 0.3, 1.0),) + TRI, ((0.3, 0.3, -1.0),) + TRI)
    assert q.kind is QueryKind.VERTEX_FACE
    assert q.all_coordinates().shape == (8, 3)


def test_domain_box_validation():
    DomainBox((0.0, 1.0), (0.0, 1.0), (0.0, 1.0))
    with pytest.raises(ValueError):
        DomainBox((0.5, 0.25), (0.0, 1.0), (0.0, 1.0))
    with pytest.raises(ValueError):
        DomainBox((0.0, 1.0), (0.0, 1.0), (0.0, 1.0), level=-1)


# --- filters (pkg/tests/test_inclusion.py:45-76 expectations) ----------------

def test_filter_constants_and_scaling():
    assert compute_filters(QueryKind.VERTEX_FACE, (1, 1, 1)).eps == (inclusion.VF_COEFF,) * 3
    assert compute_filters(QueryKind.EDGE_EDGE, (1, 1, 1)).eps == (inclusion.EE_COEFF,) * 3
    assert compute_filters(QueryKind.VERTEX_FACE, (1, 1, 1), 0.5).eps == (inclusion.VF_COEFF_MINSEP,) * 3
    assert compute_filters(QueryKind.EDGE_EDGE, (1, 1, 1), 0.5).eps == (inclusion.EE_COEFF_MINSEP,) * 3
    eps = compute_filters(QueryKind.VERTEX_FACE, (10.0, 1.0, 100.0)).eps
    assert eps == (inclusion.VF_COEFF * 1e3, inclusion.VF_COEFF, inclusion.VF_COEFF * 1e6)
    assert compute_gamma([[0.5, -3.0, 0.0], [0.25, 2.0, 100.0]]) == (1.0, 3.0, 100.0)
    for args in (((0.5, 1.0, 1.0),), ((1, 1, 1), 1.0), ((1, 1, 1), -1e-20)):
        with pytest.raises(ValueError):
            compute_filters(QueryKind.VERTEX_FACE, *args)
    with pytest.raises(ValueError):
        compute_gamma(np.zeros((0, 3)))


def test_host_filters_match_oracle():
    import oracle
    g = np.load(os.path.join(ROOT, "tests", "golden", "c3.npz"))
    L = oracle.lib()
    for i in range(0, 200, 7):
        pts = np.ascontiguousarray(g["points"][i])
        out = np.zeros(3)
        rc = L.tccd_oracle_filters(pts.ctypes.data_as(ctypes.c_void_p), int(g["kind"][i]), 0.0,
                                   out.ctypes.data_as(ctypes.c_void_p))
        assert rc == 1
        f = compute_filters(QueryKind(int(g["kind"][i])), compute_gamma(pts), 0.0)
        assert f.eps == tuple(out)


# --- workloads -----------------------------------------------------------------

@pytest.mark.parametrize("config", [0, 1, 2, 3, 4])
def test_workloads_are_index_addressable(config):
    full = W.generate(config, 70_000, 2_000)
    part = W.generate(config, 71_000, 500)
    assert np.array_equal(full.points[1000:1500], part.points)
    assert np.array_equal(full.kind[1000:1500], part.kind)
    assert full.points.shape == (2000, 8, 3) and np.isfinite(full.points).all()


def _solve_uv(e1, e2, r):
    """Exact (u, v) with u*e1 + v*e2 = r (3-vectors of Fractions), or None."""
    for i, j in ((0, 1), (0, 2), (1, 2)):
        det = e1[i] * e2[j] - e1[j] * e2[i]
        if det != 0:
            u = (r[i] * e2[j] - r[j] * e2[i]) / det
            v = (e1[i] * r[j] - e1[j] * r[i]) / det
            if all(u * e1[k] + v * e2[k] == r[k] for k in range(3)):
                return u, v
            return None
    return None


def test_planted_roots_are_exact():
    """Config-1 planted queries: F(t*, u, v) = 0 in exact rational arithmetic
    with (u, v) inside the domain (dataset.py:457-461 construction)."""
    w = W.generate(1, 0, 400)
    planted = np.flatnonzero(~np.isnan(w.planted_t))
    assert len(planted) > 100
    for i in planted:
        P = [[Fraction(float(c)) for c in p] for p in w.points[i]]
        t = Fraction(float(w.planted_t[i]))
        X = [[(1 - t) * P[k][ax] + t * P[k + 4][ax] for ax in range(3)] for k in range(4)]
        sub = lambda a, b: [a[k] - b[k] for k in range(3)]
        if w.kind[i] == 0:   # X0 = X1 + u (X2 - X1) + v (X3 - X1)
            uv = _solve_uv(sub(X[2], X[1]), sub(X[3], X[1]), sub(X[0], X[1]))
            assert uv is not None and uv[0] >= 0 and uv[1] >= 0 and uv[0] + uv[1] <= 1, i
        else:                # X0 + u (X1 - X0) = X2 + v (X3 - X2)
            d2 = sub(X[3], X[2])
            uv = _solve_uv(sub(X[1], X[0]), [-c for c in d2], sub(X[2], X[0]))
            assert uv is not None and 0 <= uv[0] <= 1 and 0 <= uv[1] <= 1, i


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 1000, 10**6 + 3):
        for world in (1, 2, 3, 8):
            bounds = [shard_bounds(n, world, r) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))


def _gloo_worker(rank, world, port, out_path):
    import torch.distributed as dist
    import oracle
    from paper_2009_13349_b200.sharding import solve_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = W.generate(3, 0, 3001)
    res = solve_sharded(w.points, w.kind, lambda p, k, **kw: oracle.solve_batch(p, k, threads=1),
                        rank=rank, world=world)
    # timing reduction used by bench.py: max over ranks
    import torch
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.savez(out_path, max_t=t.numpy(), **res)
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_gather(tmp_path):
    import socket
    import torch.multiprocessing as mp
    import oracle
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "r.npz")
    mp.spawn(_gloo_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    w = W.generate(3, 0, 3001)
    ref = oracle.solve_batch(w.points, w.kind)
    assert float(got["max_t"][0]) == 2.0
    for k in ("status", "toi", "checks", "witness"):
        assert np.array_equal(got[k], ref[k])


# --- the C-ABI library (no GPU needed to load it) ------------------------------

def _header_symbols():
    src = open(os.path.join(ROOT, "include", "tccd.h")).read()
    return sorted(set(re.findall(r"\b(tccd_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2009_13349_b200 import _lib
    L = _lib.lib()
    syms = _header_symbols()
    assert set(syms) == set(_lib.EXPORTS)
    for name in syms:
        assert hasattr(L, name), name
    assert L.tccd_abi_version() == _lib.ABI_VERSION == 3
    for code in range(0, 12):
        assert L.tccd_error_string(code)
    assert b"unknown" in L.tccd_error_string(999)


@pytest.mark.parametrize("cname,pyname", [("tccd_batch", "TccdBatch"), ("tccd_mesh", "TccdMesh")])
def test_struct_layout_matches_header(tmp_path, cname, pyname):
    """ctypes mirrors of the C-ABI structs == the C compiler's layout."""
    from paper_2009_13349_b200 import _lib
    cls = getattr(_lib, pyname)
    fields = [f for f, _ in cls._fields_]
    prog = ["#include <stdio.h>", "#include <stddef.h>", '#include "tccd.h"', "int main(void){",
            f'printf("%zu\\n", sizeof({cname}));']
    prog += [f'printf("%zu\\n", offsetof({cname}, {f}));' for f in fields]
    prog += ["return 0;}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(c)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert vals[0] == ctypes.sizeof(cls)
    for f, off in zip(fields, vals[1:]):
        assert getattr(cls, f).offset == off, f


def test_workspace_bytes_is_monotone_and_rejects_bad_sizes():
    from paper_2009_13349_b200 import _lib
    L = _lib.lib()
    a = L.tccd_workspace_bytes(1000, 1000, 4)
    b = L.tccd_workspace_bytes(1000, 1_000_000, 4)
    c = L.tccd_workspace_bytes(1000, 1_000_000, 8)
    assert 0 < a < b < c
    assert L.tccd_workspace_bytes(-1, 10, 1) == 0
    assert L.tccd_workspace_bytes(10, 0, 1) == 0
    assert L.tccd_workspace_bytes_ex(10, 10, 1, -1) == 0


def test_workspace_scales_with_the_batch():
    """Queues, lane scratch, group arenas and handover pools follow the batch
    size: one query at m_I = 1e6 needs its giant arena (2 m_I + 2 boxes) and
    little else, so the per-call drop-in is not a multi-GB allocation."""
    from paper_2009_13349_b200 import _lib
    L = _lib.lib()
    one = L.tccd_workspace_bytes(1, 1_000_000, 1)
    assert one < 400e6
    small = L.tccd_workspace_bytes(1, 1000, 1)
    assert small < 20e6
    sizes = [L.tccd_workspace_bytes(n, 1000, 1) for n in (1, 10, 1000, 100_000, 1 << 22, 1 << 26,
                                                          1 << 27)]
    assert all(a <= b for a, b in zip(sizes, sizes[1:]))
    assert sizes[-1] == sizes[-2]  # bounded by one library chunk
    # the handover pool size is a parameter; a smaller pool never grows the layout
    assert L.tccd_workspace_bytes_ex(1 << 20, 1000, 1, 1 << 16) < L.tccd_workspace_bytes(1 << 20, 1000, 1)


def test_solve_batch_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2009_13349_b200 import solve_batch
    with pytest.raises(RuntimeError):
        solve_batch(np.zeros((1, 8, 3)), 0, device="cpu")


def test_bench_launcher_starts_n_ranks():
    """`bench.py --gpus 2` re-launches itself under torch.distributed.run with
    two ranks (here: the CPU launcher self-test, gloo, no solve); the line
    reports n_gpus 2 and the two contiguous shards of the one query set."""
    import json
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--selftest-launcher", "--queries", "1001"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["shards"] == [[0, 500], [500, 1001]]
