"""Scene-level throughput on a synthetic cloth
scene: two g x g triangulated sheets moving into each other (seeded noise).

Times, with CUDA events on the launching stream after a warm-up:
  * the GPU broad phase (tccd_broad_create + emit: swept boxes, grid, pair
    search, sort, candidate queries written in the solver layout);
  * construct_active_set (broad phase + one batched narrow-phase solve);
and, for scale, the numpy host restatement of the broad phase on the same
mesh (tests/scene_host.py, the CPU reference-shaped path).  Prints one JSON
line.

    python tools/scene_bench.py [--grid 200] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_13349_b200.scene import (TriMeshPair, active_set_batch,  # noqa: E402
                                         broad_phase_batch, construct_active_set,
                                         line_search_step)


def cloth(g: int, seed: int = 0) -> TriMeshPair:
    rng = np.random.default_rng(seed)
    xs, ys = np.meshgrid(np.linspace(0, 1, g), np.linspace(0, 1, g))
    sheet = np.stack([xs.ravel(), ys.ravel(), np.zeros(g * g)], 1)
    i, j = np.meshgrid(np.arange(g - 1), np.arange(g - 1), indexing="ij")
    a = (i * g + j).ravel()
    tris = np.concatenate([np.stack([a, a + 1, a + g], 1), np.stack([a + 1, a + g + 1, a + g], 1)])
    h = 1.0 / (g - 1)
    top = sheet + np.array([0.3 * h, 0.2 * h, 2.0 * h])
    x0 = np.vstack([sheet, top])
    x1 = np.vstack([sheet + rng.normal(0, 0.05 * h, sheet.shape),
                    top + np.array([0.0, 0.0, -3.0 * h]) + rng.normal(0, 0.3 * h, top.shape)])
    return TriMeshPair(x0, x1, np.vstack([tris, tris + g * g]))


def cuda_ms(fn, reps):
    s = torch.cuda.current_stream()
    out = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        out = fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=200)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-host", action="store_true")
    args = ap.parse_args()
    mesh = cloth(args.grid)
    infl = 2e-6
    bp_ms, cs = cuda_ms(lambda: broad_phase_batch(mesh, infl), args.reps)
    act_ms, (hits, _) = cuda_ms(lambda: active_set_batch(mesh), args.reps)
    t0 = time.perf_counter()
    act = construct_active_set(mesh)
    list_ms = 1e3 * (time.perf_counter() - t0)
    line = {"scene": f"two {args.grid}x{args.grid} sheets", "vertices": mesh.n_vertices,
            "triangles": int(len(mesh.triangles)), "edges": int(len(mesh.edges)),
            "candidates": cs.m, "vf": int((cs.kind == 0).sum()), "ee": int((cs.kind == 1).sum()),
            "gpu_broad_phase_ms": bp_ms, "gpu_candidates_per_s": cs.m / (bp_ms * 1e-3),
            "active_set_batch_ms": act_ms, "active_pairs": hits.m,
            "construct_active_set_list_ms": list_ms}
    assert len(act) == hits.m
    # line_search_step (scene.py:468-583): broad phase, start-distance bounds
    # and filters of every candidate, solves at the shrinking alpha
    t0 = time.perf_counter()
    ls = line_search_step(mesh, p=0.5)
    line.update({"line_search_ms": 1e3 * (time.perf_counter() - t0), "line_search_alpha": ls.alpha,
                 "line_search_validations": ls.validations, "line_search_bounds": len(ls.bounds)})
    if not args.no_host:
        # bounded host sample: the numpy restatement on a 60 x 60 cloth
        from scene_host import broad_phase_host
        small = cloth(60)
        t0 = time.perf_counter()
        hc = broad_phase_host(small, infl)
        t = time.perf_counter() - t0
        assert hc.m == broad_phase_batch(small, infl).m
        line.update({"host_sample": "two 60x60 sheets", "host_broad_phase_ms": 1e3 * t,
                     "host_candidates_per_s": hc.m / t,
                     "host_kind": "numpy restatement (tests/scene_host.py), 1 thread"})
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
