"""Golden results of the reference's scene-level callers.

Runs ccdkit.scene (pkg/src/ccdkit/scene.py: broad_phase :225-300,
construct_active_set :303-327, primitive_distance_lb :404-419,
line_search_step :468-583) from /root/reference on seeded meshes and stores
candidate lists, active sets and line-search outcomes in scene.json.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_scene_golden.py
"""

import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from ccdkit.scene import (InfeasibleStepError, TriMeshPair, broad_phase,  # noqa: E402
                          construct_active_set, line_search_step, primitive_distance_lb)

BASE = [[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]


def meshes():
    out = {}
    for z0, z1, tag in ((0.5, -0.5, "mover_hit"), (0.5, 0.45, "mover_free"),
                        (0.5, 0.05, "mover_near"), (10.0, 9.0, "mover_far")):
        out[tag] = (np.vstack([BASE, [0.3, 0.3, z0]]), np.vstack([BASE, [0.3, 0.3, z1]]),
                    [[0, 1, 2]])
    rng = np.random.default_rng(2009)
    # two sheets of triangles approaching each other
    g = 4
    xs, ys = np.meshgrid(np.linspace(0, 1, g), np.linspace(0, 1, g))
    sheet = np.stack([xs.ravel(), ys.ravel(), np.zeros(g * g)], 1)
    tris = []
    for i in range(g - 1):
        for j in range(g - 1):
            a, b, c, d = i * g + j, i * g + j + 1, (i + 1) * g + j, (i + 1) * g + j + 1
            tris += [[a, b, c], [b, d, c]]
    tris = np.array(tris)
    top = sheet + np.array([0.05, 0.07, 0.3])
    x0 = np.vstack([sheet, top])
    x1 = np.vstack([sheet + rng.normal(0, 0.01, sheet.shape),
                    top + np.array([0.0, 0.0, -0.45]) + rng.normal(0, 0.02, top.shape)])
    out["sheets"] = (x0, x1, np.vstack([tris, tris + g * g]).tolist())
    x1b = np.vstack([sheet, top + np.array([0.0, 0.0, -0.2])])
    out["sheets_free"] = (x0, x1b, np.vstack([tris, tris + g * g]).tolist())
    # a random soup of small triangles
    m = 14
    c = rng.uniform(-0.5, 0.5, (m, 1, 3))
    v0 = (c + rng.normal(0, 0.15, (m, 3, 3))).reshape(-1, 3)
    v1 = v0 + rng.normal(0, 0.1, v0.shape)
    out["soup"] = (v0, v1, np.arange(3 * m).reshape(m, 3).tolist())
    return out


def cand_list(cands):
    return [[int(c.kind), int(c.indices[0]), int(c.indices[1])] for c in cands]


def main():
    res = {}
    for tag, (x0, x1, tris) in meshes().items():
        mesh = TriMeshPair(x0, x1, tris)
        entry = {"x0": np.asarray(x0).tolist(), "x1": np.asarray(x1).tolist(), "tris": tris}
        entry["broad"] = {str(infl): cand_list(broad_phase(mesh, infl)) for infl in (0.0, 0.05, 0.3)}
        entry["dlb"] = [primitive_distance_lb(c) for c in broad_phase(mesh, 0.3)]
        act = {}
        for sep in (0.0, 1e-3):
            act[str(sep)] = [[int(c.kind), int(c.indices[0]), int(c.indices[1]), toi,
                              list(w.t) + list(w.u) + list(w.v), w.level]
                             for c, toi, w in construct_active_set(mesh, separation=sep)]
        entry["active"] = act
        ls = {}
        for p, infl in ((0.5, None), (0.5, 0.3), (0.9, 0.1)):
            key = f"{p}_{infl}"
            try:
                r = line_search_step(mesh, p=p, inflation=infl)
                ls[key] = {"alpha": r.alpha, "p": r.p, "validations": r.validations,
                           "limiting": r.limiting,
                           "bounds": [[int(b.candidate.kind), int(b.candidate.indices[0]),
                                       int(b.candidate.indices[1]), b.distance_lb, b.separation,
                                       b.toi] for b in r.bounds]}
            except InfeasibleStepError as exc:
                ls[key] = {"infeasible": str(exc)}
        entry["line_search"] = ls
        res[tag] = entry
        print(tag, {k: len(v) for k, v in entry["broad"].items()},
              {k: len(v) for k, v in act.items()},
              {k: v.get("alpha", "inf") for k, v in ls.items()})
    with open(os.path.join(HERE, "scene.json"), "w") as fh:
        json.dump(res, fh)


if __name__ == "__main__":
    main()
