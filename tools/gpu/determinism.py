"""Run-to-run determinism probe: full config 1 solved several times with and
without the lane tier; differing queries are checked against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import oracle
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dev = torch.device("cuda", 0)
w = W.generate_parallel(cfg)
pts = torch.from_numpy(w.points).to(dev)
kind = torch.from_numpy(w.kind).to(dev)
for lanes in (True, False):
    runs = []
    for rep in range(3):
        r = solve_batch(pts, kind, device=dev, lanes=lanes, stats=True, raise_on_error=False)
        runs.append({k: v.cpu().numpy() for k, v in r.items()})
    st = runs[0]["stats"]
    print("lanes", lanes, "stats restarts", st[_lib.STAT_RESTARTS:_lib.STAT_RESTARTS+2],
          "demand", st[_lib.STAT_POOL_DEMAND:_lib.STAT_POOL_DEMAND+2],
          "lane evicted", st[_lib.STAT_LANE_EVICTED], "giant", st[_lib.STAT_GIANT_QUERIES],
          "medium", st[_lib.STAT_MEDIUM_QUERIES], flush=True)
    bad = np.zeros(w.n, bool)
    for r in runs[1:]:
        for k in ("status", "toi", "checks", "level"):
            a, b = runs[0][k], r[k]
            bad |= (a.view(np.uint8).reshape(w.n, -1) != b.view(np.uint8).reshape(w.n, -1)).any(axis=1)
    idx = np.flatnonzero(bad)
    print("lanes", lanes, "nondeterministic queries:", len(idx), idx[:20], flush=True)
    if len(idx):
        sub = idx[:200]
        ref = oracle.solve_batch(w.points[sub], w.kind[sub])
        for j, r in enumerate(runs):
            ok = (r["checks"][sub] == ref["checks"]) & (r["status"][sub] == ref["status"])
            print("  run", j, "matches oracle on", int(ok.sum()), "of", len(sub),
                  "checks", r["checks"][sub[:5]], "ref", ref["checks"][:5], flush=True)
