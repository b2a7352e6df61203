"""Which queries does a lanes-on solve leave unwritten?  Outputs are poisoned
first; the lost queries are then classified by their no-lane results."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
dev = torch.device("cuda", 0)
w = W.generate_parallel(cfg, 0, n)
pts = torch.from_numpy(w.points).to(dev)
kind = torch.from_numpy(w.kind).to(dev)
ref = {k: v.cpu().numpy() for k, v in solve_batch(pts, kind, device=dev, lanes=False,
                                                   raise_on_error=False).items()}
for rep in range(3):
    r = solve_batch(pts, kind, device=dev, poison=True, stats=True, raise_on_error=False)
    r = {k: v.cpu().numpy() for k, v in r.items()}
    st = r["stats"]
    lost = np.flatnonzero(r["status"] == 0xEE)
    wrong = np.flatnonzero((r["status"] != 0xEE) & (r["checks"] != ref["checks"]))
    print("rep", rep, "lost", len(lost), "wrong", len(wrong), "lane q", st[_lib.STAT_LANE_QUERIES],
          "done", st[_lib.STAT_LANE_DONE] + st[_lib.STAT_LANE_DONE + 1], "ev", st[_lib.STAT_LANE_EVICTED],
          "medium", st[_lib.STAT_MEDIUM_QUERIES], "giant", st[_lib.STAT_GIANT_QUERIES],
          "tier checks", st[_lib.STAT_TIER_CHECKS:_lib.STAT_TIER_CHECKS + 3], flush=True)
    if len(lost):
        c = ref["checks"][lost]
        print("   lost ref checks: min", c.min(), "median", np.median(c), "max", c.max(),
              "kinds", np.bincount(w.kind[lost], minlength=2), flush=True)
