import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W
dev = torch.device("cuda", 0)
w = W.generate_parallel(1)
pts = torch.from_numpy(w.points).to(dev)
kind = torch.from_numpy(w.kind).to(dev)
base = {k: v.cpu().numpy() for k, v in solve_batch(pts, kind, device=dev, lanes=False, raise_on_error=False).items()}
def run(sel, lanes, tag):
    s = torch.from_numpy(sel).to(dev)
    r = solve_batch(pts[s].contiguous(), kind[s].contiguous(), device=dev, lanes=lanes, poison=True, stats=True, raise_on_error=False)
    r = {k: v.cpu().numpy() for k, v in r.items()}
    wrong = np.flatnonzero(r["checks"] != base["checks"][sel])
    c = base["checks"][sel][wrong]
    print(tag, len(sel), "wrong", len(wrong), "ref checks of wrong: min", c.min() if len(c) else None,
          "max", c.max() if len(c) else None, "got", r["checks"][wrong[:6]], "ref", c[:6],
          "medium", r["stats"][_lib.STAT_MEDIUM_QUERIES], "giant", r["stats"][_lib.STAT_GIANT_QUERIES], flush=True)
perm = np.random.default_rng(1).permutation(w.n)
if sys.argv[1] == "perm":
    run(perm, False, "permuted lanes=False")
    run(perm, True, "permuted lanes=True")
else:
    c = base["checks"]
    run(np.flatnonzero(c < 1000), True, "light-only (<1000 checks)")
    run(np.flatnonzero((c >= 1000) & (c < 50000)), True, "medium-ish (1e3..5e4)")
    run(np.flatnonzero(c >= 50000), True, "giant-ish (>=5e4)")
