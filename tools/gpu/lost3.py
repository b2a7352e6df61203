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
mode = sys.argv[1]
if mode == "heavy":
    sel = np.flatnonzero(base["checks"] > 1500)
    p2 = pts[torch.from_numpy(sel).to(dev)].contiguous(); k2 = kind[torch.from_numpy(sel).to(dev)].contiguous()
    for rep in range(3):
        r = solve_batch(p2, k2, device=dev, lanes=False, poison=True, stats=True, raise_on_error=False)
        r = {k: v.cpu().numpy() for k, v in r.items()}
        wrong = np.flatnonzero(r["checks"] != base["checks"][sel])
        print("heavy subset", len(sel), "lanes=False rep", rep, "wrong", len(wrong), "medium", r["stats"][_lib.STAT_MEDIUM_QUERIES], flush=True)
else:
    for rep in range(2):
        r = solve_batch(pts, kind, device=dev, poison=True, stats=True, raise_on_error=False)
        r = {k: v.cpu().numpy() for k, v in r.items()}
        wrong = np.flatnonzero(r["checks"] != base["checks"])
        print(mode, "rep", rep, "wrong", len(wrong), "lane ev", r["stats"][_lib.STAT_LANE_EVICTED], "medium", r["stats"][_lib.STAT_MEDIUM_QUERIES], flush=True)
