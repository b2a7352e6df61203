import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W
dev = torch.device("cuda", 0)
w = W.generate_parallel(1)
planted = ~np.isnan(w.planted_t)
pts = torch.from_numpy(np.ascontiguousarray(w.points[planted])).to(dev)
kind = torch.from_numpy(np.ascontiguousarray(w.kind[planted])).to(dev)
ref = None
for lanes in (False, True):
    for rep in range(3):
        r = solve_batch(pts, kind, device=dev, poison=True, lanes=lanes, stats=True, raise_on_error=False)
        torch.cuda.synchronize()
        r = {k: v.cpu().numpy() for k, v in r.items()}
        if ref is None:
            ref = r
        st = r["stats"]
        wrong = np.flatnonzero(r["checks"] != ref["checks"])
        print("planted-only lanes", lanes, "rep", rep, "wrong vs first", len(wrong), wrong[:8],
              "lost", int((r["status"] == 0xEE).sum()), "medium", st[_lib.STAT_MEDIUM_QUERIES],
              "giant", st[_lib.STAT_GIANT_QUERIES], flush=True)
