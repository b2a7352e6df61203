import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import oracle
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W
dev = torch.device("cuda", 0)
w = W.generate_parallel(1)
c_ref = None
sel = np.arange(w.n)
ref = oracle.solve_batch(w.points[:200000], w.kind[:200000], threads=16)
pts = torch.from_numpy(w.points[:200000]).to(dev)
kind = torch.from_numpy(w.kind[:200000]).to(dev)
for lanes in ((False,) if sys.argv[1] == "noflag" else (True,)):
    r = solve_batch(pts, kind, device=dev, lanes=lanes, poison=True, raise_on_error=False)
    r = {k: v.cpu().numpy() for k, v in r.items()}
    wrong = np.flatnonzero(r["checks"] != ref["checks"])
    print(sys.argv[1], "lanes", lanes, "wrong", len(wrong), wrong[:10], r["checks"][wrong[:5]], ref["checks"][wrong[:5]],
          "status", r["status"][wrong[:5]], ref["status"][wrong[:5]], "toi", r["toi"][wrong[:5]], ref["toi"][wrong[:5]],
          "level", r["level"][wrong[:5]], "early", r["early"][wrong[:5]], "wit", r["witness"][wrong[:2]], flush=True)
    if len(wrong):
        sub = wrong[:64]
        r2 = solve_batch(pts[torch.from_numpy(sub).to(dev)].contiguous(), kind[torch.from_numpy(sub).to(dev)].contiguous(), device=dev, lanes=lanes, raise_on_error=False)
        print("   alone: wrong", int((r2["checks"].cpu().numpy() != ref["checks"][sub]).sum()), "of", len(sub), flush=True)
