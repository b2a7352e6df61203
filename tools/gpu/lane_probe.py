"""Lane-tier timing and parity probe: one chunk of a workload, stage times
from the library's events, bit-equality with the group tiers alone."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2009_13349_b200 import solve_batch, _lib, solver
from paper_2009_13349_b200 import workloads as W
cfg = int(sys.argv[1]); n = int(sys.argv[2])
w = W.generate_parallel(cfg, 0, n)
dev = torch.device("cuda", 0)
pts = torch.from_numpy(w.points).to(dev); kind = torch.from_numpy(w.kind).to(dev)
ref = solve_batch(pts, kind, device=dev, lanes=False, raise_on_error=False)
tag = os.path.basename(os.environ.get("TCCD_LIB", "default"))
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(65)]
    ev[0].record()
    info = {}
    r = solve_batch(pts, kind, device=dev, raise_on_error=False, stats=True, events=ev[1:], info=info)
    torch.cuda.synchronize()
    t = solver.stage_times(ev[0], ev[1:], info["event_stages"])
    same = all(torch.equal(r[k], ref[k]) for k in ref)
    st = r["stats"].cpu().numpy()
    lane_checks = int(st[_lib.STAT_LANE_CHECKS] + st[_lib.STAT_LANE_CHECKS + 1])
    tot = sum(t.values())
    print(f"{tag} c{cfg} n={n} rep {rep}: total {tot:.2f} " + " ".join(f"{nm} {x:.2f}" for nm, x in t.items()) +
          f" | lane {lane_checks / (t['lane'] * 1e-3) / 1e9:.1f} Gchecks/s, evicted {st[_lib.STAT_LANE_EVICTED]}, same={same}", flush=True)
