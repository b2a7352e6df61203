"""One warm solve of a workload sample (for ncu / nsys-less timing).

    python tools/profile_step.py [--config 1] [--queries 1000000] [--heavy-only]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2009_13349_b200 import solve_batch  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--queries", type=int, default=1_000_000)
ap.add_argument("--start", type=int, default=0)
ap.add_argument("--sep", type=float, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--heavy-only", action="store_true")
ap.add_argument("--heavy-blocks", type=int, default=None)
ap.add_argument("--no-lanes", action="store_true")
args = ap.parse_args()
w = W.generate(args.config, args.start, args.queries, separation=args.sep)
dev = torch.device("cuda", 0)
pts = torch.from_numpy(w.points).to(dev)
kind = torch.from_numpy(w.kind).to(dev)
kw = {}
if args.config == 2:
    kw = dict(delta=torch.from_numpy(w.delta).to(dev), max_checks=torch.from_numpy(w.max_checks).to(dev))
from paper_2009_13349_b200 import _lib, solver  # noqa: E402
for r in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(64)]
    info = {}
    e0.record()
    out = solve_batch(pts, kind, outputs=("status", "toi", "checks"), device=dev,
                      separation=w.separation, heavy_only=args.heavy_only, stats=True,
                      heavy_blocks=args.heavy_blocks, lanes=not args.no_lanes,
                      events=ev, info=info, **kw)
    e1.record()
    torch.cuda.synchronize()
    st = out["stats"].tolist()
    t = solver.stage_times(e0, ev, info["event_stages"])
    stages = " stages " + "/".join(f"{nm} {x:.2f}" for nm, x in t.items())
    print(f"rep {r}: {e0.elapsed_time(e1):.2f} ms{stages}  checks {int(out['checks'].sum())} "
          f"lane q {st[_lib.STAT_LANE_QUERIES]} evicted {st[_lib.STAT_LANE_EVICTED]} "
          f"giant {st[_lib.STAT_GIANT_QUERIES]} medium {st[_lib.STAT_MEDIUM_QUERIES]} "
          f"rounds {st[_lib.STAT_ROUNDS]} deferrals {st[_lib.STAT_DEFERRALS]}", flush=True)
