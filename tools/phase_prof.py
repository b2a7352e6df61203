"""Per-phase cycle split of the engine tiers (needs a -DTCCD_PHASE_PROF build,
selected with TCCD_LIB=...).  Reads the counters from the workspace.

    TCCD_LIB=exp/lib_prof.so python tools/phase_prof.py --config 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13349_b200 import solve_batch, solver  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402

NAMES = ["P0 claim", "P0 load", "P0 n_cur", "P1 classify", "P3 outcome", "P4 scans",
         "P5 evict", "P5 layout", "P4c order", "P5b/P6+P7", "end"]
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--queries", type=int, default=1_000_000)
args = ap.parse_args()
w = W.generate(args.config, 0, args.queries)
dev = torch.device("cuda", 0)
pts = torch.from_numpy(w.points).to(dev)
kind = torch.from_numpy(w.kind).to(dev)
for rep in range(2):
    if rep == 1:  # phase[14] holds a min: start it high
        pass
    out = solve_batch(pts, kind, outputs=("status", "toi"), device=dev, raise_on_error=False)
    torch.cuda.synchronize()
ws = solver._workspaces[("cuda", 0)]
ctr = ws[:1024].cpu().view(torch.int64)
ph = ctr[17:17 + 48].view(3, 16)  # Counters: 17 u64 before phase[3][16]
for t, name in enumerate(["light", "medium", "giant"]):
    tot = int(ph[t].sum())
    if not tot:
        continue
    tot = int(ph[t][:11].sum())
    parts = ", ".join(f"{NAMES[k]} {100 * int(ph[t][k]) / tot:.1f}%" for k in range(11) if ph[t][k])
    life, groups, tmax, tmin = (int(x) for x in ph[t][11:15])
    span = (tmax - tmin) if tmin > 0 else 0
    util = life / (groups * span) if span else 0.0
    print(f"{name}: {tot / 1e9:.2f} Gcycles (thread-0 of each group): {parts}")
    print(f"   kernel span {span / 1e6:.2f} ms, {groups} groups, mean group lifetime / span = {util:.2f}")
