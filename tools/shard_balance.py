"""Per-shard solve times of the weak-scaling bench (rank r solves queries
[r*Q, (r+1)*Q) of the workload stream), all on this one GPU: the 8-GPU
bench's time is the max over ranks, so mean / max of these is the weak-
scaling efficiency the shards' own work allows (the GPUs being
independent, with no collective on the data path).

    python tools/shard_balance.py [--config 1] [--ranks 8] [--queries 1000000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13349_b200 import solve_batch  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--queries", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
dev = torch.device("cuda", 0)
ms = []
for r in range(args.ranks):
    w = W.generate(args.config, r * args.queries, args.queries)
    pts = torch.from_numpy(w.points).to(dev)
    kind = torch.from_numpy(w.kind).to(dev)
    solve_batch(pts, kind, outputs=("status", "toi"), device=dev)
    torch.cuda.synchronize()
    t = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solve_batch(pts, kind, outputs=("status", "toi"), device=dev)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    ms.append(min(t))
    print(json.dumps({"rank": r, "ms": ms[-1]}), flush=True)
mean = sum(ms) / len(ms)
print(json.dumps({"config": args.config, "ranks": args.ranks, "queries_per_rank": args.queries,
                  "ms_per_rank": ms, "mean_ms": mean, "max_ms": max(ms),
                  "weak_scaling_efficiency_bound": mean / max(ms)}), flush=True)
