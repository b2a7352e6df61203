"""Strong scaling of config 3 as far as one GPU can show it: for N in
{1, 2, 4, 8} every contiguous shard of the one 5e7-query set (the shards
`bench.py --gpus N` gives its ranks) is solved on this GPU, one after the
other, inputs resident, CUDA events.  The N-GPU step is the slowest shard
(ranks are independent: no collective on the data path), so
Q / max-shard-time is the throughput N such GPUs deliver and
t(1) / (N * max-shard-time) the strong-scaling efficiency the work itself
allows (what it cannot show: N processes sharing one host's PCIe and
cores in the e2e path).

    python tools/strong_scaling_probe.py [--queries 50000000] [--out profiles/r02/strong_scaling_1gpu.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2009_13349_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--queries", type=int, default=50_000_000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default=None)
args = ap.parse_args()
w = W.generate_parallel(3, 0, args.queries)  # (before CUDA is initialised: fork)

import torch  # noqa: E402

from paper_2009_13349_b200 import solve_batch  # noqa: E402
from paper_2009_13349_b200 import shard_bounds  # noqa: E402

dev = torch.device("cuda", 0)
pts = torch.from_numpy(w.points).to(dev)
kind = torch.from_numpy(w.kind).to(dev)
rows = []
t1 = None
for n in (1, 2, 4, 8):
    times = []
    for r in range(n):
        lo, hi = shard_bounds(args.queries, n, r)
        # (like bench.py: one warm-up solve, then the repetitions issued back to
        # back between two events, so the host's launch work overlaps the GPU's)
        solve_batch(pts[lo:hi], kind[lo:hi], outputs=(), hits=True, device=dev, raise_on_error=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            solve_batch(pts[lo:hi], kind[lo:hi], outputs=(), hits=True, device=dev, raise_on_error=False)
        e1.record()
        torch.cuda.synchronize()
        best = e0.elapsed_time(e1) / args.reps
        times.append(round(best, 3))
    step = max(times)
    t1 = step if n == 1 else t1
    rows.append({"n_gpus": n, "shard_queries": args.queries // n, "shard_ms": times, "step_ms": step,
                 "queries_per_s": args.queries / step * 1e3,
                 "strong_scaling_efficiency": round(t1 / (n * step), 4)})
    print(json.dumps(rows[-1]), flush=True)
if args.out:
    with open(args.out, "w") as fh:
        json.dump({"workload": "config 3, one set, contiguous shards (bench.py --gpus N)",
                   "method": "every shard solved on one B200, one after the other; step = slowest shard",
                   "rows": rows}, fh, indent=1)
