"""BASELINE config 4: minimum-separation sweep.  10^7 queries drawn as config 3
(own seed stream), solved at each d in {0, 1e-16, 1e-8, 1e-5, 1e-3}; reports
queries/s, the collision rate and its change with d, checks per query, and the
solve's algorithmic FP64 rate (sum_q P_kind + checks_q * F_kind).

Filters follow the reference (inclusion.py:96-122): CCD constants at d = 0,
MSCCD constants for d > 0.  Large d is budget-bound (every query that is not
separated by more than d spends m_I = 10^6 checks), so each d runs on the
first --queries[d] queries of the stream (full 10^7 where that finishes in
seconds) and says which.  The CPU port (oracle/, all host threads) is timed on
a small prefix of the same sample and checked bit-exact against the GPU
results on it.

    python tools/sweep_c4.py [--full] [--out profiles/r02/sweep_c4.jsonl]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: CPU baseline + parity check only)
from paper_2009_13349_b200 import _lib, solve_batch  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402

F_CHECK = {0: 200, 1: 174}
P_QUERY = {0: 248, 1: 222}
SEPS = (0.0, 1e-16, 1e-8, 1e-5, 1e-3)
# queries per d (default run): budget-bound d values get a prefix sample
DEFAULT_N = {0.0: 10_000_000, 1e-16: 10_000_000, 1e-8: 10_000_000, 1e-5: 1_000_000, 1e-3: 100_000}
CPU_N = {0.0: 100_000, 1e-16: 100_000, 1e-8: 100_000, 1e-5: 2_000, 1e-3: 200}

ap = argparse.ArgumentParser()
ap.add_argument("--full", action="store_true", help="all 10^7 queries at every d")
ap.add_argument("--scale", type=float, default=1.0, help="multiply the per-d sample sizes")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--out", default=None)
args = ap.parse_args()

dev = torch.device("cuda", 0)
threads = len(os.sched_getaffinity(0))
base = W.generate_parallel(4, 0, W.CONFIGS[4]["n"] if args.full else int(max(DEFAULT_N.values()) * args.scale))
pts_all = torch.from_numpy(base.points).to(dev)
kind_all = torch.from_numpy(base.kind).to(dev)
rows = []
rate0 = None
for d in SEPS:
    n = W.CONFIGS[4]["n"] if args.full else min(int(DEFAULT_N[d] * args.scale), base.n)
    pts, kind = pts_all[:n], kind_all[:n]
    out = solve_batch(pts, kind, device=dev, separation=d, stats=True, raise_on_error=False)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solve_batch(pts, kind, outputs=("status", "toi"), device=dev, separation=d,
                    raise_on_error=False)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    t = min(times)
    st = out["status"].cpu().numpy()
    checks = out["checks"].cpu().numpy()
    k = base.kind[:n]
    flops = float(np.sum(np.where(k == 0, P_QUERY[0] + checks * F_CHECK[0],
                                  P_QUERY[1] + checks * F_CHECK[1]).astype(np.float64)))
    rate = float((st == 1).mean())
    if rate0 is None:
        rate0 = rate
    # CPU port on a prefix, bit-exact check of the GPU results there
    nc = min(CPU_N[d], n)
    t0 = time.perf_counter()
    ref = oracle.solve_batch(base.points[:nc], base.kind[:nc], 1e-6, 1_000_000, d, 1.0,
                             threads=threads)
    tc = time.perf_counter() - t0
    same = (np.array_equal(ref["status"], st[:nc]) and
            np.array_equal(ref["toi"].view(np.int64), out["toi"][:nc].cpu().numpy().view(np.int64)) and
            np.array_equal(ref["checks"], checks[:nc]))
    s = [int(x) for x in out["stats"].tolist()]
    row = {"d": d, "queries": n, "sample": "full 10^7" if n == W.CONFIGS[4]["n"] else f"first {n} of 10^7",
           "gpu_s": t, "queries_per_s": n / t, "collision_rate": rate,
           "collision_rate_change_vs_d0": rate - rate0,
           "early_terminated": int(out["early"].cpu().numpy().sum()),
           "mean_checks": float(checks.mean()), "max_checks": int(checks.max()),
           "checks_per_s": float(checks.sum()) / t,
           "solve_tflops": flops / t / 1e12,
           "boxes_per_tier": s[_lib.STAT_BOXES:_lib.STAT_BOXES + 3],
           "lane_queries": s[_lib.STAT_LANE_QUERIES], "lane_handed_over": s[_lib.STAT_LANE_HANDED],
           "medium_tier_queries": s[_lib.STAT_MEDIUM_QUERIES],
           "giant_tier_queries": s[_lib.STAT_GIANT_QUERIES],
           "handover_restarts": s[_lib.STAT_RESTARTS:_lib.STAT_RESTARTS + 2],
           "cpu_port": {"queries": nc, "threads": threads, "queries_per_s": nc / tc,
                        "bit_exact_vs_gpu": bool(same)}}
    rows.append(row)
    print(json.dumps(row), flush=True)
if args.out:
    with open(args.out, "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")
