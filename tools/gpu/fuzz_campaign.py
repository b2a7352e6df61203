"""Extended randomized parity campaign (GPU box): batches of queries from the
adversarial families of tests/test_fuzz.py, every query with its own delta,
budget, separation and t_max (dyadic ones reach the lane tier, the others the
group tiers), product path and group tiers alone against the oracle, bit for
bit on all 13 fields.

    python tools/gpu/fuzz_campaign.py [--batches 400] [--n 2048] [--out profiles/r02/fuzz_campaign.json]

The oracle (oracle/) is test infrastructure: the checker here.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from conftest import assert_same_results  # noqa: E402
from test_fuzz import BUDGETS, DELTAS, SEPS, _family  # noqa: E402
from paper_2009_13349_b200 import solve_batch  # noqa: E402

TMAX = (1.0, 0.5, 0.25, 2.0 ** -10, 2.0 ** -40, 0.75, 0.3, 0.7)
FIELDS = ("status", "toi", "tol", "codom", "checks", "early", "witness", "level")

ap = argparse.ArgumentParser()
ap.add_argument("--batches", type=int, default=400)
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--seed", type=int, default=20260913349)
ap.add_argument("--out", default=None)
args = ap.parse_args()

dev = torch.device("cuda", 0)
rng = np.random.default_rng(args.seed)
tot_q = tot_checks = lane_q = hits = early = 0
t0 = time.time()
for b in range(args.batches):
    fams = rng.integers(0, 6, rng.integers(1, 4))
    parts = [_family(rng, int(f), args.n // len(fams) + 1) for f in fams]
    pts = np.ascontiguousarray(np.concatenate(parts)[:args.n])
    n = len(pts)
    kind = rng.integers(0, 2, n).astype(np.uint8)
    delta = rng.choice(np.array(DELTAS), n)
    mc = rng.choice(np.array(BUDGETS + (7, 64, 300), dtype=np.int64), n)
    sep = rng.choice(np.array(SEPS), n)
    tm = rng.choice(np.array(TMAX), n)
    ref = oracle.solve_batch(pts, kind, delta, mc, sep, tm)
    for lanes in (True, False):
        got = solve_batch(torch.from_numpy(pts), torch.from_numpy(kind), delta=torch.from_numpy(delta),
                          max_checks=torch.from_numpy(mc), separation=torch.from_numpy(sep),
                          t_max=torch.from_numpy(tm), device=dev, raise_on_error=False, lanes=lanes,
                          stats=lanes)
        if lanes:
            from paper_2009_13349_b200 import _lib
            lane_q += int(got.pop("stats")[_lib.STAT_LANE_QUERIES])
        assert_same_results({k: got[k].numpy() for k in FIELDS}, ref, f"batch {b} lanes={lanes}")
    ok = np.asarray(ref["status"]) < 2
    tot_q += n
    tot_checks += int(np.asarray(ref["checks"])[ok].sum())
    hits += int((np.asarray(ref["status"]) == 1).sum())
    early += int(np.asarray(ref["early"])[ok].sum())
line = {"batches": args.batches, "queries": tot_q, "checks": tot_checks, "hits": hits,
        "budget_returns": early, "lane_tier_queries": lane_q, "paths": ["product", "group tiers alone"],
        "mismatches": 0, "seed": args.seed, "seconds": round(time.time() - t0, 1)}
print(json.dumps(line))
if args.out:
    with open(args.out, "w") as fh:
        fh.write(json.dumps(line) + "\n")
