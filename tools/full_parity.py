"""Full-size parity: every query of the BASELINE workloads, GPU vs the oracle,
bit for bit on all 13 result fields (status, toi, tol, codom, checks, early,
the 6 witness bounds, level).

    python tools/full_parity.py [--out profiles/r02/full_parity.jsonl] [--quick]

* configs 0, 1, 2, 3 at their BASELINE sizes (10^4, 10^6, 2*10^5, 5*10^7);
* config 4 (10^7 queries) in full at d in {0, 1e-16, 1e-8}, and seeded
  random samples of 10^5 queries at d = 1e-5 and 10^4 at d = 1e-3 (budget-
  bound queries: the oracle needs ~10^3 core-seconds per 10^5 at 1e-5);
* each set through the product path (lane tier + group tiers) and through
  the group tiers alone (lanes=False);
* the reference's acceptance checks where the workload has exact roots
  (config 1's planted half: no false negative, toi <= t*, cf.
  pkg/tests/test_acceptance.py:50-137).

The oracle (oracle/, C restatement of ccdkit._kernel.solve_kernel, pinned to
the reference's own outputs by tests/test_oracle_golden.py) is test
infrastructure: it is the checker here, never the measured path.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FIELDS = ("status", "toi", "tol", "codom", "checks", "early", "witness", "level")


def mismatches(got, ref):
    """Per-field count of queries whose bits differ (error queries compared by
    error class only, as tests/conftest.py:assert_same_results)."""
    st_ref = np.asarray(ref["status"])
    err = st_ref >= 2
    out = {"error_class": int((np.asarray(got["status"]) >= 2).astype(bool).__ne__(err).sum())}
    ok = ~err
    for k in FIELDS:
        a, b = np.asarray(got[k])[ok], np.asarray(ref[k])[ok]
        if k == "witness":
            eq = (a.view(np.int64) == b.view(np.int64)).all(axis=1)
        elif a.dtype.kind == "f":
            eq = a.view(np.int64) == b.view(np.int64)
        else:
            eq = a == b
        out[k] = int((~eq).sum())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "full_parity.jsonl"))
    ap.add_argument("--quick", action="store_true", help="1/100 sizes (smoke run)")
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()

    import torch
    import oracle
    from paper_2009_13349_b200 import solve_batch
    from paper_2009_13349_b200 import workloads as W

    dev = torch.device("cuda", 0)
    div = 100 if args.quick else 1
    cases = [dict(config=0, n=10_000), dict(config=1, n=1_000_000),
             dict(config=2, n=200_000), dict(config=3, n=50_000_000)]
    for d in (0.0, 1e-16, 1e-8):
        cases.append(dict(config=4, n=10_000_000, sep=d))
    cases.append(dict(config=4, n=10_000_000, sep=1e-5, sample=100_000, seed=5))
    cases.append(dict(config=4, n=10_000_000, sep=1e-3, sample=10_000, seed=3))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    fh = open(args.out, "a")
    for c in cases:
        n = max(1, c["n"] // div)
        sep = c.get("sep", 0.0)
        w = W.generate_parallel(c["config"], 0, n, separation=sep if c["config"] == 4 else None)
        desc = f"full {n}"
        if "sample" in c:
            m = max(1, c["sample"] // div)
            idx = np.sort(np.random.default_rng(c["seed"]).choice(n, m, replace=False))
            w = W.Workload(np.ascontiguousarray(w.points[idx]), np.ascontiguousarray(w.kind[idx]),
                           separation=sep, meta=dict(w.meta))
            desc = f"seeded sample {m} of {n} (numpy default_rng({c['seed']}).choice)"
        t0 = time.perf_counter()
        ref = oracle.solve_batch(w.points, w.kind, w.delta, w.max_checks, w.separation, w.t_max,
                                 threads=args.threads)
        t_oracle = time.perf_counter() - t0
        rec = {"config": c["config"], "separation": sep, "queries": int(w.n), "set": desc,
               "oracle_s": round(t_oracle, 2), "oracle_threads": args.threads,
               "hits": int((ref["status"] == 1).sum()), "checks_sum": int(ref["checks"].sum())}
        pts = torch.from_numpy(w.points).to(dev)
        kind = torch.from_numpy(w.kind).to(dev)
        kw = {}
        if c["config"] == 2:
            kw = dict(delta=torch.from_numpy(w.delta).to(dev),
                      max_checks=torch.from_numpy(w.max_checks).to(dev))
        for lanes in (True, False):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = solve_batch(pts, kind, device=dev, separation=w.separation, lanes=lanes,
                            raise_on_error=False, **kw)
            e1.record()
            torch.cuda.synchronize()
            got = {k: v.cpu().numpy() for k, v in r.items()}
            mm = mismatches(got, ref)
            tag = "product" if lanes else "group_tiers_only"
            rec[tag] = {"gpu_ms": round(e0.elapsed_time(e1), 2), "mismatches": mm,
                        "bit_exact": all(v == 0 for v in mm.values())}
            if lanes and c["config"] == 1:
                # the reference's acceptance checks on the product path's results
                planted = ~np.isnan(w.planted_t)
                rec["acceptance"] = {
                    "planted": int(planted.sum()),
                    "false_negatives": int((got["status"][planted] != 1).sum()),
                    "toi_after_root": int((got["toi"][planted] > w.planted_t[planted]).sum())}
            del r, got
        print(json.dumps(rec), flush=True)
        fh.write(json.dumps(rec) + "\n")
        fh.flush()
        del pts, kind, ref
        torch.cuda.empty_cache()
    fh.close()


if __name__ == "__main__":
    main()
