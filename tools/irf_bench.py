"""IRF baseline vs the inclusion solver (the paper's
"Ours vs IRF" comparison) on the same seeded workload queries.

Times, with CUDA events on the launching stream after a warm-up, one
batched solve of Q queries by each GPU method; the IRF's CPU restatement
(oracle/irf_oracle.c, all host threads) runs a bounded sample of the same
stream for scale.  Prints one JSON line per config.

    python tools/irf_bench.py [--configs 0,3] [--queries 1000000] [--max-checks 1000000]
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

from paper_2009_13349_b200 import SolverConfig, irf_batch, solve_batch  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402


def cuda_ms(fn):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    out = fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,3")
    ap.add_argument("--queries", type=int, default=1_000_000)
    ap.add_argument("--max-checks", type=int, default=1_000_000)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for cfg in (int(c) for c in args.configs.split(",")):
        w = W.generate(cfg, 0, args.queries)
        pts = torch.from_numpy(w.points).to(dev)
        kind = torch.from_numpy(w.kind).to(dev)
        sc = SolverConfig(max_checks=args.max_checks)
        ours_ms, ours = cuda_ms(lambda: solve_batch(pts, kind, sc, outputs=("status", "toi", "checks"),
                                                    device=dev))
        irf_ms, irf = cuda_ms(lambda: irf_batch(pts, kind, 1e-6, args.max_checks, 1.0, device=dev))
        line = {"config": cfg, "queries": args.queries, "max_checks": args.max_checks,
                "ours_ms": ours_ms, "ours_qps": args.queries / (ours_ms * 1e-3),
                "ours_checks": int(ours["checks"].sum()),
                "irf_ms": irf_ms, "irf_qps": args.queries / (irf_ms * 1e-3),
                "irf_checks": int(irf["checks"].sum()), "irf_early": int(irf["early"].sum()),
                "irf_over_ours_time": irf_ms / ours_ms,
                "hits_ours": int((ours["status"] == 1).sum()),
                "hits_irf": int((irf["status"] == 1).sum())}
        # CPU: the oracle IRF on consecutive chunks until cpu-seconds elapsed
        import oracle
        threads = len(os.sched_getaffinity(0))
        done, t_cpu, lo, step = 0, 0.0, 0, 32
        while t_cpu < args.cpu_seconds and lo < args.queries:
            n = min(step, args.queries - lo)
            step = min(2 * step, 20_000)  # (heavy workloads: small first chunks)
            t0 = time.perf_counter()
            oracle.irf_batch(w.points[lo:lo + n], w.kind[lo:lo + n], 1e-6, args.max_checks, 1.0,
                             threads=threads)
            t_cpu += time.perf_counter() - t0
            done += n
            lo += n
        line.update({"irf_cpu_qps": done / t_cpu, "irf_cpu_threads": threads,
                     "irf_cpu_sample": done, "irf_gpu_over_cpu": (args.queries / (irf_ms * 1e-3))
                     / (done / t_cpu)})
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
