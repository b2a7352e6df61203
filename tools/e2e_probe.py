"""Per-step breakdown of the end-to-end (host buffers) solve: H2D copy alone,
device-resident solve, and the host-input solve through the public API.

    python tools/e2e_probe.py [--config 1] [--queries 1000000] [--steps 6]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13349_b200 import solve_batch, solver  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--queries", type=int, default=1_000_000)
ap.add_argument("--steps", type=int, default=6)
args = ap.parse_args()
w = W.generate(args.config, 0, args.queries)
dev = torch.device("cuda", 0)
pts_h = torch.from_numpy(w.points).pin_memory()
kind_h = torch.from_numpy(w.kind).pin_memory()
pts = pts_h.to(dev)
kind = kind_h.to(dev)
s = torch.cuda.current_stream(dev)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record(s)
    fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b), 1e3 * (time.perf_counter() - t0)


solve_batch(pts, kind, outputs=("status", "toi"), device=dev)
for k in range(args.steps):
    h2d = timed(lambda: pts_h.to(dev, non_blocking=True))
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    dev_solve = timed(lambda: (evs[0].record(s), solve_batch(pts, kind, outputs=("status", "toi"),
                                                             device=dev, events=evs[1:])))
    stages = [evs[j].elapsed_time(evs[j + 1]) for j in range(4)]
    host_solve = timed(lambda: solve_batch(pts_h, kind_h, outputs=("status", "toi"), device=dev))
    ws = solver._workspaces.get(("cuda", 0))
    hb = solver.default_heavy_blocks(dev, args.queries, 1_000_000)
    print(f"  heavy_blocks {hb}, workspace {ws.numel() / 2**30:.2f} GiB, "
          f"free {torch.cuda.mem_get_info(dev)[0] / 2**30:.1f} GiB")
    print("  stages prologue/light/medium/giant ms: " + " / ".join(f"{x:.2f}" for x in stages))
    print(f"step {k}: h2d {h2d[0]:.2f} ms ({193e-3 * args.queries / 1e3 / h2d[0]:.1f} GB/s), "
          f"device solve {dev_solve[0]:.2f} ms, host-input solve {host_solve[0]:.2f} ms "
          f"(wall {host_solve[1]:.2f})", flush=True)

# host-side cost of the pieces solve_batch runs before its launches
for k in range(5):
    t0 = time.perf_counter()
    torch.cuda.mem_get_info(dev)
    t1 = time.perf_counter()
    solver.default_heavy_blocks(dev, args.queries, 1_000_000)
    t2 = time.perf_counter()
    solver.sm_count(dev)
    t3 = time.perf_counter()
    print(f"mem_get_info {1e3 * (t1 - t0):.3f} ms, default_heavy_blocks {1e3 * (t2 - t1):.3f} ms, "
          f"sm_count {1e3 * (t3 - t2):.3f} ms")
