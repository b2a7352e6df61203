"""Host-side cost of one non-blocking solve_batch call with pinned host
inputs (the e2e path of bench.py): per-call wall time of the Python API and
its cProfile breakdown.

    python tools/e2e_probe.py [--config 0] [--steps 20]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13349_b200 import solve_batch  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=0)
ap.add_argument("--queries", type=int, default=1_000_000)
ap.add_argument("--steps", type=int, default=20)
args = ap.parse_args()
dev = torch.device("cuda", 0)
w = W.generate(args.config, 0, args.queries)
pts_h = torch.from_numpy(w.points).pin_memory()
kind_h = torch.from_numpy(w.kind).pin_memory()


def loop():
    t = []
    res = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res.append(solve_batch(pts_h, kind_h, outputs=("status", "toi"), device=dev,
                               non_blocking=True))
        t.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    return t


loop()
t0 = time.perf_counter()
t = loop()
wall = time.perf_counter() - t0
print(f"per call host ms: {[round(1e3 * x, 2) for x in t]}; wall per step {1e3 * wall / args.steps:.2f} ms")
pr = cProfile.Profile()
pr.enable()
loop()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)

# components: copies alone on the API's copy stream, solves alone (device inputs)
from paper_2009_13349_b200 import solver  # noqa: E402
cs = solver.copy_stream(dev)
bufs = [torch.empty_like(pts_h, device=dev) for _ in range(2)]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(cs):
    e0.record(cs)
    for k in range(args.steps):
        bufs[k % 2].copy_(pts_h, non_blocking=True)
    e1.record(cs)
torch.cuda.synchronize()
print(f"copies alone: {e0.elapsed_time(e1) / args.steps:.2f} ms per step")
pts_d, kind_d = pts_h.to(dev), kind_h.to(dev)
solve_batch(pts_d, kind_d, outputs=("status", "toi"), device=dev)
torch.cuda.synchronize()
e0.record()
for k in range(args.steps):
    solve_batch(pts_d, kind_d, outputs=("status", "toi"), device=dev)
e1.record()
torch.cuda.synchronize()
print(f"solves alone: {e0.elapsed_time(e1) / args.steps:.2f} ms per step")
# copies on cs concurrently with solves on the current stream
e0.record()
cs.wait_event(e0)
with torch.cuda.stream(cs):
    for k in range(args.steps):
        bufs[k % 2].copy_(pts_h, non_blocking=True)
for k in range(args.steps):
    solve_batch(pts_d, kind_d, outputs=("status", "toi"), device=dev)
torch.cuda.current_stream().wait_stream(cs)
e1.record()
torch.cuda.synchronize()
print(f"copies || solves: {e0.elapsed_time(e1) / args.steps:.2f} ms per step")
# with the result copies (status + toi) back to pinned host memory after each solve
st_h = torch.empty(args.queries, dtype=torch.uint8).pin_memory()
toi_h = torch.empty(args.queries, dtype=torch.float64).pin_memory()
for variant in ("d2h on the solve stream", "d2h on a third stream"):
    ds = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    e0.record()
    cs.wait_event(e0)
    with torch.cuda.stream(cs):
        for k in range(args.steps):
            bufs[k % 2].copy_(pts_h, non_blocking=True)
    for k in range(args.steps):
        r = solve_batch(pts_d, kind_d, outputs=("status", "toi"), device=dev)
        if variant.startswith("d2h on the solve"):
            st_h.copy_(r["status"], non_blocking=True)
            toi_h.copy_(r["toi"], non_blocking=True)
        else:
            ds.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(ds):
                st_h.copy_(r["status"], non_blocking=True)
                toi_h.copy_(r["toi"], non_blocking=True)
    torch.cuda.current_stream().wait_stream(cs)
    torch.cuda.current_stream().wait_stream(ds)
    e1.record()
    torch.cuda.synchronize()
    print(f"copies || solves + {variant}: {e0.elapsed_time(e1) / args.steps:.2f} ms per step")
# the API's issue order: copy k on the side stream, then solve k and its
# result copies on the solve stream, then copy k + 1 ...
torch.cuda.synchronize()
e0.record()
cs.wait_event(e0)
for k in range(args.steps):
    with torch.cuda.stream(cs):
        bufs[k % 2].copy_(pts_h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(cs)
    r = solve_batch(bufs[k % 2].view(-1, 8, 3), kind_d, outputs=("status", "toi"), device=dev)
    st_h.copy_(r["status"], non_blocking=True)
    toi_h.copy_(r["toi"], non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"interleaved issue (copy k+1 after result copies k): {e0.elapsed_time(e1) / args.steps:.2f} ms per step")
