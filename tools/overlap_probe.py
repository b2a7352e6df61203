"""Does the non_blocking host-input pipeline overlap the next batch's points
copy with the current solve?  Prints host call durations and the copy-stream
timeline against the launching stream.

    python tools/overlap_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2009_13349_b200 import solve_batch, solver  # noqa: E402
from paper_2009_13349_b200 import workloads as W  # noqa: E402

w = W.generate(1, 0, 1_000_000)
dev = torch.device("cuda", 0)
pts_h = torch.from_numpy(w.points).pin_memory()
kind_h = torch.from_numpy(w.kind).pin_memory()
s = torch.cuda.current_stream(dev)
cs = solver.copy_stream(dev)
for hb in (None, 148):
    solve_batch(pts_h, kind_h, outputs=("status", "toi"), device=dev, heavy_blocks=hb)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(s)
    cs.wait_event(t0)
    marks, host = [], []
    for k in range(4):
        a = torch.cuda.Event(enable_timing=True)
        a.record(cs)  # before this step's copy on the copy stream
        h0 = time.perf_counter()
        r = solve_batch(pts_h, kind_h, outputs=("status", "toi"), device=dev, non_blocking=True,
                        heavy_blocks=hb)
        host.append(1e3 * (time.perf_counter() - h0))
        b = torch.cuda.Event(enable_timing=True)
        b.record(cs)  # after this step's copy
        marks.append((a, b, r["ready"]))
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record(s)
    torch.cuda.synchronize()
    print(f"heavy_blocks={hb}: total {t0.elapsed_time(t1) / 4:.2f} ms/step, host call ms "
          + ", ".join(f"{x:.2f}" for x in host))
    for k, (a, b, rd) in enumerate(marks):
        print(f"  step {k}: copy {t0.elapsed_time(a):.2f} -> {t0.elapsed_time(b):.2f} ms")
