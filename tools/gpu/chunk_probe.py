"""Time one config-3 solve (5e7 queries, resident) under the loaded library."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W
cfg = int(sys.argv[1]); n = int(sys.argv[2])
w = W.generate_parallel(cfg, 0, n)
dev = torch.device("cuda", 0)
pts = torch.from_numpy(w.points).to(dev); kind = torch.from_numpy(w.kind).to(dev)
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = solve_batch(pts, kind, device=dev, outputs=("status", "toi"), raise_on_error=False)
    e1.record(); torch.cuda.synchronize()
    print(os.environ.get("TCCD_LIB", "default"), cfg, n, f"{e0.elapsed_time(e1):.1f} ms", flush=True)
