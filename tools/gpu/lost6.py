import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_2009_13349_b200 import solve_batch, _lib, solver
from paper_2009_13349_b200 import workloads as W
dev = torch.device("cuda", 0)
w = W.generate_parallel(1, 0, 200000)
pts = torch.from_numpy(w.points).to(dev)
kind = torch.from_numpy(w.kind).to(dev)
r = solve_batch(pts, kind, device=dev, lanes=False, raise_on_error=False)
torch.cuda.synchronize()
ws = solver._workspaces[("cuda", 0)]
ctr = ws[:4096].cpu().view(torch.int64)
# Counters: q_count[3], q_next[3], rounds, deferred, evicted[3], boxes[3], pool[3] = 17 u64, then phase[3][16]
ph = ctr[17:17 + 48].view(3, 16)
print("light tier debug: classified-already", int(ph[0][13]), "past-cut", int(ph[0][14]), "classified-in-P1", int(ph[0][15]),
      "P3 recheck non-disjoint", int(ph[0][12]), "nn!=1", int(ph[0][11]), "flag sum", int(ph[0][10]), flush=True)
