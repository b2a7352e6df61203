import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W
n=int(sys.argv[1]) if len(sys.argv)>1 else 1000000
w=W.generate(4,0,n,separation=1e-5)
dev=torch.device('cuda',0)
pts=torch.from_numpy(w.points).to(dev); kind=torch.from_numpy(w.kind).to(dev)
for rep in range(2):
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    out=solve_batch(pts,kind,outputs=("status","toi","checks"),device=dev,separation=1e-5,stats=True,raise_on_error=False)
    e1.record(); torch.cuda.synchronize()
    st=out["stats"].tolist()
    print(f"rep {rep}: {e0.elapsed_time(e1):.1f} ms checks {int(out['checks'].sum())} giant {st[_lib.STAT_GIANT_QUERIES]} medium {st[_lib.STAT_MEDIUM_QUERIES]} restarts {st[_lib.STAT_RESTARTS:_lib.STAT_RESTARTS+2]} pool demand {st[_lib.STAT_POOL_DEMAND:_lib.STAT_POOL_DEMAND+2]}", flush=True)
