python tools/gpu/lane_probe.py 3 50000000 2>&1 | grep -v Warn | tail -1 > gpurun_out/lp25.log
python tools/gpu/lane_probe.py 1 1000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/lp25.log
python -c "
import torch,sys
sys.path.insert(0,'.')
from paper_2009_13349_b200 import solve_batch, _lib
from paper_2009_13349_b200 import workloads as W
w=W.generate_parallel(1); dev=torch.device('cuda',0)
r=solve_batch(torch.from_numpy(w.points).to(dev), torch.from_numpy(w.kind).to(dev), device=dev, stats=True, outputs=('status','toi'))
st=r['stats'].cpu().numpy()
print('c1 lane evicted', st[_lib.STAT_LANE_EVICTED], 'handed', st[_lib.STAT_LANE_HANDED], 'wasted', st[_lib.STAT_LANE_WASTED], 'restarts', st[_lib.STAT_RESTARTS:_lib.STAT_RESTARTS+2])
" >> gpurun_out/lp25.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t25.log 2>&1; echo rc=$? >> gpurun_out/t25.log
