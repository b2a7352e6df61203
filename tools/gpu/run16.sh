for L in default exp/lib_k48.so exp/lib_k32.so exp/lib_k16.so; do
  if [ $L = default ]; then E=""; else E="TCCD_LIB=$L"; fi
  env $E python tools/gpu/lane_probe.py 3 50000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/k.log
  env $E python tools/gpu/lane_probe.py 1 1000000 2>&1 | grep -v Warn | tail -1 >> gpurun_out/k.log
done
python -c "
import torch,sys
sys.path.insert(0,'.')
from paper_2009_13349_b200 import solve_batch, solver
from paper_2009_13349_b200 import workloads as W
w=W.generate_parallel(1)
dev=torch.device('cuda',0)
p=torch.from_numpy(w.points).to(dev); k=torch.from_numpy(w.kind).to(dev)
for lanes in (False, True, False, True):
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    solve_batch(p,k,device=dev,lanes=lanes,outputs=('status','toi'))
    torch.cuda.synchronize(); e0.record()
    solve_batch(p,k,device=dev,lanes=lanes,outputs=('status','toi'))
    e1.record(); torch.cuda.synchronize()
    print('config1 lanes', lanes, e0.elapsed_time(e1))
" >> gpurun_out/k.log 2>&1
