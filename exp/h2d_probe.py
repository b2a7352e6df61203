import torch, time
dev=torch.device('cuda',0)
for mb in (64, 256, 805, 2048):
    n=mb*1024*1024
    h=torch.empty(n,dtype=torch.uint8).pin_memory()
    d=torch.empty(n,dtype=torch.uint8,device=dev)
    d.copy_(h,non_blocking=True); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(8): d.copy_(h,non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(mb,'MB chunks:', 8*n/e0.elapsed_time(e1)/1e6,'GB/s')
