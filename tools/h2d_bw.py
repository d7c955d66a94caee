import torch,time
d=torch.device('cuda',0)
for mb in (1,8,32,128):
    n=mb*1024*1024//8
    h=torch.randn(n,dtype=torch.float64).pin_memory(); g=torch.empty(n,dtype=torch.float64,device=d)
    for _ in range(3): g.copy_(h,non_blocking=True)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True);e1=torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(10): g.copy_(h,non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/10
    print(f"H2D {mb} MB: {ms:.3f} ms {mb*1.048576e6/ms/1e6:.1f} GB/s")
    e0.record()
    for _ in range(10): h.copy_(g,non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/10
    print(f"D2H {mb} MB: {ms:.3f} ms {mb*1.048576e6/ms/1e6:.1f} GB/s")
