import torch, time
n=1<<20
for k in (1, 8, 16, 64, 256):
    B=torch.randn(n,k,dtype=torch.float64,device="cuda")
    X=torch.empty(k,n,dtype=torch.float64,device="cuda")
    for _ in range(3): X.copy_(B.t())
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): X.copy_(B.t())
    e1.record(); e1.synchronize()
    t=e0.elapsed_time(e1)/10
    e0.record()
    for _ in range(10): Y=X.clone()
    e1.record(); e1.synchronize()
    t2=e0.elapsed_time(e1)/10
    print(k, "transpose-copy %.1f us (%.0f GB/s)"%(t*1e3, 2*n*k*8/t/1e6), "clone %.1f us"%(t2*1e3))
