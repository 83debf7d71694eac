import torch, time
n = 256*1024*1024  # 1 GiB fp32
h = torch.empty(n, pin_memory=True); h2 = torch.empty(n, pin_memory=True)
d = torch.empty(n, device='cuda'); d2 = torch.empty(n, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best=1e9
    for _ in range(reps):
        t0=time.perf_counter(); fn(); torch.cuda.synchronize(); best=min(best,time.perf_counter()-t0)
    return best
gb = n*4/1e9
print("H2D alone GB/s", gb/t(lambda: d.copy_(h, non_blocking=True)))
print("D2H alone GB/s", gb/t(lambda: h2.copy_(d2, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
tb = t(both); print("both: aggregate GB/s", 2*gb/tb, "time", tb)
def chunked():
    k=8; c=n//k
    for i in range(k):
        with torch.cuda.stream(s1 if i%2==0 else s2): d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
print("H2D 2 streams chunked GB/s", gb/t(chunked))
