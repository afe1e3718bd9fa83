import torch, time
n = 3*3840*2160
ring = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
big = [torch.empty(256*1024*1024//8*4, dtype=torch.float64).pin_memory()]
d = torch.randn(n, dtype=torch.float64, device='cuda')
s = torch.cuda.Stream()
def run(bufs, k=16, src=d, kernels=False):
    torch.cuda.synchronize()
    x = torch.randn(64*1024*1024, device='cuda')
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(k):
        with torch.cuda.stream(s):
            bufs[i % len(bufs)][:src.numel()].copy_(src, non_blocking=True)
    e1.record(s)
    if kernels:
        for _ in range(200): x.mul_(1.0001)
    torch.cuda.synchronize()
    return k*src.numel()*8/(e0.elapsed_time(e1)/1e3)/1e9
for name, bufs in (("ring4x199MB", ring), ("one199MB", ring[:1]), ("big1GB_slice199", big)):
    run(bufs, 2)
    print(name, round(run(bufs), 1), "GB/s; with concurrent HBM kernels", round(run(bufs, kernels=True), 1))
