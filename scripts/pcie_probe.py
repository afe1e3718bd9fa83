import torch, time
n = 256*1024*1024 // 8 * 4
h = torch.empty(n, dtype=torch.float64).pin_memory(); d = torch.empty(n, dtype=torch.float64, device='cuda')
for name, fn in [('h2d', lambda: d.copy_(h, non_blocking=True)), ('d2h', lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t=time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
    print(name, n*8/dt/1e9, 'GB/s')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.float64).pin_memory(); d2 = torch.empty(n, dtype=torch.float64, device='cuda')
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
print('bidir', 2*n*8/dt/1e9, 'GB/s total')
