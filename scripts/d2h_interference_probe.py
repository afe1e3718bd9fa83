"""Does a concurrent 4K solve (device-resident, no host packing) slow the
199 MB result copy? D2H GB/s into pinned memory alone vs beside solves.

  python scripts/d2h_interference_probe.py
"""
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import paper_2110_03946_b200 as si  # noqa: E402

W, H, C = 3840, 2160, 3
n = C * W * H
ring = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
src = torch.randn(n, dtype=torch.float64, device="cuda")
cs = torch.cuda.Stream()
cs2 = torch.cuda.Stream()
f = torch.from_numpy(si.synthetic_test_image(W, H, C, 7).data).cuda()
m = torch.from_numpy(si.random_mask(W, H, 0.04, 11).known).cuda()
out = torch.empty((C, H, W), dtype=torch.float64, device="cuda")
sv = si.Solver(0)
ss = torch.cuda.Stream()
o = si.RunOptions(levels=3)


def solve_loop(k, stop):
    for _ in range(k):
        if stop.is_set():
            break
        sv.run_method_device(si.Method.MultilevelOras, f.data_ptr(), m.data_ptr(), W, H, C,
                             out.data_ptr(), o, stream=ss.cuda_stream)


def copies(k=24, split=False):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    cs2.wait_event(e0)
    h = n // 2
    for i in range(k):
        if split:  # two halves on two streams (two copy engines)
            with torch.cuda.stream(cs):
                ring[i % 4][:h].copy_(src[:h], non_blocking=True)
            with torch.cuda.stream(cs2):
                ring[i % 4][h:].copy_(src[h:], non_blocking=True)
        else:
            with torch.cuda.stream(cs):
                ring[i % 4].copy_(src, non_blocking=True)
    e2 = torch.cuda.Event()
    e2.record(cs2)
    cs.wait_event(e2)
    e1.record(cs)
    e1.synchronize()
    return round(k * n * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)


solve_loop(3, threading.Event())
copies(4)
res = {"alone": [copies(), copies()], "alone_split": [copies(split=True), copies(split=True)]}
for rep in range(2):
    for split in (False, True):
        stop = threading.Event()
        t = threading.Thread(target=solve_loop, args=(100, stop))
        t.start()
        res.setdefault("beside_solves" + ("_split" if split else ""), []).append(
            copies(split=split))
        stop.set()
        t.join()
torch.cuda.synchronize()
print(json.dumps(res), flush=True)
