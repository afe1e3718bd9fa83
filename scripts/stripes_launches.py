"""ncu launch list of one direct C5 solve and one G=1 / G=2 stripe solve
(profiler range only around the measured solves):
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
      python scripts/stripes_launches.py"""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2110_03946_b200 as si
from paper_2110_03946_b200 import stripes as S

W, H, C = 7680, 4320, 3
f = si.synthetic_test_image(W, H, C, 7)
m = si.random_mask(W, H, 0.02, 11)
o = si.RunOptions(levels=3)
solver = si.Solver(0)
df = torch.from_numpy(f.data).cuda(); dm = torch.from_numpy(m.known).cuda(); do = torch.empty_like(df)
def direct():
    solver.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(), W, H, C, do.data_ptr(), o)
G = int(os.environ.get("G", "1"))
sv = [solver] + [si.Solver(0) for _ in range(G - 1)]
comms = S.local_comms(sv)
plans = [S.level_plan(si.Method.MultilevelOras, W, H, C, o, G, r)[0] for r in range(G)]
ins = [(torch.from_numpy(np.ascontiguousarray(f.data[:, p.store_lo:p.store_hi])).cuda(),
        torch.from_numpy(np.ascontiguousarray(m.known[p.store_lo:p.store_hi])).cuda(),
        torch.empty((C, p.own_hi - p.own_lo, W), dtype=torch.float64, device="cuda")) for p in plans]
def group():
    def rank(r):
        fi, mi, oi = ins[r]
        S.run_method_striped_device(sv[r], comms[r], si.Method.MultilevelOras, fi.data_ptr(),
                                    mi.data_ptr(), W, H, C, oi.data_ptr(), o)
    th = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
    [t.start() for t in th]; [t.join() for t in th]
for _ in range(3):
    direct(); group()
torch.cuda.synchronize()
torch.cuda.profiler.start()
direct()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("stripes")
group()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
