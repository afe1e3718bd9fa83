"""Micro-benchmark of one 4K RGB finest-level sweep (K2) on the device.

  python scripts/sweep_micro.py [--fixed] [--precision fp64|fp32] [--reps 5]

--fixed forces every local CG to run exactly 30 iterations (tolerance 1e-300),
which makes timings of kernel variants comparable independent of numerics.
Prints ms per sweep, CTA-iterations, and ns per CTA-iteration.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402
from paper_2110_03946_b200 import _lib as L  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--fixed", action="store_true")
p.add_argument("--precision", default="fp64")
p.add_argument("--reps", type=int, default=5)
p.add_argument("--size", default="3840x2160")
a = p.parse_args()
w, h = (int(v) for v in a.size.split("x"))
prec = 0 if a.precision == "fp64" else 1
dt = torch.float64 if prec == 0 else torch.float32
f = si.synthetic_test_image(w, h, 3, 7)
m = si.random_mask(w, h, 0.04, 11)
s = si.Solver(0)
opts = si.RunOptions(precision=prec)
if a.fixed:
    opts.local = si.SolverConfig(1e-300, 30, 30)
# u = the prolongated initial guess of a real solve is not needed: b itself is
# a valid iterate (u = b at known pixels, 0 elsewhere).
b = torch.from_numpy(np.where(m.known[None] != 0, f.data, 0.0)).to("cuda", dt)
u = b.clone()
un = torch.empty_like(u)
dm = torch.from_numpy(m.known).cuda()
st = torch.cuda.Stream()
o = opts.to_c()
fails, its = C.c_longlong(), C.c_longlong()
nby = si.partition_domain(w, h, 32, 6).blocks_y
lib = L.load()


def sweep():
    return lib.si_device_sweep_rows(s.handle, dm.data_ptr(), b.data_ptr(), u.data_ptr(),
                                    un.data_ptr(), w, h, 3, 32, 6, 0, nby, 1, C.byref(o), 1,
                                    C.byref(fails), C.byref(its), C.c_void_p(st.cuda_stream))


torch.cuda.synchronize()
assert sweep() == 0
times = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    assert sweep() == 0
    e1.record(st)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = float(np.median(times))
print(f"sweep {a.precision} fixed={a.fixed}: {ms:.3f} ms, CTA-iterations {its.value}, "
      f"{ms * 1e6 / max(its.value, 1):.2f} ns/CTA-iteration, failures {fails.value}")
