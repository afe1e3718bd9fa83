"""Solve a few 4K RGB frames (device-resident) — the command profiled by ncu."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--frames", type=int, default=2)
p.add_argument("--precision", default="fp64")
p.add_argument("--size", default="3840x2160")
a = p.parse_args()
w, h = (int(v) for v in a.size.split("x"))
f = si.synthetic_test_image(w, h, 3, 7)
m = si.random_mask(w, h, 0.04, 11)
df = torch.from_numpy(f.data).cuda()
dm = torch.from_numpy(m.known).cuda()
out = torch.empty_like(df)
s = si.Solver(0)
o = si.RunOptions(precision=si.Precision.FP64 if a.precision == "fp64" else si.Precision.FP32)
for _ in range(a.frames):
    rep = s.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(), w, h, 3,
                              out.data_ptr(), o)
torch.cuda.synchronize()
print("levels", rep.level_iterations, "final", rep.final_relative_residual)
