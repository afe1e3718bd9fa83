"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): a 640x480 RGB multilevel ORAS solve through run_method (K1-K5
incl. the TMA + TMEM sweep), the batch entry (graph-mode levels), the
multilevel CG level solver and a 2-rank striped solve on one device."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_03946_b200 as si  # noqa: E402
from paper_2110_03946_b200 import stripes as S  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
f = si.synthetic_test_image(640, 480, 3, 7)
m = si.random_mask(640, 480, 0.05, 11)
s = si.Solver(0)
o = si.RunOptions(levels=3)
r = s.run_method(si.Method.MultilevelOras, f, m, o, reference=f)
print("run_method levels", r.report.level_iterations, "cg", r.report.local_cg_iterations)
if which in ("all", "batch"):
    b = s.run_batch(si.Method.MultilevelOras, [(f, m), (f, m)], o)
    assert np.array_equal(b[0].image.data, r.image.data)
    print("batch ok")
if which in ("all", "cg"):
    c = s.run_method(si.Method.MultilevelCg, f, m, si.RunOptions(levels=2))
    print("mlcg", c.report.iterations)
if which in ("all", "stripes"):
    img, reps = S.run_method_striped_group([s, si.Solver(0)], si.Method.MultilevelOras, f, m, o)
    assert np.array_equal(img.data, r.image.data)
    print("stripes ok")
print("done")
