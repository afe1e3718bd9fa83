import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2110_03946_b200 as si
from paper_2110_03946_b200 import stripes as S
f = si.synthetic_test_image(7680, 4320, 3, 7)
m = si.random_mask(7680, 4320, 0.02, 11)
o = si.RunOptions(levels=3)
solver = si.Solver(0)
single = solver.run_method(si.Method.MultilevelOras, f, m, o)
sv = [solver] + [si.Solver(0) for _ in range(7)]
for G in [int(g) for g in sys.argv[1:]]:
    for k in range(2):
        img, reps = S.run_method_striped_group(sv[:G], si.Method.MultilevelOras, f, m, o)
        d = np.abs(img.data - single.image.data)
        bad = np.nonzero(d.max(axis=(0, 2)))[0]
        print(G, k, reps[0].final_relative_residual, single.report.final_relative_residual,
              "maxdiff", d.max(), "bad rows", bad[:10], bad[-10:] if len(bad) else None, len(bad), flush=True)
