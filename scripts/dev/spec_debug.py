import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2110_03946_b200 as si
from paper_2110_03946_b200 import stripes as S

w, h, c = 640, 480, 3
o = si.RunOptions(levels=3, tolerance=1e-4)
frames = [(si.synthetic_test_image(w, h, c, 500 + k), si.random_mask(w, h, d, 600 + k))
          for k, d in enumerate([0.30, 0.02, 0.30, 0.05, 0.02])]
solver = si.Solver(0)
singles = [solver.run_method(si.Method.MultilevelOras, f, m, o) for f, m in frames]
print("single", [list(s.report.level_iterations) for s in singles])
sv = [si.Solver(0), si.Solver(0)]
for spec in (False, True):
    comms = S.local_comms(sv)
    for cm in comms:
        cm.set_speculation(spec)
    for k, (f, m) in enumerate(frames):
        out = si.ImageBuffer(data=np.zeros_like(f.data))
        res = [None, None]
        def rank(r):
            res[r] = S.run_method_striped(sv[r], comms[r], si.Method.MultilevelOras, f, m, o, out=out)
        th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
        [t.start() for t in th]; [t.join() for t in th]
        print("spec", spec, k, list(res[0].report.level_iterations), list(res[1].report.level_iterations),
              "same", np.array_equal(out.data, singles[k].image.data), comms[0].counters())
    for cm in comms:
        cm.close()
# group entry (fresh comms each call)
for k, (f, m) in enumerate(frames):
    img, reps = S.run_method_striped_group(sv, si.Method.MultilevelOras, f, m, o)
    print("group", k, list(reps[0].level_iterations), np.array_equal(img.data, singles[k].image.data))
