"""MIXED precision (double image / outer iteration, float local CG) against
the FP64 path and the oracle: iteration counts, trace and output deviation,
and device time per 4K frame."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402
from instances import C1, C2, C3, config_instance  # noqa: E402

s = si.Solver(0)
for cfg, name in ((C1, "C1"), (C2, "C2"), (C3, "C3")):
    f, m = config_instance(cfg)
    r64 = s.run_method(si.Method.MultilevelOras, f, m, si.RunOptions(levels=cfg[4]))
    rmx = s.run_method(si.Method.MultilevelOras, f, m,
                       si.RunOptions(levels=cfg[4], precision=si.Precision.MIXED))
    t64 = np.array([r.rel_residual for r in r64.trace.rows])
    tmx = np.array([r.rel_residual for r in rmx.trace.rows])
    d = rmx.image.data - r64.image.data
    s.set_profiling(True)
    s.kernel_stats(reset=True)
    s.run_method(si.Method.MultilevelOras, f, m,
                 si.RunOptions(levels=cfg[4], precision=si.Precision.MIXED))
    st = s.kernel_stats(reset=True)
    s.set_profiling(False)
    print(name, "levels", r64.report.level_iterations, rmx.report.level_iterations,
          "trace rel dev %.2e" % (np.abs(tmx - t64) / t64).max() if tmx.shape == t64.shape else "shape",
          "max-abs %.2e" % np.abs(d).max(), "mse %.2e" % np.mean(d * d),
          "cg its", r64.report.local_cg_iterations, rmx.report.local_cg_iterations,
          "sweep ms", round(st["sweep"]["device_ms"], 3))
