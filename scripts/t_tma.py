import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, paper_2110_03946_b200 as si
from instances import *
s = si.Solver(0)
f, m = config_instance(C1)
for prec in (si.Precision.FP64, si.Precision.FP32):
    o = si.RunOptions(levels=2, precision=prec)
    try:
        r = s.run_method(si.Method.MultilevelOras, f, m, o)
        print(prec, r.report.level_iterations)
    except Exception as e:
        print(prec, 'ERR', e); break
