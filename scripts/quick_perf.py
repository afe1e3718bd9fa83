import sys, time, numpy as np
import os; R=os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R); sys.path.insert(0, os.path.join(R,'tests'))
import paper_2110_03946_b200 as si
from instances import *
s = si.Solver(0)
for cfg, name in [(C1,'C1'),(C2,'C2'),(C3,'C3')]:
    f, m = config_instance(cfg)
    for prec in (si.Precision.FP64, si.Precision.FP32):
        o = si.RunOptions(levels=cfg[4], precision=prec)
        r = s.run_method(si.Method.MultilevelOras, f, m, o)
        ts=[]
        for k in range(3):
            t=time.time(); r = s.run_method(si.Method.MultilevelOras, f, m, o); ts.append(time.time()-t)
        s.set_profiling(True); s.kernel_stats(reset=True)
        r = s.run_method(si.Method.MultilevelOras, f, m, o)
        st = s.kernel_stats(reset=True); s.set_profiling(False)
        print(name, prec.name, 'levels', r.report.level_iterations, 'trace', [x.rel_residual for x in r.trace.rows], 'host ms', [round(t*1e3,1) for t in ts], 'cg its', r.report.local_cg_iterations, 'fails', r.report.local_failures)
        print('   ', {k:(v['launches'], round(v['device_ms'],3)) for k,v in st.items() if isinstance(v, dict)})
