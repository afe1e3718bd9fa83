"""Cost of the stripe decomposition on ONE B200 (BASELINE configs[4] shape):
the 8K RGB frame solved directly (run_method_device) and as G virtual ranks
(G host threads -- the local group's persistent C++ workers, or Python
threads with --py-threads -- one context and stream each, local
communicator: device copies ordered by events, no kernel waits on another
rank's kernel).  All
ranks share the one GPU, so this measures the decomposition's overhead
(extra launches, halo copies, per-iteration all-gathers and host
decisions), not multi-GPU scaling.  Device time: every rank's stream waits
on a start event, the main stream waits on every rank's end event.

  python scripts/stripes_overhead.py [--forced] [--reps 10]
"""
import argparse
import json
import os
import statistics
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402
from paper_2110_03946_b200 import stripes as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--forced", action="store_true")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--config", choices=["c5", "c3"], default="c5")
ap.add_argument("--ranks", default="1,2,4")
ap.add_argument("--copy-out", action="store_true", help="each rank copies its rows to an "
                "output buffer (else they stay in place: si_stripe_result_rows)")
ap.add_argument("--py-threads", action="store_true", help="one Python thread per rank "
                "calling si_run_method_striped_device (else si_run_method_striped_local_device)")
ap.add_argument("--sync", action="store_true", help="speculation off: one host round trip "
                "per outer-iteration decision")
a = ap.parse_args()
if a.config == "c3":  # configs[2]: 4K RGB, 4%
    W, H, C, dens = 3840, 2160, 3, 0.04
else:               # configs[4]: 8K RGB, 2%
    W, H, C, dens = 7680, 4320, 3, 0.02
f = si.synthetic_test_image(W, H, C, 7)
m = si.random_mask(W, H, dens, 11)
o = (si.RunOptions(levels=3, tolerance=1e-12, max_outer_iterations=2) if a.forced
     else si.RunOptions(levels=3))
main = torch.cuda.current_stream()


def timed(run_once, streams):
    for _ in range(3):
        run_once()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for st in streams:
            st.wait_event(e0)
        run_once()
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            main.wait_event(e)
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = {"workload": f"{W}x{H} RGB {dens:.0%} 3 levels" + (" forced 2 sweeps" if a.forced else ""),
       "speculation": not a.sync, "output": "copied" if a.copy_out else "in place",
       "ranks_driven_by": "python threads" if a.py_threads else "si_run_method_striped_local_device"}
solver = si.Solver(0)
df = torch.from_numpy(f.data).cuda()
dm = torch.from_numpy(m.known).cuda()
do = torch.empty_like(df)
rep = None


def direct():
    global rep
    rep = solver.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(), W, H,
                                   C, do.data_ptr(), o, stream=main.cuda_stream)


out["direct_ms"] = timed(direct, [])
out["levels"] = list(rep.level_iterations)
ref = do.cpu().numpy()
for G in (int(g) for g in a.ranks.split(",")):
    solvers = [solver] + [si.Solver(0) for _ in range(G - 1)]
    comms = S.local_comms(solvers)
    for cm in comms:
        cm.set_speculation(not a.sync)
    streams = [torch.cuda.Stream() for _ in range(G)]
    plans = [S.level_plan(si.Method.MultilevelOras, W, H, C, o, G, r)[0] for r in range(G)]
    ins = [(torch.from_numpy(np.ascontiguousarray(f.data[:, p.store_lo:p.store_hi])).cuda(),
            torch.from_numpy(np.ascontiguousarray(m.known[p.store_lo:p.store_hi])).cuda(),
            torch.empty((C, p.own_hi - p.own_lo, W), dtype=torch.float64, device="cuda"))
           for p in plans]
    torch.cuda.synchronize()

    def group():
        if not a.py_threads:  # one call: ranks 1.. on the group's persistent C++ threads
            S.run_method_striped_local_device(
                solvers, comms, si.Method.MultilevelOras, [i[0].data_ptr() for i in ins],
                [i[1].data_ptr() for i in ins], W, H, C,
                [i[2].data_ptr() for i in ins] if a.copy_out else None, o,
                streams=[st.cuda_stream for st in streams])
            return

        def rank(r):
            fi, mi, oi = ins[r]
            S.run_method_striped_device(solvers[r], comms[r], si.Method.MultilevelOras,
                                        fi.data_ptr(), mi.data_ptr(), W, H, C,
                                        oi.data_ptr() if a.copy_out else None, o,
                                        stream=streams[r].cuda_stream)
        if G == 1:  # one rank: no thread to start
            rank(0)
            return
        th = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    ms = timed(group, streams)
    rows = [ins[r][2] if a.copy_out else S.result_rows_tensor(solvers[r], C, W)
            for r in range(G)]
    same = all(np.array_equal(rows[r].cpu().numpy(), ref[:, p.own_lo:p.own_hi])
               for r, p in enumerate(plans))
    out[f"G{G}"] = {"ms": ms, "ratio_to_direct": ms / out["direct_ms"], "bit_identical": same,
                    "store_rows": [[p.store_lo, p.store_hi] for p in plans],
                    "comm": comms[0].counters()}
    for cm in comms:
        cm.close()
print(json.dumps(out))
