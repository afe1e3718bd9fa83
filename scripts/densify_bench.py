"""Voronoi densification (masks.hpp:155-212) timing: device loop vs the
reference on the host cores, same inputs; checks the masks are identical.

python scripts/densify_bench.py [--sizes 1920x1080,3840x2160] [--no-ref]
Prints one JSON object per size.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1920x1080,3840x2160")
    ap.add_argument("--target", type=float, default=0.04)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--ref-max-pixels", type=int, default=2_100_000)
    args = ap.parse_args()
    solver = si.Solver(0)
    for spec in args.sizes.split(","):
        w, h = (int(v) for v in spec.split("x"))
        f = si.synthetic_test_image(w, h, 3, 7)
        solver.voronoi_densify(f, args.target, 11)  # warm
        times = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            res = solver.voronoi_densify(f, args.target, 11)
            times.append(time.perf_counter() - t0)
        solver.set_profiling(True)
        solver.kernel_stats(reset=True)
        solver.voronoi_densify(f, args.target, 11)
        st = solver.kernel_stats(reset=True)
        solver.set_profiling(False)
        line = {"workload": f"voronoi_densify {w}x{h} RGB target {args.target} seed 11",
                "sweeps": res.sweeps, "known": res.mask.known_count(),
                "gpu_ms": 1e3 * statistics.median(times),
                "gpu_ms_per_sweep": 1e3 * statistics.median(times) / max(res.sweeps, 1),
                "kernel_ms": {k: round(v["device_ms"], 3) for k, v in st.items()
                              if isinstance(v, dict) and v["launches"]}}
        if not args.no_ref and w * h <= args.ref_max_pixels:
            from oracle import pyoracle as P
            if P.ref_available():
                P.ref().ref_set_threads(0)
                t0 = time.perf_counter()
                rm, rs, _ = P.ref_voronoi_densify(f.data, args.target, 11)
                line["ref_ms"] = 1e3 * (time.perf_counter() - t0)
                line["ref_threads"] = P.ref().ref_thread_count()
                line["ref_sweeps"] = rs
                line["mask_identical"] = bool(np.array_equal(rm, res.mask.known))
                line["speedup_vs_ref"] = line["ref_ms"] / line["gpu_ms"]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
