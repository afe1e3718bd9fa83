"""The paper's comparison (multilevel ORAS vs multilevel CG)
on one B200 and on the reference CPU path, same inputs.

  python scripts/mlcg_bench.py [--sizes 1920x1080,3840x2160] [--no-ref]
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
import torch  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1920x1080,3840x2160")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--ref-max-pixels", type=int, default=2_100_000)
    args = ap.parse_args()
    solver = si.Solver(0)
    stream = torch.cuda.current_stream()
    for spec in args.sizes.split(","):
        w, h = (int(v) for v in spec.split("x"))
        levels = 3 if w * h > 4_000_000 else 2
        f = si.synthetic_test_image(w, h, 3, 7)
        m = si.random_mask(w, h, 0.04, 11)
        df = torch.from_numpy(f.data).cuda()
        dm = torch.from_numpy(m.known).cuda()
        out = torch.empty_like(df)
        line = {"workload": f"{w}x{h} RGB 4% mask, {levels} levels"}
        for name, method in (("mloras", si.Method.MultilevelOras), ("mlcg", si.Method.MultilevelCg)):
            o = si.RunOptions(levels=levels)
            solver.run_method_device(method, df.data_ptr(), dm.data_ptr(), w, h, 3, out.data_ptr(), o,
                                     stream=stream.cuda_stream)
            ts = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rep = solver.run_method_device(method, df.data_ptr(), dm.data_ptr(), w, h, 3,
                                               out.data_ptr(), o, stream=stream.cuda_stream)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            line[f"gpu_{name}_ms"] = statistics.median(ts)
            line[f"gpu_{name}_levels"] = list(rep.level_iterations)
            if not args.no_ref and w * h <= args.ref_max_pixels:
                from oracle import pyoracle as P
                if P.ref_available():
                    P.ref().ref_set_threads(0)
                    t0 = time.perf_counter()
                    P.ref_run_method(name, f.data, m.known, levels=levels,
                                     flavour=2 if name == "mlcg" else 1)
                    line[f"ref_{name}_ms"] = 1e3 * (time.perf_counter() - t0)
        line["gpu_mlcg_over_mloras"] = line["gpu_mlcg_ms"] / line["gpu_mloras_ms"]
        if "ref_mlcg_ms" in line:
            line["ref_mlcg_over_mloras"] = line["ref_mlcg_ms"] / line["ref_mloras_ms"]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
