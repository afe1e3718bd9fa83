"""Every BASELINE.json configuration that fits one B200, device-resident,
next to the reference's own run_method on the host cores (oracle/_ref, all
threads), with the GPU result checked against the reference output.

  python scripts/configs_bench.py [--configs c1,c2,c3,c5,c5f] [--no-ref]

c5f is SURVEY.md §8d's forced-sweep C5 variant (tolerance 1e-12,
max_outer_iterations 2): two finest sweeps on the 8K frame.
Prints one JSON object per configuration.
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

CONFIGS = {
    "c1": dict(w=256, h=256, c=1, d=0.05, levels=2),
    "c2": dict(w=1920, h=1080, c=3, d=0.04, levels=2),
    "c3": dict(w=3840, h=2160, c=3, d=0.04, levels=3),
    "c5": dict(w=7680, h=4320, c=3, d=0.02, levels=3),
    "c5f": dict(w=7680, h=4320, c=3, d=0.02, levels=3, tolerance=1e-12, max_outer_iterations=2),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c5,c5f")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    from oracle import pyoracle as P
    if P.ref_available():
        P.use_tuned_reference()  # -march tuned for the host CPU when supported
    solver = si.Solver(0)
    stream = torch.cuda.current_stream()
    for name in args.configs.split(","):
        cfg = CONFIGS[name]
        w, h, c = cfg["w"], cfg["h"], cfg["c"]
        kw = {k: cfg[k] for k in ("tolerance", "max_outer_iterations") if k in cfg}
        opts = si.RunOptions(levels=cfg["levels"], **kw)
        f = si.synthetic_test_image(w, h, c, 7)
        m = si.random_mask(w, h, cfg["d"], 11)
        df = torch.from_numpy(f.data).cuda()
        dm = torch.from_numpy(m.known).cuda()
        out = torch.empty_like(df)

        def run():
            return solver.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(),
                                            w, h, c, out.data_ptr(), opts,
                                            stream=stream.cuda_stream)

        rep = run()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = run()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        line = {"config": name, "workload": f"{w}x{h}x{c}, {cfg['d']:.0%} mask, {cfg['levels']} levels"
                + (f", {kw}" if kw else ""),
                "gpu_ms": statistics.median(times), "frames_per_s": 1e3 / statistics.median(times),
                "level_iterations": list(rep.level_iterations),
                "local_cg_iterations": rep.local_cg_iterations}
        if not args.no_ref:
            from oracle import pyoracle as P
            if P.ref_available():
                P.ref().ref_set_threads(0)
                okw = {k: v for k, v in kw.items()}
                t0 = time.perf_counter()
                ref = P.ref_run_method("mloras", f.data, m.known, levels=cfg["levels"], **okw)
                line["ref_ms"] = 1e3 * (time.perf_counter() - t0)
                line["ref_threads"] = P.ref().ref_thread_count()
                line["speedup_vs_ref"] = line["ref_ms"] / line["gpu_ms"]
                got = out.cpu().numpy()
                d = got - ref.image
                line["max_abs_vs_ref"] = float(np.abs(d).max())
                line["mse_vs_ref"] = float(np.mean(d * d))
                line["finest_iterations_equal"] = ref.iterations == rep.iterations
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
