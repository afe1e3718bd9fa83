#!/usr/bin/env python
"""Benchmark: 4K RGB multilevel-ORAS inpainting frames/s on B200 (BASELINE.json).

A step is one full solve of one 3840x2160 RGB frame with a 4% random mask
(BASELINE.json configs[2], the paper headline): pyramid + every level's
outer ORAS iterations to the reference's residual tolerance (1e-3 finest,
1e-2 coarse, 3 levels, 32x32 blocks, overlap 6, alpha 0.25), exactly the
reference's run_method(Method::MultilevelOras) with default RunOptions.

  value : frames/s with inputs resident in HBM (si_run_method_device),
          --inflight independent frames at a time (default 4: one context,
          stream and host thread each), CUDA events on the launching stream
          bracketing every lane's stream, max over ranks.
  e2e   : frames/s through the public host batch API (si_run_method_batch)
          from pinned host buffers, H2D of each frame's inputs and D2H of its
          result inside the timing.
Multi-GPU (torchrun): independent frames per rank (configs[3]); no
collective on the data path ("scaling": "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# measured DFMA peak (scripts/fp64_peak.cu, profiles/r02_fp64_peak.json)
FP64_PEAK_TF = 34.2
METRIC = "4K RGB inpaint frames/s at fixed residual tol; fraction of HBM roofline"
W4K, H4K, C4K, DENSITY, LEVELS = 3840, 2160, 3, 0.04, 3


# One config dict for both arms (the driver compares them verbatim).
CONFIG = {"workload": "3840x2160 RGB, 4% random mask, 3-level ORAS, tol 1e-3 (BASELINE configs[2]); "
                      "per rank independent frames (configs[3])",
          "block": 32, "overlap": 6, "alpha": 0.25, "levels": LEVELS,
          "seeds": "image 7+k, mask 11+k (frame k = rank*64 + j)",
          "l2": "inputs larger than L2 (199 MB f64 input, ~0.8 GB working set)"}


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json (driver-measured copy bandwidth),
    else the B200_PROFILING.md fallback."""
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(peaks["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback"


def level_sizes(w, h, levels):
    """build_pyramid's level pixel counts (multilevel.hpp:90-93), finest first."""
    out = [(w, h)]
    while len(out) < levels and out[-1][0] >= 2 and out[-1][1] >= 2:
        out.append(((out[-1][0] + 1) // 2, (out[-1][1] + 1) // 2))
    return [a * b for a, b in out]


def survey_frame_bytes(level_iters, w=W4K, h=H4K, c=C4K, s=8):
    """Algorithmic HBM bytes of one frame by SURVEY.md §8d: per level k_L sweeps
    ((2Cs+1) N_L each), k_L+1 residual checks and one r0 pass ((Cs+1) N_L
    each), the restrictions (Cs+1)(N_L + N_{L+1}) and the prolongations plus
    snap Cs N_{L+1} + (2Cs+1) N_L."""
    n = level_sizes(w, h, len(level_iters))
    tot = 0.0
    for lvl, k in enumerate(level_iters):
        tot += (k * (2 * c * s + 1) + (k + 2) * (c * s + 1)) * n[lvl]
    for lvl in range(len(n) - 1):
        tot += (c * s + 1) * (n[lvl] + n[lvl + 1])
        tot += c * s * n[lvl + 1] + (2 * c * s + 1) * n[lvl]
    return tot


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--precision", default="fp64", choices=["fp64", "fp32", "mixed"])
    p.add_argument("--frames", type=int, default=4, help="distinct frames per rank")
    # frames in flight (round 2, 4K fp64, frames/s): 1 -> 325, 2 -> 340, 3 -> 343, 4 -> 346
    p.add_argument("--inflight", type=int, default=4,
                   help="frames in flight per rank (one context, stream and host thread each)")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-c5", action="store_true", help="skip the configs[4] stripe leg")
    p.add_argument("--selfcheck", action="store_true",
                   help="launch/rendezvous check only (gloo, no GPU): rank 0 prints n_gpus")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def frame_seeds(rank, j):
    """Frame k = rank*64 + j uses seeds (7+k, 11+k) as SURVEY.md §8d C4."""
    k = rank * 64 + j
    return 7 + k, 11 + k


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled through NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int, period_s: float = 0.005):
        self.device = device
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = None
        self._thread = None
        self.error = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() \
                else self.device
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons",
                                  getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
        except Exception as e:  # NVML unavailable: report, never fail the bench
            self.error = str(e)[:120]
            return
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    if get_reasons is not None:
                        bits = get_reasons(h)
                        for bit, name in self.REASONS.items():
                            if bits & bit:
                                self.reasons.add(name)
                except Exception:
                    pass
                self._stop.wait(self.period)

        self._thread = threading.Thread(target=run, daemon=True)
        self._thread.start()

    def stop(self):
        if self._thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["nvml unavailable: " + (self.error or "?")]}
        self._stop.set()
        self._thread.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU legs
def cpu_reference_run(frames, steps, warmup, budget_s):
    """Time the reference's own CPU run_method (oracle/_ref, all host threads);
    falls back to the single-threaded C restatement when _ref is absent."""
    from oracle import pyoracle as P
    build = None
    if P.ref_available():
        build = P.use_tuned_reference()
        lib = P.ref()
        lib.ref_set_threads(0)
        cores = int(lib.ref_thread_count())
        kind = "reference"

        def solve(f, m):
            return P.ref_run_method("mloras", f, m, levels=LEVELS)
    else:
        cores, kind = 1, "port"

        def solve(f, m):
            return P.oracle_solve(f, m, levels=LEVELS)
    times = []
    t_start = time.perf_counter()
    iters = None
    for s in range(warmup + steps):
        f, m = frames[s % len(frames)]
        t0 = time.perf_counter()
        res = solve(f, m)
        dt = time.perf_counter() - t0
        iters = res.iterations
        if s >= warmup:
            times.append(dt)
        if time.perf_counter() - t_start > budget_s and times:
            break
    return {"times": times, "cores": cores, "kind": kind, "finest_iterations": iters,
            "build": build}


def host_frames(n, rank=0):
    import paper_2110_03946_b200 as si
    out = []
    for j in range(n):
        sf, sm = frame_seeds(rank, j)
        f = si.synthetic_test_image(W4K, H4K, C4K, sf)
        m = si.random_mask(W4K, H4K, DENSITY, sm)
        out.append((f, m))
    return out


def ref_frames(n, rank=0):
    """Reference-arm inputs from the reference's OWN generators
    (synthetic.hpp:14-59, masks.hpp:25-43 in oracle/_ref/libref.so): the arm
    never loads this repository's library."""
    from oracle import pyoracle as P
    out = []
    for j in range(n):
        sf, sm = frame_seeds(rank, j)
        out.append((P.ref_synthetic_test_image(W4K, H4K, C4K, sf),
                    P.ref_random_mask(W4K, H4K, DENSITY, sm)))
    return out


def run_reference_arm(args, world, rank):
    """The reference's own CPU run_method (oracle/_ref/libref.so = the
    unmodified headers, -O3 tuned for the box's CPU) on all host threads.
    Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return 0
    from oracle import pyoracle as P
    P.use_tuned_reference()  # before the first reference call loads a build
    frames = ref_frames(min(args.frames, 2))
    r = cpu_reference_run(frames, args.steps, args.warmup, budget_s=240.0)
    ms = 1e3 * sum(r["times"]) / len(r["times"])
    fps = 1e3 / ms
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": len(r["times"]), "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(CONFIG),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": r["cores"],
                         "kind": r["kind"], "build": r.get("build"),
                         "sample": f"{len(r['times'])} full 4K RGB frames (run_method mloras)"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "outer_iterations_finest": r["finest_iterations"],
    }
    if r["kind"] == "reference" and not args.no_cpu_baseline:
        # SURVEY.md §8d protocol: the same frame at 1 thread, and C5 (8K, 2%)
        # on all threads, in the same run
        lib = P.ref()
        lib.ref_set_threads(1)
        f, m = frames[0]
        t0 = time.perf_counter()
        P.ref_run_method("mloras", f, m, levels=LEVELS)
        line["cpu_baseline_1thread"] = {"value": 1.0 / (time.perf_counter() - t0),
                                        "unit": "frames/s", "cores": 1,
                                        "sample": "1 full 4K RGB frame"}
        lib.ref_set_threads(0)
        f5 = P.ref_synthetic_test_image(7680, 4320, 3, 7)
        m5 = P.ref_random_mask(7680, 4320, 0.02, 11)
        t0 = time.perf_counter()
        res5 = P.ref_run_method("mloras", f5, m5, levels=LEVELS)
        line["c5_reference"] = {"ms_per_frame": 1e3 * (time.perf_counter() - t0),
                                "cores": r["cores"], "finest_iterations": res5.iterations,
                                "workload": "7680x4320 RGB, 2% mask, 3 levels (configs[4])"}
    print(json.dumps(line), flush=True)
    return 0


def c5_leg(args, world, rank, local, dist, solver):
    """BASELINE configs[4]: ONE 7680x4320 RGB frame (2% mask, 3 levels)
    striped over the `world` ranks (si_run_method_striped_device: each rank
    holds, ingests, restricts, sweeps and prolongs only its rows; NCCL
    all-gathers of the partial norms and halo rows between neighbours).
    Device-resident, CUDA events on the solve stream, max over ranks; plus
    the forced-sweep variant (tolerance 1e-12, max_outer 2) and a bit-identity
    check of the assembled image against the single-GPU run_method."""
    import hashlib
    import torch
    import paper_2110_03946_b200 as si
    from paper_2110_03946_b200 import stripes as S
    w, h, c = 7680, 4320, 3
    f = si.synthetic_test_image(w, h, c, 7)
    m = si.random_mask(w, h, 0.02, 11)
    comm = S.nccl_comm(solver, dist) if dist is not None else S.local_comms([solver])[0]
    dev = f"cuda:{local}"
    stream = torch.cuda.current_stream()
    out = {"workload": "7680x4320 RGB, 2% random mask, 3-level ORAS (BASELINE configs[4]), "
                       "one frame striped over n_gpus ranks", "comm": comm.kind,
           "output": "each rank's finest rows left in its level storage "
                     "(si_stripe_result_rows; hashed after the timed region)"}
    for name, o in (("tol", si.RunOptions(levels=LEVELS)),
                    ("forced", si.RunOptions(levels=LEVELS, tolerance=1e-12,
                                             max_outer_iterations=2))):
        pl = S.level_plan(si.Method.MultilevelOras, w, h, c, o, world, rank)[0]
        df = torch.from_numpy(np.ascontiguousarray(f.data[:, pl.store_lo:pl.store_hi])).to(dev)
        dm = torch.from_numpy(np.ascontiguousarray(m.known[pl.store_lo:pl.store_hi])).to(dev)

        def run():  # the rank's rows stay in its level storage (result_rows)
            return S.run_method_striped_device(solver, comm, si.Method.MultilevelOras,
                                               df.data_ptr(), dm.data_ptr(), w, h, c,
                                               None, o, stream=stream.cuda_stream)
        for _ in range(max(args.warmup, 3)):
            rep = run()
        steps = max(3, min(args.steps, 20))
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            rep = run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        # bit identity against the single-GPU solve (hash of each rank's rows)
        mine = hashlib.sha256(S.result_rows_tensor(solver, c, w).cpu().numpy().tobytes()
                              ).hexdigest()
        spans = [(pl.own_lo, pl.own_hi)]
        if dist is not None:
            got = [None] * world
            dist.all_gather_object(got, (mine, pl.own_lo, pl.own_hi))
        else:
            got = [(mine, pl.own_lo, pl.own_hi)]
        same = None
        if rank == 0:
            ref = solver.run_method(si.Method.MultilevelOras, f, m, o)
            same = all(hashlib.sha256(np.ascontiguousarray(ref.image.data[:, a:b]).tobytes())
                       .hexdigest() == hx for hx, a, b in got)
            same = same and list(rep.level_iterations) == list(ref.report.level_iterations)
        n_px = w * h
        out[name] = {"ms_per_frame": ms, "frames_per_s": 1e3 / ms, "steps": steps,
                     "level_iterations": list(rep.level_iterations),
                     "bit_identical_to_1gpu": same,
                     "store_rows_rank0": [pl.store_lo, pl.store_hi],
                     "hbm_frac_rank_avg": survey_frame_bytes(list(rep.level_iterations), w, h, c)
                     / world / (ms / 1e3) / 1e9 / hbm_peak()[0]}
        del df, dm
    comm.close()
    if world == 1:
        out["virtual_g2"] = c5_virtual_g2(args, solver, f, m, w, h, c, out["tol"]["ms_per_frame"])
    return out


def c5_virtual_g2(args, solver, f, m, w, h, c, ms_one):
    """The stripe decomposition's overhead on one GPU: the configs[4] frame as
    TWO ranks of a local group sharing this GPU (si_run_method_striped_local_device,
    rows in place), CUDA events on both rank streams; not a scaling number."""
    import torch
    import paper_2110_03946_b200 as si
    from paper_2110_03946_b200 import stripes as S
    o = si.RunOptions(levels=LEVELS)
    sv = [solver, si.Solver(solver.device)]
    comms = S.local_comms(sv)
    streams = [torch.cuda.Stream() for _ in sv]
    plans = [S.level_plan(si.Method.MultilevelOras, w, h, c, o, 2, r)[0] for r in range(2)]
    ins = [(torch.from_numpy(np.ascontiguousarray(f.data[:, p.store_lo:p.store_hi])).cuda(),
            torch.from_numpy(np.ascontiguousarray(m.known[p.store_lo:p.store_hi])).cuda())
           for p in plans]
    main = torch.cuda.current_stream()

    def run():
        return S.run_method_striped_local_device(
            sv, comms, si.Method.MultilevelOras, [i[0].data_ptr() for i in ins],
            [i[1].data_ptr() for i in ins], w, h, c, None, o,
            streams=[st.cuda_stream for st in streams])
    for _ in range(max(args.warmup, 3)):
        run()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 20))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for st in streams:
        st.wait_event(e0)
    for _ in range(steps):
        reps = run()
    for st in streams:
        ev = torch.cuda.Event()
        ev.record(st)
        main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    img = np.zeros_like(f.data)
    for r, p in enumerate(plans):
        img[:, p.own_lo:p.own_hi] = S.result_rows_tensor(sv[r], c, w).cpu().numpy()
    ref = solver.run_method(si.Method.MultilevelOras, f, m, o)
    res = {"ms_per_frame": ms, "ratio_to_one_rank": ms / ms_one, "steps": steps,
           "bit_identical_to_1gpu": bool(np.array_equal(img, ref.image.data)) and
           list(reps[0].level_iterations) == list(ref.report.level_iterations),
           "speculative_solves": comms[0].counters()["speculative"],
           "note": "two ranks on ONE GPU (local communicator): decomposition overhead"}
    for cm in comms:
        cm.close()
    return res


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1;
    rank 0 prints the line, the exit code is the launcher's."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.selfcheck:  # the multi-rank launch path without a GPU (tests/test_bench_cli.py)
        import torch
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("gloo")
            t = torch.tensor([float(rank)])
            dist.all_reduce(t)
            ranks = int(t.item())
            dist.destroy_process_group()
        else:
            ranks = 0
        if rank == 0:
            print(json.dumps({"selfcheck": True, "n_gpus": world,
                              "rank_sum": ranks}), flush=True)
        return 0

    import torch
    import paper_2110_03946_b200 as si

    torch.cuda.set_device(local)
    dist = None
    if world > 1 or "WORLD_SIZE" in os.environ:  # under torchrun (even one rank: NCCL paths)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    prec = {"fp64": si.Precision.FP64, "fp32": si.Precision.FP32,
            "mixed": si.Precision.MIXED}[args.precision]
    opts = si.RunOptions(levels=LEVELS, precision=prec)
    solver = si.Solver(local)
    stream = torch.cuda.current_stream()

    frames = host_frames(args.frames, rank)
    dev = []
    for f, m in frames:
        df = torch.from_numpy(f.data).to(f"cuda:{local}")
        dm = torch.from_numpy(m.known).to(f"cuda:{local}")
        dev.append((df, dm))
    # independent frames in flight: lane i has its own context, stream and
    # output; lane 0 is the profiled/e2e solver on torch's current stream
    inflight = max(1, args.inflight)
    solvers = [solver] + [si.Solver(local) for _ in range(inflight - 1)]
    streams = [stream] + [torch.cuda.Stream(device=local) for _ in range(inflight - 1)]
    outs = [torch.empty((C4K, H4K, W4K), dtype=torch.float64, device=f"cuda:{local}")
            for _ in range(inflight)]

    def step(j, lane=0):
        df, dm = dev[j % len(dev)]
        return solvers[lane].run_method_device(si.Method.MultilevelOras, df.data_ptr(),
                                               dm.data_ptr(), W4K, H4K, C4K,
                                               outs[lane].data_ptr(), opts,
                                               stream=streams[lane].cuda_stream)

    for lane in range(inflight):
        for j in range(max(args.warmup, 3)):
            rep = step(j, lane)
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region
    clocks = ClockSampler(local)
    # (no per-kernel events inside the timed region; they are collected in a
    # separate profiled pass below)
    for sv in solvers:
        sv.set_profiling(False)
        sv.kernel_stats(reset=True)
    iters = [None] * args.steps
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s in streams[1:]:
        s.wait_event(ev0)

    def run_lane(lane):
        for j in range(lane, args.steps, inflight):
            iters[j] = tuple(step(j, lane).level_iterations)

    if inflight == 1:
        run_lane(0)
    else:  # ctypes releases the GIL: the lanes' host loops overlap
        lanes = [threading.Thread(target=run_lane, args=(i,)) for i in range(inflight)]
        for t in lanes:
            t.start()
        for t in lanes:
            t.join()
    for s in streams[1:]:
        e = torch.cuda.Event()
        e.record(s)
        stream.wait_event(e)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    if any(x is None for x in iters):
        raise RuntimeError("a frame lane failed inside the timed region")
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    launches = sum(int(sv.kernel_stats(reset=True)["total_launches"]) for sv in solvers)

    # ---- single-frame latency (one lane, nothing else in flight)
    lat = []
    for j in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(j)
        e1.record(stream)
        torch.cuda.synchronize()
        lat.append(e0.elapsed_time(e1))
    latency_ms = statistics.median(lat)

    # ---- per-kernel device times (CUDA events on the launching stream) over
    # a separate pass of the same frames: the roofline numbers below
    prof_steps = min(args.steps, 4)
    solver.set_profiling(True)
    cg_its = []
    for j in range(prof_steps):
        cg_its.append(step(j).local_cg_iterations)
    torch.cuda.synchronize()
    solver.set_profiling(False)
    stats = solver.kernel_stats(reset=True)
    ms_per_step = ms_total / args.steps
    value = world * args.steps / (ms_total / 1e3)

    # ---- end to end through the public host API (pinned buffers), BASELINE
    # configs[3]: a batch of 64 frames (k = 0..63, seeds 7+k / 11+k) sharded
    # round-robin over the ranks (batch.run_sharded: frame k -> rank k mod G,
    # no data-path collective), each rank's share in one Solver.run_batch
    # call; every frame's H2D (mask + known samples) and D2H (result) are
    # inside the timed region, overlapped with the neighbouring solves.
    from paper_2110_03946_b200 import batch
    e2e_frames = args.e2e_steps or 64
    mine = batch.frames_for_rank(e2e_frames, world, rank)
    n = W4K * H4K
    distinct = {}
    for k in mine[:4]:  # inputs of up to 4 distinct frames per rank, cycled
        sf, sm = 7 + k, 11 + k
        hf = torch.empty((C4K, H4K, W4K), dtype=torch.float64).pin_memory()
        hm = torch.empty((H4K, W4K), dtype=torch.uint8).pin_memory()
        hf.numpy()[...] = si.synthetic_test_image(W4K, H4K, C4K, sf).data
        hm.numpy()[...] = si.random_mask(W4K, H4K, DENSITY, sm).known
        distinct[k] = (si.ImageBuffer(data=hf.numpy()), si.InpaintingMask(known=hm.numpy()))
    keys = list(distinct)
    pinned_in = [distinct[k] for k in keys]
    # outputs: a ring of pinned buffers (a frame's result is read back before
    # the frame RING steps later is produced: the pipeline holds two slots)
    ring = 4
    pinned_out = []
    for j in range(ring):
        ho = torch.empty((C4K, H4K, W4K), dtype=torch.float64).pin_memory()
        pinned_out.append(si.ImageBuffer(data=ho.numpy()))
    batch_out = [pinned_out[j % ring] for j in range(len(mine))]
    solver.run_batch(si.Method.MultilevelOras, pinned_in[:2], opts, batch_out[:2])  # warm
    local_run = batch.run_sharded(
        e2e_frames, lambda k: distinct[keys[mine.index(k) % len(keys)]],
        lambda fr: solver.run_batch(si.Method.MultilevelOras, fr, opts, batch_out), dist)
    e2e_res = list(local_run["frames"].values())
    e2e_value = local_run["frames_per_s"]

    # ---- the plain drop-in call, one frame at a time: run_method on pageable
    # numpy buffers (methods.hpp:57-88's signature; the library uploads the
    # known samples and copies the result out through pinned chunks)
    rm_frames = [(si.ImageBuffer(data=np.array(f.data)), si.InpaintingMask(known=np.array(m.known)))
                 for f, m in (pinned_in[j % len(pinned_in)] for j in range(2))]
    solver.run_method(si.Method.MultilevelOras, *rm_frames[0], opts)  # warm
    rm_n = 8
    barrier()
    t0 = time.perf_counter()
    for j in range(rm_n):
        rm_res = solver.run_method(si.Method.MultilevelOras, *rm_frames[j % 2], opts)
    t_rm = max_over_ranks(time.perf_counter() - t0)
    rm_value = world * rm_n / t_rm

    # ---- the same through the CLI's wire format (P6 pixels + P4 mask in, P6
    # out; read_pnm/write_pnm decode and quantise run on the device)
    pnm_in, pnm_out = [], []
    for j in range(len(pinned_in)):
        px = torch.empty((H4K, W4K, C4K), dtype=torch.uint8).pin_memory()
        pb = torch.empty((H4K, (W4K + 7) // 8), dtype=torch.uint8).pin_memory()
        px.numpy()[...] = si.quantise_pnm(pinned_in[j][0])
        pb.numpy()[...] = si.pack_pbm(pinned_in[j][1])
        pnm_in.append((px.numpy(), pb.numpy()))
    for j in range(ring):
        pnm_out.append(torch.empty((H4K, W4K, C4K), dtype=torch.uint8).pin_memory().numpy())
    pnm_frames = [pnm_in[j % len(pnm_in)] for j in range(len(mine))]
    pnm_out = [pnm_out[j % ring] for j in range(len(mine))]
    solver.run_pnm_batch(si.Method.MultilevelOras, pnm_frames[:2], opts, pnm_out[:2])  # warm
    barrier()
    t0 = time.perf_counter()
    solver.run_pnm_batch(si.Method.MultilevelOras, pnm_frames, opts, pnm_out)
    t_pnm = max_over_ranks(time.perf_counter() - t0)
    pnm_value = e2e_frames / t_pnm

    # ---- roofline of the dominant kernel (K2 sweep)
    sw = stats["sweep"]
    fp64_tf = (15.0 * 1024 * float(np.sum(cg_its)) / (sw["device_ms"] / 1e3) / 1e12
               if sw["device_ms"] else None)
    peak, peak_src = hbm_peak()
    achieved = (sw["algorithmic_bytes"] / (sw["device_ms"] / 1e3) / 1e9) if sw["device_ms"] else 0.0
    traffic, traffic_alg, fp64_pct = None, None, None
    tfile = os.path.join(ROOT, "profiles", "sweep_dram_traffic.json")
    if os.path.exists(tfile) and prec == si.Precision.FP64:  # ncu capture of the fp64 sweep
        try:
            tj = json.load(open(tfile))
            traffic, traffic_alg = tj.get("dram_bytes_per_launch"), tj.get("algorithmic_bytes_per_launch")
            fp64_pct = tj.get("fp64_pipe_pct_of_peak")
        except ValueError:
            pass
    total_dev = sum(v["device_ms"] for k, v in stats.items() if isinstance(v, dict))
    frame_bytes_survey = survey_frame_bytes(list(iters[-1]),
                                            s=4 if prec == si.Precision.FP32 else 8)

    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {si.Precision.FP64: "f64", si.Precision.FP32: "f32",
                  si.Precision.MIXED: "f64 (local CG f32)"}[prec], "data": "synthetic",
        "config": dict(CONFIG),
        "lanes": {"frames_per_rank": len(dev), "frames_in_flight": inflight,
                  "latency_ms_one_frame": latency_ms},
        "roofline": {"bound": "hbm", "kernel": "oras_sweep_kernel", "achieved": achieved,
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_launch": "finest-level sweep, ncu dram__bytes_read+write",
                     "traffic_algorithmic": traffic_alg,
                     "frame_hbm_frac": frame_bytes_survey / (ms_per_step / 1e3) / 1e9 / peak,
                     "frame_bytes": frame_bytes_survey,
                     "frame_bytes_formula": "SURVEY.md 8d per-frame formula with the measured k_L",
                     "sweep_share_of_step": sw["device_ms"] / max(total_dev, 1e-9),
                     # informational: 15 FP64 flops per cell per local CG iteration
                     # (stencil 5, two dots 4, three axpys 6) x 1,024 cells, counted
                     # on the device (report.local_cg_iterations)
                     "sweep_fp64_tflops": fp64_tf,
                     "fp64_peak_tflops": FP64_PEAK_TF,
                     "sweep_fp64_frac": fp64_tf / FP64_PEAK_TF if fp64_tf else None,
                     "fp64_peak_source": "scripts/fp64_peak.cu on a B200 of this pool "
                                         "(8 DFMA chains/thread, 1965 MHz): "
                                         "profiles/r02_fp64_peak.json",
                     "onchip_bound": {"pipe": "fp64", "pct_of_peak": fp64_pct,
                                      "source": "ncu --set full, first finest-level sweep"}},
        "e2e": {"value": e2e_value, "unit": "frames/s",
                "h2d_bytes_per_step": int(np.mean([r.report.h2d_bytes for r in e2e_res])),
                "d2h_bytes_per_step": int(np.mean([r.report.d2h_bytes for r in e2e_res])),
                "api": "si_run_method_batch (host f64 planar + u8 mask in, f64 out; pinned); "
                       "a frame crosses PCIe as its mask + the f values at known pixels "
                       "(the only ones the solver reads, multilevel.hpp:84-88), packed on "
                       "host threads inside the timed region; outer iterations decided on "
                       "the device (cached CUDA graphs with conditional nodes)",
                "frames": e2e_frames, "frames_per_rank": len(mine),
                "scaling": "strong (configs[3]: the 64-frame batch sharded over n_gpus)",
                "inputs": "frames k = 0..63 (seeds 7+k, 11+k); up to 4 distinct inputs per "
                          "rank, cycled"},
        "e2e_run_method": {"value": rm_value, "unit": "frames/s",
                           "h2d_bytes_per_step": int(rm_res.report.h2d_bytes),
                           "d2h_bytes_per_step": int(rm_res.report.d2h_bytes),
                           "api": "si_run_method (the drop-in run_method) on pageable numpy "
                                  "buffers, one frame per call, copies included",
                           "frames": rm_n},
        "e2e_pnm": {"value": pnm_value, "unit": "frames/s",
                    "h2d_bytes_per_step": int(C4K * n + H4K * ((W4K + 7) // 8)),
                    "d2h_bytes_per_step": int(C4K * n),
                    "api": "si_run_pnm_batch (P6 + P4 payloads in, P6 out; pinned)",
                    "frames": e2e_frames},
        "gpu_launches": launches,
        "clocks": clk,
        "outer_iterations_per_level": list(iters[-1]) if iters else None,
        "kernel_ms_per_step": {k: v["device_ms"] / prof_steps for k, v in stats.items()
                               if isinstance(v, dict) and v["launches"]},
    }

    if not args.no_c5:
        try:
            line["c5"] = c5_leg(args, world, rank, local, dist, solver)
        except Exception as e:  # the configs[4] leg never takes the headline line down
            line["c5"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_run([(frames[0][0].data, frames[0][1].known)], steps=3, warmup=0,
                                  budget_s=20.0)
            ms = 1e3 * statistics.median(r["times"])
            line["cpu_baseline"] = {"value": 1e3 / ms, "unit": "frames/s", "cores": r["cores"],
                                    "kind": r["kind"], "build": r.get("build"),
                                    "sample": f"{len(r['times'])} full 4K RGB frame(s), median"}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    solver.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
