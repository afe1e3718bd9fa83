"""One 8K RGB frame striped over G GPUs (BASELINE.json configs[4], SURVEY.md
§8e): every pyramid level split by block rows, halo exchange and residual
all-reduce over torch.distributed (NCCL), results bit-identical to one GPU.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node G \\
      --master-addr 127.0.0.1 --master-port 29531 scripts/stripes_bench.py [--forced]

--forced: the C5 forced-sweep variant (tolerance 1e-12, max_outer 2), which
exercises the finest-level halo exchange (the default C5 needs 0 finest
sweeps).  Rank 0 prints one JSON line: ms per frame (max over ranks, CUDA
events), level iterations and whether the result equals the 1-GPU solve.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402
from paper_2110_03946_b200 import stripes as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="7680x4320")
    ap.add_argument("--density", type=float, default=0.02)
    ap.add_argument("--forced", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", local))
    w, h = (int(v) for v in args.size.split("x"))
    f = si.synthetic_test_image(w, h, 3, 7)
    m = si.random_mask(w, h, args.density, 11)
    df = torch.from_numpy(f.data).cuda()
    dm = torch.from_numpy(m.known).cuda()
    opts = si.RunOptions(levels=3)
    if args.forced:
        opts.tolerance = 1e-12
        opts.max_outer_iterations = 2
    solver = si.Solver(local)
    comm = S.TorchComm(dist, device=torch.device("cuda", local))
    backend = S.DeviceBackend(solver)
    stream = torch.cuda.current_stream()

    u, rep = S.solve_striped(df, dm, comm, backend, opts)  # warm-up
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        u, rep = S.solve_striped(df, dm, comm, backend, opts)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
    plan = rep.plans[0]
    spans = [(p.own_lo, p.own_hi) for p in
             (S.stripe_plan(h, *S.clamped(w, h, 32, 6), world, r) for r in range(world))]
    full = S.gather_full(comm, u, plan, spans)
    line = None
    if rank == 0:
        one = si.Solver(local).run_method_device(si.Method.MultilevelOras, df.data_ptr(),
                                                 dm.data_ptr(), w, h, 3,
                                                 torch.empty_like(df).data_ptr(), opts)
        ref_out = torch.empty_like(df)
        si.Solver(local).run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(),
                                           w, h, 3, ref_out.data_ptr(), opts)
        torch.cuda.synchronize()
        line = {"workload": f"{w}x{h} RGB, {args.density:.0%} mask, 3 levels"
                + (", forced 2 finest sweeps" if args.forced else ""),
                "n_gpus": world, "ms_per_frame": statistics.median(times),
                "level_iterations": rep.level_iterations,
                "one_gpu_level_iterations": list(one.level_iterations),
                "identical_to_one_gpu": bool(torch.equal(full, ref_out))}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
