"""Throughput of independent 4K frames solved one at a time vs two in flight
(two contexts = two streams, one host thread each; device-resident inputs).

  python scripts/concurrency_probe.py [--frames 40]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import paper_2110_03946_b200 as si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=40)
    args = ap.parse_args()
    W, H, C = 3840, 2160, 3
    dev = []
    for k in range(4):
        f = si.synthetic_test_image(W, H, C, 7 + k)
        m = si.random_mask(W, H, 0.04, 11 + k)
        dev.append((torch.from_numpy(f.data).cuda(), torch.from_numpy(m.known).cuda()))
    o = si.RunOptions(levels=3)
    solvers = [si.Solver(0), si.Solver(0)]
    outs = [torch.empty((C, H, W), dtype=torch.float64, device="cuda") for _ in range(2)]

    def run(sv, out, frames):
        for j in frames:
            df, dm = dev[j % len(dev)]
            sv.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(), W, H, C,
                                 out.data_ptr(), o)

    for sv, out in zip(solvers, outs):
        run(sv, out, range(3))
    torch.cuda.synchronize()
    res = {}
    t0 = time.perf_counter()
    run(solvers[0], outs[0], range(args.frames))
    torch.cuda.synchronize()
    res["sequential_fps"] = args.frames / (time.perf_counter() - t0)
    for inflight in (2,):
        t0 = time.perf_counter()
        ths = [threading.Thread(target=run, args=(solvers[i], outs[i],
                                                 range(i, args.frames, inflight)))
               for i in range(inflight)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        torch.cuda.synchronize()
        res[f"inflight{inflight}_fps"] = args.frames / (time.perf_counter() - t0)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
