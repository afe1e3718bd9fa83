"""A/B of the batch entry's upload strategies on one GPU (4K RGB f64, 4%
mask, pinned buffers): frames/s of si_run_method_batch per setting, plus the
host cost of packing one frame.

  python scripts/e2e_probe.py            # runs every setting in a subprocess
  python scripts/e2e_probe.py --one      # one measurement with the current env
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(frames_n=32):
    import numpy as np
    import torch
    import paper_2110_03946_b200 as si
    W, H, C = 3840, 2160, 3
    solver = si.Solver(0)
    ins, outs = [], []
    for j in range(2):
        f = si.synthetic_test_image(W, H, C, 7 + j)
        m = si.random_mask(W, H, 0.04, 11 + j)
        hf = torch.empty((C, H, W), dtype=torch.float64).pin_memory()
        hm = torch.empty((H, W), dtype=torch.uint8).pin_memory()
        hf.numpy()[...] = f.data
        hm.numpy()[...] = m.known
        ins.append((si.ImageBuffer(data=hf.numpy()), si.InpaintingMask(known=hm.numpy())))
    for j in range(4):
        outs.append(si.ImageBuffer(data=torch.empty((C, H, W), dtype=torch.float64)
                                   .pin_memory().numpy()))
    o = si.RunOptions(levels=3)
    fr = [ins[j % 2] for j in range(frames_n)]
    ou = [outs[j % 4] for j in range(frames_n)]
    solver.run_batch(si.Method.MultilevelOras, fr[:2], o, ou[:2])
    t0 = time.perf_counter()
    res = solver.run_batch(si.Method.MultilevelOras, fr, o, ou)
    dt = time.perf_counter() - t0
    # single frame through si_run_method from pageable numpy buffers (the
    # reference caller's std::vector): latency per call
    fp = si.synthetic_test_image(W, H, C, 7)
    mp = si.random_mask(W, H, 0.04, 11)
    solver.run_method(si.Method.MultilevelOras, fp, mp, o)
    ts = []
    for _ in range(5):
        t1 = time.perf_counter()
        solver.run_method(si.Method.MultilevelOras, fp, mp, o)
        ts.append((time.perf_counter() - t1) * 1e3)
    single_ms = sorted(ts)[2]
    t1 = time.perf_counter()
    for _ in range(5):
        si.pack_known_samples(*ins[0])
    pack_ms = (time.perf_counter() - t1) / 5 * 1e3
    print(json.dumps({"fps": frames_n / dt,
                      "solve_ms_mean": float(np.mean([r.report.elapsed_ms for r in res])),
                      "h2d_mb": res[0].report.h2d_bytes / 1e6,
                      "single_frame_ms_pageable": single_ms,
                      "pack_ms_16threads_py": pack_ms,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("SI_")}}),
          flush=True)


def main():
    if "--one" in sys.argv:
        one()
        return
    settings = [{"SI_NO_KNOWN_PACK": "1"}] + [{"SI_PACK_THREADS": str(t)} for t in (4, 8)]
    for st in settings:
        env = dict(os.environ, **st)
        subprocess.run([sys.executable, __file__, "--one"], env=env, check=False)


if __name__ == "__main__":
    main()
