"""e2e through si_run_method_batch with the frames split over L independent
contexts (one host thread each, interleaved frames): does a second solve
stream lift the f64 batch above the single pipeline?

  python scripts/e2e_lanes_probe.py [--frames 64]
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
    ap.add_argument("--frames", type=int, default=64)
    args = ap.parse_args()
    W, H, C = 3840, 2160, 3
    ins = []
    for k in range(2):
        hf = torch.empty((C, H, W), dtype=torch.float64).pin_memory()
        hm = torch.empty((H, W), dtype=torch.uint8).pin_memory()
        hf.numpy()[...] = si.synthetic_test_image(W, H, C, 7 + k).data
        hm.numpy()[...] = si.random_mask(W, H, 0.04, 11 + k).known
        ins.append((si.ImageBuffer(data=hf.numpy()), si.InpaintingMask(known=hm.numpy())))
    outs = [si.ImageBuffer(data=torch.empty((C, H, W), dtype=torch.float64).pin_memory().numpy())
            for _ in range(8)]
    o = si.RunOptions(levels=3)
    res = {}
    for lanes in (1, 2, 1, 2):
        svs = [si.Solver(0) for _ in range(lanes)]
        parts = [list(range(i, args.frames, lanes)) for i in range(lanes)]

        def run(i, warm=False):
            idx = parts[i][:2] if warm else parts[i]
            svs[i].run_batch(si.Method.MultilevelOras, [ins[j % 2] for j in idx], o,
                             [outs[(4 * i + n) % 8] for n in range(len(idx))])

        for i in range(lanes):
            run(i, warm=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ts = [threading.Thread(target=run, args=(i,)) for i in range(lanes)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        torch.cuda.synchronize()
        fps = args.frames / (time.perf_counter() - t0)
        res.setdefault(f"lanes{lanes}_fps", []).append(round(fps, 1))
        for s in svs:
            s.close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
