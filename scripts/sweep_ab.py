"""A/B timing of library variants on the C3 frame (4K RGB fp64, 3 levels):
median device ms of the sweeps and of the whole frame (device-resident entry),
plus the parity fingerprint against tests/golden/c3.npz.
Usage: SI_LIB_PATH=variants/lib_x.so python scripts/sweep_ab.py [reps]"""
import os
import statistics
import sys

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
import torch  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 7
g = np.load(os.path.join(R, "tests", "golden", "c3.npz"))
f = si.synthetic_test_image(3840, 2160, 3, 7)
m = si.random_mask(3840, 2160, 0.04, 11)
s = si.Solver(0)
df = torch.from_numpy(f.data).cuda()
dm = torch.from_numpy(m.known).cuda()
out = torch.empty_like(df)
o = si.RunOptions(levels=3)
st = torch.cuda.current_stream()


def run():
    return s.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(), 3840, 2160,
                               3, out.data_ptr(), o, stream=st.cuda_stream)


for _ in range(3):
    rep = run()
frame = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    rep = run()
    e1.record(st)
    torch.cuda.synchronize()
    frame.append(e0.elapsed_time(e1))
s.set_profiling(True)
sw = []
kinds = {}
for _ in range(reps):
    s.kernel_stats(reset=True)
    run()
    torch.cuda.synchronize()
    ks = s.kernel_stats(reset=True)
    sw.append(ks["sweep"]["device_ms"])
    for k, v in ks.items():
        if isinstance(v, dict) and v["launches"]:
            kinds.setdefault(k, []).append(v["device_ms"])
s.set_profiling(False)
img = out.cpu().numpy()
ok = (list(rep.level_iterations) == [int(v) for v in g["level_iterations"]] and
      rep.local_solves == int(g["local_solves"]) and
      np.all(np.abs(img.sum(axis=(1, 2)) - g["channel_sum"]) <= 1e-12 * np.abs(g["channel_sum"])) and
      np.abs(img.reshape(-1)[g["sample_index"]] - g["sample_value"]).max() <= 1e-9)
print(f"{os.environ.get('SI_LIB_PATH', 'default')}: frame {statistics.median(frame):.3f} ms, "
      f"sweeps {statistics.median(sw):.3f} ms, cg_its {rep.local_cg_iterations}, "
      f"fails {rep.local_failures}, parity {'OK' if ok else 'FAIL'}; "
      + ", ".join(f"{k} {statistics.median(v):.3f}" for k, v in kinds.items()))
