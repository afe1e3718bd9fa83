"""Where the plain drop-in run_method's time goes on a 4K RGB frame (host
pageable numpy buffers, one frame per call): the same call with a pinned
output, with pinned input+output, and the device-resident solve alone."""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_03946_b200 as si  # noqa: E402
from paper_2110_03946_b200 import _lib as L  # noqa: E402

W, H, Ch = 3840, 2160, 3
f = si.synthetic_test_image(W, H, Ch, 7)
m = si.random_mask(W, H, 0.04, 11)
s = si.Solver(0)
lib = L.load()
o = si.RunOptions().to_c()
n = W * H * Ch


def pinned(nbytes):
    p = C.c_void_p()
    assert lib.si_host_alloc(nbytes, C.byref(p)) == 0
    return p


def call(fp, mp, outp):
    rep = L.si_report()
    st = lib.si_run_method(s.handle, int(si.Method.MultilevelOras), fp, mp, W, H, Ch, C.byref(o),
                           None, outp, C.byref(rep), L.TRACE_FN(), None)
    assert st == 0, lib.si_last_error()


def timed(fn, reps=6):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


out = {}
out["pageable_new_output_each_call_ms"] = timed(
    lambda: s.run_method(si.Method.MultilevelOras, f, m, si.RunOptions()))
po = np.empty_like(f.data)
out["pageable_reused_output_ms"] = timed(lambda: call(f.data.ctypes.data, m.known.ctypes.data,
                                                       po.ctypes.data))
pout = pinned(n * 8)
out["pinned_output_ms"] = timed(lambda: call(f.data.ctypes.data, m.known.ctypes.data, pout.value))
pin_f = pinned(n * 8)
C.memmove(pin_f.value, f.data.ctypes.data, n * 8)
pin_m = pinned(W * H)
C.memmove(pin_m.value, m.known.ctypes.data, W * H)
out["pinned_in_out_ms"] = timed(lambda: call(pin_f.value, pin_m.value, pout.value))
df = torch.from_numpy(f.data).cuda()
dm = torch.from_numpy(m.known).cuda()
do = torch.empty_like(df)
st = torch.cuda.current_stream()


def dev():
    s.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(), W, H, Ch,
                        do.data_ptr(), si.RunOptions(), stream=st.cuda_stream)
    torch.cuda.synchronize()


out["device_resident_ms"] = timed(dev)
print(out)
