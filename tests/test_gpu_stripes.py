"""GPU: the C++ stripe engine (csrc/stripes.cuh, BASELINE configs[4]).

G ranks run as host threads of this process on ONE B200 over the local
communicator (device copies ordered by events: no kernel waits on another
rank's kernel).  Every case must reproduce the single-GPU run_method:
  * per-level outer counts, local solves and local failures equal;
  * the image bit-identical (the only difference is the summation order of
    the global residual norm, which can only change a stop decision at the
    threshold itself);
  * trace rows within 1e-12 relative.
The single-GPU solve is itself pinned to the reference (test_gpu_headline.py).
"""
import numpy as np
import pytest

import paper_2110_03946_b200 as si
from paper_2110_03946_b200 import stripes as S

pytestmark = pytest.mark.gpu

_SOLVERS = []


def solvers(n):
    while len(_SOLVERS) < n:
        _SOLVERS.append(si.Solver(0))
    return _SOLVERS[:n]


def check_same(single, img, reps, G):
    for r in reps:
        assert list(r.level_iterations) == list(single.report.level_iterations)
        assert r.iterations == single.report.iterations
        assert r.converged == single.report.converged
        assert r.local_solves == single.report.local_solves
        assert r.local_failures == single.report.local_failures
        assert r.local_cg_iterations == single.report.local_cg_iterations
        assert abs(r.final_relative_residual - single.report.final_relative_residual) <= \
            1e-12 * abs(single.report.final_relative_residual) + 1e-18
    assert np.array_equal(img.data, single.image.data), np.abs(img.data - single.image.data).max()


CASES = [
    # w, h, c, density, method, options
    (640, 480, 3, 0.05, si.Method.MultilevelOras, dict(levels=3)),
    (1000, 600, 3, 0.04, si.Method.MultilevelOras, dict(tolerance=1e-6)),
    (777, 333, 3, 0.04, si.Method.MultilevelOras, dict()),          # odd widths: cp.async paths
    (512, 700, 1, 0.03, si.Method.Oras, dict(tolerance=1e-5)),
    (400, 300, 2, 0.05, si.Method.Ras, dict(tolerance=1e-5)),
    (300, 200, 3, 0.05, si.Method.MultilevelOras, dict(block_size=16, overlap=3, levels=4)),
    (260, 190, 3, 0.04, si.Method.MultilevelOras, dict(block_size=64, overlap=10)),  # K2g
    (640, 360, 3, 0.04, si.Method.MultilevelOras, dict(precision=si.Precision.FP32)),
    (640, 360, 3, 0.04, si.Method.MultilevelOras, dict(precision=si.Precision.MIXED)),
    (200, 150, 3, 0.05, si.Method.MultilevelOras,
     dict(averaging=si.CoarseAveraging.AllPixels, normalizer=si.ResidualNormalizer.RhsNorm)),
]


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_striped_group_matches_single_gpu(solver, case, G):
    w, h, c, d, method, kw = CASES[case]
    f = si.synthetic_test_image(w, h, c, 100 + case)
    m = si.random_mask(w, h, d, 200 + case)
    o = si.RunOptions(**kw)
    single = solver.run_method(method, f, m, o)
    img, reps = S.run_method_striped_group(solvers(G), method, f, m, o)
    check_same(single, img, reps, G)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_c5_striped_matches_single_gpu(solver, G):
    """configs[4]: 7680x4320 RGB, 2% (0 finest sweeps)."""
    f = si.synthetic_test_image(7680, 4320, 3, 7)
    m = si.random_mask(7680, 4320, 0.02, 11)
    o = si.RunOptions(levels=3)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    img, reps = S.run_method_striped_group(solvers(G), si.Method.MultilevelOras, f, m, o)
    check_same(single, img, reps, G)


@pytest.mark.parametrize("G", [2, 8])
def test_c5_forced_sweeps_striped_matches_single_gpu(solver, G):
    """configs[4] forced-sweep variant: two sweeps on every level, so the
    finest-level halo exchange runs."""
    f = si.synthetic_test_image(7680, 4320, 3, 7)
    m = si.random_mask(7680, 4320, 0.02, 11)
    o = si.RunOptions(levels=3, tolerance=1e-12, max_outer_iterations=2)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    assert single.report.level_iterations[0] == 2
    img, reps = S.run_method_striped_group(solvers(G), si.Method.MultilevelOras, f, m, o)
    check_same(single, img, reps, G)


def test_more_ranks_than_block_rows(solver):
    """Ranks without blocks on a level still join every collective."""
    f = si.synthetic_test_image(96, 70, 2, 3)
    m = si.random_mask(96, 70, 0.08, 4)
    o = si.RunOptions(levels=3)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    img, reps = S.run_method_striped_group(solvers(8), si.Method.MultilevelOras, f, m, o)
    check_same(single, img, reps, 8)


def test_nccl_comm_single_rank(solver):
    """The NCCL communicator at world 1 (the only NCCL shape one GPU can run:
    ranks of a multi-rank NCCL group would wait on each other's kernels)."""
    import ctypes as C
    import torch  # noqa: F401  (its NCCL is loaded first and reused by the library)
    from paper_2110_03946_b200 import _lib as L
    lib = L.load()
    idbuf = (C.c_ubyte * L.SI_NCCL_ID_BYTES)()
    assert lib.si_nccl_unique_id(idbuf) == 0
    h = C.c_void_p()
    assert lib.si_stripe_comm_init_nccl(solver.handle, 1, 0, idbuf, C.byref(h)) == 0, \
        lib.si_last_error()
    comm = S.StripeComm(h, 1, 0, "nccl")
    f = si.synthetic_test_image(640, 480, 3, 9)
    m = si.random_mask(640, 480, 0.05, 10)
    o = si.RunOptions(levels=3, tolerance=1e-5)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    for _ in range(3):  # the repeats speculate (NCCL calls after a stop are no-ops)
        res = S.run_method_striped(solver, comm, si.Method.MultilevelOras, f, m, o)
        check_same(single, res.image, [res.report], 1)
        assert len(res.trace.rows) == single.report.iterations + 1
    assert comm.counters()["speculative"] == 2
    comm.close()


def test_striped_device_entry_rows(solver):
    """si_run_method_striped_device: store rows in, own rows out, on a
    2-rank local group driven from two threads."""
    import threading
    import torch
    w, h, c = 640, 480, 3
    f = si.synthetic_test_image(w, h, c, 31)
    m = si.random_mask(w, h, 0.05, 32)
    o = si.RunOptions(levels=3)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    sv = solvers(2)
    comms = S.local_comms(sv)
    out = np.zeros_like(f.data)
    reps = [None, None]

    def rank(r):
        pl = S.level_plan(si.Method.MultilevelOras, w, h, c, o, 2, r)[0]
        df = torch.from_numpy(np.ascontiguousarray(f.data[:, pl.store_lo:pl.store_hi])).cuda()
        dm = torch.from_numpy(np.ascontiguousarray(m.known[pl.store_lo:pl.store_hi])).cuda()
        do = torch.empty((c, pl.own_hi - pl.own_lo, w), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        reps[r] = S.run_method_striped_device(sv[r], comms[r], si.Method.MultilevelOras,
                                              df.data_ptr(), dm.data_ptr(), w, h, c,
                                              do.data_ptr(), o)
        out[:, pl.own_lo:pl.own_hi] = do.cpu().numpy()

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for cm in comms:
        cm.close()
    check_same(single, si.ImageBuffer(data=out), reps, 2)


def test_cg_methods_are_not_striped(solver):
    f = si.synthetic_test_image(64, 64, 1, 1)
    m = si.random_mask(64, 64, 0.05, 2)
    with pytest.raises(si.SolverError):
        S.run_method_striped_group(solvers(2), si.Method.MultilevelCg, f, m, si.RunOptions())


def test_empty_mask_fails_on_every_rank(solver):
    f = si.synthetic_test_image(64, 64, 1, 1)
    m = si.InpaintingMask(64, 64, 0)
    with pytest.raises(si.InvalidArgument, match="no known pixels"):
        S.run_method_striped_group(solvers(2), si.Method.MultilevelOras, f, m, si.RunOptions())


# ---- device-decided iterations: speculation and its recovery -------------------

def _group_persistent(solvers_, comms, method, f, m, o):
    """One collective solve over persistent communicators (threads)."""
    import threading
    G = len(solvers_)
    out = si.ImageBuffer(data=np.zeros_like(f.data))
    res = [None] * G
    err = [None] * G

    def rank(r):
        try:
            res[r] = S.run_method_striped(solvers_[r], comms[r], method, f, m, o, out=out)
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out, res


SPEC_CASES = [
    # w, h, c, method, options, G
    (640, 480, 3, si.Method.MultilevelOras, dict(levels=3), 2),
    (777, 333, 3, si.Method.MultilevelOras, dict(tolerance=1e-6), 3),
    (512, 700, 1, si.Method.Oras, dict(tolerance=1e-5), 2),
    (260, 190, 3, si.Method.MultilevelOras, dict(block_size=64, overlap=10), 2),  # K2g
    (640, 360, 3, si.Method.MultilevelOras, dict(precision=si.Precision.MIXED), 4),
    (640, 360, 3, si.Method.MultilevelOras, dict(precision=si.Precision.FP32), 2),
    (96, 70, 2, si.Method.MultilevelOras, dict(levels=3), 8),  # ranks without rows
    (300, 200, 3, si.Method.MultilevelOras,
     dict(averaging=si.CoarseAveraging.AllPixels, normalizer=si.ResidualNormalizer.RhsNorm), 3),
    (400, 300, 2, si.Method.Ras, dict(tolerance=1e-5), 2),
]


@pytest.mark.parametrize("case", range(len(SPEC_CASES)))
def test_speculative_repeat_matches_single_gpu(solver, case):
    """The second solve of the same shape/options issues every level's
    iterations without host round trips: same image, counts and trace."""
    w, h, c, method, kw, G = SPEC_CASES[case]
    f = si.synthetic_test_image(w, h, c, 300 + case)
    m = si.random_mask(w, h, 0.04, 400 + case)
    o = si.RunOptions(**kw)
    single = solver.run_method(method, f, m, o)
    sv = solvers(G)
    comms = S.local_comms(sv)
    try:
        for k in range(3):
            img, res = _group_persistent(sv, comms, method, f, m, o)
            check_same(single, img, [r.report for r in res], G)
            for r in res:
                assert len(r.trace.rows) == single.report.iterations + 1
                for a, b in zip(r.trace.rows, single.trace.rows):
                    assert a.iteration == b.iteration
                    assert abs(a.rel_residual - b.rel_residual) <= \
                        1e-12 * abs(b.rel_residual) + 1e-18
                ts = [row.time_ms for row in r.trace.rows]
                assert ts[0] >= 0 and all(b >= a for a, b in zip(ts, ts[1:]))
        for cm in comms:
            cnt = cm.counters()
            assert cnt["solves"] == 3 and cnt["speculative"] == 2 and cnt["resumes"] == 0, cnt
    finally:
        for cm in comms:
            cm.close()


def test_misspeculation_resumes_and_redoes_finer_levels(solver):
    """Frames of one shape whose level counts differ: a level that needs more
    iterations than the previous frame took is resumed and the finer levels
    are redone; every frame equals its single-GPU solve."""
    w, h, c = 640, 480, 3
    o = si.RunOptions(levels=3, tolerance=1e-4)
    frames = [(si.synthetic_test_image(w, h, c, 500 + k), si.random_mask(w, h, d, 600 + k))
              for k, d in enumerate([0.30, 0.02, 0.30, 0.05, 0.02])]
    singles = [solver.run_method(si.Method.MultilevelOras, f, m, o) for f, m in frames]
    counts = [list(s.report.level_iterations) for s in singles]
    assert any(any(b > a for a, b in zip(counts[k], counts[k + 1]))
               for k in range(len(counts) - 1)), counts  # some level is under-predicted
    sv = solvers(2)
    comms = S.local_comms(sv)
    try:
        for (f, m), single in zip(frames, singles):
            img, res = _group_persistent(sv, comms, si.Method.MultilevelOras, f, m, o)
            check_same(single, img, [r.report for r in res], 2)
        cnt = comms[0].counters()
        assert cnt["speculative"] == len(frames) - 1 and cnt["resumes"] >= 1, cnt
        assert comms[1].counters() == cnt
    finally:
        for cm in comms:
            cm.close()


def test_speculation_off_matches(solver):
    f = si.synthetic_test_image(640, 480, 3, 9)
    m = si.random_mask(640, 480, 0.05, 10)
    o = si.RunOptions(levels=3, tolerance=1e-5)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    sv = solvers(2)
    comms = S.local_comms(sv)
    try:
        for cm in comms:
            cm.set_speculation(False)
        for _ in range(2):
            img, res = _group_persistent(sv, comms, si.Method.MultilevelOras, f, m, o)
            check_same(single, img, [r.report for r in res], 2)
        assert comms[0].counters()["speculative"] == 0
    finally:
        for cm in comms:
            cm.close()


@pytest.mark.parametrize("forced", [False, True])
def test_c5_speculative_repeat(solver, forced):
    """configs[4] (and its forced-sweep variant) solved twice over the same
    two-rank group: the second solve speculates and stays bit-identical."""
    f = si.synthetic_test_image(7680, 4320, 3, 7)
    m = si.random_mask(7680, 4320, 0.02, 11)
    o = (si.RunOptions(levels=3, tolerance=1e-12, max_outer_iterations=2) if forced
         else si.RunOptions(levels=3))
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    sv = solvers(2)
    comms = S.local_comms(sv)
    try:
        for _ in range(2):
            img, res = _group_persistent(sv, comms, si.Method.MultilevelOras, f, m, o)
            check_same(single, img, [r.report for r in res], 2)
        assert comms[0].counters()["speculative"] == 1
    finally:
        for cm in comms:
            cm.close()


@pytest.mark.parametrize("G", [1, 2, 3])
def test_result_rows_in_place(solver, G):
    """A device solve without an output buffer leaves each rank's rows in
    its storage (si_stripe_result_rows): same rows as the single-GPU image,
    including after a speculative repeat with an odd finest sweep count."""
    import threading
    import torch
    w, h, c = 640, 480, 3
    f = si.synthetic_test_image(w, h, c, 41)
    m = si.random_mask(w, h, 0.05, 42)
    o = si.RunOptions(levels=3, tolerance=1e-5)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    sv = solvers(G)
    comms = S.local_comms(sv)
    plans = [S.level_plan(si.Method.MultilevelOras, w, h, c, o, G, r)[0] for r in range(G)]
    ins = [(torch.from_numpy(np.ascontiguousarray(f.data[:, p.store_lo:p.store_hi])).cuda(),
            torch.from_numpy(np.ascontiguousarray(m.known[p.store_lo:p.store_hi])).cuda())
           for p in plans]
    torch.cuda.synchronize()
    reps = [None] * G
    try:
        for _ in range(2):
            def rank(r):
                reps[r] = S.run_method_striped_device(sv[r], comms[r], si.Method.MultilevelOras,
                                                      ins[r][0].data_ptr(), ins[r][1].data_ptr(),
                                                      w, h, c, None, o)
            th = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            out = np.zeros_like(f.data)
            for r, p in enumerate(plans):
                out[:, p.own_lo:p.own_hi] = S.result_rows_tensor(sv[r], c, w).cpu().numpy()
            check_same(single, si.ImageBuffer(data=out), reps, G)
    finally:
        for cm in comms:
            cm.close()


def test_fp32_needs_an_output_buffer(solver):
    import torch
    f = si.synthetic_test_image(64, 48, 1, 1)
    m = si.random_mask(64, 48, 0.1, 2)
    comm = S.local_comms([solver])[0]
    try:
        df = torch.from_numpy(f.data).cuda()
        dm = torch.from_numpy(m.known).cuda()
        with pytest.raises(si.InvalidArgument, match="FP32"):
            S.run_method_striped_device(solver, comm, si.Method.MultilevelOras, df.data_ptr(),
                                        dm.data_ptr(), 64, 48, 1, None,
                                        si.RunOptions(precision=si.Precision.FP32))
    finally:
        comm.close()


@pytest.mark.parametrize("G", [1, 2, 4])
def test_local_device_group_call(solver, G):
    """si_run_method_striped_local_device: the whole group in one call (the
    group's persistent threads), repeated (speculative), rows in place and
    copied out."""
    import torch
    w, h, c = 777, 333, 3
    f = si.synthetic_test_image(w, h, c, 51)
    m = si.random_mask(w, h, 0.04, 52)
    o = si.RunOptions(levels=3, tolerance=1e-5)
    single = solver.run_method(si.Method.MultilevelOras, f, m, o)
    sv = solvers(G)
    comms = S.local_comms(sv)
    plans = [S.level_plan(si.Method.MultilevelOras, w, h, c, o, G, r)[0] for r in range(G)]
    ins = [(torch.from_numpy(np.ascontiguousarray(f.data[:, p.store_lo:p.store_hi])).cuda(),
            torch.from_numpy(np.ascontiguousarray(m.known[p.store_lo:p.store_hi])).cuda(),
            torch.empty((c, p.own_hi - p.own_lo, w), dtype=torch.float64, device="cuda"))
           for p in plans]
    torch.cuda.synchronize()
    try:
        for k in range(3):
            copy = k == 1
            reps = S.run_method_striped_local_device(
                sv, comms, si.Method.MultilevelOras, [i[0].data_ptr() for i in ins],
                [i[1].data_ptr() for i in ins], w, h, c,
                [i[2].data_ptr() for i in ins] if copy else None, o)
            out = np.zeros_like(f.data)
            for r, p in enumerate(plans):
                rows = ins[r][2] if copy else S.result_rows_tensor(sv[r], c, w)
                out[:, p.own_lo:p.own_hi] = rows.cpu().numpy()
            check_same(single, si.ImageBuffer(data=out), reps, G)
        assert comms[0].counters()["speculative"] == 2
    finally:
        for cm in comms:
            cm.close()


def test_local_device_group_error_reaches_caller(solver):
    import torch
    f = si.synthetic_test_image(64, 64, 1, 1)
    m = si.InpaintingMask(64, 64, 0)
    sv = solvers(2)
    comms = S.local_comms(sv)
    plans = [S.level_plan(si.Method.MultilevelOras, 64, 64, 1, None, 2, r)[0] for r in range(2)]
    ins = [(torch.from_numpy(np.ascontiguousarray(f.data[:, p.store_lo:p.store_hi])).cuda(),
            torch.from_numpy(np.ascontiguousarray(m.known[p.store_lo:p.store_hi])).cuda())
           for p in plans]
    try:
        with pytest.raises(si.InvalidArgument, match="no known pixels"):
            S.run_method_striped_local_device(sv, comms, si.Method.MultilevelOras,
                                              [i[0].data_ptr() for i in ins],
                                              [i[1].data_ptr() for i in ins], 64, 64, 1)
    finally:
        for cm in comms:
            cm.close()


def test_cpp_dropin_striped_two_threads(tmp_path, solver):
    """include/schwarz_b200.hpp: StripeComm::local + run_method_striped from
    two C++ threads (two contexts on one GPU), solved twice (the second
    speculates); the assembled image equals the single-GPU run_method."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include <thread>
#include "schwarz_b200.hpp"
namespace sb = schwarz_b200;
int main() {
  auto f = sb::synthetic_test_image(640, 480, 3, 9);
  auto m = sb::random_mask(640, 480, 0.05, 10);
  sb::RunOptions o; o.tolerance = 1e-5;
  auto single = sb::run_method(sb::Method::MultilevelOras, f, m, o);
  sb::Context c0(0), c1(0);
  auto comms = sb::StripeComm::local({&c0, &c1});
  int ok = 1;
  for (int rep = 0; rep < 2; ++rep) {
    sb::SolveResult r[2];
    std::thread t([&] { r[1] = sb::run_method_striped(sb::Method::MultilevelOras, f, m, o, comms[1], c1); });
    r[0] = sb::run_method_striped(sb::Method::MultilevelOras, f, m, o, comms[0], c0);
    t.join();
    for (size_t i = 0; i < f.data.size(); ++i) {
      const double v = r[0].image.data[i] + r[1].image.data[i];  // own rows are disjoint
      if (v != single.image.data[i]) ok = 0;
    }
    for (auto& x : r)
      if (x.report.level_iterations != single.report.level_iterations ||
          x.report.local_cg_iterations != single.report.local_cg_iterations ||
          x.trace.rows.size() != single.trace.rows.size()) ok = 0;
  }
  long long cnt[3];
  si_stripe_comm_counters(comms[0].get(), cnt);
  std::printf("%d %lld %lld\n", ok, cnt[0], cnt[1]);
  return 0;
}
''')
    lib_dir = os.path.join(root, "paper_2110_03946_b200")
    exe = str(tmp_path / "t")
    cc = subprocess.run(["g++", "-std=c++17", "-O2", "-pthread", "-I", os.path.join(root, "include"),
                         str(src), os.path.join(lib_dir, "libschwarz_b200.so"),
                         f"-Wl,-rpath,{lib_dir}", "-o", exe], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stderr
    assert run.stdout.split() == ["1", "2", "1"], run.stdout


def test_invalid_local_options_fail_like_the_reference(solver):
    """Invalid local CG options are rejected when the first sweep is about to
    run (cg_solve's check, cg.hpp:75-80), on every rank (the stripe engine
    never speculates with options the sweep would reject)."""
    f = si.synthetic_test_image(320, 240, 3, 61)
    m = si.random_mask(320, 240, 0.05, 62)
    o = si.RunOptions(levels=2)
    o.local.tolerance = 0.0
    with pytest.raises(si.InvalidArgument, match="tolerance must be positive"):
        solver.run_method(si.Method.MultilevelOras, f, m, o)
    sv = solvers(2)
    comms = S.local_comms(sv)
    try:
        with pytest.raises(si.InvalidArgument, match="tolerance must be positive"):
            _group_persistent(sv, comms, si.Method.MultilevelOras, f, m, o)
    finally:
        for cm in comms:
            cm.close()
