"""End-to-end GPU parity of run_method / solve_schwarz / multilevel_solve.

Bar (stated per assertion):
  fp64: equal outer-iteration counts on every level; every trace row within
        1e-9 relative; output max-abs <= 1e-9 and MSE <= 1e-18.
  fp32: equal counts; trace rows within 1e-4 relative; output max-abs <= 5e-4
        and MSE <= 1e-10.
  mixed (double outer iteration, float local CG): equal counts; trace rows
        within 1e-5 relative; output max-abs <= 1e-4 and MSE <= 1e-12.
Behavioural tests port schwarz_test.cpp / multilevel_test.cpp /
acceptance_test.cpp properties to the GPU path.
"""
import os

import numpy as np
import pytest

import paper_2110_03946_b200 as si
from instances import C1, C2, config_instance, random_instance

pytestmark = pytest.mark.gpu

FP64 = dict(trace=1e-9, maxabs=1e-9, mse=1e-18)
FP32 = dict(trace=1e-4, maxabs=5e-4, mse=1e-10)
# double image / outer iteration, float local CG: the local solves stop at
# 1e-2, so float changes them at ~1e-7 relative
MIXED = dict(trace=1e-5, maxabs=1e-4, mse=1e-12)


def compare(res, ora, bar, levels=True):
    rep = res.report
    if levels:
        assert rep.level_iterations == ora.level_iterations, (rep.level_iterations,
                                                              ora.level_iterations)
    assert rep.iterations == ora.iterations
    got = np.array([r.rel_residual for r in res.trace.rows])
    assert got.shape == ora.trace.shape
    # |d rel| <= tol_rel * rel + 1e-15: the residual of a well-converged
    # iterate carries ~eps*|u|/r0 of absolute rounding noise.
    err = np.abs(got - ora.trace)
    assert (err <= bar["trace"] * np.abs(ora.trace) + 1e-15).all(), err / np.abs(ora.trace)
    diff = res.image.data - ora.image
    assert np.abs(diff).max() <= bar["maxabs"]
    assert np.mean(diff * diff) <= bar["mse"]
    assert rep.converged == ora.converged


def opts_dict(o: si.RunOptions, method):
    return dict(tolerance=o.tolerance, levels=o.levels if si.is_multilevel(method) else 1,
                block_size=o.block_size, overlap=o.overlap, alpha=o.alpha,
                coarse_tolerance=o.coarse_tolerance, averaging=int(o.averaging),
                local_tolerance=o.local.tolerance, local_max_iterations=o.local.max_iterations,
                local_check_interval=o.local.residual_check_interval,
                max_outer_iterations=o.max_outer_iterations, normalizer=int(o.normalizer),
                flavour=(2 if method in (si.Method.Cg, si.Method.MultilevelCg) else
                         0 if method == si.Method.Ras else 1),
                cg_max_iterations=o.cg_max_iterations, cg_check_interval=o.cg_check_interval)


@pytest.mark.parametrize("precision,bar", [(si.Precision.FP64, FP64), (si.Precision.FP32, FP32),
                                           (si.Precision.MIXED, MIXED)])
def test_c1_mloras_matches_oracle(solver, oracle, precision, bar):
    """BASELINE config 1: 256x256 grey, 5%, 2 levels (the CPU reference case)."""
    f, m = config_instance(C1)
    o = si.RunOptions(levels=2, precision=precision)
    res = solver.run_method(si.Method.MultilevelOras, f, m, o)
    ora = oracle.oracle_solve(f.data, m.known, **opts_dict(o, si.Method.MultilevelOras))
    assert ora.level_iterations == [2, 2]
    compare(res, ora, bar)
    assert res.report.local_cg_iterations == ora.local_cg_iterations or precision == si.Precision.FP32


@pytest.mark.slow
@pytest.mark.parametrize("precision,bar", [(si.Precision.FP64, FP64), (si.Precision.FP32, FP32),
                                           (si.Precision.MIXED, MIXED)])
def test_c2_mloras_matches_oracle(solver, oracle, precision, bar):
    """BASELINE config 2: 1920x1080 RGB, 4%, 2 levels."""
    f, m = config_instance(C2)
    o = si.RunOptions(levels=2, precision=precision)
    res = solver.run_method(si.Method.MultilevelOras, f, m, o)
    ora = oracle.oracle_solve(f.data, m.known, **opts_dict(o, si.Method.MultilevelOras))
    assert ora.level_iterations == [1, 2]
    compare(res, ora, bar)


RANDOM_CASES = [
    # (w, h, c, density, method, options)
    (64, 64, 1, 0.1, si.Method.Oras, dict(tolerance=1e-6, block_size=16, overlap=4)),
    (64, 48, 3, 0.07, si.Method.Oras, dict(tolerance=1e-6, block_size=16, overlap=4)),
    (40, 40, 3, 0.1, si.Method.Ras, dict(tolerance=1e-6, block_size=16, overlap=4)),
    (96, 96, 1, 0.05, si.Method.MultilevelOras, dict(block_size=16, overlap=3)),
    (48, 48, 1, 0.08, si.Method.MultilevelOras, dict(tolerance=1e-8, block_size=16, overlap=4)),
    (512, 512, 1, 0.05, si.Method.MultilevelOras, dict()),
    (123, 77, 3, 0.04, si.Method.MultilevelOras, dict(levels=4)),
    (9, 3, 1, 0.5, si.Method.MultilevelOras, dict(levels=5)),
    (33, 17, 2, 0.3, si.Method.MultilevelOras, dict(averaging=si.CoarseAveraging.AllPixels,
                                                    normalizer=si.ResidualNormalizer.RhsNorm)),
    (300, 170, 3, 0.02, si.Method.MultilevelOras, dict(alpha=0.5, block_size=24, overlap=5)),
    # degenerate shapes: clamped partitions down to 1x1 blocks
    (1, 2, 1, 0.5, si.Method.MultilevelOras, dict()),
    (1, 37, 2, 0.2, si.Method.MultilevelOras, dict(max_outer_iterations=60)),
    (53, 1, 1, 0.2, si.Method.Oras, dict(block_size=8, overlap=2, max_outer_iterations=60)),
    (2, 2, 3, 0.5, si.Method.MultilevelOras, dict(levels=3)),
    # staging paths: odd stride / odd W - B (cooperative) vs even anchors (TMA box)
    (777, 333, 3, 0.04, si.Method.MultilevelOras, dict()),
    (1000, 600, 3, 0.04, si.Method.MultilevelOras, dict()),
    (200, 150, 3, 0.05, si.Method.Oras, dict(overlap=5)),
    (180, 90, 8, 0.05, si.Method.MultilevelOras, dict(overlap=2, levels=2)),
    # blocks beyond 32x32 (K2g)
    (260, 190, 3, 0.04, si.Method.MultilevelOras, dict(block_size=64, overlap=10)),
    (120, 100, 1, 0.05, si.Method.Oras, dict(block_size=40, overlap=6)),
]


@pytest.mark.parametrize("w,h,c,d,method,kw", RANDOM_CASES)
def test_random_instances_match_oracle(solver, oracle, w, h, c, d, method, kw):
    f, m = random_instance(w, h, d, c, 1000 + w + h)
    o = si.RunOptions(**kw)
    res = solver.run_method(method, f, m, o)
    ora = oracle.oracle_solve(f.data, m.known, **opts_dict(o, method))
    compare(res, ora, FP64)


@pytest.mark.parametrize("w,h,c,d,method,kw", [RANDOM_CASES[i] for i in (0, 3, 6, 9, 14, 16)])
def test_random_instances_mixed_precision(solver, oracle, w, h, c, d, method, kw):
    """MIXED: double image and outer iteration, float local CG."""
    f, m = random_instance(w, h, d, c, 1000 + w + h)
    o = si.RunOptions(precision=si.Precision.MIXED, **kw)
    res = solver.run_method(method, f, m, o)
    ora = oracle.oracle_solve(f.data, m.known, **opts_dict(o, method))
    compare(res, ora, MIXED)


def test_acceptance_oracle_equivalence_dense(solver):
    """acceptance_test.cpp:39-67: mloras at tol 1e-8 agrees with a dense direct
    solve over 50 instances (8..32 pixels a side, 5-50% known)."""
    rng = np.random.default_rng(101)
    worst = 0.0
    for inst in range(50):
        w, h = rng.integers(8, 33, 2)
        c = 1 if inst % 2 == 0 else 3
        f = si.synthetic_test_image(int(w), int(h), c, 1000 + inst)
        m = si.random_mask(int(w), int(h), float(rng.uniform(0.05, 0.5)), 77 + inst)
        res = solver.run_method(si.Method.MultilevelOras, f, m,
                                si.RunOptions(tolerance=1e-8, max_outer_iterations=5000))
        assert res.report.converged
        exact = dense_inpaint(m.known, f.data)
        worst = max(worst, np.abs(res.image.data - exact).max())
    assert worst <= 1e-6


def dense_inpaint(mask, f):
    """tests/support/oracle.hpp:15-51 with numpy in place of Eigen's LU."""
    h, w = mask.shape
    n = w * h
    A = np.zeros((n, n))
    for y in range(h):
        for x in range(w):
            i = y * w + x
            if mask[y, x]:
                A[i, i] = 1.0
                continue
            deg = 0
            for xx, yy in ((x - 1, y), (x + 1, y), (x, y - 1), (x, y + 1)):
                if 0 <= xx < w and 0 <= yy < h:
                    A[i, yy * w + xx] -= 1.0
                    deg += 1
            A[i, i] = deg
    out = np.empty_like(f)
    for c in range(f.shape[0]):
        b = np.where(mask.reshape(-1) != 0, f[c].reshape(-1), 0.0)
        out[c] = np.linalg.solve(A, b).reshape(h, w)
    return out


# ---------------------------------------------------------------- behaviour
def tight(flavour=si.SchwarzFlavour.Oras, tol=1e-6, alpha=0.25, **kw):
    return si.SchwarzSolveOptions(si.SchwarzOptions(flavour, alpha, max_outer_iterations=5000,
                                                    **kw), tol)


def test_alpha_one_reproduces_ras_bitwise(solver):
    """schwarz_test.cpp:109-122."""
    f, m = random_instance(40, 40, 0.1, 3, 17)
    part = si.partition_domain(40, 40, 16, 4)
    ras = solver.solve_schwarz(f, m, part, tight(si.SchwarzFlavour.Ras))
    oras = solver.solve_schwarz(f, m, part, tight(si.SchwarzFlavour.Oras, alpha=1.0))
    assert ras.report.iterations == oras.report.iterations
    assert np.array_equal(ras.image.data, oras.image.data)


def test_single_block_exact_local_solve_one_iteration(solver):
    """schwarz_test.cpp:124-133."""
    f, m = random_instance(24, 24, 0.2, 1, 19)
    part = si.partition_domain(24, 24, 24, 4)
    assert part.size() == 1
    opt = tight(tol=1e-8, local=si.SolverConfig(1e-12, 100000, 50))
    res = solver.solve_schwarz(f, m, part, opt)
    assert res.report.converged and res.report.iterations == 1


def test_fixed_point_of_exact_solution(solver):
    """schwarz_test.cpp:135-150: run_schwarz_level from the dense solution."""
    f, m = random_instance(16, 16, 0.25, 1, 23)
    u = dense_inpaint(m.known, f.data)
    b = np.where(m.known[None] != 0, f.data, 0.0)
    r0 = solver.canonical_r0(m, b)
    part = si.partition_domain(16, 16, 8, 2)
    rep = solver.run_schwarz_level(m, part, b, u, r0, 1e-8, si.SchwarzOptions())
    assert rep.converged and rep.iterations == 0


def test_partition_independence(solver):
    """schwarz_test.cpp:152-166 / acceptance criterion 4."""
    f, m = random_instance(64, 64, 0.08, 1, 29)
    a = solver.solve_schwarz(f, m, si.partition_domain(64, 64, 16, 4), tight(tol=1e-8))
    b = solver.solve_schwarz(f, m, si.partition_domain(64, 64, 32, 6), tight(tol=1e-8))
    assert a.report.converged and b.report.converged
    assert np.abs(a.image.data - b.image.data).max() <= 1e-6


def test_oras_needs_no_more_iterations_than_ras(solver):
    """schwarz_test.cpp:168-178."""
    f, m = random_instance(64, 64, 0.05, 1, 31)
    part = si.partition_domain(64, 64, 16, 4)
    ras = solver.solve_schwarz(f, m, part, tight(si.SchwarzFlavour.Ras))
    oras = solver.solve_schwarz(f, m, part, tight())
    assert ras.report.converged and oras.report.converged
    assert oras.report.iterations <= ras.report.iterations


def test_maximum_principle_and_constants(solver):
    """schwarz_test.cpp:180-204."""
    f, m = random_instance(48, 32, 0.1, 1, 37)
    res = solver.solve_schwarz(f, m, si.partition_domain(48, 32, 16, 4), tight(tol=1e-8))
    assert res.report.converged
    kv = f.data[0][m.known != 0]
    assert res.image.data.min() >= kv.min() - 1e-6 and res.image.data.max() <= kv.max() + 1e-6
    flat = si.ImageBuffer(20, 20, 1, 0.4)
    mask = si.random_mask(20, 20, 0.1, 41)
    res = solver.solve_schwarz(flat, mask, si.partition_domain(20, 20, 8, 2), tight(tol=1e-8))
    assert np.abs(res.image.data - 0.4).max() <= 1e-6


def test_full_mask_returns_input_with_zero_iterations(solver):
    """schwarz_test.cpp:206-215."""
    mask = si.InpaintingMask(12, 12, 1)
    img = si.synthetic_test_image(12, 12, 1, 2)
    res = solver.solve_schwarz(img, mask, si.partition_domain(12, 12, 6, 2), tight(tol=1e-3))
    assert res.report.converged and res.report.iterations == 0
    assert np.array_equal(res.image.data, img.data)


def test_trace_rows_decrease_to_tolerance(solver):
    """schwarz_test.cpp:217-237 (with PSNR rows)."""
    f, m = random_instance(64, 64, 0.1, 1, 43)
    res = solver.solve_schwarz(f, m, si.partition_domain(64, 64, 16, 4), tight(), reference=f)
    rows = res.trace.rows
    assert res.report.converged and len(rows) >= 2
    assert rows[0].iteration == 0 and rows[0].rel_residual == 1.0
    for i in range(1, len(rows)):
        assert rows[i].rel_residual < rows[i - 1].rel_residual
        assert rows[i].time_ms >= rows[i - 1].time_ms
        assert rows[i].iteration == i and rows[i].psnr is not None
    assert rows[-1].rel_residual <= 1e-6
    assert rows[-1].psnr > rows[0].psnr


def test_neumann_cut_stays_robust(solver):
    """schwarz_test.cpp:257-268: alpha = 0 must not raise."""
    f, m = random_instance(24, 24, 0.3, 1, 53)
    opt = tight(alpha=0.0)
    opt.schwarz.max_outer_iterations = 500
    solver.solve_schwarz(f, m, si.partition_domain(24, 24, 8, 2), opt)


def test_levels_one_matches_direct_schwarz_bitwise(solver):
    """multilevel_test.cpp:161-182."""
    f, m = random_instance(40, 30, 0.1, 3, 7)
    mopt = si.MultilevelSolveOptions(levels=1, tolerance=1e-6, block_size=12, overlap=3)
    ml = solver.multilevel_solve(f, m, si.LevelSolver.Oras, mopt)
    sopt = si.SchwarzSolveOptions(tolerance=1e-6)
    sl = solver.solve_schwarz(f, m, si.partition_domain(40, 30, 12, 3), sopt)
    assert ml.report.iterations == sl.report.iterations
    assert np.array_equal(ml.image.data, sl.image.data)


def test_constant_image_zero_finest_iterations(solver):
    """multilevel_test.cpp:184-200."""
    flat = si.ImageBuffer(32, 32, 1, 0.7)
    mask = si.random_mask(32, 32, 0.1, 9)
    res = solver.multilevel_solve(flat, mask, si.LevelSolver.Oras,
                                  si.MultilevelSolveOptions(levels=3, block_size=8, overlap=2))
    assert res.report.converged and res.report.iterations == 0
    assert np.abs(res.image.data - 0.7).max() <= 0.01


def test_coarse_initialisation_cuts_finest_iterations(solver):
    """multilevel_test.cpp:202-218."""
    f, m = random_instance(96, 96, 0.05, 1, 11)
    flat = solver.multilevel_solve(f, m, si.LevelSolver.Oras,
                                   si.MultilevelSolveOptions(levels=1, block_size=16, overlap=3))
    nested = solver.multilevel_solve(f, m, si.LevelSolver.Oras,
                                     si.MultilevelSolveOptions(levels=3, block_size=16, overlap=3))
    assert flat.report.converged and nested.report.converged
    assert nested.report.iterations < flat.report.iterations


def test_errors_mirror_reference(solver):
    f, m = random_instance(16, 16, 0.2, 1, 1)
    with pytest.raises(si.InvalidArgument, match="no known pixels"):
        solver.run_method(si.Method.MultilevelOras, f, si.InpaintingMask(16, 16))
    with pytest.raises(si.InvalidArgument, match="tolerances must be positive"):
        solver.run_method(si.Method.MultilevelOras, f, m, si.RunOptions(tolerance=0.0))
    with pytest.raises(si.InvalidArgument, match="dimensions differ"):
        solver.run_method(si.Method.Oras, f, si.InpaintingMask(8, 16, 1))
    with pytest.raises(si.InvalidArgument, match="alpha must be finite"):
        solver.run_method(si.Method.Oras, f, m, si.RunOptions(alpha=float("nan")))
    with pytest.raises(si.SolverError, match="singular system"):  # reduction.hpp:109-110
        solver.run_method(si.Method.MultilevelCg, f, si.InpaintingMask(16, 16))


def test_non_convergence_is_reported_not_raised(solver):
    f, m = random_instance(64, 64, 0.05, 1, 3)
    res = solver.run_method(si.Method.Oras, f, m, si.RunOptions(tolerance=1e-12,
                                                               max_outer_iterations=2))
    assert not res.report.converged and res.report.iterations == 2
    assert "did not converge" in res.report.diagnostic


def test_batch_equals_individual_solves(solver):
    """si_run_method_batch (overlapped copies) == run_method frame by frame, bitwise."""
    frames = [random_instance(96, 64, 0.05, 3, 300 + k) for k in range(5)]
    o = si.RunOptions(levels=2)
    batch = solver.run_batch(si.Method.MultilevelOras, frames, o)
    for (f, m), b in zip(frames, batch):
        single = solver.run_method(si.Method.MultilevelOras, f, m, o)
        assert np.array_equal(single.image.data, b.image.data)
        assert single.report.level_iterations == b.report.level_iterations
        assert b.report.converged


def _device_solve(solver, method, f, m, o):
    """run_method through the device entry (dense on-device ingest)."""
    import torch
    df = torch.from_numpy(np.ascontiguousarray(f.data)).cuda()
    dm = torch.from_numpy(np.ascontiguousarray(m.known)).cuda()
    out = torch.empty_like(df)
    rep = solver.run_method_device(method, df.data_ptr(), dm.data_ptr(), f.width, f.height,
                                   f.channels, out.data_ptr(), o)
    torch.cuda.synchronize()
    return out.cpu().numpy(), rep


def test_known_sample_upload_matches_dense_ingest(solver):
    """si_run_method ships a sparse frame as mask + known samples (scatter
    kernel on the device); the result equals the dense device ingest bitwise,
    NaN at unknown pixels and mask bytes other than 1 included."""
    w, h, c = 701, 389, 3
    f = si.synthetic_test_image(w, h, c, 5)
    m = si.random_mask(w, h, 0.04, 6)
    m.known[m.known != 0] = 200
    f.data[:, m.known == 0] = np.nan
    o = si.RunOptions()
    res = solver.run_method(si.Method.MultilevelOras, f, m, o)
    want, rep = _device_solve(solver, si.Method.MultilevelOras, f, m, o)
    assert np.array_equal(res.image.data, want)
    assert res.report.level_iterations == rep.level_iterations
    K = int((m.known != 0).sum())
    tiles = (w * h + 4095) // 4096
    assert res.report.h2d_bytes == (tiles * 4 + 15) // 16 * 16 + K * c * 8 + w * h
    assert res.report.d2h_bytes == w * h * c * 8


def test_batch_known_sample_and_dense_frames(solver):
    """A batch mixing sparse frames (known-sample upload) and dense ones
    (mask density above 1/8: plain upload) equals the device path frame by
    frame, bitwise; the reports carry each frame's PCIe bytes."""
    w, h, c = 300, 200, 3
    dens = [0.04, 0.5, 0.02, 0.2, 0.04, 0.01]
    frames = []
    for k, d in enumerate(dens):
        f = si.synthetic_test_image(w, h, c, 40 + k)
        m = si.random_mask(w, h, d, 50 + k)
        f.data[:, m.known == 0] = np.inf
        frames.append((f, m))
    o = si.RunOptions()
    batch = solver.run_batch(si.Method.MultilevelOras, frames, o)
    for (f, m), b in zip(frames, batch):
        want, rep = _device_solve(solver, si.Method.MultilevelOras, f, m, o)
        assert np.array_equal(b.image.data, want)
        assert b.report.level_iterations == rep.level_iterations
        K = int((m.known != 0).sum())
        if K * 8 <= w * h:
            tiles = (w * h + 4095) // 4096
            assert b.report.h2d_bytes == (tiles * 4 + 15) // 16 * 16 + K * c * 8 + w * h
        else:
            assert b.report.h2d_bytes == w * h * c * 8 + w * h


@pytest.mark.parametrize("method,kw", [
    (si.Method.MultilevelOras, dict()),
    (si.Method.MultilevelOras, dict(levels=4, tolerance=1e-6)),
    (si.Method.MultilevelOras, dict(tolerance=1e-12, max_outer_iterations=3)),  # cap, odd
    (si.Method.Oras, dict(tolerance=1e-4)),
    (si.Method.Ras, dict(max_outer_iterations=0)),
    (si.Method.MultilevelOras, dict(precision=si.Precision.FP32)),
    (si.Method.MultilevelOras, dict(precision=si.Precision.MIXED, alpha=0.5, overlap=3)),
    (si.Method.MultilevelOras, dict(normalizer=si.ResidualNormalizer.RhsNorm, levels=2)),
    (si.Method.MultilevelCg, dict(levels=2)),   # host-driven CG levels in the batch
])
def test_batch_device_driven_levels_match_host_loop(solver, method, kw):
    """The batch entry runs the outer iteration as cached CUDA graphs with
    conditional nodes (decisions on the device); results and every report
    field equal the host-driven loop of the device entry, bitwise."""
    w, h, c = 230, 170, 3
    frames = []
    for k in range(4):
        f = si.synthetic_test_image(w, h, c, 60 + k)
        m = si.random_mask(w, h, 0.05, 70 + k)
        frames.append((f, m))
    o = si.RunOptions(**kw)
    batch = solver.run_batch(method, frames + frames[:2], o)  # repeats hit the graph cache
    for (f, m), b in zip(frames + frames[:2], batch):
        want, rep = _device_solve(solver, method, f, m, o)
        assert np.array_equal(b.image.data, want)
        r = b.report
        assert r.level_iterations == rep.level_iterations
        assert r.level_final_rel == rep.level_final_rel
        assert r.level_converged == rep.level_converged
        assert (r.iterations, r.final_relative_residual, r.converged) == \
            (rep.iterations, rep.final_relative_residual, rep.converged)
        assert (r.local_solves, r.local_failures, r.local_cg_iterations) == \
            (rep.local_solves, rep.local_failures, rep.local_cg_iterations)
        assert r.diagnostic == rep.diagnostic


@pytest.mark.parametrize("w,h,c", [(231, 171, 1), (97, 401, 5), (64, 33, 2)])
def test_batch_device_driven_odd_shapes(solver, w, h, c):
    """Odd widths (cooperative tile staging instead of TMA), many channels
    and clamped coarse partitions through the graph-mode batch."""
    frames = [(si.synthetic_test_image(w, h, c, 90 + k), si.random_mask(w, h, 0.06, 95 + k))
              for k in range(3)]
    o = si.RunOptions(levels=3)
    batch = solver.run_batch(si.Method.MultilevelOras, frames, o)
    for (f, m), b in zip(frames, batch):
        want, rep = _device_solve(solver, si.Method.MultilevelOras, f, m, o)
        assert np.array_equal(b.image.data, want)
        assert b.report.level_iterations == rep.level_iterations
        assert b.report.local_cg_iterations == rep.local_cg_iterations


@pytest.mark.parametrize("pinned_out", [False, True])
def test_batch_many_distinct_frames_no_slot_race(solver, pinned_out):
    """16 distinct small frames (the queueing thread runs far ahead of the
    device): every frame's inputs, outputs and report stay its own."""
    import torch
    w, h, c = 320, 200, 3
    frames = [(si.synthetic_test_image(w, h, c, 200 + k), si.random_mask(w, h, 0.03 + 0.01 * (k % 5),
                                                                         300 + k))
              for k in range(16)]
    outs = None
    if pinned_out:
        outs = [si.ImageBuffer(data=torch.empty((c, h, w), dtype=torch.float64).pin_memory().numpy())
                for _ in frames]
    o = si.RunOptions()
    batch = solver.run_batch(si.Method.MultilevelOras, frames, o, outs)
    for (f, m), b in zip(frames, batch):
        want, rep = _device_solve(solver, si.Method.MultilevelOras, f, m, o)
        assert np.array_equal(b.image.data, want)
        assert b.report.level_iterations == rep.level_iterations


def test_batch_empty_mask_in_a_later_frame_raises(solver):
    w, h = 300, 200
    good = (si.synthetic_test_image(w, h, 3, 1), si.random_mask(w, h, 0.05, 2))
    bad = (si.synthetic_test_image(w, h, 3, 3), si.InpaintingMask(w, h))
    with pytest.raises(si.InvalidArgument, match="no known pixels"):
        solver.run_batch(si.Method.MultilevelOras, [good, good, bad, good])
    # the context stays usable
    res = solver.run_batch(si.Method.MultilevelOras, [good])
    want, _ = _device_solve(solver, si.Method.MultilevelOras, *good, si.RunOptions())
    assert np.array_equal(res[0].image.data, want)


def test_known_sample_upload_empty_mask_raises(solver):
    f = si.synthetic_test_image(400, 300, 1, 1)
    m = si.InpaintingMask(400, 300)
    with pytest.raises(si.InvalidArgument, match="no known pixels"):
        solver.run_method(si.Method.MultilevelOras, f, m)
    with pytest.raises(si.InvalidArgument, match="no known pixels"):
        solver.run_batch(si.Method.MultilevelOras, [(f, m)])


# ---------------------------------------------------------------- multilevel CG
CG_CASES = [
    (si.Method.MultilevelCg, C1, dict(levels=2)),
    (si.Method.Cg, (64, 48, 3, 0.07, 1), dict(tolerance=1e-6)),
    (si.Method.MultilevelCg, (123, 77, 3, 0.04, 3), dict(cg_check_interval=1)),
    (si.Method.MultilevelCg, (96, 96, 1, 0.3, 3), dict(tolerance=1e-8, cg_check_interval=3)),
    (si.Method.Cg, (40, 30, 2, 0.1, 1), dict(cg_max_iterations=5)),   # hits the cap
]


@pytest.mark.parametrize("method,cfg,kw", CG_CASES)
def test_cg_level_solver_matches_oracle(solver, oracle, method, cfg, kw):
    """run_cg_level + cg_solve_lockstep (multilevel.hpp:162-209, cg.hpp:192-291)."""
    w, h, c, d, _ = cfg
    f, m = random_instance(w, h, d, c, 500 + w)
    o = si.RunOptions(**kw)
    res = solver.run_method(method, f, m, o)
    ora = oracle.oracle_solve(f.data, m.known, **opts_dict(o, method))
    compare(res, ora, FP64, levels=False)


@pytest.mark.slow
def test_c2_mlcg_matches_oracle(solver, oracle):
    f, m = config_instance(C2)
    o = si.RunOptions(levels=2)
    res = solver.run_method(si.Method.MultilevelCg, f, m, o)
    ora = oracle.oracle_solve(f.data, m.known, **opts_dict(o, si.Method.MultilevelCg))
    assert ora.iterations == 17
    compare(res, ora, FP64, levels=False)


# ---------------------------------------------------------------- PNM wire format
@pytest.mark.parametrize("w,h,c", [(160, 120, 3), (97, 61, 1), (256, 256, 3)])
def test_pnm_batch_matches_decoded_pipeline(solver, oracle, w, h, c):
    """read_pnm -> run_method -> write_pnm (pnm.hpp) with decode/quantise on the
    device equals the same pipeline through the f64 API (bit-exact bytes), and
    the CPU oracle's pipeline up to rounding-boundary bytes."""
    frames, decoded = [], []
    for k in range(3):
        f, m = random_instance(w, h, 0.06, c, 40 + k)
        px = si.quantise_pnm(f)
        frames.append((px, si.pack_pbm(m)))
        fd = (px.astype(np.float64) / 255.0)
        fd = fd[None] if c == 1 else np.moveaxis(fd, -1, 0)
        decoded.append((si.ImageBuffer(data=fd), m))
    reps, outs = solver.run_pnm_batch(si.Method.MultilevelOras, frames, si.RunOptions(levels=2))
    for (fd, m), rep, out in zip(decoded, reps, outs):
        ref = solver.run_method(si.Method.MultilevelOras, fd, m, si.RunOptions(levels=2))
        assert rep.level_iterations == ref.report.level_iterations
        assert np.array_equal(out, si.quantise_pnm(ref.image))
        ora = oracle.oracle_solve(fd.data, m.known, levels=2)
        diff = np.abs(out.astype(int) - si.quantise_pnm(si.ImageBuffer(data=ora.image)).astype(int))
        assert diff.max() <= 1 and np.count_nonzero(diff) <= max(1, diff.size // 10000)


@pytest.mark.parametrize("precision,overlap", [(0, 6), (1, 6), (0, 5), (1, 3)])
def test_tma_and_cooperative_staging_agree_bitwise(tmp_path, precision, overlap):
    """The sweep and residual kernels stage tiles by TMA (box start aligned
    down to 16 bytes left of each block, any anchor) and cooperatively
    otherwise (SI_NO_TMA=1 forces the latter): same arithmetic, so
    bit-identical results, fp64 and fp32, even and odd block strides."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_2110_03946_b200 as si\n"
        "from instances import random_instance\n"
        "f, m = random_instance(640, 480, 0.04, 3, 5)\n"
        "o = si.RunOptions(overlap=%d, precision=si.Precision(%d))\n"
        "r = si.Solver(0).run_method(si.Method.MultilevelOras, f, m, o)\n"
        "np.save(sys.argv[1], r.image.data)\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
         os.path.dirname(os.path.abspath(__file__)), overlap, precision)
    outs = []
    for k, env_extra in enumerate(({}, {"SI_NO_TMA": "1"})):
        path = str(tmp_path / f"u{k}.npy")
        env = dict(os.environ, **env_extra)
        run = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True,
                             text=True, timeout=300)
        assert run.returncode == 0, run.stderr
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


def test_cpp_dropin_header_on_device(tmp_path, solver):
    """include/schwarz_b200.hpp used the way a reference caller would
    (run_method, voronoi_densify) gives the Python/C-ABI results."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "t.cpp"
    src.write_text(
        '#include <cstdio>\n#include "schwarz_b200.hpp"\n'
        'int main() { namespace sb = schwarz_b200;\n'
        '  auto f = sb::synthetic_test_image(256, 256, 1, 7);\n'
        '  auto m = sb::random_mask(256, 256, 0.05, 11);\n'
        '  sb::RunOptions o; o.levels = 2;\n'
        '  auto r = sb::run_method(sb::Method::MultilevelOras, f, m, o);\n'
        '  double s = 0; for (double v : r.image.data) s += v;\n'
        '  std::printf("%d %d %.17g\\n", r.report.level_iterations[0], r.report.level_iterations[1], s);\n'
        '  auto g = sb::synthetic_test_image(64, 64, 1, 3);\n'
        '  sb::DensifyOptions d; d.max_sweeps = 50;\n'
        '  auto res = sb::voronoi_densify(g, 0.08, 17, d);\n'
        '  size_t k = 0; for (auto b : res.mask.known) k += b != 0;\n'
        '  std::printf("%d %d %zu\\n", res.sweeps, (int)res.reached_target, k);\n'
        '  auto m2 = sb::random_mask(256, 256, 0.05, 12);\n'
        '  auto b = sb::run_batch(sb::Method::MultilevelOras, {{&f, &m}, {&f, &m2}, {&f, &m}}, o);\n'
        '  int same = b[0].image.data == r.image.data && b[2].image.data == r.image.data;\n'
        '  std::printf("%d %d\\n", same, b[1].report.level_iterations[0]);\n'
        '  return 0; }\n')
    lib_dir = os.path.join(root, "paper_2110_03946_b200")
    exe = str(tmp_path / "t")
    cc = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(root, "include"), str(src),
                         os.path.join(lib_dir, "libschwarz_b200.so"), f"-Wl,-rpath,{lib_dir}",
                         "-o", exe], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stderr
    l1, l2, l3 = run.stdout.strip().splitlines()
    same, it_b1 = (int(v) for v in l3.split())
    assert same == 1  # run_batch == run_method, bitwise
    ref2 = solver.run_method(si.Method.MultilevelOras, si.synthetic_test_image(256, 256, 1, 7),
                             si.random_mask(256, 256, 0.05, 12), si.RunOptions(levels=2))
    assert it_b1 == ref2.report.level_iterations[0]
    it0, it1, checksum = l1.split()
    f = si.synthetic_test_image(256, 256, 1, 7)
    m = si.random_mask(256, 256, 0.05, 11)
    ref = solver.run_method(si.Method.MultilevelOras, f, m, si.RunOptions(levels=2))
    assert [int(it0), int(it1)] == ref.report.level_iterations
    assert float(checksum) == pytest.approx(float(ref.image.data.sum()), rel=1e-12)
    sweeps, reached, known = (int(v) for v in l2.split())
    dens = solver.voronoi_densify(si.synthetic_test_image(64, 64, 1, 3), 0.08, 17,
                                  si.DensifyOptions(max_sweeps=50))
    assert (sweeps, bool(reached), known) == (dens.sweeps, dens.reached_target,
                                              dens.mask.known_count())


@pytest.mark.parametrize("precision", [si.Precision.FP64, si.Precision.FP32, si.Precision.MIXED])
def test_bitwise_deterministic_across_runs_and_contexts(solver, precision):
    """The reference is bitwise identical for any thread count
    (schwarz_test.cpp:239-255, README.md:131-137); here every reduction has a
    fixed order, so repeated solves and independent contexts agree bit for bit."""
    f = si.synthetic_test_image(777, 333, 3, 21)
    m = si.random_mask(777, 333, 0.04, 22)
    o = si.RunOptions(precision=precision)
    a = solver.run_method(si.Method.MultilevelOras, f, m, o)
    b = solver.run_method(si.Method.MultilevelOras, f, m, o)
    other = si.Solver(0)
    c = other.run_method(si.Method.MultilevelOras, f, m, o)
    other.close()
    for r in (b, c):
        assert np.array_equal(a.image.data, r.image.data)
        assert [x.rel_residual for x in a.trace.rows] == [x.rel_residual for x in r.trace.rows]
        assert a.report.local_cg_iterations == r.report.local_cg_iterations


def test_concurrent_contexts_in_flight_match_sequential(solver):
    """bench.py's frames-in-flight mode: independent contexts, each on its own
    stream and host thread, solving device-resident frames at the same time
    give the bit-identical images and reports of one-at-a-time solves."""
    import threading

    import torch
    w, h, c = 640, 360, 3
    frames = []
    for k in range(4):
        f = si.synthetic_test_image(w, h, c, 40 + k)
        m = si.random_mask(w, h, 0.04, 50 + k)
        frames.append((torch.from_numpy(f.data).cuda(), torch.from_numpy(m.known).cuda()))
    o = si.RunOptions(levels=3)

    def solve(sv, j, out, stream):
        df, dm = frames[j]
        rep = sv.run_method_device(si.Method.MultilevelOras, df.data_ptr(), dm.data_ptr(), w, h,
                                   c, out.data_ptr(), o, stream=stream)
        return rep

    seq_out = [torch.empty((c, h, w), dtype=torch.float64, device="cuda") for _ in frames]
    seq_rep = [solve(solver, j, seq_out[j], torch.cuda.current_stream().cuda_stream)
               for j in range(len(frames))]
    torch.cuda.synchronize()

    lanes = [si.Solver(0), si.Solver(0)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    par_out = [torch.empty_like(x) for x in seq_out]
    par_rep = [None] * len(frames)

    def run(lane):
        for _ in range(3):  # repeated so the lanes' kernels really overlap
            for j in range(lane, len(frames), 2):
                par_rep[j] = solve(lanes[lane], j, par_out[j], streams[lane].cuda_stream)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    for lane in lanes:
        lane.close()
    for j in range(len(frames)):
        assert par_rep[j] is not None
        assert torch.equal(seq_out[j], par_out[j])
        assert par_rep[j].level_iterations == seq_rep[j].level_iterations
        assert par_rep[j].final_relative_residual == seq_rep[j].final_relative_residual


def test_many_channels(solver, oracle):
    """Channels are independent CTAs of one launch; the mapped scalar slots
    grow with the channel count (16 and 80 channels against the oracle)."""
    for c, (w, h) in ((16, (96, 80)), (80, (40, 33))):
        f, m = random_instance(w, h, 0.05, c, 5)
        o = si.RunOptions(levels=2)
        res = solver.run_method(si.Method.MultilevelOras, f, m, o)
        ora = oracle.oracle_solve(f.data, m.known, **opts_dict(o, si.Method.MultilevelOras))
        compare(res, ora, FP64)


def test_cpp_dropin_lower_seams(tmp_path, solver, oracle):
    """The C++ drop-in's lower seams, called the way the reference's own
    callers call them: tools/alpha_calibrate.cpp's body (solve_schwarz on
    partition_domain, SchwarzSolveOptions, alpha_calibrate.cpp:17-30),
    multilevel_solve with each LevelSolver (multilevel.hpp:239-241), and
    canonical_r0 + run_schwarz_level with a row sink (schwarz.hpp:266-270,
    333-345).  Counts equal the Python/C-ABI path and the oracle; images
    equal the Python path bit for bit (same library)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include <vector>
#include "schwarz_b200.hpp"
namespace si = schwarz_b200;
static double sum(const si::ImageBuffer& a) { double s = 0; for (double v : a.data) s += v; return s; }
int main() {
  // alpha_calibrate.cpp:17-30, verbatim call shapes
  const si::ImageBuffer image = si::synthetic_test_image(256, 256, 3, 7);
  const si::InpaintingMask mask = si::random_mask(256, 256, 0.05, 11);
  const auto partition = si::partition_domain(256, 256, 32, 6);
  auto outer_iterations = [&](si::SchwarzFlavour flavour, double alpha) {
    si::SchwarzSolveOptions opt;
    opt.schwarz.flavour = flavour;
    opt.schwarz.alpha = alpha;
    opt.schwarz.max_outer_iterations = 5000;
    opt.tolerance = 1e-6;
    const auto result = si::solve_schwarz(image, mask, partition, opt);
    return result.report.converged ? result.report.iterations : -1;
  };
  std::printf("%d %d %d\n", outer_iterations(si::SchwarzFlavour::Ras, 1.0),
              outer_iterations(si::SchwarzFlavour::Oras, 0.25),
              outer_iterations(si::SchwarzFlavour::Oras, 2.0));
  // multilevel_solve with every level solver
  si::MultilevelSolveOptions ml;
  ml.levels = 3;
  for (si::LevelSolver s : {si::LevelSolver::Oras, si::LevelSolver::Ras, si::LevelSolver::Cg}) {
    const auto r = si::multilevel_solve(image, mask, s, ml);
    std::printf("%d %.17g %d\n", r.report.iterations, sum(r.image), (int)r.trace.rows.size());
  }
  // canonical_r0 + run_schwarz_level: the finest seam with u in/out
  si::InpaintingOperator op(mask);
  std::vector<si::ChannelVector> b(3, si::ChannelVector(256 * 256, 0.0)), u;
  for (int c = 0; c < 3; ++c)
    for (size_t i = 0; i < b[c].size(); ++i) b[c][i] = mask.known[i] ? image.channel(c)[i] : 0.0;
  u = b;
  const double r0 = si::canonical_r0(op, b, si::ResidualNormalizer::InitialGuess);
  int rows = 0;
  double last = -1;
  si::SchwarzOptions so;
  const auto st = si::run_schwarz_level(op, partition, b, u, r0, 1e-4, so,
                                        [&](int it, double rel) { rows = it + 1; last = rel; });
  double su = 0;
  for (auto& c : u) for (double v : c) su += v;
  std::printf("%.17g %d %d %d %.17g %lld %.17g\n", r0, st.iterations, (int)st.converged, rows,
              last, st.local_solves, su);
  return 0;
}
''')
    lib_dir = os.path.join(root, "paper_2110_03946_b200")
    exe = str(tmp_path / "t")
    cc = subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "include"), str(src),
                         os.path.join(lib_dir, "libschwarz_b200.so"), f"-Wl,-rpath,{lib_dir}",
                         "-o", exe], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stderr
    lines = run.stdout.strip().splitlines()
    f = si.synthetic_test_image(256, 256, 3, 7)
    m = si.random_mask(256, 256, 0.05, 11)
    part = si.partition_domain(256, 256, 32, 6)
    # alpha_calibrate: outer counts vs the Python path and the oracle
    want = []
    for flav, alpha in ((si.SchwarzFlavour.Ras, 1.0), (si.SchwarzFlavour.Oras, 0.25),
                        (si.SchwarzFlavour.Oras, 2.0)):
        opt = si.SchwarzSolveOptions(tolerance=1e-6)
        opt.schwarz.flavour, opt.schwarz.alpha, opt.schwarz.max_outer_iterations = flav, alpha, 5000
        r = solver.solve_schwarz(f, m, part, opt)
        ora = oracle.oracle_solve(f.data, m.known, levels=1, tolerance=1e-6, alpha=alpha,
                                  flavour=int(flav), max_outer_iterations=5000)
        assert r.report.iterations == ora.iterations
        want.append(r.report.iterations if r.report.converged else -1)
    assert [int(v) for v in lines[0].split()] == want
    for line, ls in zip(lines[1:4], (si.LevelSolver.Oras, si.LevelSolver.Ras, si.LevelSolver.Cg)):
        r = solver.multilevel_solve(f, m, ls, si.MultilevelSolveOptions(levels=3))
        it, s, rows = line.split()
        assert int(it) == r.report.iterations and int(rows) == len(r.trace.rows)
        assert float(s) == pytest.approx(float(r.image.data.sum()), rel=1e-13)
    r0, its, conv, rows, last, solves, su = lines[4].split()
    b = np.where(m.known[None] != 0, f.data, 0.0)
    assert float(r0) == pytest.approx(solver.canonical_r0(m, b), rel=1e-14)
    u = b.copy()
    tr = si.ConvergenceTrace()
    rep = solver.run_schwarz_level(m, part, b, u, float(r0), 1e-4, si.SchwarzOptions(), trace=tr)
    assert int(its) == rep.iterations and int(rows) == len(tr.rows) == rep.iterations + 1
    assert bool(int(conv)) == rep.converged and int(solves) == rep.local_solves
    assert float(last) == pytest.approx(tr.rows[-1].rel_residual, rel=1e-14)
    assert float(su) == pytest.approx(float(u.sum()), rel=1e-13)


def test_repeated_headline_solves_are_bit_identical(solver):
    """Race check in place of compute-sanitizer (closed on this GPU pool):
    the 4K frame solved repeatedly, and on a second context running
    concurrently on its own host thread, gives bit-identical images, trace
    rows, PSNR rows and counters -- any race in K2's barrier-free
    warp-boundary exchange, the TMEM-resident CG vectors or the reductions
    would show up as a difference."""
    import threading
    f = si.synthetic_test_image(3840, 2160, 3, 8)
    m = si.random_mask(3840, 2160, 0.04, 12)
    o = si.RunOptions(levels=3)
    runs = [solver.run_method(si.Method.MultilevelOras, f, m, o, reference=f) for _ in range(3)]
    other = si.Solver(0)
    conc = [None, None]

    def go(k, s):
        conc[k] = s.run_method(si.Method.MultilevelOras, f, m, o, reference=f)

    ts = [threading.Thread(target=go, args=(0, solver)), threading.Thread(target=go, args=(1, other))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    other.close()
    base = runs[0]
    for r in runs[1:] + conc:
        assert np.array_equal(r.image.data, base.image.data)
        assert [x.rel_residual for x in r.trace.rows] == [x.rel_residual for x in base.trace.rows]
        assert [x.psnr for x in r.trace.rows] == [x.psnr for x in base.trace.rows]
        assert r.report.local_cg_iterations == base.report.local_cg_iterations
        assert r.report.local_failures == base.report.local_failures


@pytest.mark.parametrize("size", [(3840, 2160, 3, 0.04), (640, 480, 3, 0.05)])
def test_data_movement_switches_are_bit_identical(size):
    """The pair pass deriving b from u0 and the unwritten level-0 b change
    only data movement: with SI_NO_PAIR_DERIVE / SI_NO_INGEST_FUSION (b0
    written and read back) the device path's image and report are the same
    bits."""
    import hashlib
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    w, h, c, d = size
    code = (
        "import sys, json, hashlib; sys.path.insert(0, %r)\n"
        "import torch\n"
        "import paper_2110_03946_b200 as si\n"
        "f = si.synthetic_test_image(%d, %d, %d, 7); m = si.random_mask(%d, %d, %r, 11)\n"
        "df = torch.from_numpy(f.data).cuda(); dm = torch.from_numpy(m.known).cuda()\n"
        "do = torch.empty_like(df)\n"
        "r = si.Solver(0).run_method_device(si.Method.MultilevelOras, df.data_ptr(),\n"
        "    dm.data_ptr(), %d, %d, %d, do.data_ptr(), si.RunOptions())\n"
        "torch.cuda.synchronize()\n"
        "print(json.dumps({'img': hashlib.sha256(do.cpu().numpy().tobytes()).hexdigest(),\n"
        "  'levels': list(r.level_iterations), 'rel': r.final_relative_residual.hex(),\n"
        "  'cg': r.local_cg_iterations, 'fails': r.local_failures}))\n"
    ) % (root, w, h, c, w, h, d, w, h, c)
    outs = []
    for env in ({}, {"SI_NO_PAIR_DERIVE": "1"}, {"SI_NO_INGEST_FUSION": "1"}):
        run = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                             timeout=300, env={**os.environ, **env})
        assert run.returncode == 0, run.stderr[-2000:]
        outs.append(json.loads(run.stdout.strip().splitlines()[-1]))
    assert outs[1] == outs[0]
    assert outs[2] == outs[0]
