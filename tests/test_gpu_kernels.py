"""GPU parity of the individual kernels against the CPU oracle, through the C ABI.

Each test names the reference test or function it ports
(/root/reference/proj/tests/*.cpp, proj/include/schwarz_inpaint/*.hpp).
Integer/index work (partition, masks) must be bit-exact; floating-point
work states its tolerance inline.
"""
import numpy as np
import pytest

import paper_2110_03946_b200 as si
from instances import random_instance, random_vector

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- K1 residual
@pytest.mark.parametrize("w,h,c,d,seed", [(64, 48, 1, 0.1, 1), (97, 33, 3, 0.3, 2),
                                          (2, 1, 1, 1.0, 3), (5, 1, 2, 0.5, 4),
                                          (300, 200, 3, 0.04, 5)])
def test_residual_sumsq_matches_oracle(solver, oracle, w, h, c, d, seed):
    img, mask = random_instance(w, h, d, c, seed)
    rng = np.random.default_rng(seed)
    u = rng.uniform(0, 1, (c, h, w))
    b = np.where(mask.known[None] != 0, img.data, 0.0)
    got = solver.residual_sumsq(mask.known, u, b)
    for k in range(c):
        want = oracle.oracle_residual_sumsq(mask.known, u[k], b[k])
        # only the summation order differs (tree vs lane_sum): 1e-13 relative
        assert got[k] == pytest.approx(want, rel=1e-13, abs=1e-300)


# ---------------------------------------------------------------- K3 restriction
def test_restriction_two_by_two_rules(solver):
    """multilevel_test.cpp:13-41 (Restriction.TwoByTwoAveragingRules)."""
    mask = np.zeros((2, 4), np.uint8)
    vals = np.zeros((1, 2, 4))
    for x, y, v in [(0, 0, 0.2), (1, 0, 0.4), (0, 1, 0.6), (1, 1, 0.8), (2, 1, 0.3)]:
        mask[y, x] = 1
        vals[0, y, x] = v
    cm, cv = solver.restrict_level(mask, vals, si.CoarseAveraging.KnownOnly)
    assert cm.shape == (1, 2) and cm.all()
    assert abs(cv[0, 0, 0] - 0.5) <= 1e-15 and abs(cv[0, 0, 1] - 0.3) <= 1e-15
    cm, cv = solver.restrict_level(mask, vals, si.CoarseAveraging.AllPixels)
    assert abs(cv[0, 0, 1] - 0.3 / 4.0) <= 1e-15 and abs(cv[0, 0, 0] - 0.5) <= 1e-15


def test_restriction_empty_and_odd(solver):
    """multilevel_test.cpp:43-68."""
    cm, cv = solver.restrict_level(np.zeros((4, 4), np.uint8), np.zeros((1, 4, 4)))
    assert cm.sum() == 0 and (cv == 0).all()
    mask = np.zeros((5, 5), np.uint8)
    vals = np.zeros((1, 5, 5))
    mask[4, 4] = 1
    vals[0, 4, 4] = 0.9
    for avg in (si.CoarseAveraging.KnownOnly, si.CoarseAveraging.AllPixels):
        cm, cv = solver.restrict_level(mask, vals, avg)
        assert cm.shape == (3, 3) and cm[2, 2] == 1
        assert abs(cv[0, 2, 2] - 0.9) <= 1e-15


@pytest.mark.parametrize("avg", [0, 1])
def test_restriction_bitwise_vs_oracle(solver, oracle, avg):
    """OR rule + known-only mean (multilevel_test.cpp:70-95), bit-exact."""
    for trial in range(40):
        w, h = 3 + trial % 13, 3 + (trial * 7) % 11
        img, mask = random_instance(w, h, 0.02 + 0.6 * (trial % 10) / 10.0, 2, 1000 + trial)
        vals = np.where(mask.known[None] != 0, img.data, 0.0)
        cm, cv = solver.restrict_level(mask.known, vals, avg)
        om, ov = oracle.oracle_restrict(mask.known, vals, avg)
        assert np.array_equal(cm, om)
        assert np.array_equal(cv, ov)


def test_restriction_rejects_tiny(solver):
    with pytest.raises(si.InvalidArgument, match="at least 2x2"):
        solver.restrict_level(np.ones((1, 5), np.uint8), np.zeros((1, 1, 5)))


# ---------------------------------------------------------------- K4 prolongation
def test_prolongation_constant_and_bilinear(solver):
    """multilevel_test.cpp:125-152."""
    fine = solver.prolongate(np.full(6, 0.5), 3, 2, 6, 4)
    assert (fine == 0.5).all()
    fine = solver.prolongate(np.array([1.0, 2.0, 3.0, 4.0]), 2, 2, 4, 4).reshape(4, 4)
    assert fine[0, 0] == 1.0 and fine[0, 3] == 2.0 and fine[3, 0] == 3.0 and fine[3, 3] == 4.0
    assert fine[0, 1] == pytest.approx(0.75 * 1.0 + 0.25 * 2.0, abs=1e-15)
    assert fine[0, 2] == pytest.approx(0.25 * 1.0 + 0.75 * 2.0, abs=1e-15)
    assert fine[1, 0] == pytest.approx(0.75 * 1.0 + 0.25 * 3.0, abs=1e-15)
    assert fine[1, 1] == pytest.approx(0.75 * 0.75 * 1 + 0.25 * 0.75 * 2 + 0.75 * 0.25 * 3 +
                                       0.25 * 0.25 * 4, abs=1e-15)


def test_prolongation_rejects_mismatch(solver):
    """multilevel_test.cpp:154-159."""
    for args in [(2, 2, 5, 4), (2, 2, 4, 7)]:
        with pytest.raises(si.InvalidArgument):
            solver.prolongate(np.zeros(4), *args)


@pytest.mark.parametrize("fw,fh", [(73, 45), (8, 8), (3, 1), (640, 361), (1920, 1080), (260, 131)])
def test_prolongation_bitwise_vs_oracle(solver, oracle, fw, fh):
    """Even coarse widths take the persistent TMA-ring kernel, odd ones the
    one-shot kernel; both bit-identical to the oracle (multilevel.hpp:101-128)."""
    cw, ch = (fw + 1) // 2, (fh + 1) // 2
    coarse = np.random.default_rng(fw).uniform(0, 1, (ch, cw))
    got = solver.prolongate(coarse, cw, ch, fw, fh).reshape(fh, fw)
    want = oracle.oracle_prolongate(coarse, fw, fh)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- local operator
def test_robin_diagonal_at_cut_edges(solver):
    """schwarz_test.cpp:35-64 (LocalOperator.RobinDiagonalAtCutEdges)."""
    mask = np.zeros((3, 6), np.uint8)

    def col(flavour, alpha, j):
        e = np.zeros(9)
        e[j] = 1.0
        return solver.local_operator_apply(mask, 3, 1, 0, flavour, alpha, e)

    R, O = si.SchwarzFlavour.Ras, si.SchwarzFlavour.Oras
    cut = 1 * 3 + 2
    assert col(R, 0.5, cut)[cut] == 4.0
    assert col(O, 1.0, cut)[cut] == 4.0
    assert col(O, 0.5, cut)[cut] == 3.5
    assert col(O, 0.0, cut)[cut] == 3.0
    assert col(O, 0.5, 0)[0] == 2.0 and col(R, 0.5, 0)[0] == 2.0
    assert col(R, 0.5, 2)[2] == 3.0 and col(O, 0.5, 2)[2] == 2.5


def test_local_operator_known_rows_identity_and_symmetry(solver, oracle):
    """schwarz_test.cpp:66-94."""
    img, mask = random_instance(20, 20, 0.3, 1, 3)
    v = random_vector(64, 5)
    out = solver.local_operator_apply(mask.known, 8, 2, 3, si.SchwarzFlavour.Oras, 0.25, v)
    part = si.partition_domain(20, 20, 8, 2)
    sd = part.subdomains[3]
    known = mask.known[sd.y0:sd.y0 + 8, sd.x0:sd.x0 + 8].reshape(-1)
    assert np.array_equal(out[known != 0], v[known != 0])
    img, mask = random_instance(14, 14, 0.2, 1, 8)
    part = si.partition_domain(14, 14, 7, 2)
    for idx in range(part.size()):
        cols = np.stack([solver.local_operator_apply(mask.known, 7, 2, idx, si.SchwarzFlavour.Oras,
                                                     0.7, np.eye(49)[j]) for j in range(49)], 1)
        sd = part.subdomains[idx]
        unk = mask.known[sd.y0:sd.y0 + 7, sd.x0:sd.x0 + 7].reshape(-1) == 0
        sub = cols[np.ix_(unk, unk)]
        assert np.array_equal(sub, sub.T)


# ---------------------------------------------------------------- K2 sweep
@pytest.mark.parametrize("w,h,c,d,block,overlap,flavour,seed", [
    (64, 64, 1, 0.05, 16, 4, 1, 1),
    (96, 80, 3, 0.05, 32, 6, 1, 2),
    (50, 40, 2, 0.2, 32, 6, 1, 3),     # shifted last blocks
    (37, 23, 1, 0.3, 8, 3, 0, 4),      # RAS, small blocks
    (40, 40, 3, 0.1, 16, 4, 1, 5),
    (33, 31, 1, 0.02, 31, 0, 1, 6),    # single block, overlap 0
    (100, 70, 3, 0.01, 10, 3, 1, 7),
    (12, 12, 1, 0.0, 6, 2, 1, 8),      # almost empty mask
])
def test_single_sweep_matches_oracle(solver, oracle, w, h, c, d, block, overlap, flavour, seed):
    img, mask = random_instance(w, h, d, c, seed)
    b = np.where(mask.known[None] != 0, img.data, 0.0)
    u = b.copy()
    got, gfail, gits = solver.schwarz_sweep(mask.known, b, u, block, overlap, flavour)
    want, ofail, oits = oracle.oracle_sweep(mask.known, b, u, block, overlap, flavour=flavour)
    # fp64: only dot-product summation order differs inside the local CG.
    assert np.abs(got - want).max() <= 1e-10
    assert gits == oits and gfail == ofail


def test_sweep_arbitrary_u_and_b(solver, oracle):
    """The general formulas (known cells keep r = b - u, b != 0 at unknowns)."""
    rng = np.random.default_rng(11)
    img, mask = random_instance(70, 45, 0.15, 2, 12)
    b = rng.uniform(-1, 1, (2, 45, 70))
    u = rng.uniform(-1, 1, (2, 45, 70))
    got, _, _ = solver.schwarz_sweep(mask.known, b, u, 16, 5)
    want, _, _ = oracle.oracle_sweep(mask.known, b, u, 16, 5)
    assert np.abs(got - want).max() <= 1e-9


@pytest.mark.parametrize("w,h,c,d,block,overlap,flavour,seed", [
    (100, 90, 2, 0.05, 40, 8, 1, 21),   # K2g: blocks beyond 32x32
    (130, 70, 3, 0.03, 64, 12, 1, 22),
    (48, 48, 1, 0.1, 48, 0, 1, 23),     # one block, overlap 0
    (150, 97, 1, 0.2, 33, 5, 0, 24),    # RAS, shifted last blocks
])
def test_large_block_sweep_matches_oracle(solver, oracle, w, h, c, d, block, overlap, flavour,
                                          seed):
    img, mask = random_instance(w, h, d, c, seed)
    b = np.where(mask.known[None] != 0, img.data, 0.0)
    u = b.copy()
    got, gfail, gits = solver.schwarz_sweep(mask.known, b, u, block, overlap, flavour)
    want, ofail, oits = oracle.oracle_sweep(mask.known, b, u, block, overlap, flavour=flavour)
    assert np.abs(got - want).max() <= 1e-10
    assert gits == oits and gfail == ofail
    rng = np.random.default_rng(seed)
    b = rng.uniform(-1, 1, b.shape)
    u = rng.uniform(-1, 1, b.shape)
    got, _, _ = solver.schwarz_sweep(mask.known, b, u, block, overlap, flavour)
    want, _, _ = oracle.oracle_sweep(mask.known, b, u, block, overlap, flavour=flavour)
    assert np.abs(got - want).max() <= 1e-9


def test_division_shortcut_is_ieee_exact(solver):
    """beta = rr_new/rr runs as div_by_recip(rr_new, rr, RN(1/rr)); it must equal
    the IEEE quotient bit for bit (fp64 and fp32)."""
    import ctypes as C
    from paper_2110_03946_b200 import _lib as L
    bad = C.c_longlong(-1)
    assert L.load().si_selftest(solver.handle, 0, 50_000_000, C.byref(bad)) == 0
    assert bad.value == 0
