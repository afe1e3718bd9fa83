"""GPU parity of the Voronoi densification caller (SURVEY.md §8f item 4,
masks.hpp:45-215) through the C ABI (si_assign_nearest_site,
si_voronoi_densify).

Bar: the nearest-site assignment is integer work and must be bit-exact.  The
densified mask is compared byte for byte with the reference's (golden
fixtures from tests/golden/make_golden.py): the ranking consumes cell error
sums of a guide solve that matches the CPU to ~1e-12, so a flip needs two
cells within that distance; where the guide error is pure rounding noise
(the flat image) only the reference test's own properties are asserted.
"""
import os

import numpy as np
import pytest

import paper_2110_03946_b200 as si
from test_oracle import DENS, MG, densify_input

pytestmark = pytest.mark.gpu


def test_assignment_matches_reference_fixtures(solver):
    for i, (w, h, d, seed) in enumerate(MG.ASSIGN_CASES):
        m = si.InpaintingMask(known=DENS[f"assign{i}_mask"])
        a = solver.assign_nearest_site(m)
        assert np.array_equal(a.site_of, DENS[f"assign{i}_site_of"]), i
        assert np.array_equal(a.sites, np.flatnonzero(m.known.ravel()))


def test_assignment_random_masks_match_oracle(solver, oracle):
    rng = np.random.default_rng(3)
    for t in range(20):
        w, h = (int(v) for v in rng.integers(1, 400, 2))
        d = float(rng.choice([0.001, 0.01, 0.05, 0.3, 1.0]))
        d = max(d, 1.5 / (w * h))
        m = si.random_mask(w, h, min(d, 1.0), 100 + t)
        a = solver.assign_nearest_site(m)
        sites, site_of = oracle.oracle_assign_nearest_site(m.known)
        assert np.array_equal(a.sites, sites) and np.array_equal(a.site_of, site_of), (w, h, d)


def test_assignment_ties_and_ownership(solver):
    """masks_test.cpp:79-103."""
    m = si.InpaintingMask(7, 7)
    m.known[3, 1] = m.known[3, 5] = 1
    a = solver.assign_nearest_site(m)
    assert len(a.sites) == 2 and (a.site_of[:, 3] == 0).all()
    m = si.random_mask(40, 40, 0.06, 9)
    a = solver.assign_nearest_site(m)
    assert (a.site_of.ravel()[a.sites] == np.arange(len(a.sites))).all()
    assert (a.site_of >= 0).all()


def test_assignment_large_frame_properties(solver):
    """4K mask at 4%: every site owns itself and a sample of pixels agrees
    with brute force over all sites."""
    m = si.random_mask(3840, 2160, 0.04, 11)
    a = solver.assign_nearest_site(m)
    assert (a.site_of.ravel()[a.sites] == np.arange(len(a.sites))).all()
    ys, xs = np.divmod(a.sites.astype(np.int64), 3840)
    rng = np.random.default_rng(0)
    for p in rng.choice(3840 * 2160, 200, replace=False):
        py, px = divmod(int(p), 3840)
        d = (ys - py) ** 2 + (xs - px) ** 2
        assert a.site_of.ravel()[p] == int(np.argmin(d))


def test_assignment_rejects_empty_mask(solver):
    with pytest.raises(si.InvalidArgument, match="no known pixels"):
        solver.assign_nearest_site(si.InpaintingMask(8, 8))


@pytest.mark.parametrize("i", [0, 1, 2, 4, 5])
def test_densify_matches_reference(solver, i):
    spec, target, seed, dopts, sopts = MG.DENSIFY_CASES[i]
    f = si.ImageBuffer(data=densify_input(spec))
    opt = si.DensifyOptions(**dopts)
    for k, v in sopts.items():
        setattr(opt.solve, k, v)
    res = solver.voronoi_densify(f, target, seed, opt)
    gs, greached, gcount = DENS[f"densify{i}_stats"]
    assert (res.sweeps, int(res.reached_target), res.mask.known_count()) == (gs, greached, gcount)
    assert np.array_equal(res.mask.known, DENS[f"densify{i}_mask"])


def test_densify_flat_image_terminates(solver):
    """masks_test.cpp:159-166."""
    res = solver.voronoi_densify(si.ImageBuffer(32, 32, 1, 0.25), 0.1, 3)
    assert res.reached_target and res.mask.known_count() == round(0.1 * 32 * 32)


def test_densify_deterministic_and_monotone(solver):
    """masks_test.cpp:105-132."""
    img = si.synthetic_test_image(48, 48, 1, 5)
    opt = si.DensifyOptions(initial_density=0.02)
    a = solver.voronoi_densify(img, 0.10, 23, opt)
    b = solver.voronoi_densify(img, 0.10, 23, opt)
    assert np.array_equal(a.mask.known, b.mask.known) and a.sweeps == b.sweeps
    seeded = si.random_mask(48, 48, 0.02, 23)
    assert (a.mask.known[seeded.known != 0] == 1).all()


def test_densify_beats_random_mask(solver):
    """masks_test.cpp:134-157: error-guided placement beats uniform sampling."""
    img = si.synthetic_test_image(128, 128, 1, 7)
    rnd = si.random_mask(128, 128, 0.05, 31)
    ada = solver.voronoi_densify(img, 0.05, 31).mask
    assert ada.known_count() == rnd.known_count()
    o = si.RunOptions(tolerance=1e-4, block_size=16, overlap=3)
    a = solver.run_method(si.Method.MultilevelOras, img, rnd, o)
    b = solver.run_method(si.Method.MultilevelOras, img, ada, o)
    assert a.report.converged and b.report.converged
    assert si.psnr(img, b.image) > si.psnr(img, a.image) + 1.0


def test_densify_rejects_bad_targets(solver):
    """masks_test.cpp:168-176."""
    img = si.synthetic_test_image(16, 16, 1, 1)
    for t in (0.0, 1.2):
        with pytest.raises(si.InvalidArgument, match="target density"):
            solver.voronoi_densify(img, t, 1)
    with pytest.raises(si.InvalidArgument, match="initial density"):
        solver.voronoi_densify(img, 0.1, 1, si.DensifyOptions(initial_density=0.5))
