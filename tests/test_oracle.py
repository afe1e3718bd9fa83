"""CPU: pin the oracle (oracle/si_oracle.c) against the reference.

1. against the committed fixtures in tests/golden/ (produced from the
   unmodified reference by tests/golden/make_golden.py) — always runs;
2. against the compiled reference itself (oracle/_ref/libref.so) on a sweep
   of random instances and options — runs where _ref was built.
The restatement follows the reference's expression order and deterministic
sums, so agreement is expected to be bit-exact; the asserted bound is 1e-12.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2110_03946_b200 as si

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INPUTS = json.load(open(os.path.join(GOLD, "inputs.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen(w, h, c, d, si_, sm_):
    return si.synthetic_test_image(w, h, c, si_).data, si.random_mask(w, h, d, sm_).known


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_generators_reproduce_reference_inputs(name):
    """si_synthetic_test_image / si_random_mask emit the reference's bytes."""
    cfg = INPUTS[name]
    f, m = gen(cfg["w"], cfg["h"], cfg["c"], cfg["d"], 7, 11)
    assert sha(m) == cfg["mask"]
    assert int(m.sum()) == round(cfg["d"] * cfg["w"] * cfg["h"])
    assert sha(f) == cfg["image"]


def check_solve(got, gold_trace, gold_levels, tol=1e-12):
    assert got.level_iterations == list(gold_levels)
    assert got.trace.shape == gold_trace.shape
    assert np.allclose(got.trace, gold_trace, rtol=tol, atol=0)


def test_oracle_c1_full_output(oracle):
    g = np.load(os.path.join(GOLD, "c1.npz"))
    f, m = gen(256, 256, 1, 0.05, 7, 11)
    res = oracle.oracle_solve(f, m, levels=2)
    check_solve(res, g["trace"], g["level_iterations"])
    assert np.abs(res.image - g["image"]).max() <= 1e-12
    assert res.local_solves == int(g["local_solves"])
    assert res.local_failures == int(g["local_failures"])


@pytest.mark.parametrize("name,levels", [("c2", 2), ("c3", 3)])
def test_oracle_large_configs(oracle, name, levels):
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    cfg = INPUTS[name]
    f, m = gen(cfg["w"], cfg["h"], cfg["c"], cfg["d"], 7, 11)
    res = oracle.oracle_solve(f, m, levels=levels)
    check_solve(res, g["trace"], g["level_iterations"])
    assert np.allclose(res.image.sum(axis=(1, 2)), g["channel_sum"], rtol=1e-12, atol=0)
    assert np.abs(res.image.reshape(-1)[g["sample_index"]] - g["sample_value"]).max() <= 1e-12
    assert res.local_failures == int(g["local_failures"])


def test_oracle_small_cases(oracle):
    g = np.load(os.path.join(GOLD, "small.npz"))
    i = 0
    while f"case{i}_image" in g:
        cfg = INPUTS[f"small{i}"]
        f, m = gen(cfg["w"], cfg["h"], cfg["c"], cfg["d"], cfg["seed_image"], cfg["seed_mask"])
        res = oracle.oracle_solve(f, m, **cfg["options"])
        check_solve(res, g[f"case{i}_trace"], g[f"case{i}_levels"])
        assert np.abs(res.image - g[f"case{i}_image"]).max() <= 1e-12, i
        solves, fails, conv = g[f"case{i}_stats"]
        assert (res.local_solves, res.local_failures, int(res.converged)) == (solves, fails, conv)
        i += 1
    assert i == 12


def test_oracle_cg_cases(oracle):
    """The CG level solver restatement (reduction.hpp, cg.hpp:192-291) against
    run_method("cg"/"mlcg") of the reference."""
    g = np.load(os.path.join(GOLD, "cg.npz"))
    i = 0
    while f"case{i}_image" in g:
        cfg = INPUTS[f"cg{i}"]
        f, m = gen(cfg["w"], cfg["h"], cfg["c"], cfg["d"], cfg["seed_image"], cfg["seed_mask"])
        res = oracle.oracle_solve(f, m, flavour=2, **cfg["options"])
        its, conv = g[f"case{i}_iterations"]
        assert (res.iterations, int(res.converged)) == (its, conv)
        assert np.allclose(res.trace, g[f"case{i}_trace"], rtol=1e-12, atol=0)
        assert np.abs(res.image - g[f"case{i}_image"]).max() <= 1e-12
        i += 1
    assert i == 4


def test_oracle_kernels_bitwise(oracle):
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    for avg in (0, 1):
        cm, cv = oracle.oracle_restrict(g["restrict_in_mask"], g["restrict_in_values"], avg)
        assert np.array_equal(cm, g[f"restrict{avg}_mask"])
        assert np.array_equal(cv, g[f"restrict{avg}_values"])
    fine = oracle.oracle_prolongate(g["prolong_in"], 73, 45)
    assert np.array_equal(fine, g["prolong_out"])


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLD), "..", "oracle", "_ref",
                                                    "libref.so")),
                    reason="compiled reference (oracle/_ref) not present")
def test_oracle_matches_compiled_reference_sweep(oracle):
    """Random option sweep: restatement vs the reference, bit for bit."""
    rng = np.random.default_rng(1)
    mism = 0
    for t in range(25):
        w, h = (int(v) for v in rng.integers(5, 70, 2))
        c = int(rng.choice([1, 3]))
        d = float(rng.uniform(0.02, 0.5))
        f = oracle.ref_synthetic_test_image(w, h, c, 100 + t)
        m = oracle.ref_random_mask(w, h, d, 200 + t)
        opts = dict(levels=int(rng.integers(1, 5)), block_size=int(rng.integers(2, 33)),
                    flavour=int(rng.integers(0, 2)), alpha=float(rng.choice([0.25, 0.5, 1.0, 2.0])),
                    averaging=int(rng.integers(0, 2)), normalizer=int(rng.integers(0, 2)),
                    tolerance=float(rng.choice([1e-3, 1e-6])), max_outer_iterations=300)
        opts["overlap"] = int(rng.integers(0, opts["block_size"]))
        a = oracle.oracle_solve(f, m, **opts)
        b = oracle.ref_solve_levels(f, m, **opts)
        assert a.level_iterations == b.level_iterations
        assert np.allclose(a.trace, b.trace, rtol=1e-12, atol=0)
        assert np.abs(a.image - b.image).max() <= 1e-12
        mism += not np.array_equal(a.image, b.image)
    assert mism == 0  # bit-exact in practice


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLD), "..", "oracle", "_ref",
                                                    "libref.so")),
                    reason="compiled reference (oracle/_ref) not present")
def test_ref_driver_levels_loop_equals_run_method(oracle):
    f = oracle.ref_synthetic_test_image(120, 90, 3, 3)
    m = oracle.ref_random_mask(120, 90, 0.05, 4)
    a = oracle.ref_run_method("mloras", f, m, levels=3)
    b = oracle.ref_solve_levels(f, m, levels=3)
    assert np.array_equal(a.image, b.image) and np.array_equal(a.trace, b.trace)


# ---------------------------------------------------------------- densification
DENS = np.load(os.path.join(GOLD, "densify.npz"))


def _densify_cases():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLD, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg


MG = _densify_cases()


def densify_input(spec):
    if spec[0] == "flat":
        _, w, h, v = spec
        return np.full((1, h, w), v)
    w, h, c, seed = spec
    return si.synthetic_test_image(w, h, c, seed).data


def test_oracle_assignment_matches_reference_fixtures(oracle):
    """assign_nearest_site (masks.hpp:54-139): the restatement equals the
    reference on masks_test.cpp's trials plus larger and degenerate masks."""
    for i, (w, h, d, seed) in enumerate(MG.ASSIGN_CASES):
        m = si.random_mask(w, h, d, seed).known
        assert np.array_equal(m, DENS[f"assign{i}_mask"])
        sites, site_of = oracle.oracle_assign_nearest_site(m)
        assert np.array_equal(site_of, DENS[f"assign{i}_site_of"]), i
        assert np.array_equal(sites, np.flatnonzero(m.ravel()))


def test_oracle_assignment_brute_force_and_ties(oracle):
    """masks_test.cpp:79-103: the equidistant column goes to the lower site;
    every site owns itself; brute force agrees."""
    m = np.zeros((7, 7), np.uint8)
    m[3, 1] = m[3, 5] = 1
    _, site_of = oracle.oracle_assign_nearest_site(m)
    assert (site_of[:, 3] == 0).all()
    m = si.random_mask(40, 40, 0.06, 9).known
    sites, site_of = oracle.oracle_assign_nearest_site(m)
    assert (site_of.ravel()[sites] == np.arange(len(sites))).all()
    ys, xs = np.divmod(sites, 40)
    py, px = np.mgrid[0:40, 0:40]
    d = (py[..., None] - ys) ** 2 + (px[..., None] - xs) ** 2
    assert np.array_equal(site_of, np.argmin(d, axis=-1))  # argmin: first (lowest) index on ties


@pytest.mark.parametrize("i", range(6))
def test_oracle_densify_matches_reference_fixtures(oracle, i):
    """voronoi_densify (masks.hpp:155-212) restated in C equals the reference's
    mask and sweep count from the same seed mask."""
    spec, target, seed, dopts, sopts = MG.DENSIFY_CASES[i]
    f = densify_input(spec)
    c, h, w = f.shape
    init = oracle.densify_seed_density(target, w * h, dopts.get("initial_density", 0.0))
    seed_mask = si.random_mask(w, h, init, seed).known
    kw = {k: v for k, v in dopts.items() if k != "initial_density"}
    mask, sweeps = oracle.oracle_voronoi_densify(f, seed_mask, target, **kw, **sopts)
    gs, greached, gcount = DENS[f"densify{i}_stats"]
    assert sweeps == gs and int(mask.sum()) == gcount
    assert np.array_equal(mask, DENS[f"densify{i}_mask"])
