"""Generate tests/golden/ fixtures from the UNMODIFIED reference.

Runs only where the reference was compiled (oracle/_ref/libref.so, built by
oracle/Makefile from /root/reference/proj/include).  Every fixture records
the reference's own outputs on seeded inputs from its own generators:

  inputs.json   sha256 of synthetic_test_image / random_mask bytes per config
  c1.npz        256x256 grey, 5%, 2 levels: full output, trace, level counts
  c2.npz/c3.npz 1080p / 4K RGB: trace, level counts, local-solve statistics,
                per-channel sums and 4096 sampled output pixels
  c4k{1,2,3}.npz  4K RGB frames k = 1..3 of BASELINE configs[3] (seeds 7+k, 11+k)
  c5.npz        8K RGB, 2%, 3 levels (BASELINE configs[4]); same fields
  c5f.npz       C5 forced-sweep variant (tolerance 1e-12, max_outer_iterations 2)
  psnr.npz      run_method with a reference image: per-row rel and PSNR
                (metrics.hpp:30-56, multilevel.hpp:252-261)
  small.npz     12 small instances over the option space, full outputs
  kernels.npz   restriction / prolongation / local-operator probes
  densify.npz   assign_nearest_site / voronoi_densify (masks.hpp) outputs

Usage: python tests/golden/make_golden.py [--only densify|psnr|big|c5|c5f|c4k1 ...]
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as P  # noqa: E402

CONFIGS = {
    "c1": dict(w=256, h=256, c=1, d=0.05, levels=2),
    "c2": dict(w=1920, h=1080, c=3, d=0.04, levels=2),
    "c3": dict(w=3840, h=2160, c=3, d=0.04, levels=3),
}

# Headline-scale fixtures added in round 2: seeds (7+k, 11+k)
BIG = {
    "c4k1": dict(w=3840, h=2160, c=3, d=0.04, k=1, opts=dict(levels=3)),
    "c4k2": dict(w=3840, h=2160, c=3, d=0.04, k=2, opts=dict(levels=3)),
    "c4k3": dict(w=3840, h=2160, c=3, d=0.04, k=3, opts=dict(levels=3)),
    "c5": dict(w=7680, h=4320, c=3, d=0.02, k=0, opts=dict(levels=3)),
    "c5f": dict(w=7680, h=4320, c=3, d=0.02, k=0,
                opts=dict(levels=3, tolerance=1e-12, max_outer_iterations=2)),
}

# run_method(..., reference) trace rows with PSNR: (w, h, c, d, seed_img, seed_mask, method, opts)
PSNR_CASES = [
    (256, 256, 1, 0.05, 7, 11, "mloras", dict(levels=2)),
    (320, 240, 3, 0.04, 21, 22, "mloras", dict(levels=3, tolerance=1e-5)),
    (200, 120, 3, 0.06, 23, 24, "oras", dict(tolerance=1e-4)),
    (160, 96, 2, 0.08, 25, 26, "mlcg", dict(levels=2, flavour=2)),
]

SMALL = [
    # w, h, c, density, seed, options
    (64, 64, 1, 0.1, 1, dict(levels=1, tolerance=1e-6, block_size=16, overlap=4)),
    (64, 48, 3, 0.07, 2, dict(levels=1, tolerance=1e-6, block_size=16, overlap=4)),
    (40, 40, 3, 0.1, 3, dict(levels=1, tolerance=1e-6, block_size=16, overlap=4, flavour=0)),
    (96, 96, 1, 0.05, 4, dict(levels=3, block_size=16, overlap=3)),
    (48, 48, 1, 0.08, 5, dict(levels=3, tolerance=1e-8, block_size=16, overlap=4)),
    (123, 77, 3, 0.04, 6, dict(levels=4)),
    (9, 3, 1, 0.5, 7, dict(levels=5)),
    (33, 17, 2, 0.3, 8, dict(levels=3, averaging=1, normalizer=1)),
    (150, 90, 3, 0.02, 9, dict(levels=3, alpha=0.5, block_size=24, overlap=5)),
    (50, 40, 2, 0.2, 10, dict(levels=2, block_size=32, overlap=6)),
    (77, 31, 1, 0.15, 11, dict(levels=2, block_size=8, overlap=3, alpha=2.0)),
    (128, 128, 3, 0.05, 12, dict(levels=3, local_max_iterations=10, local_check_interval=4)),
]


CG_CASES = [
    # w, h, c, density, seed, method, options
    (256, 256, 1, 0.05, 1, "mlcg", dict(levels=2)),
    (64, 48, 3, 0.07, 2, "cg", dict(levels=1, tolerance=1e-6)),
    (123, 77, 3, 0.04, 3, "mlcg", dict(levels=3, cg_check_interval=1)),
    (40, 30, 2, 0.1, 4, "cg", dict(levels=1, cg_max_iterations=5)),
]


DENSIFY_CASES = [
    # image (w, h, c, seed) or ("flat", w, h, value), target, seed, DensifyOptions fields, solve
    ((64, 64, 1, 3), 0.08, 17, dict(max_sweeps=50), {}),
    ((48, 48, 1, 5), 0.10, 23, dict(initial_density=0.02), {}),
    ((128, 128, 1, 7), 0.05, 31, {}, {}),
    (("flat", 32, 32, 0.25), 0.10, 3, {}, {}),
    ((96, 80, 3, 9), 0.06, 5, dict(cell_fraction=0.3), dict(levels=2, block_size=16, overlap=3)),
    ((200, 150, 3, 11), 0.04, 8, dict(inner_tolerance=1e-4), {}),
]

ASSIGN_CASES = [  # masks_test.cpp:65-77 trials, then larger and degenerate masks
    *[(5 + 4 * (t % 5), 4 + 3 * (t % 4), 0.1 + 0.05 * t, 500 + t) for t in range(12)],
    (300, 200, 0.03, 5), (257, 129, 0.004, 6), (64, 64, 1.0 / 4096, 7), (1, 1, 1.0, 8),
]


def densify_image(spec):
    if spec[0] == "flat":
        _, w, h, v = spec
        return np.full((1, h, w), v)
    w, h, c, seed = spec
    return P.ref_synthetic_test_image(w, h, c, seed)


def densify_fixtures():
    out = {}
    for i, (spec, target, seed, dopts, sopts) in enumerate(DENSIFY_CASES):
        f = densify_image(spec)
        mask, sweeps, reached = P.ref_voronoi_densify(f, target, seed, **dopts, **sopts)
        out[f"densify{i}_mask"] = mask
        out[f"densify{i}_stats"] = np.array([sweeps, int(reached), int(mask.sum())])
    for i, (w, h, d, seed) in enumerate(ASSIGN_CASES):
        m = P.ref_random_mask(w, h, d, seed)
        sites, site_of = P.ref_assign_nearest_site(m)
        out[f"assign{i}_mask"] = m
        out[f"assign{i}_site_of"] = site_of
    np.savez_compressed(os.path.join(HERE, "densify.npz"), **out)
    print("densify fixtures:", [int(out[f"densify{i}_stats"][0]) for i in range(len(DENSIFY_CASES))])


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def instance(w, h, c, d, seed_img, seed_mask):
    return P.ref_synthetic_test_image(w, h, c, seed_img), P.ref_random_mask(w, h, d, seed_mask)


def big_fixtures(names=None):
    """Headline-size fixtures: counts, trace, local statistics, sums, samples."""
    hashes = {}
    for name, cfg in BIG.items():
        if names and name not in names:
            continue
        k = cfg["k"]
        f, m = instance(cfg["w"], cfg["h"], cfg["c"], cfg["d"], 7 + k, 11 + k)
        run = P.ref_run_method("mloras", f, m, **cfg["opts"])
        lv = P.ref_solve_levels(f, m, **cfg["opts"])
        assert np.array_equal(run.image, lv.image) and np.array_equal(run.trace, lv.trace)
        rng = np.random.default_rng(1234)
        idx = rng.choice(f.size, size=4096, replace=False)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), trace=run.trace,
            level_iterations=np.array(lv.level_iterations), iterations=run.iterations,
            final_rel=run.final_rel, converged=run.converged, local_solves=lv.local_solves,
            local_failures=lv.local_failures, channel_sum=run.image.sum(axis=(1, 2)),
            channel_sumsq=(run.image ** 2).sum(axis=(1, 2)), sample_index=idx,
            sample_value=run.image.reshape(-1)[idx])
        hashes[name] = {"image": sha(f), "mask": sha(m), "w": cfg["w"], "h": cfg["h"],
                        "c": cfg["c"], "d": cfg["d"], "seed_image": 7 + k, "seed_mask": 11 + k,
                        "options": cfg["opts"]}
        print(name, lv.level_iterations, run.trace, flush=True)
    return hashes


def psnr_fixtures():
    out = {}
    for i, (w, h, c, d, si_, sm_, meth, opts) in enumerate(PSNR_CASES):
        f, m = instance(w, h, c, d, si_, sm_)
        run = P.ref_run_method(meth, f, m, reference=f, **opts)
        assert np.isfinite(run.psnr).all()
        out[f"case{i}_trace"] = run.trace
        out[f"case{i}_psnr"] = run.psnr
        out[f"case{i}_image"] = run.image
    np.savez_compressed(os.path.join(HERE, "psnr.npz"), **out)
    print("psnr fixtures:", [len(out[f"case{i}_psnr"]) for i in range(len(PSNR_CASES))])


def merge_hashes(extra):
    path = os.path.join(HERE, "inputs.json")
    cur = json.load(open(path)) if os.path.exists(path) else {}
    cur.update(extra)
    with open(path, "w") as fh:
        json.dump(cur, fh, indent=1, sort_keys=True)


def main():
    if not P.ref_available():
        sys.exit("oracle/_ref/libref.so missing: run `make -C oracle` where /root/reference exists")
    P.ref().ref_set_threads(0)
    if "--only" in sys.argv:
        what = sys.argv[sys.argv.index("--only") + 1:]
        if "densify" in what:
            densify_fixtures()
        if "psnr" in what:
            psnr_fixtures()
        big = [w for w in what if w in BIG] or (list(BIG) if "big" in what else [])
        if big:
            merge_hashes(big_fixtures(big))
        return
    densify_fixtures()
    psnr_fixtures()
    densify_fixtures()
    hashes = {}
    for name, cfg in CONFIGS.items():
        f, m = instance(cfg["w"], cfg["h"], cfg["c"], cfg["d"], 7, 11)
        hashes[name] = {"image": sha(f), "mask": sha(m), **cfg}
        run = P.ref_run_method("mloras", f, m, levels=cfg["levels"])
        lv = P.ref_solve_levels(f, m, levels=cfg["levels"])
        assert np.array_equal(run.image, lv.image) and np.array_equal(run.trace, lv.trace)
        rng = np.random.default_rng(1234)
        idx = rng.choice(f.size, size=min(4096, f.size), replace=False)
        fields = dict(trace=run.trace, level_iterations=np.array(lv.level_iterations),
                      iterations=run.iterations, final_rel=run.final_rel,
                      converged=run.converged, local_solves=lv.local_solves,
                      local_failures=lv.local_failures, channel_sum=run.image.sum(axis=(1, 2)),
                      channel_sumsq=(run.image ** 2).sum(axis=(1, 2)), sample_index=idx,
                      sample_value=run.image.reshape(-1)[idx])
        if name == "c1":
            fields["image"] = run.image
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **fields)
        print(name, lv.level_iterations, run.trace)

    small = {}
    for i, (w, h, c, d, seed, opts) in enumerate(SMALL):
        f, m = instance(w, h, c, max(d, 1.5 / (w * h)), 1000 + seed, 77 + seed)
        lv = P.ref_solve_levels(f, m, **opts)
        small[f"case{i}_image"] = lv.image
        small[f"case{i}_trace"] = lv.trace
        small[f"case{i}_levels"] = np.array(lv.level_iterations)
        small[f"case{i}_stats"] = np.array([lv.local_solves, lv.local_failures, int(lv.converged)])
        hashes[f"small{i}"] = {"image": sha(f), "mask": sha(m), "w": w, "h": h, "c": c,
                               "d": max(d, 1.5 / (w * h)), "seed_image": 1000 + seed,
                               "seed_mask": 77 + seed, "options": opts}
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small)

    # multilevel CG (the paper's baseline method) through run_method itself
    cg = {}
    for i, (w, h, c, d, seed, meth, opts) in enumerate(CG_CASES):
        f, m = instance(w, h, c, d, 2000 + seed, 99 + seed)
        run = P.ref_run_method(meth, f, m, flavour=2, **opts)
        cg[f"case{i}_image"] = run.image
        cg[f"case{i}_trace"] = run.trace
        cg[f"case{i}_iterations"] = np.array([run.iterations, int(run.converged)])
        hashes[f"cg{i}"] = {"image": sha(f), "mask": sha(m), "w": w, "h": h, "c": c, "d": d,
                            "seed_image": 2000 + seed, "seed_mask": 99 + seed, "method": meth,
                            "options": opts}
    np.savez_compressed(os.path.join(HERE, "cg.npz"), **cg)

    # kernel probes: restriction (both averagings), prolongation, local operator
    k = {}
    f, m = instance(29, 23, 2, 0.3, 5, 6)
    vals = np.where(m[None] != 0, f, 0.0)
    for avg in (0, 1):
        cm = np.empty((12, 15), np.uint8)
        cv = np.empty((2, 12, 15))
        assert P.ref().ref_restrict_level(m.ravel(), vals.ravel(), 29, 23, 2, avg, cm.ravel(),
                                          cv.ravel()) == 0
        k[f"restrict{avg}_mask"], k[f"restrict{avg}_values"] = cm, cv
    k["restrict_in_mask"], k["restrict_in_values"] = m, vals
    coarse = np.random.default_rng(5).uniform(0, 1, (23, 37))
    fine = np.empty((45, 73))
    assert P.ref().ref_prolongate(coarse.ravel(), 37, 23, 73, 45, fine.ravel()) == 0
    k["prolong_in"], k["prolong_out"] = coarse, fine
    v = np.random.default_rng(9).uniform(-1, 1, 64)
    out = np.empty(64)
    assert P.ref().ref_local_operator_apply(m.ravel(), 29, 23, 8, 2, 5, 1, 0.25, v, out) == 0
    k["localop_mask"], k["localop_in"], k["localop_out"] = m, v, out
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **k)

    hashes.update(big_fixtures())
    merge_hashes(hashes)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
