"""CPU: the stripe decomposition of one image (BASELINE configs[4], SURVEY.md
§8e) -- the C++ plan (si_stripe_level_plan, host only) and a numpy model of
the C++ executor (tests/stripes_cpu_model.py) over G ranks as threads and as
gloo processes (world size 2).  Rows outside a rank's store are NaN in the
model, so a pass proves the plan's windows, halos and transfers suffice; the
gathered image must equal the single-rank run and the oracle's multilevel
solve bit for bit (same blocks, same arithmetic).  The GPU executor itself
is tested in test_gpu_stripes.py.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2110_03946_b200 as si
from paper_2110_03946_b200 import stripes as S

W, H, CH = 160, 120, 2
OPTS = dict(levels=3, block_size=16, overlap=4)


def instance(w=W, h=H, c=CH):
    f = si.synthetic_test_image(w, h, c, 21)
    m = si.random_mask(w, h, 0.06, 5)
    return f.data, m.known


SHAPES = [(3840, 2160, 3), (7680, 4320, 3), (160, 120, 2), (777, 333, 1), (96, 70, 1),
          (1000, 600, 3), (33, 17, 2)]


@pytest.mark.parametrize("w,h,c", SHAPES)
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plan_invariants(w, h, c, world):
    o = si.RunOptions(levels=3)
    plans = [S.level_plan(si.Method.MultilevelOras, w, h, c, o, world, r) for r in range(world)]
    depth = len(plans[0])
    lh = [h]
    for _ in range(1, depth):
        lh.append((lh[-1] + 1) // 2)
    for l in range(depth):
        covered = np.zeros(lh[l], np.int32)
        for r in range(world):
            p = plans[r][l]
            covered[p.own_lo:p.own_hi] += 1
            if p.k1 > p.k0:
                # the window holds own +- 1 and lies inside the store
                assert p.win_lo <= max(0, p.own_lo - 1) and p.win_hi >= min(lh[l], p.own_hi + 1)
                assert p.store_lo <= p.win_lo and p.win_hi <= p.store_hi
            if p.need_hi > p.need_lo:
                assert p.store_lo <= p.need_lo and p.need_hi <= p.store_hi
            if l + 1 < depth:  # restriction source of the coarser store
                q = plans[r][l + 1]
                if q.store_hi > q.store_lo:
                    assert p.store_lo <= 2 * q.store_lo
                    assert min(2 * q.store_hi, lh[l]) <= p.store_hi
        assert (covered == 1).all()  # owned rows tile the level
        assert plans[0][l].k0 == 0
    # stores scale as 1/G: a rank holds its share plus halo rows of every
    # level (the coarse halos double on the way down: <= 4 x ~40 rows)
    if world > 1 and h >= 1000:
        for r in range(world):
            p = plans[r][0]
            assert p.store_hi - p.store_lo <= h / world + 160


def test_plan_rejects_cg_and_bad_ranks():
    with pytest.raises(si.SolverError):
        S.level_plan(si.Method.MultilevelCg, 64, 64, 1, None, 2, 0)
    with pytest.raises(si.InvalidArgument):
        S.level_plan(si.Method.MultilevelOras, 64, 64, 1, None, 2, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_threads_model_matches_single_rank_and_oracle(world):
    import stripes_cpu_model as M
    from oracle import pyoracle as P
    f, m = instance()
    o = si.RunOptions(**OPTS)
    single = M.run_threads(1, f, m, o)
    multi = M.run_threads(world, f, m, o)
    img1, img = M.assemble(single), M.assemble(multi)
    assert np.isfinite(img).all()
    assert np.array_equal(img, img1)
    for _, rep in multi:
        assert rep["level_iterations"] == single[0][1]["level_iterations"]
    ora = P.oracle_solve(f, m, **OPTS)
    assert multi[0][1]["level_iterations"] == ora.level_iterations
    assert np.array_equal(img, ora.image)


def test_threads_model_forced_sweeps_odd_shape():
    """Every level sweeps twice (halo exchange on every level), odd sizes."""
    import stripes_cpu_model as M
    from oracle import pyoracle as P
    f, m = instance(131, 97, 1)
    kw = dict(levels=3, block_size=16, overlap=4, tolerance=1e-12, coarse_tolerance=1e-12,
              max_outer_iterations=2)
    o = si.RunOptions(**kw)
    multi = M.run_threads(3, f, m, o)
    ora = P.oracle_solve(f, m, **kw)
    assert multi[0][1]["level_iterations"] == ora.level_iterations == [2, 2, 2]
    assert np.array_equal(M.assemble(multi), ora.image)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import stripes_cpu_model as M
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f, m = instance()
        u, rep = M.solve_model(f, m, M.GlooComm(dist), si.RunOptions(**OPTS))
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u,
                 levels=np.array(rep["level_iterations"]), trace=np.array(rep["trace"]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_oracle(tmp_path):
    from oracle import pyoracle as P
    mp.spawn(_gloo_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    parts = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(2)]
    img = np.nansum(np.stack([p["u"] for p in parts]), axis=0)
    f, m = instance()
    ora = P.oracle_solve(f, m, **OPTS)
    for p in parts:
        assert list(p["levels"]) == ora.level_iterations
        assert np.allclose(p["trace"], ora.trace, rtol=1e-12, atol=0)
    assert np.array_equal(img, ora.image)
