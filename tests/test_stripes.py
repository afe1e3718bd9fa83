"""Stripe decomposition of one image (BASELINE configs[4]).

CPU: the orchestrator (stripes.solve_striped) with G = 2, 3 ranks as threads
(ThreadComm) and as gloo processes (TorchComm), oracle compute backend;
the gathered result must equal the single-rank run bit for bit and match
the oracle's multilevel solve.  GPU: the same orchestrator on the device
kernels, G virtual ranks on one B200, against si_run_method (bit-identical:
only the norm's summation order differs).
"""
import os
import socket
import threading

import numpy as np
import pytest

import paper_2110_03946_b200 as si
from paper_2110_03946_b200 import stripes as S

W, H, CH = 160, 120, 2
OPTS = dict(levels=2, block_size=16, overlap=4)


def instance():
    f = si.synthetic_test_image(W, H, CH, 21)
    m = si.random_mask(W, H, 0.06, 5)
    return f.data, m.known


def test_stripe_plans_tile_rows():
    for h, b, o in [(2160, 32, 6), (4320, 32, 6), (120, 16, 4), (540, 32, 6), (1080, 32, 6)]:
        for world in (1, 2, 3, 4, 8):
            plans = [S.stripe_plan(h, b, o, world, r) for r in range(world)]
            assert all(p.valid for p in plans), (h, world)
            covered = np.zeros(h, np.int32)
            for p in plans:
                covered[p.own_lo:p.own_hi] += 1
                assert p.win_lo <= p.own_lo and p.own_hi <= p.win_hi
            assert (covered == 1).all()
            assert plans[0].k0 == 0 and plans[-1].k1 == plans[0].blocks_y


def _run_threads(world, backend_factory, f, m, opts):
    comms = S.ThreadComm.group(world)
    out = [None] * world
    err = []

    def run(r):
        try:
            be = backend_factory(r)
            u, rep = S.solve_striped(f, m, comms[r], be, si.RunOptions(**opts))
            w_, h_ = u.shape[2], u.shape[1]
            plan = rep.plans[0]
            spans = [(p.own_lo, p.own_hi) for p in
                     (S.stripe_plan(h_, *S.clamped(w_, h_, opts["block_size"], opts["overlap"]),
                                    world, q) for q in range(world))]
            S.gather_full(comms[r], u, plan, spans)
            out[r] = (u, rep)
        except Exception as e:  # surface worker failures
            err.append(e)
            comms[r].s.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_threads_match_single_rank_and_oracle(world):
    from stripes_cpu_backend import OracleBackend
    from oracle import pyoracle as P
    f, m = instance()
    single = _run_threads(1, lambda r: OracleBackend(), f, m, OPTS)[0]
    multi = _run_threads(world, lambda r: OracleBackend(), f, m, OPTS)
    for u, rep in multi:
        assert rep.level_iterations == single[1].level_iterations
        assert np.array_equal(u, single[0])
        assert np.allclose(rep.trace, single[1].trace, rtol=1e-12, atol=0)
    ora = P.oracle_solve(f, m, **OPTS)
    assert single[1].level_iterations == ora.level_iterations
    assert np.abs(single[0] - ora.image).max() <= 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, out_dir):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    from stripes_cpu_backend import OracleBackend
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = S.TorchComm(dist)
        f, m = instance()
        tf = torch.from_numpy(f)  # torch tensors so send/recv carry them
        tm = torch.from_numpy(m)

        class TorchOracle(OracleBackend):
            def copy(self, a):
                return a.clone() if hasattr(a, "clone") else torch.from_numpy(np.array(a))

            def ingest(self, f_, mask):
                b, k = OracleBackend.ingest(self, f_.numpy(), mask.numpy())
                return torch.from_numpy(b), k

            def restrict(self, mask, vals, averaging):
                cm, cv = OracleBackend.restrict(self, mask.numpy(), vals.numpy(), averaging)
                return torch.from_numpy(cm), torch.from_numpy(cv)

            def prolong_snap(self, coarse, fmask, fvals):
                return torch.from_numpy(OracleBackend.prolong_snap(
                    self, coarse.numpy(), fmask.numpy(), fvals.numpy()))

            def residual_rows(self, mask, u, b, r0, r1, mode=0):
                return OracleBackend.residual_rows(self, mask.numpy(), u.numpy(), b.numpy(), r0,
                                                   r1, mode)

            def sweep_rows(self, mask, b, u_old, u_new, *a):
                un = u_new.numpy()
                OracleBackend.sweep_rows(self, mask.numpy(), b.numpy(), u_old.numpy(), un, *a)
                return 0, 0

        u, rep = S.solve_striped(tf, tm, comm, TorchOracle(), si.RunOptions(**OPTS))
        w_, h_ = W, H
        plans = [S.stripe_plan(h_, *S.clamped(w_, h_, 16, 4), world, q) for q in range(world)]
        S.gather_full(comm, u, rep.plans[0], [(p.own_lo, p.own_hi) for p in plans])
        if rank == 0:
            np.save(os.path.join(out_dir, "u.npy"), u.numpy())
            np.save(os.path.join(out_dir, "lv.npy"), np.array(rep.level_iterations))
    finally:
        dist.destroy_process_group()


def test_gloo_processes_match_single_rank(tmp_path):
    import torch.multiprocessing as mp
    from stripes_cpu_backend import OracleBackend
    f, m = instance()
    single = _run_threads(1, lambda r: OracleBackend(), f, m, OPTS)[0]
    mp.spawn(_gloo_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    u = np.load(os.path.join(tmp_path, "u.npy"))
    assert list(np.load(os.path.join(tmp_path, "lv.npy"))) == single[1].level_iterations
    assert np.array_equal(u, single[0])


@pytest.mark.gpu
@pytest.mark.parametrize("world,w,h,c,levels", [(2, 640, 480, 3, 3), (3, 1024, 600, 3, 3),
                                                (4, 1920, 1080, 3, 2)])
def test_device_stripes_match_single_gpu(world, w, h, c, levels):
    import torch
    f = si.synthetic_test_image(w, h, c, 9)
    m = si.random_mask(w, h, 0.04, 10)
    ref = si.default_solver().run_method(si.Method.MultilevelOras, f, m, si.RunOptions(levels=levels))
    df = torch.from_numpy(f.data).cuda()
    dm = torch.from_numpy(m.known).cuda()
    opts = dict(levels=levels, block_size=32, overlap=6)
    out = _run_threads(world, lambda r: S.DeviceBackend(si.Solver(0)), df, dm, opts)
    for u, rep in out:
        assert rep.level_iterations == ref.report.level_iterations, (rep.trace, rep.plans)
        assert np.array_equal(u.cpu().numpy(), ref.image.data)
        got = np.array(rep.trace)
        want = np.array([r.rel_residual for r in ref.trace.rows])
        assert np.allclose(got, want, rtol=1e-12, atol=1e-16)
