"""TEST INFRASTRUCTURE: a numpy model of the C++ stripe executor
(paper_2110_03946_b200/csrc/stripes.cuh) for CPU multi-rank tests.

It takes the decomposition from the library itself (si_stripe_level_plan,
host-only) and runs the executor's steps with the C oracle as the compute:
every level array is full-size but holds NaN outside the rank's store rows,
and a sweep's or prolongation's result is kept only on the rows the C++ code
writes.  Any read of a row the plan does not make valid therefore poisons
the result, so a pass proves the plan's windows, halos, prolongation needs
and transfers are sufficient.  Communicators: gloo (torch.distributed) or
threads of one process.
"""
import threading

import numpy as np

import paper_2110_03946_b200 as si
from oracle import pyoracle as P
from paper_2110_03946_b200 import stripes as S


def minus(a, b):
    """[a) \\ [b) as up to two (lo, hi) spans."""
    lo, hi = a
    if hi <= lo:
        return []
    ilo, ihi = max(lo, b[0]), min(hi, b[1])
    if ihi <= ilo:
        return [a]
    out = []
    if lo < ilo:
        out.append((lo, ilo))
    if ihi < hi:
        out.append((ihi, hi))
    return out


def xfers(own, want, rank):
    """plan_xfers (stripes.cuh): recvs = my wanted rows owned by p, sends =
    p's wanted rows I own, in (peer, span) order."""
    sends, recvs = [], []
    for p in range(len(own)):
        if p == rank:
            continue
        for a in want[rank]:
            lo, hi = max(a[0], own[p][0]), min(a[1], own[p][1])
            if hi > lo:
                recvs.append((p, lo, hi))
        for a in want[p]:
            lo, hi = max(a[0], own[rank][0]), min(a[1], own[rank][1])
            if hi > lo:
                sends.append((p, lo, hi))
    return sends, recvs


class GlooComm:
    def __init__(self, dist):
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def allgather(self, vals):
        import torch
        t = torch.tensor(vals, dtype=torch.float64)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        return np.stack([p.numpy() for p in parts])

    def exchange(self, arr, sends, recvs):
        import torch
        ops, bufs = [], []
        for p, lo, hi in recvs:
            b = torch.empty(arr[:, lo:hi].shape, dtype=torch.float64)
            bufs.append((lo, hi, b))
            ops.append(self.dist.P2POp(self.dist.irecv, b, p))
        for p, lo, hi in sends:
            ops.append(self.dist.P2POp(self.dist.isend,
                                       torch.from_numpy(np.ascontiguousarray(arr[:, lo:hi])), p))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        for lo, hi, b in bufs:
            arr[:, lo:hi] = b.numpy()


class ThreadComm:
    """world ranks as threads; a shared slot table and a barrier."""

    class Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = {}

    def __init__(self, shared, rank):
        self.s, self.rank, self.world = shared, rank, shared.world

    @classmethod
    def group(cls, world):
        sh = cls.Shared(world)
        return [cls(sh, r) for r in range(world)]

    def allgather(self, vals):
        self.s.slots[("ag", self.rank)] = np.array(vals, dtype=np.float64)
        self.s.barrier.wait()
        out = np.stack([self.s.slots[("ag", r)] for r in range(self.world)])
        self.s.barrier.wait()
        return out

    def exchange(self, arr, sends, recvs):
        self.s.slots[("x", self.rank)] = arr
        self.s.barrier.wait()
        got = [(lo, hi, self.s.slots[("x", p)][:, lo:hi].copy()) for p, lo, hi in recvs]
        self.s.barrier.wait()
        for lo, hi, v in got:
            arr[:, lo:hi] = v


def residual_sumsq_rows(mask, u, b, lo, hi, mode=0):
    """(b - A u)^2 summed over rows [lo, hi) per channel (operators.hpp:38-66);
    mode 1: ||b||^2 (RhsNorm)."""
    if mode == 1:
        return np.array([np.sum(b[k, lo:hi] ** 2) for k in range(b.shape[0])])
    out = []
    for k in range(u.shape[0]):
        uk = u[k]
        s = np.zeros_like(uk)
        deg = np.zeros_like(uk)
        s[:, 1:] += uk[:, :-1]; deg[:, 1:] += 1
        s[:, :-1] += uk[:, 1:]; deg[:, :-1] += 1
        s[1:, :] += uk[:-1, :]; deg[1:, :] += 1
        s[:-1, :] += uk[1:, :]; deg[:-1, :] += 1
        r = b[k] - np.where(mask != 0, uk, deg * uk - s)
        out.append(np.sum(r[lo:hi] ** 2))
    return np.array(out)


def nan_outside(arr, lo, hi):
    out = np.full_like(arr, np.nan)
    out[:, lo:hi] = arr[:, lo:hi]
    return out


def solve_model(f, mask, comm, options, method=si.Method.MultilevelOras):
    """The executor of stripes.cuh on one rank.  f (C, H, W), mask (H, W):
    the full host image (only store rows are used).  Returns (u, report):
    u holds the finest own rows (NaN elsewhere)."""
    o = options
    C_, H, W = f.shape
    G, me = comm.world, comm.rank
    plans = [S.level_plan(method, W, H, C_, o, G, r) for r in range(G)]
    depth = len(plans[0])
    flavour = 0 if method == si.Method.Ras else 1
    sp = lambda l, r, a: (getattr(plans[r][l], a + "_lo"), getattr(plans[r][l], a + "_hi"))
    shapes = [(W, H)]
    for _ in range(1, depth):
        shapes.append(((shapes[-1][0] + 1) // 2, (shapes[-1][1] + 1) // 2))
    # pyramid of the store rows: level 0 from f, then restriction
    masks = [mask]
    lo, hi = sp(0, me, "store")
    vals = [nan_outside(np.where(mask[None] != 0, f, 0.0), lo, hi)]
    for l in range(1, depth):
        cm, cv = P.oracle_restrict(masks[-1], np.nan_to_num(vals[-1], nan=np.nan),
                                   int(o.averaging))
        lo, hi = sp(l, me, "store")
        cv = nan_outside(cv, lo, hi)
        assert np.isfinite(cv[:, lo:hi]).all(), f"restriction read unstored rows at level {l}"
        masks.append(cm)
        vals.append(cv)
    # known-pixel check over the level-0 own rows
    lo, hi = sp(0, me, "own")
    known = comm.allgather([float(np.count_nonzero(mask[lo:hi]))]).sum()
    if known == 0:
        raise si.InvalidArgument("build_rhs: mask has no known pixels")
    rep = dict(level_iterations=[0] * depth, trace=[], converged=False, local_solves=0)
    u = None
    for level in range(depth - 1, -1, -1):
        pl = plans[me][level]
        own = sp(level, me, "own")
        w, h = shapes[level]
        m, b = masks[level], vals[level]
        if level == depth - 1:
            u = b.copy()  # canonical start u0 = b (multilevel.hpp:267-273)
        tol = o.tolerance if level == 0 else o.coarse_tolerance
        own_all = [sp(level, r, "own") for r in range(G)]
        want = [minus(sp(level, r, "win"), own_all[r]) for r in range(G)]
        halo_s, halo_r = xfers(own_all, want, me)
        r0 = None
        outer = 0
        nbx = si.partition_domain(w, h, pl.block, pl.overlap).blocks_x
        while True:
            if own[1] > own[0]:
                sums = residual_sumsq_rows(m, u, b, *own)
                r0s = residual_sumsq_rows(m, b, b, *own, mode=int(o.normalizer))
                assert np.isfinite(sums).all() and np.isfinite(r0s).all()
            else:
                sums = r0s = np.zeros(C_)
            g = comm.allgather(np.concatenate([sums, r0s]))
            tot = np.zeros(C_)
            tr0 = np.zeros(C_)
            for r in range(G):  # fixed rank order
                tot += g[r, :C_]
                tr0 += g[r, C_:]
            if r0 is None:
                r0 = si.api.L.load().si_joint_norm(
                    np.ascontiguousarray(tr0).ctypes.data_as(si.api.C.POINTER(si.api.C.c_double)),
                    C_)
            jn = si.api.L.load().si_joint_norm(
                np.ascontiguousarray(tot).ctypes.data_as(si.api.C.POINTER(si.api.C.c_double)), C_)
            rel = jn / r0 if r0 > 0 else 0.0
            if level == 0:
                rep["trace"].append(rel)
            rep["level_iterations"][level] = outer
            if rel <= tol:
                if level == 0:
                    rep["converged"] = True
                break
            if outer >= o.max_outer_iterations:
                break
            new = np.full_like(u, np.nan)
            if pl.k1 > pl.k0:
                full, _, _ = P.oracle_sweep(m, np.nan_to_num(b, nan=np.nan), u, pl.block,
                                            pl.overlap, flavour=flavour, alpha=o.alpha,
                                            local_tolerance=o.local.tolerance,
                                            local_max_iterations=o.local.max_iterations,
                                            local_check_interval=o.local.residual_check_interval)
                new[:, own[0]:own[1]] = full[:, own[0]:own[1]]
                assert np.isfinite(new[:, own[0]:own[1]]).all(), \
                    f"sweep read unstored rows at level {level}"
                rep["local_solves"] += nbx * (pl.k1 - pl.k0) * C_
            u = new
            comm.exchange(u, halo_s, halo_r)
            outer += 1
        if level > 0:
            want = [[s for s in minus(sp(level, r, "need"), sp(level, r, "win"))]
                    for r in range(G)]
            s_, r_ = xfers(own_all, want, me)
            comm.exchange(u, s_, r_)
            fw_lo, fw_hi = sp(level - 1, me, "win")
            fwid, fhei = shapes[level - 1]
            fine = np.full((C_, fhei, fwid), np.nan)
            if fw_hi > fw_lo:
                pro = np.stack([P.oracle_prolongate(u[k], fwid, fhei) for k in range(C_)])
                fm, fb = masks[level - 1], vals[level - 1]
                pro = np.where(fm[None] != 0, fb, pro)
                fine[:, fw_lo:fw_hi] = pro[:, fw_lo:fw_hi]
                assert np.isfinite(fine[:, fw_lo:fw_hi]).all(), \
                    f"prolongation read unstored rows at level {level}"
            u = fine
    lo, hi = sp(0, me, "own")
    return nan_outside(u, lo, hi), rep


def run_threads(world, f, mask, options, method=si.Method.MultilevelOras):
    comms = ThreadComm.group(world)
    out, err = [None] * world, []

    def run(r):
        try:
            out[r] = solve_model(f, mask, comms[r], options, method)
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


def assemble(results):
    img = np.nansum(np.stack([u for u, _ in results]), axis=0)
    return img
