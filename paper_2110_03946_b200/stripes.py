"""One very large image over G GPUs: horizontal stripes with halo exchange
(BASELINE.json configs[4]).

Every level of the pyramid is split by block rows of its own (clamped)
partition: rank g owns block rows [k0, k1) and the pixel rows those blocks own
(`si_stripe_plan`).  Each rank keeps full-size level buffers but only computes
its stripe, so the per-block arithmetic is identical to the single-GPU solve
and the result is bit-identical to it whenever the stop decisions agree (the
only difference is the summation order of the global residual norm).

Per outer iteration of a level (run_schwarz_level, schwarz.hpp:288-320):
  1. partial per-channel sums of (b - A u)^2 over the owned rows,
  2. all-reduce(sum) -> every rank takes the same rel <= tol decision,
  3. sweep of the owned block rows (u_old -> u_new on owned rectangles),
  4. halo exchange: the window rows owned by the neighbours g-1 / g+1.
Between levels the coarse iterate is all-gathered (coarse levels are 4x and
16x smaller), then prolongated and snapped locally.

The orchestration is written once against two small interfaces:
  * a communicator (`TorchComm` over torch.distributed — NCCL on B200s, gloo on
    CPU — or `ThreadComm`, G ranks as threads of one process), and
  * a compute backend (`DeviceBackend`: the CUDA kernels of libschwarz_b200.so
    on torch CUDA tensors; the CPU tests plug in a numpy/oracle backend).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _lib as L
from .api import RunOptions, _check


@dataclass
class StripePlan:
    blocks_y: int
    k0: int
    k1: int
    own_lo: int
    own_hi: int
    win_lo: int
    win_hi: int
    valid: bool


def stripe_plan(h: int, block: int, overlap: int, world: int, rank: int) -> StripePlan:
    out = (C.c_int * 8)()
    _check(L.load().si_stripe_plan(h, block, overlap, world, rank, out))
    return StripePlan(*out[:7], bool(out[7]))


def clamped(w: int, h: int, block: int, overlap: int):
    """clamped_partition (multilevel.hpp:146-150)."""
    be = min(block, min(w, h))
    return be, max(0, min(overlap, be - 1))


def level_shapes(w: int, h: int, levels: int):
    """build_pyramid's level sizes (multilevel.hpp:90-93)."""
    shapes = [(w, h)]
    while len(shapes) < levels:
        cw, ch = shapes[-1]
        if cw < 2 or ch < 2:
            break
        shapes.append(((cw + 1) // 2, (ch + 1) // 2))
    return shapes


def joint_norm(sums) -> float:
    """sqrt(sum_c sqrt(s_c)^2) with the reference's fma accumulate
    (schwarz.hpp:290-295), computed by the library's host code."""
    arr = np.ascontiguousarray(sums, dtype=np.float64)
    return L.load().si_joint_norm(arr.ctypes.data_as(C.POINTER(C.c_double)), arr.size)


# ----------------------------------------------------------------- communicators
class TorchComm:
    """torch.distributed (NCCL between B200s, gloo on CPU)."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device

    def allreduce_sum(self, vals: np.ndarray) -> np.ndarray:
        import torch
        t = torch.tensor(vals, dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t)
        return t.cpu().numpy()

    def exchange(self, sends: dict, recv_shapes: dict, like):
        """sends: {peer: tensor}; recv_shapes: {peer: shape} -> {peer: tensor}."""
        ops, out = [], {}
        for peer, shape in recv_shapes.items():
            out[peer] = like.new_empty(shape)
            ops.append(self.dist.P2POp(self.dist.irecv, out[peer], peer))
        for peer, t in sends.items():
            ops.append(self.dist.P2POp(self.dist.isend, t.contiguous(), peer))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return out

    def allgather_rows(self, arr, lo: int, hi: int, spans):
        """Fill rows [lo_r, hi_r) of every rank r into arr (C, H, W) in place."""
        import torch
        parts = []
        for r, (a, b) in enumerate(spans):
            parts.append(arr[:, a:b, :].contiguous() if r == self.rank else
                         arr.new_empty((arr.shape[0], b - a, arr.shape[2])))
        for r, (a, b) in enumerate(spans):
            if b > a:
                self.dist.broadcast(parts[r], src=r)
                if r != self.rank:
                    arr[:, a:b, :] = parts[r]
        return arr


class ThreadComm:
    """G ranks as threads of one process (single GPU or CPU emulation)."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = {}

    def __init__(self, shared: "ThreadComm._Shared", rank: int):
        self.s = shared
        self.rank = rank
        self.world = shared.world

    @classmethod
    def group(cls, world: int) -> List["ThreadComm"]:
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def _publish(self, key, value):
        self.s.slots[(key, self.rank)] = value
        self.s.barrier.wait()

    def _done(self):
        self.s.barrier.wait()

    def allreduce_sum(self, vals: np.ndarray) -> np.ndarray:
        self._publish("ar", np.asarray(vals, dtype=np.float64).copy())
        tot = np.zeros_like(np.asarray(vals, dtype=np.float64))
        for r in range(self.world):  # fixed order: identical on every rank
            tot = tot + self.s.slots[("ar", r)]
        self._done()
        return tot

    def exchange(self, sends: dict, recv_shapes: dict, like):
        self._publish("x", {peer: _copy(t) for peer, t in sends.items()})
        out = {peer: self.s.slots[("x", peer)][self.rank] for peer in recv_shapes}
        self._done()
        return out

    def allgather_rows(self, arr, lo: int, hi: int, spans):
        self._publish("ag", _copy(arr[:, lo:hi, :]))
        for r, (a, b) in enumerate(spans):
            if r != self.rank and b > a:
                arr[:, a:b, :] = self.s.slots[("ag", r)]
        self._done()
        return arr


def _copy(t):
    return t.clone() if hasattr(t, "clone") else np.array(t, copy=True)


# ----------------------------------------------------------------- device backend
class DeviceBackend:
    """The CUDA kernels of libschwarz_b200.so on torch CUDA tensors."""

    def __init__(self, solver, precision: int = 0, stream=None):
        import torch
        self.torch = torch
        self.solver = solver
        self.lib = solver._lib
        self.h = solver.handle
        self.precision = precision
        self.dtype = torch.float64 if precision == 0 else torch.float32
        self.dev = torch.device("cuda", solver.device)
        self.stream = stream

    def _pre(self):
        # torch work issued by the orchestrator (copies, halo writes) is on
        # torch's current stream; the library runs on its own stream and
        # returns synchronised, so ordering needs only this wait.
        self.torch.cuda.current_stream(self.dev).synchronize()

    def empty(self, c, h, w):
        return self.torch.empty((c, h, w), dtype=self.dtype, device=self.dev)

    def empty_mask(self, h, w):
        return self.torch.empty((h, w), dtype=self.torch.uint8, device=self.dev)

    def ingest(self, f, mask):
        self._pre()
        c, h, w = f.shape
        b = self.empty(c, h, w)
        known = C.c_longlong()
        _check(self.lib.si_device_ingest(self.h, f.data_ptr(), mask.data_ptr(), w, h, c,
                                         self.precision, b.data_ptr(), C.byref(known),
                                         self.stream))
        return b, known.value

    def restrict(self, mask, vals, averaging):
        self._pre()
        c, h, w = vals.shape
        cw, ch = (w + 1) // 2, (h + 1) // 2
        cm, cv = self.empty_mask(ch, cw), self.empty(c, ch, cw)
        _check(self.lib.si_device_restrict(self.h, mask.data_ptr(), vals.data_ptr(), w, h, c,
                                           averaging, self.precision, cm.data_ptr(),
                                           cv.data_ptr(), self.stream))
        return cm, cv

    def prolong_snap(self, coarse, fmask, fvals):
        self._pre()
        c, ch, cw = coarse.shape
        _, fh, fw = fvals.shape
        fine = self.empty(c, fh, fw)
        _check(self.lib.si_device_prolong_snap(self.h, coarse.data_ptr(), cw, ch, fw, fh, c,
                                               fmask.data_ptr(), fvals.data_ptr(), self.precision,
                                               fine.data_ptr(), self.stream))
        return fine

    def residual_rows(self, mask, u, b, row0, row1, mode=0):
        self._pre()
        c, h, w = u.shape
        sums = np.zeros(c)
        _check(self.lib.si_device_residual_rows(self.h, mask.data_ptr(), u.data_ptr(),
                                                b.data_ptr(), w, h, c, row0, row1, mode, 1,
                                                self.precision,
                                                sums.ctypes.data_as(C.POINTER(C.c_double)),
                                                self.stream))
        return sums

    def sweep_rows(self, mask, b, u_old, u_new, block, overlap, by0, by1, flavour, opts):
        self._pre()
        c, h, w = u_old.shape
        o = opts.to_c()
        fails, its = C.c_longlong(), C.c_longlong()
        _check(self.lib.si_device_sweep_rows(self.h, mask.data_ptr(), b.data_ptr(),
                                             u_old.data_ptr(), u_new.data_ptr(), w, h, c, block,
                                             overlap, by0, by1, flavour, C.byref(o), 1,
                                             C.byref(fails), C.byref(its), self.stream))
        return fails.value, its.value

    def copy(self, t):
        return t.clone()


# ----------------------------------------------------------------- the solve
@dataclass
class StripeReport:
    level_iterations: List[int]
    trace: List[float]
    converged: bool
    local_failures: int
    local_cg_iterations: int
    plans: List[StripePlan]


def solve_striped(f, mask, comm, backend, options: Optional[RunOptions] = None,
                  flavour: int = 1):
    """multilevel_solve (multilevel.hpp:239-310) with every level striped over
    comm.world ranks.  f: (C, H, W) float64 and mask (H, W) uint8 on the
    backend's device, replicated on every rank.  Returns (u, report): u holds
    the finest solution on the rank's owned rows; use gather_full() for all."""
    o = options or RunOptions()
    C_, H, W = f.shape
    shapes = level_shapes(W, H, o.levels)
    depth = len(shapes)
    b0, known = backend.ingest(f, mask)
    if known == 0:
        raise ValueError("build_rhs: mask has no known pixels")
    masks, vals = [mask], [b0]
    for l in range(1, depth):
        cm, cv = backend.restrict(masks[-1], vals[-1], int(o.averaging))
        masks.append(cm)
        vals.append(cv)
    rep = StripeReport([0] * depth, [], False, 0, 0, [])
    u = None
    for level in range(depth - 1, -1, -1):
        w, h = shapes[level]
        be, oe = clamped(w, h, o.block_size, o.overlap)
        plan = stripe_plan(h, be, oe, comm.world, comm.rank)
        if not plan.valid:
            raise ValueError(f"level {level}: stripes too thin for {comm.world} ranks")
        rep.plans.insert(0, plan)
        m, b = masks[level], vals[level]
        if level == depth - 1:
            u = backend.copy(b)  # canonical start u0 = b (multilevel.hpp:267-273)
        finest = level == 0
        tol = o.tolerance if finest else o.coarse_tolerance
        plans = [stripe_plan(h, be, oe, comm.world, r) for r in range(comm.world)]
        spans = [(p.own_lo, p.own_hi) for p in plans]
        r0 = joint_norm(comm.allreduce_sum(
            backend.residual_rows(m, b, b, plan.own_lo, plan.own_hi,
                                  1 if int(o.normalizer) == 1 else 0)))
        u_alt = backend.copy(u)
        outer = 0
        while True:
            sums = comm.allreduce_sum(backend.residual_rows(m, u, b, plan.own_lo, plan.own_hi))
            rel = joint_norm(sums) / r0 if r0 > 0 else 0.0
            if finest:
                rep.trace.append(rel)
            rep.level_iterations[level] = outer
            if rel <= tol:
                if finest:
                    rep.converged = True
                break
            if outer >= o.max_outer_iterations:
                break
            fails, its = backend.sweep_rows(m, b, u, u_alt, be, oe, plan.k0, plan.k1, flavour, o)
            rep.local_failures += fails
            rep.local_cg_iterations += its
            u, u_alt = u_alt, u
            _exchange_halos(comm, u, plans)
            outer += 1
        if not finest:
            comm.allgather_rows(u, plan.own_lo, plan.own_hi, spans)
            fw, fh = shapes[level - 1]
            u = backend.prolong_snap(u, masks[level - 1], vals[level - 1])
    return u, rep


def _exchange_halos(comm, u, plans: List[StripePlan]):
    """Rows of my window owned by rank-1 / rank+1 come from them; I send them
    the rows I own inside their windows (stripe_plan guarantees no other rank
    is involved)."""
    r = comm.rank
    me = plans[r]
    sends, recv = {}, {}
    for peer in (r - 1, r + 1):
        if not 0 <= peer < comm.world:
            continue
        pp = plans[peer]
        lo, hi = max(pp.win_lo, me.own_lo), min(pp.win_hi, me.own_hi)
        if hi > lo:
            sends[peer] = u[:, lo:hi, :]
        lo2, hi2 = max(me.win_lo, pp.own_lo), min(me.win_hi, pp.own_hi)
        if hi2 > lo2:
            recv[peer] = (lo2, hi2)
    got = comm.exchange(sends, {p: (u.shape[0], b - a, u.shape[2]) for p, (a, b) in recv.items()},
                        u)
    for p, (a, b) in recv.items():
        u[:, a:b, :] = got[p]


def gather_full(comm, u, plan: StripePlan, spans):
    """All ranks end with the full finest image."""
    return comm.allgather_rows(u, plan.own_lo, plan.own_hi, spans)
