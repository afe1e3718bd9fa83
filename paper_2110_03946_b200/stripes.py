"""One very large image over G GPUs: horizontal stripes with halo exchange
(BASELINE.json configs[4]) -- Python mirror of the C ABI.

The solve itself is C++ and CUDA (`csrc/stripes.cuh`, `si_run_method_striped*`):
every pyramid level is split into G stripes of whole block rows of that
level's own partition (partition_domain, partition.hpp:46-106); each rank
allocates, ingests, restricts, sweeps and prolongs only its rows (plus
halos).  Per outer iteration (run_schwarz_level, schwarz.hpp:288-320) the
G x C partial residual sums are all-gathered, every rank takes the same stop
decision on the device (fixed rank order), sweeps its block rows and
exchanges halo rows with the owners; repeated solves of one shape issue
their iterations without host round trips (speculation, resumed when a
level needs more).  The image equals the single-GPU solve bit for bit
whenever the stop decisions agree.

Communicators:
  * `nccl_comm(solver, dist)`: one process per GPU; rank 0 makes the NCCL
    id, torch.distributed broadcasts it, the library drives NCCL
    (ncclAllGather + grouped ncclSend/ncclRecv on the solve stream);
  * `local_comms(solvers)`: G ranks as host threads of this process (any
    devices, including G ranks on one GPU); device copies ordered by events;
    `run_method_striped_local_device` drives the whole group in one call.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L
from .api import (ConvergenceTrace, ImageBuffer, InpaintingMask, InvalidArgument, Method,
                  RunOptions, SolveResult, Solver, _check, _report, _require_same_grid)

PLAN_INTS = 12


@dataclass
class StripeLevel:
    """Rows of one level held by one rank (global row coordinates)."""
    k0: int
    k1: int            # block rows [k0, k1)
    own_lo: int
    own_hi: int        # rows the rank owns (owned rows of all ranks tile the level)
    win_lo: int
    win_hi: int        # rows its sweeps and residual stencil read
    need_lo: int
    need_hi: int       # rows of this level its prolongation onto the finer window reads
    store_lo: int
    store_hi: int      # rows it allocates / ingests / restricts
    block: int
    overlap: int       # clamped partition (multilevel.hpp:146-150)


def level_plan(method: Method, w: int, h: int, c: int, options: Optional[RunOptions],
               world: int, rank: int) -> List[StripeLevel]:
    """si_stripe_level_plan: the decomposition the C++ executor uses (index 0 =
    finest).  Host only."""
    o = (options or RunOptions()).to_c()
    depth = C.c_int()
    out = (C.c_int * (L.SI_MAX_LEVELS * PLAN_INTS))()
    _check(L.load().si_stripe_level_plan(int(method), w, h, c, C.byref(o), world, rank,
                                         C.byref(depth), out))
    return [StripeLevel(*out[l * PLAN_INTS:(l + 1) * PLAN_INTS]) for l in range(depth.value)]


class StripeComm:
    """Owns an si_stripe_comm handle."""

    def __init__(self, handle, world: int, rank: int, kind: str):
        self.handle = handle
        self.world = world
        self.rank = rank
        self.kind = kind

    def set_speculation(self, enabled: bool) -> None:
        """Issue each level's outer iterations without host round trips, as
        many as the last solve of the same shape and options took (default
        on; every rank of a group must agree)."""
        _check(L.load().si_stripe_comm_set_speculation(self.handle, 1 if enabled else 0))

    def counters(self) -> dict:
        """Solves run on this communicator, how many speculated, and how many
        levels had to be resumed."""
        out = (C.c_longlong * 3)()
        _check(L.load().si_stripe_comm_counters(self.handle, out))
        return {"solves": out[0], "speculative": out[1], "resumes": out[2]}

    def close(self):
        if self.handle:
            L.load().si_stripe_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_comm(solver: Solver, dist, device=None) -> StripeComm:
    """NCCL communicator over the ranks of torch.distributed `dist` (one
    process per GPU): rank 0's id is broadcast through `dist`."""
    import torch
    lib = L.load()
    world, rank = dist.get_world_size(), dist.get_rank()
    idbuf = (C.c_ubyte * L.SI_NCCL_ID_BYTES)()
    if rank == 0:
        _check(lib.si_nccl_unique_id(idbuf))
    dev = device if device is not None else (
        torch.device("cuda", solver.device) if dist.get_backend() == "nccl" else None)
    t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=0)
    idbuf = (C.c_ubyte * L.SI_NCCL_ID_BYTES)(*t.cpu().tolist())
    h = C.c_void_p()
    _check(lib.si_stripe_comm_init_nccl(solver.handle, world, rank, idbuf, C.byref(h)))
    return StripeComm(h, world, rank, "nccl")


def local_comms(solvers: Sequence[Solver]) -> List[StripeComm]:
    """G = len(solvers) ranks as threads of this process (rank r on solvers[r])."""
    world = len(solvers)
    ctxs = (C.c_void_p * world)(*[s.handle for s in solvers])
    hs = (C.c_void_p * world)()
    _check(L.load().si_stripe_comm_init_local(ctxs, world, hs))
    return [StripeComm(C.c_void_p(hs[r]), world, r, "local") for r in range(world)]


def run_method_striped(solver: Solver, comm: StripeComm, method: Method, f: ImageBuffer,
                       mask: InpaintingMask, options: Optional[RunOptions] = None,
                       out: Optional[ImageBuffer] = None, trace: Optional[ConvergenceTrace] = None
                       ) -> SolveResult:
    """Collective run_method over comm's ranks (every rank calls it with the
    full host image; only its rows are uploaded).  The returned image holds
    this rank's own finest rows (others untouched); the report carries the
    global counts."""
    options = options or RunOptions()
    _require_same_grid(f, mask)
    out = out or ImageBuffer(data=np.zeros_like(f.data))
    if out.data.shape != f.data.shape:
        raise InvalidArgument("run_method_striped: output shape differs from the image")
    rep = L.si_report()
    o = options.to_c()
    tr = trace if trace is not None else ConvergenceTrace()
    cb = Solver._sink(tr, False)
    _check(L.load().si_run_method_striped(solver.handle, comm.handle, int(method),
                                          f.data.ctypes.data, mask.known.ctypes.data, f.width,
                                          f.height, f.channels, C.byref(o), out.data.ctypes.data,
                                          C.byref(rep), cb, None))
    return SolveResult(out, tr, _report(rep))


def run_method_striped_device(solver: Solver, comm: StripeComm, method: Method, f_rows_ptr: int,
                              mask_rows_ptr: int, w: int, h: int, c: int,
                              out_rows_ptr: Optional[int], options: Optional[RunOptions] = None,
                              stream=None):
    """Device-resident: rows [store_lo, store_hi) of f / mask in, rows
    [own_lo, own_hi) of the result out (level_plan(...)[0]).  out_rows_ptr
    None (FP64 / MIXED): the rows stay in the solver's storage, see
    result_rows()."""
    options = options or RunOptions()
    rep = L.si_report()
    o = options.to_c()
    _check(L.load().si_run_method_striped_device(solver.handle, comm.handle, int(method),
                                                 f_rows_ptr, mask_rows_ptr, w, h, c, C.byref(o),
                                                 out_rows_ptr, C.byref(rep), stream))
    return _report(rep)


def run_method_striped_local_device(solvers: Sequence[Solver], comms: Sequence[StripeComm],
                                    method: Method, f_rows_ptrs, mask_rows_ptrs, w: int, h: int,
                                    c: int, out_rows_ptrs=None,
                                    options: Optional[RunOptions] = None, streams=None):
    """Every rank of a local group in one call (ranks 1.. on the group's
    persistent host threads): per-rank device rows as in
    run_method_striped_device; out_rows_ptrs None = rows in place.  Returns
    every rank's report."""
    options = options or RunOptions()
    G = len(solvers)
    if len(comms) != G:
        raise InvalidArgument("run_method_striped_local_device: one communicator per solver")
    vp = C.c_void_p * G
    rep = (L.si_report * G)()
    o = options.to_c()
    outs = None if out_rows_ptrs is None else vp(*out_rows_ptrs)
    sts = None if streams is None else vp(*streams)
    _check(L.load().si_run_method_striped_local_device(
        vp(*[cm.handle for cm in comms]), vp(*[s.handle for s in solvers]), G, int(method),
        vp(*f_rows_ptrs), vp(*mask_rows_ptrs), w, h, c, C.byref(o), outs, rep, sts))
    return [_report(rep[r]) for r in range(G)]


def result_rows(solver: Solver):
    """(device pointer, plane stride in doubles, rows) of this rank's finest
    own rows after a striped solve without an output buffer (valid until the
    solver's next call); pointer 0 when the rank owns no rows."""
    p = C.c_void_p()
    stride = C.c_size_t()
    rows = C.c_int()
    _check(L.load().si_stripe_result_rows(solver.handle, C.byref(p), C.byref(stride),
                                          C.byref(rows)))
    return (p.value or 0), stride.value, rows.value


def result_rows_tensor(solver: Solver, c: int, w: int):
    """result_rows() as a torch view [c, rows, w] (float64, no copy)."""
    import torch
    ptr, stride, rows = result_rows(solver)
    if not ptr:
        return torch.empty((c, 0, w), dtype=torch.float64, device=f"cuda:{solver.device}")

    class _Rows:
        __cuda_array_interface__ = {"shape": (c, rows, w), "typestr": "<f8", "data": (ptr, False),
                                    "version": 2, "strides": (8 * stride, 8 * w, 8)}
    return torch.as_tensor(_Rows(), device=f"cuda:{solver.device}")


def run_method_striped_group(solvers: Sequence[Solver], method: Method, f: ImageBuffer,
                             mask: InpaintingMask, options: Optional[RunOptions] = None):
    """G = len(solvers) ranks as threads of this process: the whole image and
    every rank's report."""
    options = options or RunOptions()
    _require_same_grid(f, mask)
    world = len(solvers)
    out = ImageBuffer(data=np.zeros_like(f.data))
    ctxs = (C.c_void_p * world)(*[s.handle for s in solvers])
    reps = (L.si_report * world)()
    o = options.to_c()
    _check(L.load().si_run_method_striped_group(ctxs, world, int(method), f.data.ctypes.data,
                                                mask.known.ctypes.data, f.width, f.height,
                                                f.channels, C.byref(o), out.data.ctypes.data,
                                                reps))
    return out, [_report(reps[r]) for r in range(world)]
