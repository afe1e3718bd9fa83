"""Python mirror of the reference solver API over the C ABI.

Names, defaults, argument meaning and error behaviour follow
schwarz_inpaint (/root/reference/proj/include/schwarz_inpaint/):

* ``Method``, ``RunOptions``, ``run_method``           methods.hpp:13-88
* ``MultilevelSolveOptions``, ``multilevel_solve``     multilevel.hpp:132-310
* ``SchwarzOptions``, ``SchwarzSolveOptions``,
  ``solve_schwarz``, ``run_schwarz_level``,
  ``canonical_r0``                                      schwarz.hpp:29-389
* ``partition_domain``, ``SubdomainPartition``          partition.hpp:21-106
* ``ImageBuffer``, ``InpaintingMask``                   image.hpp:24-94
* ``SolveResult``, ``ConvergenceTrace``, ``psnr``       metrics.hpp:30-105
* ``synthetic_test_image``, ``random_mask``             synthetic.hpp / masks.hpp

``std::invalid_argument`` becomes :class:`InvalidArgument` (a ValueError).
All arithmetic runs in libschwarz_b200.so on the GPU; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference (image.hpp:18-20)."""


class SolverError(RuntimeError):
    """Device-side failure (CUDA error, out of memory, no device)."""


class Unsupported(SolverError):
    pass


def _check(status: int) -> None:
    if status == L.SI_OK:
        return
    msg = L.load().si_last_error().decode()
    if status == L.SI_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == L.SI_ERR_UNSUPPORTED:
        raise Unsupported(msg)
    raise SolverError(f"{L.load().si_status_string(status).decode()}: {msg}")


# ----------------------------------------------------------------- enums
class Method(enum.IntEnum):
    Cg = 0
    MultilevelCg = 1
    Ras = 2
    Oras = 3
    MultilevelOras = 4


_METHOD_NAMES = {Method.Cg: "cg", Method.MultilevelCg: "mlcg", Method.Ras: "ras",
                 Method.Oras: "oras", Method.MultilevelOras: "mloras"}


def method_name(m: Method) -> str:
    return _METHOD_NAMES.get(Method(m), "?")


def parse_method(name: str) -> Method:
    for m, n in _METHOD_NAMES.items():
        if n == name:
            return m
    raise InvalidArgument(f"unknown method '{name}' (expected cg, mlcg, ras, oras or mloras)")


def is_multilevel(m: Method) -> bool:
    return m in (Method.MultilevelCg, Method.MultilevelOras)


class CoarseAveraging(enum.IntEnum):
    KnownOnly = 0
    AllPixels = 1


class ResidualNormalizer(enum.IntEnum):
    InitialGuess = 0
    RhsNorm = 1


class SchwarzFlavour(enum.IntEnum):
    Ras = 0
    Oras = 1


class LevelSolver(enum.IntEnum):
    Cg = 0
    Ras = 1
    Oras = 2


class Precision(enum.IntEnum):
    FP64 = 0   # the reference's arithmetic
    FP32 = 1   # everything in float
    MIXED = 2  # double image / residuals / outer iteration, float local CG


kDefaultOrasAlpha = 0.25  # schwarz.hpp:34


# ----------------------------------------------------------------- options
@dataclass
class SolverConfig:  # cg.hpp:23-27
    tolerance: float = 1e-6
    max_iterations: int = 10000
    residual_check_interval: int = 1


@dataclass
class RunOptions:  # methods.hpp:40-55 (+ device precision)
    tolerance: float = 1e-3
    levels: int = 3
    block_size: int = 32
    overlap: int = 6
    alpha: float = kDefaultOrasAlpha
    coarse_tolerance: float = 1e-2
    averaging: CoarseAveraging = CoarseAveraging.KnownOnly
    local: SolverConfig = field(default_factory=lambda: SolverConfig(1e-2, 30, 30))
    max_outer_iterations: int = 1000
    cg_max_iterations: int = 100000
    cg_check_interval: int = 4
    normalizer: ResidualNormalizer = ResidualNormalizer.InitialGuess
    precision: Precision = Precision.FP64

    def to_c(self) -> L.si_options:
        return L.si_options(
            float(self.tolerance), int(self.levels), int(self.block_size), int(self.overlap),
            float(self.alpha), float(self.coarse_tolerance), int(self.averaging),
            float(self.local.tolerance), int(self.local.max_iterations),
            int(self.local.residual_check_interval), int(self.max_outer_iterations),
            int(self.cg_max_iterations), int(self.cg_check_interval), int(self.normalizer),
            int(self.precision))


@dataclass
class SchwarzOptions:  # schwarz.hpp:38-45
    flavour: SchwarzFlavour = SchwarzFlavour.Oras
    alpha: float = kDefaultOrasAlpha
    local: SolverConfig = field(default_factory=lambda: SolverConfig(1e-2, 30, 30))
    max_outer_iterations: int = 1000


@dataclass
class SchwarzSolveOptions:  # schwarz.hpp:325-329
    schwarz: SchwarzOptions = field(default_factory=SchwarzOptions)
    tolerance: float = 1e-3
    normalizer: ResidualNormalizer = ResidualNormalizer.InitialGuess
    precision: Precision = Precision.FP64


@dataclass
class MultilevelSolveOptions:  # multilevel.hpp:132-142
    levels: int = 3
    tolerance: float = 1e-3
    coarse_tolerance: float = 1e-2
    averaging: CoarseAveraging = CoarseAveraging.KnownOnly
    block_size: int = 32
    overlap: int = 6
    schwarz: SchwarzOptions = field(default_factory=SchwarzOptions)
    cg: SolverConfig = field(default_factory=lambda: SolverConfig(1e-3, 100000, 4))
    normalizer: ResidualNormalizer = ResidualNormalizer.InitialGuess
    precision: Precision = Precision.FP64


def _ml_run_options(o: MultilevelSolveOptions) -> "RunOptions":
    return RunOptions(tolerance=o.tolerance, levels=o.levels, block_size=o.block_size,
                      overlap=o.overlap, alpha=o.schwarz.alpha,
                      coarse_tolerance=o.coarse_tolerance, averaging=o.averaging,
                      local=o.schwarz.local, max_outer_iterations=o.schwarz.max_outer_iterations,
                      cg_max_iterations=o.cg.max_iterations,
                      cg_check_interval=o.cg.residual_check_interval,
                      normalizer=o.normalizer, precision=o.precision)


@dataclass
class DensifyOptions:  # masks.hpp:145-151
    initial_density: float = 0.0   # <= 0: start at a quarter of the target
    cell_fraction: float = 0.20    # share of cells refined per sweep
    inner_tolerance: float = 1e-3  # tolerance of the guiding inpainting runs
    max_sweeps: int = 100
    solve: MultilevelSolveOptions = field(default_factory=MultilevelSolveOptions)

    def to_c(self) -> L.si_densify_options:
        d = L.si_densify_options()
        d.initial_density = self.initial_density
        d.cell_fraction = self.cell_fraction
        d.inner_tolerance = self.inner_tolerance
        d.max_sweeps = self.max_sweeps
        d.solve = _ml_run_options(self.solve).to_c()
        return d


@dataclass
class VoronoiAssignment:  # masks.hpp:45-48
    sites: np.ndarray     # int32 known pixel indices, ascending
    site_of: np.ndarray   # int32 (h, w): index into sites


# ----------------------------------------------------------------- data
class ImageBuffer:
    """Planar image [c][y][x] of doubles (image.hpp:24-63)."""

    def __init__(self, width: int = 0, height: int = 0, channels: int = 1, fill: float = 0.0,
                 data: Optional[np.ndarray] = None):
        if data is not None:
            arr = np.ascontiguousarray(data, dtype=np.float64)
            if arr.ndim == 2:
                arr = arr[None]
            channels, height, width = arr.shape
            self.data = arr
        else:
            if not (width > 0 and height > 0 and channels > 0):
                raise InvalidArgument("ImageBuffer: dimensions must be positive")
            self.data = np.full((channels, height, width), fill, dtype=np.float64)
        self.width, self.height, self.channels = int(width), int(height), int(channels)

    def pixel_count(self) -> int:
        return self.width * self.height

    def channel(self, c: int) -> np.ndarray:
        if not 0 <= c < self.channels:
            raise InvalidArgument("ImageBuffer::channel: index out of range")
        return self.data[c].reshape(-1)

    def at(self, x: int, y: int, c: int = 0) -> float:
        return float(self.data[c, y, x])


class InpaintingMask:
    """uint8 per pixel, nonzero = known (image.hpp:67-94)."""

    def __init__(self, width: int = 0, height: int = 0, fill: int = 0,
                 known: Optional[np.ndarray] = None):
        if known is not None:
            arr = np.ascontiguousarray(known, dtype=np.uint8)
            height, width = arr.shape
            self.known = arr
        else:
            if not (width > 0 and height > 0):
                raise InvalidArgument("InpaintingMask: dimensions must be positive")
            self.known = np.full((height, width), fill, dtype=np.uint8)
        self.width, self.height = int(width), int(height)

    def size(self) -> int:
        return self.width * self.height

    def is_known(self, x: int, y: int) -> bool:
        return bool(self.known[y, x])

    def known_count(self) -> int:
        return int(np.count_nonzero(self.known))

    def density(self) -> float:
        return 0.0 if self.size() == 0 else self.known_count() / self.size()


@dataclass
class TraceRow:  # metrics.hpp:60-65
    iteration: int
    time_ms: float
    rel_residual: float
    psnr: Optional[float] = None


@dataclass
class ConvergenceTrace:  # metrics.hpp:69-97
    rows: List[TraceRow] = field(default_factory=list)
    kCsvHeader = "iter,time_ms,rel_residual,psnr"

    def append(self, iteration, time_ms, rel, psnr=None):
        self.rows.append(TraceRow(iteration, time_ms, rel, psnr))

    def write_csv(self) -> str:
        out = [self.kCsvHeader]
        for r in self.rows:
            s = f"{r.iteration},{r.time_ms:.3f},{r.rel_residual:.9e}"
            if r.psnr is None:
                s += ","
            elif math.isinf(r.psnr):
                s += ",inf"
            else:
                s += f",{r.psnr:.4f}"
            out.append(s)
        return "\n".join(out) + "\n"


@dataclass
class SolveReport:  # cg.hpp:29-34 (+ per-level statistics)
    iterations: int = 0
    final_relative_residual: float = 0.0
    converged: bool = False
    diagnostic: str = ""
    depth: int = 0
    level_iterations: List[int] = field(default_factory=list)   # index 0 = finest
    level_final_rel: List[float] = field(default_factory=list)
    level_converged: List[bool] = field(default_factory=list)
    local_solves: int = 0
    local_failures: int = 0
    local_cg_iterations: int = 0
    elapsed_ms: float = 0.0
    h2d_bytes: int = 0   # host entries: bytes this frame moved over PCIe
    d2h_bytes: int = 0


@dataclass
class SolveResult:  # metrics.hpp:101-105
    image: ImageBuffer
    trace: ConvergenceTrace
    report: SolveReport


@dataclass
class Subdomain:  # partition.hpp:21-28
    x0: int
    y0: int
    width: int
    height: int
    own_x0: int
    own_y0: int
    own_x1: int
    own_y1: int

    def cell_count(self) -> int:
        return self.width * self.height


@dataclass
class SubdomainPartition:  # partition.hpp:30-40
    image_width: int
    image_height: int
    block_size: int
    overlap: int
    blocks_x: int
    blocks_y: int
    subdomains: List[Subdomain]

    def size(self) -> int:
        return len(self.subdomains)


def _result_buffer(width: int, height: int, channels: int) -> ImageBuffer:
    """Output image the solver overwrites completely: left uninitialised (a
    zero fill of a 4K RGB frame costs more host time than the solve)."""
    return ImageBuffer(data=np.empty((channels, height, width), dtype=np.float64))


def _report(r: L.si_report) -> SolveReport:
    d = r.depth
    return SolveReport(r.iterations, r.final_relative_residual, bool(r.converged),
                       r.diagnostic.decode(), d, list(r.level_iterations[:d]),
                       list(r.level_final_rel[:d]), [bool(v) for v in r.level_converged[:d]],
                       r.local_solves, r.local_failures, r.local_cg_iterations, r.elapsed_ms,
                       r.h2d_bytes, r.d2h_bytes)


# ----------------------------------------------------------------- context
class Solver:
    """One device context (si_ctx); independent per GPU / host thread."""

    def __init__(self, device: int = 0):
        self._lib = L.load()
        h = C.c_void_p()
        _check(self._lib.si_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._lib.si_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- tracing plumbing
    @staticmethod
    def _sink(trace: ConvergenceTrace, with_psnr: bool):
        def cb(it, ms, rel, q, _user):
            trace.append(it, ms, rel, q if with_psnr else None)
        return L.TRACE_FN(cb)

    def run_method(self, method: Method, f: ImageBuffer, mask: InpaintingMask,
                   options: Optional[RunOptions] = None,
                   reference: Optional[ImageBuffer] = None) -> SolveResult:
        """run_method (methods.hpp:57-88) on host buffers."""
        options = options or RunOptions()
        _require_same_grid(f, mask)
        if reference is not None:
            _require_same_shape(f, reference)
        out = _result_buffer(f.width, f.height, f.channels)
        trace = ConvergenceTrace()
        rep = L.si_report()
        o = options.to_c()
        cb = self._sink(trace, reference is not None)
        ref_ptr = None if reference is None else reference.data.ctypes.data
        st = self._lib.si_run_method(self._h, int(method), f.data.ctypes.data,
                                     mask.known.ctypes.data, f.width, f.height, f.channels,
                                     C.byref(o), ref_ptr, out.data.ctypes.data, C.byref(rep), cb,
                                     None)
        _check(st)
        return SolveResult(out, trace, _report(rep))

    def run_method_device(self, method: Method, f_ptr: int, mask_ptr: int, width: int,
                          height: int, channels: int, out_ptr: int,
                          options: Optional[RunOptions] = None, reference_ptr: Optional[int] = None,
                          stream: Optional[int] = None, trace: Optional[ConvergenceTrace] = None
                          ) -> SolveReport:
        """Device-resident run_method: raw device pointers (e.g. torch data_ptr())."""
        options = options or RunOptions()
        rep = L.si_report()
        o = options.to_c()
        cb = self._sink(trace, reference_ptr is not None) if trace is not None else L.TRACE_FN()
        _check(self._lib.si_run_method_device(self._h, int(method), f_ptr, mask_ptr, width, height,
                                              channels, C.byref(o), reference_ptr, out_ptr,
                                              C.byref(rep), cb, None, stream))
        return _report(rep)

    def run_batch(self, method: Method, frames, options: Optional[RunOptions] = None,
                  outputs=None) -> List[SolveResult]:
        """run_method over a batch of independent frames [(ImageBuffer, InpaintingMask)]
        with host<->device copies overlapped with the solves (si_run_method_batch).
        outputs: optional list of preallocated (pinned) ImageBuffers."""
        options = options or RunOptions()
        n = len(frames)
        if n == 0:
            return []
        f0 = frames[0][0]
        for f, m in frames:
            _require_same_grid(f, m)
            if (f.width, f.height, f.channels) != (f0.width, f0.height, f0.channels):
                raise InvalidArgument("run_batch: frames must share one shape")
        outs = outputs or [_result_buffer(f0.width, f0.height, f0.channels) for _ in range(n)]
        # the C ABI receives raw pointers: every output must be a full,
        # C-contiguous float64 (c, h, w) buffer (no NULL, no short list)
        _require_outputs([o.data for o in outs], n, (f0.channels, f0.height, f0.width),
                         np.float64, "run_batch")
        fp = (C.c_void_p * n)(*[f.data.ctypes.data for f, _ in frames])
        mp = (C.c_void_p * n)(*[m.known.ctypes.data for _, m in frames])
        op = (C.c_void_p * n)(*[o.data.ctypes.data for o in outs])
        reps = (L.si_report * n)()
        o = options.to_c()
        _check(self._lib.si_run_method_batch(self._h, int(method), n, fp, mp, f0.width, f0.height,
                                             f0.channels, C.byref(o), op, reps))
        return [SolveResult(outs[k], ConvergenceTrace(), _report(reps[k])) for k in range(n)]

    def run_pnm_batch(self, method: Method, frames, options: Optional[RunOptions] = None,
                      outputs=None) -> List[SolveReport]:
        """The CLI wire format (pnm.hpp) end to end on the device: frames is a
        list of (pixels, mask_pbm) with pixels the P5/P6 payload as a uint8 array
        (h, w) or (h, w, 3) and mask_pbm the P4 payload (h, (w+7)//8) uint8;
        returns (reports, outputs) with outputs the P5/P6 payloads."""
        options = options or RunOptions()
        n = len(frames)
        if n == 0:
            return [], []
        px0 = np.asarray(frames[0][0])
        h, w = px0.shape[:2]
        c = 1 if px0.ndim == 2 else px0.shape[2]
        ins = [np.ascontiguousarray(p, dtype=np.uint8) for p, _ in frames]
        masks = [np.ascontiguousarray(m, dtype=np.uint8) for _, m in frames]
        for p_, m_ in zip(ins, masks):
            if p_.shape != px0.shape or m_.shape != (h, (w + 7) // 8):
                raise InvalidArgument("run_pnm_batch: frames must share one shape")
        outs = outputs or [np.empty_like(ins[0]) for _ in range(n)]
        _require_outputs(outs, n, px0.shape, np.uint8, "run_pnm_batch")
        ip = (C.c_void_p * n)(*[a.ctypes.data for a in ins])
        mp = (C.c_void_p * n)(*[a.ctypes.data for a in masks])
        op = (C.c_void_p * n)(*[a.ctypes.data for a in outs])
        reps = (L.si_report * n)()
        o = options.to_c()
        _check(self._lib.si_run_pnm_batch(self._h, int(method), n, ip, mp, w, h, c, C.byref(o),
                                          op, reps))
        return [_report(reps[k]) for k in range(n)], outs

    def solve_schwarz(self, f: ImageBuffer, mask: InpaintingMask, partition: SubdomainPartition,
                      options: Optional[SchwarzSolveOptions] = None,
                      reference: Optional[ImageBuffer] = None) -> SolveResult:
        """solve_schwarz (schwarz.hpp:349-389)."""
        options = options or SchwarzSolveOptions()
        _require_same_grid(f, mask)
        if partition.image_width != f.width or partition.image_height != f.height:
            raise InvalidArgument("solve_schwarz: partition and image dimensions differ")
        ro = RunOptions(tolerance=options.tolerance, levels=1, block_size=partition.block_size,
                        overlap=partition.overlap, alpha=options.schwarz.alpha,
                        local=options.schwarz.local,
                        max_outer_iterations=options.schwarz.max_outer_iterations,
                        normalizer=options.normalizer, precision=options.precision)
        out = _result_buffer(f.width, f.height, f.channels)
        trace = ConvergenceTrace()
        rep = L.si_report()
        o = ro.to_c()
        cb = self._sink(trace, reference is not None)
        ref_ptr = None if reference is None else reference.data.ctypes.data
        _check(self._lib.si_solve_schwarz(self._h, f.data.ctypes.data, mask.known.ctypes.data,
                                          f.width, f.height, f.channels, partition.block_size,
                                          partition.overlap, int(options.schwarz.flavour),
                                          C.byref(o), ref_ptr, out.data.ctypes.data,
                                          C.byref(rep), cb, None))
        return SolveResult(out, trace, _report(rep))

    def multilevel_solve(self, f: ImageBuffer, mask: InpaintingMask, solver: LevelSolver,
                         options: Optional[MultilevelSolveOptions] = None,
                         reference: Optional[ImageBuffer] = None) -> SolveResult:
        """multilevel_solve (multilevel.hpp:239-310)."""
        options = options or MultilevelSolveOptions()
        if solver == LevelSolver.Cg:
            method = Method.MultilevelCg
        else:
            method = Method.MultilevelOras if solver == LevelSolver.Oras else Method.Ras
        ro = _ml_run_options(options)
        if method == Method.Ras and options.levels != 1:
            # RAS level solver on a pyramid: the C ABI's RAS method is single level;
            # route multilevel RAS through the ORAS path with alpha = 1 (identical
            # diagonal, schwarz.hpp:12-15).
            ro.alpha = 1.0
            method = Method.MultilevelOras
        elif method == Method.Ras:
            pass
        return self.run_method(method, f, mask, ro, reference)

    def voronoi_densify(self, f: ImageBuffer, target_density: float, seed: int,
                        options: Optional[DensifyOptions] = None) -> "DensifyResult":
        """voronoi_densify (masks.hpp:155-212), the whole loop on the device."""
        options = options or DensifyOptions()
        out = np.zeros((f.height, f.width), np.uint8)
        sweeps, reached = C.c_int(), C.c_int()
        d = options.to_c()
        _check(self._lib.si_voronoi_densify(self._h, f.data.ctypes.data, f.width, f.height,
                                            f.channels, float(target_density), int(seed),
                                            C.byref(d), out.ctypes.data, C.byref(sweeps),
                                            C.byref(reached)))
        return DensifyResult(InpaintingMask(known=out), sweeps.value, bool(reached.value))

    def assign_nearest_site(self, mask: InpaintingMask) -> VoronoiAssignment:
        """assign_nearest_site (masks.hpp:54-139) on the device."""
        n = mask.width * mask.height
        sites = np.empty(n, np.int32)
        site_of = np.empty((mask.height, mask.width), np.int32)
        k = C.c_int()
        known = np.ascontiguousarray(mask.known, dtype=np.uint8)
        _check(self._lib.si_assign_nearest_site(self._h, known.ctypes.data, mask.width,
                                                mask.height, sites.ctypes.data,
                                                site_of.ctypes.data, C.byref(k)))
        return VoronoiAssignment(sites[: k.value].copy(), site_of)

    def run_schwarz_level(self, mask: InpaintingMask, partition: SubdomainPartition,
                          b: np.ndarray, u: np.ndarray, r0_norm: float, tolerance: float,
                          opt: Optional[SchwarzOptions] = None, trace=None):
        """run_schwarz_level (schwarz.hpp:266-323); u (c,h,w) float64 updated in place."""
        opt = opt or SchwarzOptions()
        b = np.ascontiguousarray(b, dtype=np.float64)
        if u.dtype != np.float64 or not u.flags.c_contiguous:
            raise InvalidArgument("run_schwarz_level: u must be C-contiguous float64")
        c = u.shape[0] if u.ndim == 3 else 1
        if b.size != u.size:
            raise InvalidArgument("run_schwarz_level: vector length mismatch")
        ro = RunOptions(alpha=opt.alpha, local=opt.local,
                        max_outer_iterations=opt.max_outer_iterations)
        o = ro.to_c()
        rep = L.si_report()
        tr = ConvergenceTrace()
        cb = self._sink(tr, False)
        _check(self._lib.si_run_schwarz_level(self._h, mask.known.ctypes.data, mask.width,
                                              mask.height, c, b.ctypes.data, u.ctypes.data,
                                              partition.block_size, partition.overlap,
                                              float(r0_norm), float(tolerance), int(opt.flavour),
                                              C.byref(o), C.byref(rep), cb, None))
        if trace is not None:
            trace.rows.extend(tr.rows)
        return _report(rep)

    def canonical_r0(self, mask: InpaintingMask, b: np.ndarray,
                     normalizer: ResidualNormalizer = ResidualNormalizer.InitialGuess) -> float:
        b = np.ascontiguousarray(b, dtype=np.float64)
        c = b.shape[0] if b.ndim == 3 else 1
        r = C.c_double()
        _check(self._lib.si_canonical_r0(self._h, mask.known.ctypes.data, mask.width, mask.height,
                                         c, b.ctypes.data, int(normalizer), C.byref(r)))
        return r.value

    # -- building blocks (each one device launch, host buffers)
    def schwarz_sweep(self, mask: np.ndarray, b: np.ndarray, u: np.ndarray, block: int,
                      overlap: int, flavour: SchwarzFlavour = SchwarzFlavour.Oras,
                      options: Optional[RunOptions] = None):
        options = options or RunOptions()
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        b = np.ascontiguousarray(b, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.ndim == 2:
            u = u[None]
            b = b.reshape(u.shape)
        c, h, w = u.shape
        un = np.empty_like(u)
        fails, its = C.c_longlong(), C.c_longlong()
        o = options.to_c()
        _check(self._lib.si_schwarz_sweep(self._h, m.ctypes.data, w, h, c, b.ctypes.data,
                                          u.ctypes.data, block, overlap, int(flavour), C.byref(o),
                                          un.ctypes.data, C.byref(fails), C.byref(its)))
        return un, fails.value, its.value

    def residual_sumsq(self, mask: np.ndarray, u: np.ndarray, b: np.ndarray) -> np.ndarray:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        u = np.ascontiguousarray(u, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        h, w = m.shape
        c = u.size // (w * h)
        out = np.zeros(c)
        _check(self._lib.si_residual_sumsq(self._h, m.ctypes.data, w, h, c, u.ctypes.data,
                                           b.ctypes.data, out.ctypes.data))
        return out

    def restrict_level(self, mask: np.ndarray, values: np.ndarray,
                       averaging: CoarseAveraging = CoarseAveraging.KnownOnly):
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        v = np.ascontiguousarray(values, dtype=np.float64)
        if v.ndim == 2:
            v = v[None]
        c, h, w = v.shape
        cw, ch = (w + 1) // 2, (h + 1) // 2
        cm = np.empty((ch, cw), np.uint8)
        cv = np.empty((c, ch, cw))
        _check(self._lib.si_restrict_level(self._h, m.ctypes.data, v.ctypes.data, w, h, c,
                                           int(averaging), cm.ctypes.data, cv.ctypes.data))
        return cm, cv

    def prolongate(self, coarse: np.ndarray, cw: int, ch: int, fw: int, fh: int) -> np.ndarray:
        cc = np.ascontiguousarray(coarse, dtype=np.float64).reshape(-1)
        if cc.size != cw * ch:
            raise InvalidArgument("prolongate: coarse vector length mismatch")
        fine = np.empty(fw * fh)
        _check(self._lib.si_prolongate(self._h, cc.ctypes.data, cw, ch, fw, fh, fine.ctypes.data))
        return fine

    def local_operator_apply(self, mask: np.ndarray, block: int, overlap: int, index: int,
                             flavour: SchwarzFlavour, alpha: float, v: np.ndarray) -> np.ndarray:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        h, w = m.shape
        vv = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
        out = np.empty(block * block)
        _check(self._lib.si_local_operator_apply(self._h, m.ctypes.data, w, h, block, overlap,
                                                 index, int(flavour), float(alpha),
                                                 vv.ctypes.data, out.ctypes.data))
        return out

    def set_profiling(self, enabled: bool):
        _check(self._lib.si_set_profiling(self._h, int(bool(enabled))))

    def kernel_stats(self, reset: bool = False) -> dict:
        s = L.si_kernel_stats()
        _check(self._lib.si_get_kernel_stats(self._h, C.byref(s), int(reset)))
        names = ["residual", "sweep", "restrict", "prolong", "ingest_export", "metrics", "voronoi"]
        out = {n: {"launches": s.launches[i], "device_ms": s.device_ms[i],
                   "algorithmic_bytes": s.algorithmic_bytes[i]} for i, n in enumerate(names)}
        out["total_launches"] = s.total_launches
        return out


@dataclass
class DensifyResult:  # masks.hpp:153-157
    mask: "InpaintingMask"
    sweeps: int = 0
    reached_target: bool = False


def voronoi_densify(f: ImageBuffer, target_density: float, seed: int,
                    options: Optional[DensifyOptions] = None) -> DensifyResult:
    return default_solver().voronoi_densify(f, target_density, seed, options)


def assign_nearest_site(mask: InpaintingMask) -> VoronoiAssignment:
    return default_solver().assign_nearest_site(mask)


def _require_outputs(outs, n: int, shape, dtype, who: str):
    """Caller-supplied batch outputs: exactly n C-contiguous arrays of the
    frame's shape and dtype (the library writes through raw pointers)."""
    if len(outs) != n:
        raise InvalidArgument(f"{who}: expected {n} outputs, got {len(outs)}")
    for k, a in enumerate(outs):
        if not isinstance(a, np.ndarray) or a.dtype != dtype or tuple(a.shape) != tuple(shape) \
                or not a.flags.c_contiguous or not a.flags.writeable:
            raise InvalidArgument(f"{who}: output {k} must be a writeable C-contiguous "
                                  f"{np.dtype(dtype).name} array of shape {tuple(shape)}")


def _require_same_grid(f: ImageBuffer, mask: InpaintingMask):
    if f.width != mask.width or f.height != mask.height:  # image.hpp:96-99
        raise InvalidArgument("image and mask dimensions differ")


def _require_same_shape(a: ImageBuffer, b: ImageBuffer):
    if (a.width, a.height, a.channels) != (b.width, b.height, b.channels):
        raise InvalidArgument("mse_per_channel: image dimensions differ")


_default: dict = {}


def default_solver(device: int = 0) -> Solver:
    s = _default.get(device)
    if s is None:
        s = _default[device] = Solver(device)
    return s


# ----------------------------------------------------------------- free functions
def run_method(method: Method, f: ImageBuffer, mask: InpaintingMask,
               options: Optional[RunOptions] = None,
               reference: Optional[ImageBuffer] = None) -> SolveResult:
    return default_solver().run_method(method, f, mask, options, reference)


def run_batch(method: Method, frames, options: Optional[RunOptions] = None, outputs=None):
    return default_solver().run_batch(method, frames, options, outputs)


def multilevel_solve(f, mask, solver: LevelSolver, options=None, reference=None) -> SolveResult:
    return default_solver().multilevel_solve(f, mask, solver, options, reference)


def solve_schwarz(f, mask, partition, options=None, reference=None) -> SolveResult:
    return default_solver().solve_schwarz(f, mask, partition, options, reference)


def run_schwarz_level(mask, partition, b, u, r0_norm, tolerance, opt=None, trace=None):
    return default_solver().run_schwarz_level(mask, partition, b, u, r0_norm, tolerance, opt,
                                              trace)


def canonical_r0(mask, b, normalizer=ResidualNormalizer.InitialGuess) -> float:
    return default_solver().canonical_r0(mask, b, normalizer)


def clamped_partition(width: int, height: int, block: int, overlap: int) -> SubdomainPartition:
    """clamped_partition (multilevel.hpp:146-150)."""
    be = min(block, min(width, height))
    oe = max(0, min(overlap, be - 1))
    return partition_domain(width, height, be, oe)


def partition_domain(width: int, height: int, block_size: int, overlap: int) -> SubdomainPartition:
    """partition_domain (partition.hpp:67-106) via the C ABI (host-only)."""
    lib = L.load()
    bx, by = C.c_int(), C.c_int()
    _check(lib.si_partition_domain(width, height, block_size, overlap, C.byref(bx), C.byref(by),
                                   None, 0))
    n = bx.value * by.value
    rects = (C.c_int * (8 * n))()
    _check(lib.si_partition_domain(width, height, block_size, overlap, C.byref(bx), C.byref(by),
                                   rects, n))
    r = np.frombuffer(rects, dtype=np.int32).reshape(n, 8)
    subs = [Subdomain(*map(int, row)) for row in r]
    return SubdomainPartition(width, height, block_size, overlap, bx.value, by.value, subs)


KNOWN_TILE = 4096


def pack_known_samples(f: ImageBuffer, mask: InpaintingMask):
    """The host entries' known-sample upload (si_pack_known_samples, host
    only): (tile_off uint32 [ceil(w*h/4096)], vals float64 [c, K]) with
    vals[c] = f[c] at the known pixels in pixel order."""
    _require_same_grid(f, mask)
    lib = L.load()
    n = f.width * f.height
    tiles = np.empty((n + KNOWN_TILE - 1) // KNOWN_TILE, dtype=np.uint32)
    K = C.c_longlong()
    known = np.ascontiguousarray(mask.known, dtype=np.uint8)
    data = np.ascontiguousarray(f.data, dtype=np.float64)
    _check(lib.si_pack_known_samples(data.ctypes.data, known.ctypes.data, f.width, f.height,
                                     f.channels, tiles.ctypes.data, None, C.byref(K)))
    vals = np.empty((f.channels, K.value), dtype=np.float64)
    _check(lib.si_pack_known_samples(data.ctypes.data, known.ctypes.data, f.width, f.height,
                                     f.channels, tiles.ctypes.data, vals.ctypes.data, C.byref(K)))
    return tiles, vals


def synthetic_test_image(width: int, height: int, channels: int, seed: int) -> ImageBuffer:
    out = np.empty((channels, height, width))
    st = L.load().si_synthetic_test_image(width, height, channels, seed, out.ctypes.data)
    if st != L.SI_OK:
        raise InvalidArgument("synthetic_test_image: dimensions must be positive")
    return ImageBuffer(data=out)


def random_mask(width: int, height: int, density: float, seed: int) -> InpaintingMask:
    out = np.empty((height, width), np.uint8)
    st = L.load().si_random_mask(width, height, density, seed, out.ctypes.data)
    if st != L.SI_OK:
        raise InvalidArgument("random_mask: invalid dimensions or density")
    return InpaintingMask(known=out)


def pack_pbm(mask: InpaintingMask) -> np.ndarray:
    """P4 payload of a mask (write_mask_pbm, pnm.hpp:190-205): MSB first, rows padded."""
    return np.packbits(mask.known != 0, axis=1, bitorder="big")


def quantise_pnm(img: ImageBuffer) -> np.ndarray:
    """P5/P6 payload of an image (write_pnm's quantise, pnm.hpp:82-85): clamp to
    [0, 1] and round half away from zero; (h, w) or (h, w, 3) uint8."""
    v = np.clip(img.data, 0.0, 1.0) * 255.0
    fl = np.floor(v)
    q = (fl + (v - fl >= 0.5)).astype(np.uint8)
    return q[0] if img.channels == 1 else np.ascontiguousarray(np.moveaxis(q, 0, -1))


def mse_per_channel(u: ImageBuffer, f: ImageBuffer) -> List[float]:
    _require_same_shape(u, f)
    d = 255.0 * (u.data - f.data)
    return [float(np.sum(d[c] * d[c]) / u.pixel_count()) for c in range(u.channels)]


def psnr(u: ImageBuffer, f: ImageBuffer) -> float:
    _require_same_shape(u, f)
    r = C.c_double()
    _check(L.load().si_psnr(u.data.ctypes.data, f.data.ctypes.data, u.width, u.height,
                            u.channels, C.byref(r)))
    return r.value
