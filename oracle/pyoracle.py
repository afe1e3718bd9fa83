"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the CPU parity oracle.

Two CPU implementations of the reference's multilevel ORAS path live here:

* ``liboracle.so`` — ``si_oracle.c``, a plain-C restatement (the "port").
* ``_ref/libref.so`` — the UNMODIFIED reference headers
  (/root/reference/proj/include) driven by ``ref_driver.cpp``; present only
  where it was built (this container, or a GPU box that received the built
  file inside the gpurun snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2110_03946_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")
REF_SPR_SO = os.path.join(HERE, "_ref", "libref_spr.so")   # -march=sapphirerapids
_ref_path = REF_SO

MAX_LEVELS = 32


class Options(C.Structure):
    """Field-for-field RunOptions (methods.hpp:40-55) + flavour."""

    _fields_ = [
        ("tolerance", C.c_double),
        ("levels", C.c_int),
        ("block_size", C.c_int),
        ("overlap", C.c_int),
        ("alpha", C.c_double),
        ("coarse_tolerance", C.c_double),
        ("averaging", C.c_int),
        ("local_tolerance", C.c_double),
        ("local_max_iterations", C.c_int),
        ("local_check_interval", C.c_int),
        ("max_outer_iterations", C.c_int),
        ("normalizer", C.c_int),
        ("flavour", C.c_int),
        ("cg_max_iterations", C.c_int),
        ("cg_check_interval", C.c_int),
    ]


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("final_rel", C.c_double),
        ("converged", C.c_int),
        ("depth", C.c_int),
        ("level_iterations", C.c_int * MAX_LEVELS),
        ("level_final_rel", C.c_double * MAX_LEVELS),
        ("level_converged", C.c_int * MAX_LEVELS),
        ("local_solves", C.c_longlong),
        ("local_failures", C.c_longlong),
        ("local_cg_iterations", C.c_longlong),
        ("trace_rows", C.c_int),
        ("error", C.c_int),
    ]


def default_options(**kw) -> Options:
    o = Options(1e-3, 3, 32, 6, 0.25, 1e-2, 0, 1e-2, 30, 30, 1000, 0, 1, 100000, 4)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref/libref.so where the reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


_P = np.ctypeslib.ndpointer
_f64 = _P(dtype=np.float64, flags="C_CONTIGUOUS")
_u8 = _P(dtype=np.uint8, flags="C_CONTIGUOUS")


def _load_oracle():
    if not os.path.exists(ORACLE_SO):
        build()
    lib = C.CDLL(ORACLE_SO)
    lib.or_multilevel_solve.argtypes = [_f64, _u8, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(Options), _f64, C.POINTER(Report),
                                        _f64, C.c_int]
    lib.or_residual_sumsq.argtypes = [_u8, C.c_int, C.c_int, _f64, _f64]
    lib.or_residual_sumsq.restype = C.c_double
    lib.or_restrict_level.argtypes = [_u8, _f64, C.c_int, C.c_int, C.c_int, C.c_int, _u8, _f64]
    lib.or_prolongate.argtypes = [_f64, C.c_int, C.c_int, C.c_int, C.c_int, _f64]
    lib.or_schwarz_sweep.argtypes = [_u8, C.c_int, C.c_int, C.c_int, _f64, _f64, C.c_int,
                                     C.c_int, C.POINTER(Options), _f64,
                                     C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
    lib.or_local_operator_apply.argtypes = [_u8, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, C.c_int, C.c_double, _f64, _f64]
    lib.or_partition_axis.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(C.c_int)]
    _i32 = _P(dtype=np.int32, flags="C_CONTIGUOUS")
    lib.or_assign_nearest_site.argtypes = [_u8, C.c_int, C.c_int, _i32, _i32, C.POINTER(C.c_int)]
    lib.or_voronoi_densify.argtypes = [_f64, C.c_int, C.c_int, C.c_int, _u8, C.c_longlong,
                                       C.c_double, C.c_double, C.c_int, C.POINTER(Options), _u8,
                                       C.POINTER(C.c_int)]
    return lib


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        _oracle = _load_oracle()
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _cpu_flags() -> set:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def use_tuned_reference() -> str:
    """Select the reference build tuned for this host (the `-march=native`
    of the benchmark protocol) when the CPU supports it; call
    before the first ref().  Returns a description of the build in use."""
    global _ref_path
    if _ref is None and os.path.exists(REF_SPR_SO) and \
            {"avx512f", "avx512_fp16", "amx_tile"} <= _cpu_flags():
        _ref_path = REF_SPR_SO
    return ref_build()


def ref_build() -> str:
    return ("g++ -std=c++20 -O3 " +
            ("-march=sapphirerapids" if _ref_path == REF_SPR_SO else "-march=x86-64-v3") +
            " -pthread (" + os.path.relpath(_ref_path, os.path.dirname(HERE)) + ")")


def ref():
    """The compiled reference (raises if it was never built here)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(_ref_path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_synthetic_test_image.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _f64]
        lib.ref_random_mask.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, _u8]
        lib.ref_set_threads.argtypes = [C.c_int]
        lib.ref_thread_count.restype = C.c_int
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        lib.ref_run_method.argtypes = [C.c_int, _f64, _u8, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(Options), C.c_void_p, _f64, ip, dp, ip,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, ip, dp]
        lib.ref_multilevel_levels.argtypes = [_f64, _u8, C.c_int, C.c_int, C.c_int,
                                              C.POINTER(Options), _f64, C.POINTER(Report),
                                              _f64, C.c_int]
        lib.ref_partition_domain.argtypes = [C.c_int] * 4 + [ip, ip, C.POINTER(C.c_int), C.c_int]
        lib.ref_restrict_level.argtypes = [_u8, _f64, C.c_int, C.c_int, C.c_int, C.c_int, _u8,
                                           _f64]
        lib.ref_prolongate.argtypes = [_f64, C.c_int, C.c_int, C.c_int, C.c_int, _f64]
        lib.ref_local_operator_apply.argtypes = [_u8, C.c_int, C.c_int, C.c_int, C.c_int,
                                                 C.c_int, C.c_int, C.c_double, _f64, _f64]
        lib.ref_run_schwarz_level.argtypes = [_u8, C.c_int, C.c_int, C.c_int, _f64, _f64,
                                              C.c_int, C.c_int, C.c_double, C.c_double,
                                              C.POINTER(Options), ip, dp, ip,
                                              C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                              _f64, C.c_int, ip]
        lib.ref_canonical_r0.argtypes = [_u8, C.c_int, C.c_int, C.c_int, _f64, C.c_int]
        lib.ref_canonical_r0.restype = C.c_double
        _i32 = _P(dtype=np.int32, flags="C_CONTIGUOUS")
        lib.ref_assign_nearest_site.argtypes = [_u8, C.c_int, C.c_int, _i32, _i32, ip]
        lib.ref_voronoi_densify.argtypes = [_f64, C.c_int, C.c_int, C.c_int, C.c_double,
                                            C.c_uint64, C.c_double, C.c_double, C.c_double,
                                            C.c_int, C.POINTER(Options), _u8, ip, ip]
        _ref = lib
    return _ref


# ---------------------------------------------------------------- results
@dataclass
class Solve:
    image: np.ndarray                 # (c, h, w) float64
    iterations: int
    final_rel: float
    converged: bool
    trace: np.ndarray                 # finest-level rel per outer iteration
    level_iterations: list = field(default_factory=list)   # index 0 = finest
    depth: int = 0
    local_solves: int = 0
    local_failures: int = 0
    local_cg_iterations: int = 0
    elapsed_ms: float = 0.0
    psnr: object = None               # per trace row (ref_run_method with a reference)


def _flat(f: np.ndarray):
    f = np.ascontiguousarray(f, dtype=np.float64)
    if f.ndim == 2:
        f = f[None]
    return f


def oracle_solve(f: np.ndarray, mask: np.ndarray, **opts) -> Solve:
    """Multilevel (levels>=1) ORAS/RAS solve with the C restatement."""
    f = _flat(f)
    c, h, w = f.shape
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    o = default_options(**opts)
    out = np.empty_like(f)
    rep = Report()
    cap = max(o.max_outer_iterations, 0) + 2 if o.flavour != 2 else o.cg_max_iterations + 2
    trace = np.zeros(cap)
    rc = oracle().or_multilevel_solve(f.ravel(), m.ravel(), w, h, c, C.byref(o), out.ravel(),
                                      C.byref(rep), trace, cap)
    if rc != 0:
        raise ValueError("oracle: invalid argument")
    return Solve(out, rep.iterations, rep.final_rel, bool(rep.converged),
                 trace[: min(rep.trace_rows, cap)].copy(),
                 [rep.level_iterations[i] for i in range(rep.depth)], rep.depth,
                 rep.local_solves, rep.local_failures, rep.local_cg_iterations)


def ref_solve_levels(f: np.ndarray, mask: np.ndarray, **opts) -> Solve:
    """The reference's multilevel loop with per-level counts (ref_driver)."""
    f = _flat(f)
    c, h, w = f.shape
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    o = default_options(**opts)
    out = np.empty_like(f)
    rep = Report()
    cap = o.max_outer_iterations + 2
    trace = np.zeros(cap)
    rc = ref().ref_multilevel_levels(f.ravel(), m.ravel(), w, h, c, C.byref(o), out.ravel(),
                                     C.byref(rep), trace, cap)
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    return Solve(out, rep.iterations, rep.final_rel, bool(rep.converged),
                 trace[: min(rep.trace_rows, cap)].copy(),
                 [rep.level_iterations[i] for i in range(rep.depth)], rep.depth,
                 rep.local_solves, rep.local_failures)


METHODS = {"cg": 0, "mlcg": 1, "ras": 2, "oras": 3, "mloras": 4}


def ref_run_method(method: str, f: np.ndarray, mask: np.ndarray, reference=None,
                   **opts) -> Solve:
    """schwarz_inpaint::run_method exactly as a user calls it."""
    f = _flat(f)
    c, h, w = f.shape
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    o = default_options(**opts)
    out = np.empty_like(f)
    it, conv, rows = C.c_int(), C.c_int(), C.c_int()
    fr, ms = C.c_double(), C.c_double()
    cap = max(o.max_outer_iterations, 100000) + 2
    trace = np.zeros(cap)
    psnr = np.full(cap, np.nan)
    refbuf = None if reference is None else _flat(reference)
    rc = ref().ref_run_method(METHODS[method], f.ravel(), m.ravel(), w, h, c, C.byref(o),
                              None if refbuf is None else refbuf.ctypes.data, out.ravel(),
                              C.byref(it), C.byref(fr), C.byref(conv), trace.ctypes.data,
                              None, psnr.ctypes.data, cap, C.byref(rows), C.byref(ms))
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    n = min(rows.value, cap)
    s = Solve(out, it.value, fr.value, bool(conv.value), trace[:n].copy())
    s.psnr = psnr[:n].copy()  # metrics.hpp:30-56 per trace row (NaN without a reference)
    s.elapsed_ms = ms.value
    return s


def ref_synthetic_test_image(w: int, h: int, c: int, seed: int) -> np.ndarray:
    out = np.empty((c, h, w))
    if ref().ref_synthetic_test_image(w, h, c, seed, out.ravel()) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_random_mask(w: int, h: int, density: float, seed: int) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    if ref().ref_random_mask(w, h, density, seed, out.ravel()) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out


def oracle_sweep(mask, b, u, block, overlap, **opts):
    """One outer ORAS sweep on a fixed partition; returns (u_new, failures, cg_its)."""
    b = _flat(b)
    u = _flat(u)
    c, h, w = u.shape
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    o = default_options(**opts)
    un = np.empty_like(u)
    fails, its = C.c_longlong(), C.c_longlong()
    oracle().or_schwarz_sweep(m.ravel(), w, h, c, b.ravel(), u.ravel(), block, overlap,
                              C.byref(o), un.ravel(), C.byref(fails), C.byref(its))
    return un, fails.value, its.value


def oracle_residual_sumsq(mask, u, b) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    h, w = mask.shape
    return oracle().or_residual_sumsq(np.ascontiguousarray(mask, dtype=np.uint8).ravel(), w, h,
                                      u.ravel(), b.ravel())


def oracle_restrict(mask, values, averaging=0):
    values = _flat(values)
    c, h, w = values.shape
    cw, ch = (w + 1) // 2, (h + 1) // 2
    cm = np.empty((ch, cw), np.uint8)
    cv = np.empty((c, ch, cw))
    oracle().or_restrict_level(np.ascontiguousarray(mask, np.uint8).ravel(), values.ravel(), w,
                               h, c, averaging, cm.ravel(), cv.ravel())
    return cm, cv


def oracle_prolongate(coarse, fw, fh):
    coarse = np.ascontiguousarray(coarse, np.float64)
    ch, cw = coarse.shape
    fine = np.empty((fh, fw))
    oracle().or_prolongate(coarse.ravel(), cw, ch, fw, fh, fine.ravel())
    return fine


def oracle_partition_axis(extent, block, overlap):
    n = extent + 2
    a = (C.c_int * n)()
    e = (C.c_int * n)()
    cnt = C.c_int()
    oracle().or_partition_axis(extent, block, overlap, a, C.byref(cnt), e)
    return list(a[: cnt.value]), list(e[: cnt.value])


# ---------------------------------------------------------------- densification
def _assign(fn, mask):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    h, w = m.shape
    sites = np.empty(w * h, np.int32)
    site_of = np.empty(w * h, np.int32)
    k = C.c_int()
    if fn(m.ravel(), w, h, sites, site_of, C.byref(k)) != 0:
        raise ValueError("assign_nearest_site: mask has no known pixels")
    return sites[: k.value].copy(), site_of.reshape(h, w)


def oracle_assign_nearest_site(mask):
    """(sites, site_of) of the C restatement (masks.hpp:54-139)."""
    return _assign(oracle().or_assign_nearest_site, mask)


def ref_assign_nearest_site(mask):
    return _assign(ref().ref_assign_nearest_site, mask)


def densify_seed_density(target: float, n: int, initial: float = 0.0) -> float:
    """Starting density of voronoi_densify (masks.hpp:166-167)."""
    init = initial if initial > 0.0 else target / 4.0
    return 1.5 / n if init * n < 1.0 else init


def densify_target(target: float, n: int) -> int:
    """target_k of masks.hpp:163-165 (llround = half away from zero)."""
    v = target * n
    k = int(np.floor(v + 0.5)) if v >= 0 else int(np.ceil(v - 0.5))
    return max(1, min(n, k))


def oracle_voronoi_densify(f, seed_mask, target, cell_fraction=0.20, inner_tolerance=1e-3,
                           max_sweeps=100, **opts):
    """voronoi_densify of the C restatement from the seed mask; (mask, sweeps)."""
    f = _flat(f)
    c, h, w = f.shape
    o = default_options(**opts)
    out = np.empty((h, w), np.uint8)
    sw = C.c_int()
    seed = np.ascontiguousarray(seed_mask, dtype=np.uint8)
    if oracle().or_voronoi_densify(f.ravel(), w, h, c, seed.ravel(), densify_target(target, w * h),
                                   cell_fraction, inner_tolerance, max_sweeps, C.byref(o),
                                   out.ravel(), C.byref(sw)) != 0:
        raise ValueError("oracle: invalid argument")
    return out, sw.value


def ref_voronoi_densify(f, target, seed, initial_density=0.0, cell_fraction=0.20,
                        inner_tolerance=1e-3, max_sweeps=100, **opts):
    """schwarz_inpaint::voronoi_densify; returns (mask, sweeps, reached)."""
    f = _flat(f)
    c, h, w = f.shape
    o = default_options(**opts)
    out = np.empty((h, w), np.uint8)
    sw, rc_ = C.c_int(), C.c_int()
    if ref().ref_voronoi_densify(f.ravel(), w, h, c, target, seed, initial_density, cell_fraction,
                                 inner_tolerance, max_sweeps, C.byref(o), out.ravel(),
                                 C.byref(sw), C.byref(rc_)) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out, sw.value, bool(rc_.value)
