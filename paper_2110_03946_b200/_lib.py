"""ctypes binding of libschwarz_b200.so (C ABI: include/schwarz_b200.h).

The library is the only compute path: if it cannot be loaded (or built in
place with nvcc) every solver call fails loudly.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

MAX_LEVELS = 32
SI_MAX_LEVELS = MAX_LEVELS
SI_NCCL_ID_BYTES = 128

SI_OK = 0
SI_ERR_INVALID_ARGUMENT = 1
SI_ERR_CUDA = 2
SI_ERR_OOM = 3
SI_ERR_UNSUPPORTED = 4
SI_ERR_NO_DEVICE = 5
SI_ERR_RUNTIME = 6


class si_options(C.Structure):
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
        ("cg_max_iterations", C.c_int),
        ("cg_check_interval", C.c_int),
        ("normalizer", C.c_int),
        ("precision", C.c_int),
    ]


class si_report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("final_relative_residual", C.c_double),
        ("converged", C.c_int),
        ("diagnostic", C.c_char * 128),
        ("depth", C.c_int),
        ("level_iterations", C.c_int * MAX_LEVELS),
        ("level_final_rel", C.c_double * MAX_LEVELS),
        ("level_converged", C.c_int * MAX_LEVELS),
        ("local_solves", C.c_longlong),
        ("local_failures", C.c_longlong),
        ("local_cg_iterations", C.c_longlong),
        ("elapsed_ms", C.c_double),
        ("h2d_bytes", C.c_longlong),
        ("d2h_bytes", C.c_longlong),
    ]


class si_kernel_stats(C.Structure):
    _fields_ = [
        ("launches", C.c_longlong * 8),
        ("device_ms", C.c_double * 8),
        ("algorithmic_bytes", C.c_double * 8),
        ("total_launches", C.c_longlong),
    ]


class si_densify_options(C.Structure):
    _fields_ = [
        ("initial_density", C.c_double),
        ("cell_fraction", C.c_double),
        ("inner_tolerance", C.c_double),
        ("max_sweeps", C.c_int),
        ("solve", si_options),
    ]


TRACE_FN = C.CFUNCTYPE(None, C.c_int, C.c_double, C.c_double, C.c_double, C.c_void_p)

_vp = C.c_void_p
_i = C.c_int
_d = C.c_double
_ip = C.POINTER(C.c_int)
_llp = C.POINTER(C.c_longlong)
_dp = C.POINTER(C.c_double)

# name -> (restype, argtypes); every symbol declared in include/schwarz_b200.h
SIGNATURES = {
    "si_abi_version": (_i, []),
    "si_last_error": (C.c_char_p, []),
    "si_status_string": (C.c_char_p, [_i]),
    "si_default_options": (None, [C.POINTER(si_options)]),
    "si_validate_options": (_i, [_i, C.POINTER(si_options)]),
    "si_create": (_i, [_i, C.POINTER(_vp)]),
    "si_destroy": (None, [_vp]),
    "si_trim": (_i, [_vp]),
    "si_run_method": (_i, [_vp, _i, _vp, _vp, _i, _i, _i, C.POINTER(si_options), _vp, _vp,
                           C.POINTER(si_report), TRACE_FN, _vp]),
    "si_run_method_device": (_i, [_vp, _i, _vp, _vp, _i, _i, _i, C.POINTER(si_options), _vp,
                                  _vp, C.POINTER(si_report), TRACE_FN, _vp, _vp]),
    "si_run_method_batch": (_i, [_vp, _i, _i, C.POINTER(_vp), C.POINTER(_vp), _i, _i, _i,
                                 C.POINTER(si_options), C.POINTER(_vp), C.POINTER(si_report)]),
    "si_run_pnm_batch": (_i, [_vp, _i, _i, C.POINTER(_vp), C.POINTER(_vp), _i, _i, _i,
                              C.POINTER(si_options), C.POINTER(_vp), C.POINTER(si_report)]),
    "si_solve_schwarz": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(si_options), _vp,
                              _vp, C.POINTER(si_report), TRACE_FN, _vp]),
    "si_run_schwarz_level": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _i, _i, _d, _d, _i,
                                  C.POINTER(si_options), C.POINTER(si_report), TRACE_FN, _vp]),
    "si_canonical_r0": (_i, [_vp, _vp, _i, _i, _i, _vp, _i, _dp]),
    "si_schwarz_sweep": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _i, _i, _i, C.POINTER(si_options),
                              _vp, _llp, _llp]),
    "si_residual_sumsq": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "si_restrict_level": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "si_prolongate": (_i, [_vp, _vp, _i, _i, _i, _i, _vp]),
    "si_local_operator_apply": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _i, _d, _vp, _vp]),
    "si_nccl_unique_id": (_i, [_vp]),
    "si_stripe_comm_init_nccl": (_i, [_vp, _i, _i, _vp, C.POINTER(_vp)]),
    "si_stripe_comm_init_local": (_i, [C.POINTER(_vp), _i, C.POINTER(_vp)]),
    "si_stripe_comm_destroy": (None, [_vp]),
    "si_stripe_comm_set_speculation": (_i, [_vp, _i]),
    "si_stripe_result_rows": (_i, [_vp, C.POINTER(_vp), C.POINTER(C.c_size_t), _ip]),
    "si_stripe_comm_counters": (_i, [_vp, _llp]),
    "si_stripe_level_plan": (_i, [_i, _i, _i, _i, C.POINTER(si_options), _i, _i, _ip, _ip]),
    "si_run_method_striped": (_i, [_vp, _vp, _i, _vp, _vp, _i, _i, _i, C.POINTER(si_options),
                                   _vp, C.POINTER(si_report), TRACE_FN, _vp]),
    "si_run_method_striped_device": (_i, [_vp, _vp, _i, _vp, _vp, _i, _i, _i,
                                          C.POINTER(si_options), _vp, C.POINTER(si_report), _vp]),
    "si_run_method_striped_local_device": (_i, [C.POINTER(_vp), C.POINTER(_vp), _i, _i,
                                                C.POINTER(_vp), C.POINTER(_vp), _i, _i, _i,
                                                C.POINTER(si_options), C.POINTER(_vp),
                                                C.POINTER(si_report), C.POINTER(_vp)]),
    "si_run_method_striped_group": (_i, [C.POINTER(_vp), _i, _i, _vp, _vp, _i, _i, _i,
                                         C.POINTER(si_options), _vp, C.POINTER(si_report)]),
    "si_partition_domain": (_i, [_i, _i, _i, _i, _ip, _ip, _ip, _i]),
    "si_pack_known_samples": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _llp]),
    "si_synthetic_test_image": (_i, [_i, _i, _i, C.c_uint64, _vp]),
    "si_random_mask": (_i, [_i, _i, _d, C.c_uint64, _vp]),
    "si_default_densify_options": (None, [C.POINTER(si_densify_options)]),
    "si_voronoi_densify": (_i, [_vp, _vp, _i, _i, _i, _d, C.c_uint64,
                                C.POINTER(si_densify_options), _vp, _ip, _ip]),
    "si_assign_nearest_site": (_i, [_vp, _vp, _i, _i, _vp, _vp, _ip]),
    "si_joint_norm": (_d, [_dp, _i]),
    "si_psnr": (_i, [_vp, _vp, _i, _i, _i, _dp]),
    "si_set_profiling": (_i, [_vp, _i]),
    "si_selftest": (_i, [_vp, _i, C.c_longlong, _llp]),
    "si_get_kernel_stats": (_i, [_vp, C.POINTER(si_kernel_stats), _i]),
    "si_host_alloc": (_i, [C.c_size_t, C.POINTER(_vp)]),
    "si_host_free": (_i, [_vp]),
}

_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    return os.environ.get("SI_LIB_PATH") or _build.LIB


def load(build_if_missing: bool = True):
    """Load (building in place first if missing or stale) the CUDA library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing and (not os.path.exists(_build.LIB) or
                                 os.environ.get("SI_REBUILD") == "1"):
            _build.build(force=os.environ.get("SI_REBUILD") == "1")
        path = lib_path()
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: build it with "
                               "`python -m paper_2110_03946_b200.build` (nvcc, sm_100a)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.si_abi_version() != 2:
            raise RuntimeError("libschwarz_b200.so ABI mismatch")
        _lib = lib
        return lib
