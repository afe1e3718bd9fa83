"""paper_2110_03946_b200 — B200-native multilevel ORAS inpainting (arXiv 2110.03946).

A drop-in for the solver path of the reference C++ library schwarz-inpaint:
``run_method(Method.MultilevelOras, f, mask, RunOptions())`` and its lower
seams.  The compute lives in ``libschwarz_b200.so`` (hand-written sm_100a
CUDA behind the C ABI in ``include/schwarz_b200.h``); this package is the
Python mirror of the reference interface.
"""
from .api import (  # noqa: F401
    CoarseAveraging, ConvergenceTrace, DensifyOptions, DensifyResult, ImageBuffer, InpaintingMask, InvalidArgument, LevelSolver,
    Method, MultilevelSolveOptions, Precision, ResidualNormalizer, RunOptions, SchwarzFlavour,
    SchwarzOptions, SchwarzSolveOptions, SolveReport, SolveResult, Solver, SolverConfig,
    SolverError, Subdomain, SubdomainPartition, TraceRow, Unsupported, canonical_r0,
    clamped_partition, default_solver, is_multilevel, kDefaultOrasAlpha, method_name,
    mse_per_channel, multilevel_solve, pack_known_samples, pack_pbm, quantise_pnm, parse_method,
    partition_domain,
    psnr, random_mask, run_batch, run_method, run_schwarz_level, solve_schwarz,
    synthetic_test_image, VoronoiAssignment, assign_nearest_site, voronoi_densify)

__all__ = [n for n in dir() if not n.startswith("_")]
