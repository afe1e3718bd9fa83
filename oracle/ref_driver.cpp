// TEST INFRASTRUCTURE ONLY — C-ABI harness around the UNMODIFIED reference.
//
// Compiled by oracle/Makefile against the reference headers where they lie
// (/root/reference/proj/include, header-only C++20) into oracle/_ref/libref.so.
// Nothing from the reference is copied here: this file only calls its public
// API (schwarz_inpaint::run_method, build_pyramid, run_schwarz_level, ...)
// and marshals plain arrays so Python tests / bench.py can drive it through
// ctypes.  It exists (a) to pin the C restatement in oracle/si_oracle.c,
// (b) to generate tests/golden/ fixtures, and (c) as bench.py's reference
// CPU arm ("cpu_baseline.kind": "reference").
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "schwarz_inpaint/masks.hpp"
#include "schwarz_inpaint/methods.hpp"
#include "schwarz_inpaint/multilevel.hpp"
#include "schwarz_inpaint/parallel.hpp"
#include "schwarz_inpaint/partition.hpp"
#include "schwarz_inpaint/schwarz.hpp"
#include "schwarz_inpaint/synthetic.hpp"

namespace si = schwarz_inpaint;

namespace {
thread_local std::string g_err;

struct RefOptions {  // same field order as or_options in si_oracle.h
  double tolerance;
  int levels;
  int block_size;
  int overlap;
  double alpha;
  double coarse_tolerance;
  int averaging;
  double local_tolerance;
  int local_max_iterations;
  int local_check_interval;
  int max_outer_iterations;
  int normalizer;
  int flavour;
  int cg_max_iterations;
  int cg_check_interval;
};

struct RefReport {  // same layout as or_report
  int iterations;
  double final_rel;
  int converged;
  int depth;
  int level_iterations[32];
  double level_final_rel[32];
  int level_converged[32];
  long long local_solves;
  long long local_failures;
  long long local_cg_iterations;
  int trace_rows;
  int error;
};

si::ImageBuffer make_image(const double* f, int w, int h, int c) {
  si::ImageBuffer img(w, h, c);
  std::memcpy(img.data.data(), f, sizeof(double) * img.data.size());
  return img;
}

si::InpaintingMask make_mask(const uint8_t* m, int w, int h) {
  si::InpaintingMask mask(w, h);
  std::memcpy(mask.known.data(), m, mask.known.size());
  return mask;
}

si::RunOptions run_options(const RefOptions* o) {
  si::RunOptions r;
  r.tolerance = o->tolerance;
  r.levels = o->levels;
  r.block_size = o->block_size;
  r.overlap = o->overlap;
  r.alpha = o->alpha;
  r.coarse_tolerance = o->coarse_tolerance;
  r.averaging = o->averaging ? si::CoarseAveraging::AllPixels : si::CoarseAveraging::KnownOnly;
  r.local = si::SolverConfig{o->local_tolerance, o->local_max_iterations, o->local_check_interval};
  r.max_outer_iterations = o->max_outer_iterations;
  r.normalizer = o->normalizer ? si::ResidualNormalizer::RhsNorm
                               : si::ResidualNormalizer::InitialGuess;
  r.cg_max_iterations = o->cg_max_iterations;
  r.cg_check_interval = o->cg_check_interval;
  return r;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { si::parallel::set_thread_count(n); }
int ref_thread_count() { return si::parallel::thread_count(); }

int ref_synthetic_test_image(int w, int h, int c, uint64_t seed, double* out) {
  try {
    auto img = si::synthetic_test_image(w, h, c, seed);
    std::memcpy(out, img.data.data(), sizeof(double) * img.data.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_random_mask(int w, int h, double density, uint64_t seed, uint8_t* out) {
  try {
    auto m = si::random_mask(w, h, density, seed);
    std::memcpy(out, m.known.data(), m.known.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// run_method(method, f, mask, options) exactly as a user calls it
// (methods.hpp:57-88); method: 0 cg, 1 mlcg, 2 ras, 3 oras, 4 mloras.
// Returns 0 ok, 1 invalid argument.  Also reports time_ms per trace row.
int ref_run_method(int method, const double* f, const uint8_t* mask, int w, int h, int c,
                   const RefOptions* opt, const double* reference, double* out, int* iterations,
                   double* final_rel, int* converged, double* trace_rel, double* trace_ms,
                   double* trace_psnr, int trace_cap, int* trace_rows, double* elapsed_ms) {
  try {
    const auto img = make_image(f, w, h, c);
    const auto m = make_mask(mask, w, h);
    const auto ro = run_options(opt);
    si::ImageBuffer ref_img;
    if (reference) ref_img = make_image(reference, w, h, c);
    si::Stopwatch clock;
    const auto res = si::run_method(static_cast<si::Method>(method), img, m, ro,
                                    reference ? &ref_img : nullptr);
    if (elapsed_ms) *elapsed_ms = clock.elapsed_ms();
    std::memcpy(out, res.image.data.data(), sizeof(double) * res.image.data.size());
    *iterations = res.report.iterations;
    *final_rel = res.report.final_relative_residual;
    *converged = res.report.converged;
    const int rows = static_cast<int>(res.trace.rows.size());
    *trace_rows = rows;
    for (int i = 0; i < rows && i < trace_cap; ++i) {
      if (trace_rel) trace_rel[i] = res.trace.rows[i].rel_residual;
      if (trace_ms) trace_ms[i] = res.trace.rows[i].time_ms;
      if (trace_psnr)
        trace_psnr[i] = res.trace.rows[i].psnr ? *res.trace.rows[i].psnr : std::nan("");
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// The multilevel loop of multilevel_solve (multilevel.hpp:239-310) re-driven
// through the reference's public pieces so per-level outer counts and the
// local-solve statistics become visible.  Its trace and output equal
// run_method's (checked in tests/test_oracle.py).
int ref_multilevel_levels(const double* f, const uint8_t* mask, int w, int h, int c,
                          const RefOptions* opt, double* out, RefReport* rep, double* trace_rel,
                          int trace_cap) {
  try {
    std::memset(rep, 0, sizeof(*rep));
    const auto img = make_image(f, w, h, c);
    const auto m = make_mask(mask, w, h);
    const auto pyramid = si::build_pyramid(
        img, m, opt->levels,
        opt->averaging ? si::CoarseAveraging::AllPixels : si::CoarseAveraging::KnownOnly);
    const int depth = static_cast<int>(pyramid.size());
    rep->depth = depth;
    const std::size_t nc = static_cast<std::size_t>(c);
    std::vector<si::ChannelVector> u;
    for (int level = depth - 1; level >= 0; --level) {
      const auto& problem = pyramid[level];
      if (level == depth - 1) {
        u.assign(nc, si::ChannelVector());
        for (std::size_t k = 0; k < nc; ++k)
          u[k] = si::build_rhs(problem.values.channel(static_cast<int>(k)), problem.mask);
      }
      const bool finest = level == 0;
      const double tol = finest ? opt->tolerance : opt->coarse_tolerance;
      si::InpaintingOperator op(problem.mask);
      std::vector<si::ChannelVector> b(nc);
      for (std::size_t k = 0; k < nc; ++k)
        b[k] = si::build_rhs(problem.values.channel(static_cast<int>(k)), problem.mask);
      const auto part = si::clamped_partition(problem.mask.width, problem.mask.height,
                                              opt->block_size, opt->overlap);
      si::SchwarzOptions sopt;
      sopt.flavour = opt->flavour ? si::SchwarzFlavour::Oras : si::SchwarzFlavour::Ras;
      sopt.alpha = opt->alpha;
      sopt.local = si::SolverConfig{opt->local_tolerance, opt->local_max_iterations,
                                    opt->local_check_interval};
      sopt.max_outer_iterations = opt->max_outer_iterations;
      const double r0 = si::canonical_r0(
          op, b,
          opt->normalizer ? si::ResidualNormalizer::RhsNorm : si::ResidualNormalizer::InitialGuess);
      auto sink = [&](int, double rel) {
        if (!finest) return;
        if (trace_rel && rep->trace_rows < trace_cap) trace_rel[rep->trace_rows] = rel;
        rep->trace_rows++;
      };
      const auto stats = si::run_schwarz_level(op, part, b, u, r0, tol, sopt, sink);
      rep->level_iterations[level] = stats.iterations;
      rep->level_final_rel[level] = stats.final_rel;
      rep->level_converged[level] = stats.converged;
      rep->local_solves += stats.local_solves;
      rep->local_failures += stats.local_failures;
      if (finest) {
        rep->iterations = stats.iterations;
        rep->final_rel = stats.final_rel;
        rep->converged = stats.converged;
      } else {
        const auto& next = pyramid[level - 1];
        for (std::size_t k = 0; k < nc; ++k) {
          u[k] = si::prolongate(u[k], problem.mask.width, problem.mask.height, next.mask.width,
                                next.mask.height);
          auto values = next.values.channel(static_cast<int>(k));
          for (std::size_t i = 0; i < next.mask.size(); ++i)
            if (next.mask.known[i]) u[k][i] = values[i];
        }
      }
    }
    for (std::size_t k = 0; k < nc; ++k)
      std::memcpy(out + k * static_cast<std::size_t>(w) * h, u[k].data(),
                  sizeof(double) * u[k].size());
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    rep->error = 1;
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    rep->error = 2;
    return 2;
  }
}

int ref_partition_domain(int w, int h, int block, int overlap, int* blocks_x, int* blocks_y,
                         int* rects, int cap) {
  try {
    const auto part = si::partition_domain(w, h, block, overlap);
    *blocks_x = part.blocks_x;
    *blocks_y = part.blocks_y;
    for (std::size_t i = 0; i < part.size() && static_cast<int>(i) < cap; ++i) {
      const auto& sd = part.subdomains[i];
      int* r = rects + 8 * i;
      r[0] = sd.x0; r[1] = sd.y0; r[2] = sd.width; r[3] = sd.height;
      r[4] = sd.own_x0; r[5] = sd.own_y0; r[6] = sd.own_x1; r[7] = sd.own_y1;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_restrict_level(const uint8_t* mask, const double* values, int w, int h, int c,
                       int averaging, uint8_t* cmask, double* cvalues) {
  try {
    const auto lp = si::restrict_level(
        make_mask(mask, w, h), make_image(values, w, h, c),
        averaging ? si::CoarseAveraging::AllPixels : si::CoarseAveraging::KnownOnly);
    std::memcpy(cmask, lp.mask.known.data(), lp.mask.known.size());
    std::memcpy(cvalues, lp.values.data.data(), sizeof(double) * lp.values.data.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_prolongate(const double* coarse, int cw, int ch, int fw, int fh, double* fine) {
  try {
    const auto v = si::prolongate(std::span<const double>(coarse, static_cast<std::size_t>(cw) * ch),
                                  cw, ch, fw, fh);
    std::memcpy(fine, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_local_operator_apply(const uint8_t* mask, int w, int h, int block, int overlap, int index,
                             int flavour, double alpha, const double* v, double* out) {
  try {
    const auto part = si::partition_domain(w, h, block, overlap);
    const auto op = si::build_local_operator(
        make_mask(mask, w, h), part, static_cast<std::size_t>(index),
        flavour ? si::SchwarzFlavour::Oras : si::SchwarzFlavour::Ras, alpha);
    op.apply(std::span<const double>(v, op.size()), std::span<double>(out, op.size()));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// run_schwarz_level (schwarz.hpp:266-323) with caller-supplied u, b, r0:
// the reference's finest public seam.  u is updated in place.
int ref_run_schwarz_level(const uint8_t* mask, int w, int h, int c, const double* b_in, double* u_io,
                          int block, int overlap, double r0, double tol, const RefOptions* opt,
                          int* iterations, double* final_rel, int* converged,
                          long long* local_solves, long long* local_failures, double* trace_rel,
                          int trace_cap, int* trace_rows) {
  try {
    const std::size_t n = static_cast<std::size_t>(w) * h;
    si::InpaintingOperator op(make_mask(mask, w, h));
    const auto part = si::partition_domain(w, h, block, overlap);
    std::vector<si::ChannelVector> b(c), u(c);
    for (int k = 0; k < c; ++k) {
      b[k].assign(b_in + k * n, b_in + (k + 1) * n);
      u[k].assign(u_io + k * n, u_io + (k + 1) * n);
    }
    si::SchwarzOptions sopt;
    sopt.flavour = opt->flavour ? si::SchwarzFlavour::Oras : si::SchwarzFlavour::Ras;
    sopt.alpha = opt->alpha;
    sopt.local = si::SolverConfig{opt->local_tolerance, opt->local_max_iterations,
                                  opt->local_check_interval};
    sopt.max_outer_iterations = opt->max_outer_iterations;
    int rows = 0;
    auto sink = [&](int, double rel) {
      if (trace_rel && rows < trace_cap) trace_rel[rows] = rel;
      ++rows;
    };
    const auto st = si::run_schwarz_level(op, part, b, u, r0, tol, sopt, sink);
    for (int k = 0; k < c; ++k) std::memcpy(u_io + k * n, u[k].data(), sizeof(double) * n);
    *iterations = st.iterations;
    *final_rel = st.final_rel;
    *converged = st.converged;
    *local_solves = st.local_solves;
    *local_failures = st.local_failures;
    *trace_rows = rows;
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

double ref_canonical_r0(const uint8_t* mask, int w, int h, int c, const double* b_in,
                        int normalizer) {
  const std::size_t n = static_cast<std::size_t>(w) * h;
  si::InpaintingOperator op(make_mask(mask, w, h));
  std::vector<si::ChannelVector> b(c);
  for (int k = 0; k < c; ++k) b[k].assign(b_in + k * n, b_in + (k + 1) * n);
  return si::canonical_r0(op, b,
                          normalizer ? si::ResidualNormalizer::RhsNorm
                                     : si::ResidualNormalizer::InitialGuess);
}

// assign_nearest_site (masks.hpp:54-139) as the reference computes it.
int ref_assign_nearest_site(const uint8_t* mask, int w, int h, int32_t* sites, int32_t* site_of,
                            int* num_sites) {
  try {
    auto a = si::assign_nearest_site(make_mask(mask, w, h));
    std::memcpy(sites, a.sites.data(), sizeof(int32_t) * a.sites.size());
    std::memcpy(site_of, a.site_of.data(), sizeof(int32_t) * a.site_of.size());
    *num_sites = static_cast<int>(a.sites.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// voronoi_densify (masks.hpp:155-212); the guide solver's options come from
// RefOptions (MultilevelSolveOptions, multilevel.hpp:132-142).
int ref_voronoi_densify(const double* f, int w, int h, int c, double target, uint64_t seed,
                        double initial_density, double cell_fraction, double inner_tolerance,
                        int max_sweeps, const RefOptions* o, uint8_t* mask_out, int* sweeps,
                        int* reached) {
  try {
    si::DensifyOptions d;
    d.initial_density = initial_density;
    d.cell_fraction = cell_fraction;
    d.inner_tolerance = inner_tolerance;
    d.max_sweeps = max_sweeps;
    d.solve.levels = o->levels;
    d.solve.tolerance = o->tolerance;
    d.solve.coarse_tolerance = o->coarse_tolerance;
    d.solve.averaging = o->averaging ? si::CoarseAveraging::AllPixels
                                     : si::CoarseAveraging::KnownOnly;
    d.solve.block_size = o->block_size;
    d.solve.overlap = o->overlap;
    d.solve.schwarz.alpha = o->alpha;
    d.solve.schwarz.local =
        si::SolverConfig{o->local_tolerance, o->local_max_iterations, o->local_check_interval};
    d.solve.schwarz.max_outer_iterations = o->max_outer_iterations;
    d.solve.normalizer = o->normalizer ? si::ResidualNormalizer::RhsNorm
                                       : si::ResidualNormalizer::InitialGuess;
    auto r = si::voronoi_densify(make_image(f, w, h, c), target, seed, d);
    std::memcpy(mask_out, r.mask.known.data(), r.mask.known.size());
    *sweeps = r.sweeps;
    *reached = r.reached_target ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
