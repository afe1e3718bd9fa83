// schwarz_b200.hpp — C++ drop-in for the reference's solver front door.
//
// Header-only wrapper over the C ABI (schwarz_b200.h).  It reproduces the
// reference's types and entry points (namespace schwarz_inpaint ->
// schwarz_b200) so a caller of
//     schwarz_inpaint::run_method(Method::MultilevelOras, f, mask, options)
// (methods.hpp:57-88) switches by changing the include and the namespace:
//   * ImageBuffer / InpaintingMask      image.hpp:24-94 (same planar layout)
//   * RunOptions / SolverConfig / Method methods.hpp:13-55, cg.hpp:23-27
//   * SolveResult / ConvergenceTrace    metrics.hpp:58-105
//   * SubdomainPartition                partition.hpp:21-106
// Errors: SI_ERR_INVALID_ARGUMENT -> std::invalid_argument (same message the
// reference throws); other failures -> std::runtime_error.  Non-convergence
// is reported in SolveReport, never thrown.
// Link with libschwarz_b200.so.
#pragma once

#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "schwarz_b200.h"

namespace schwarz_b200 {

namespace detail {
inline void throw_status(si_status s) {
  if (s == SI_OK) return;
  const std::string msg = si_last_error();
  if (s == SI_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string(si_status_string(s)) + ": " + msg);
}
inline void check_arg(bool ok, const std::string& msg) {
  if (!ok) throw std::invalid_argument(msg);
}
}  // namespace detail

struct ImageBuffer {
  int width = 0, height = 0, channels = 1;
  std::vector<double> data;
  ImageBuffer() = default;
  ImageBuffer(int w, int h, int ch, double fill = 0.0) : width(w), height(h), channels(ch) {
    detail::check_arg(w > 0 && h > 0 && ch > 0, "ImageBuffer: dimensions must be positive");
    data.assign(static_cast<size_t>(w) * h * ch, fill);
  }
  size_t pixel_count() const { return static_cast<size_t>(width) * height; }
  double& at(int x, int y, int c = 0) { return data[c * pixel_count() + static_cast<size_t>(y) * width + x]; }
  double at(int x, int y, int c = 0) const { return data[c * pixel_count() + static_cast<size_t>(y) * width + x]; }
};

struct InpaintingMask {
  int width = 0, height = 0;
  std::vector<uint8_t> known;
  InpaintingMask() = default;
  InpaintingMask(int w, int h, uint8_t fill = 0) : width(w), height(h) {
    detail::check_arg(w > 0 && h > 0, "InpaintingMask: dimensions must be positive");
    known.assign(static_cast<size_t>(w) * h, fill);
  }
  size_t size() const { return static_cast<size_t>(width) * height; }
  bool is_known(int x, int y) const { return known[static_cast<size_t>(y) * width + x] != 0; }
};

enum class Method { Cg = 0, MultilevelCg = 1, Ras = 2, Oras = 3, MultilevelOras = 4 };
enum class CoarseAveraging { KnownOnly = 0, AllPixels = 1 };
enum class ResidualNormalizer { InitialGuess = 0, RhsNorm = 1 };
enum class Precision { FP64 = 0, FP32 = 1, MIXED = 2 };  // MIXED: float local CG, double outer iteration

inline constexpr double kDefaultOrasAlpha = 0.25;

struct SolverConfig {
  double tolerance = 1e-6;
  int max_iterations = 10000;
  int residual_check_interval = 1;
};

struct RunOptions {
  double tolerance = 1e-3;
  int levels = 3;
  int block_size = 32;
  int overlap = 6;
  double alpha = kDefaultOrasAlpha;
  double coarse_tolerance = 1e-2;
  CoarseAveraging averaging = CoarseAveraging::KnownOnly;
  SolverConfig local{1e-2, 30, 30};
  int max_outer_iterations = 1000;
  int cg_max_iterations = 100000;
  int cg_check_interval = 4;
  ResidualNormalizer normalizer = ResidualNormalizer::InitialGuess;
  Precision precision = Precision::FP64;  // device arithmetic; FP64 = the reference's

  si_options to_c() const {
    si_options o;
    o.tolerance = tolerance;
    o.levels = levels;
    o.block_size = block_size;
    o.overlap = overlap;
    o.alpha = alpha;
    o.coarse_tolerance = coarse_tolerance;
    o.averaging = static_cast<int>(averaging);
    o.local_tolerance = local.tolerance;
    o.local_max_iterations = local.max_iterations;
    o.local_check_interval = local.residual_check_interval;
    o.max_outer_iterations = max_outer_iterations;
    o.cg_max_iterations = cg_max_iterations;
    o.cg_check_interval = cg_check_interval;
    o.normalizer = static_cast<int>(normalizer);
    o.precision = static_cast<int>(precision);
    return o;
  }
};

struct TraceRow {
  int iteration = 0;
  double time_ms = 0.0;
  double rel_residual = 0.0;
  std::optional<double> psnr;
};

struct ConvergenceTrace {
  std::vector<TraceRow> rows;
  void append(int it, double ms, double rel, std::optional<double> q = std::nullopt) {
    rows.push_back({it, ms, rel, q});
  }
};

struct SolveReport {
  int iterations = 0;
  double final_relative_residual = 0.0;
  bool converged = false;
  std::string diagnostic;
  std::vector<int> level_iterations;  // index 0 = finest (B200 extension)
  long long local_solves = 0, local_failures = 0, local_cg_iterations = 0;
};

struct SolveResult {
  ImageBuffer image;
  ConvergenceTrace trace;
  SolveReport report;
};

struct Subdomain {
  int x0 = 0, y0 = 0, width = 0, height = 0;
  int own_x0 = 0, own_y0 = 0, own_x1 = 0, own_y1 = 0;
};

struct SubdomainPartition {
  int image_width = 0, image_height = 0, block_size = 0, overlap = 0, blocks_x = 0, blocks_y = 0;
  std::vector<Subdomain> subdomains;
  size_t size() const { return subdomains.size(); }
};

// One device context per thread (the reference's single global thread pool
// becomes one CUDA context per host thread / GPU).
class Context {
 public:
  explicit Context(int device = 0) { detail::throw_status(si_create(device, &ctx_)); }
  ~Context() { si_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  si_ctx* get() const { return ctx_; }

  static Context& thread_default() {
    thread_local Context ctx(0);
    return ctx;
  }

 private:
  si_ctx* ctx_ = nullptr;
};

namespace detail {
inline void trace_sink(int it, double ms, double rel, double q, void* user) {
  auto* t = static_cast<ConvergenceTrace*>(user);
  t->append(it, ms, rel, std::isnan(q) ? std::nullopt : std::optional<double>(q));
}
inline SolveReport to_report(const si_report& r) {
  SolveReport out;
  out.iterations = r.iterations;
  out.final_relative_residual = r.final_relative_residual;
  out.converged = r.converged != 0;
  out.diagnostic = r.diagnostic;
  out.level_iterations.assign(r.level_iterations, r.level_iterations + r.depth);
  out.local_solves = r.local_solves;
  out.local_failures = r.local_failures;
  out.local_cg_iterations = r.local_cg_iterations;
  return out;
}
}  // namespace detail

// run_method (methods.hpp:57-88).
inline SolveResult run_method(Method method, const ImageBuffer& f, const InpaintingMask& mask,
                              const RunOptions& options, const ImageBuffer* reference = nullptr,
                              Context& ctx = Context::thread_default()) {
  detail::check_arg(f.width == mask.width && f.height == mask.height,
                    "image and mask dimensions differ");
  SolveResult res;
  res.image = ImageBuffer(f.width, f.height, f.channels);
  si_report rep;
  const si_options o = options.to_c();
  detail::throw_status(si_run_method(ctx.get(), static_cast<int>(method), f.data.data(),
                                     mask.known.data(), f.width, f.height, f.channels, &o,
                                     reference ? reference->data.data() : nullptr,
                                     res.image.data.data(), &rep, &detail::trace_sink,
                                     &res.trace));
  res.report = detail::to_report(rep);
  return res;
}

// Many independent frames of one shape (the CLI's inpaint over a list of
// files, main.cpp:101) through si_run_method_batch: each frame's upload and
// the previous frame's result copy overlap the current solve, and the outer
// iterations are decided on the device.  Same results as run_method per
// frame; no trace rows (the batch entry has no trace sink).
inline std::vector<SolveResult> run_batch(
    Method method, const std::vector<std::pair<const ImageBuffer*, const InpaintingMask*>>& frames,
    const RunOptions& options, Context& ctx = Context::thread_default()) {
  std::vector<SolveResult> res(frames.size());
  if (frames.empty()) return res;
  const ImageBuffer& f0 = *frames[0].first;
  std::vector<const double*> fp;
  std::vector<const uint8_t*> mp;
  std::vector<double*> op;
  for (size_t k = 0; k < frames.size(); ++k) {
    const ImageBuffer& f = *frames[k].first;
    const InpaintingMask& m = *frames[k].second;
    detail::check_arg(f.width == m.width && f.height == m.height,
                      "image and mask dimensions differ");
    detail::check_arg(f.width == f0.width && f.height == f0.height && f.channels == f0.channels,
                      "run_batch: frames must share one shape");
    res[k].image = ImageBuffer(f.width, f.height, f.channels);
    fp.push_back(f.data.data());
    mp.push_back(m.known.data());
    op.push_back(res[k].image.data.data());
  }
  std::vector<si_report> reps(frames.size());
  const si_options o = options.to_c();
  detail::throw_status(si_run_method_batch(ctx.get(), static_cast<int>(method),
                                           static_cast<int>(frames.size()), fp.data(), mp.data(),
                                           f0.width, f0.height, f0.channels, &o, op.data(),
                                           reps.data()));
  for (size_t k = 0; k < frames.size(); ++k) res[k].report = detail::to_report(reps[k]);
  return res;
}

// partition_domain (partition.hpp:67-106).
inline SubdomainPartition partition_domain(int w, int h, int block, int overlap) {
  SubdomainPartition p;
  detail::throw_status(si_partition_domain(w, h, block, overlap, &p.blocks_x, &p.blocks_y,
                                           nullptr, 0));
  std::vector<int> r(8 * static_cast<size_t>(p.blocks_x) * p.blocks_y);
  detail::throw_status(si_partition_domain(w, h, block, overlap, &p.blocks_x, &p.blocks_y,
                                           r.data(), p.blocks_x * p.blocks_y));
  p.image_width = w;
  p.image_height = h;
  p.block_size = block;
  p.overlap = overlap;
  for (size_t i = 0; i < r.size(); i += 8)
    p.subdomains.push_back({r[i], r[i + 1], r[i + 2], r[i + 3], r[i + 4], r[i + 5], r[i + 6], r[i + 7]});
  return p;
}

inline ImageBuffer synthetic_test_image(int w, int h, int c, uint64_t seed) {
  ImageBuffer img(w, h, c);
  detail::throw_status(si_synthetic_test_image(w, h, c, seed, img.data.data()));
  return img;
}

inline InpaintingMask random_mask(int w, int h, double density, uint64_t seed) {
  InpaintingMask m(w, h);
  const si_status s = si_random_mask(w, h, density, seed, m.known.data());
  if (s != SI_OK) throw std::invalid_argument("random_mask: invalid dimensions or density");
  return m;
}

// VoronoiAssignment / assign_nearest_site (masks.hpp:45-139).
struct VoronoiAssignment {
  std::vector<std::int32_t> sites;    // known pixel indices, ascending
  std::vector<std::int32_t> site_of;  // pixel -> index into sites
};

inline VoronoiAssignment assign_nearest_site(const InpaintingMask& mask,
                                             Context& ctx = Context::thread_default()) {
  VoronoiAssignment a;
  const size_t n = static_cast<size_t>(mask.width) * mask.height;
  a.sites.resize(n);
  a.site_of.resize(n);
  int m = 0;
  detail::throw_status(si_assign_nearest_site(ctx.get(), mask.known.data(), mask.width,
                                              mask.height, a.sites.data(), a.site_of.data(), &m));
  a.sites.resize(static_cast<size_t>(m));
  return a;
}

// DensifyOptions / DensifyResult / voronoi_densify (masks.hpp:145-212).
struct DensifyOptions {
  double initial_density = 0.0;   // <= 0: start at a quarter of the target
  double cell_fraction = 0.20;    // share of cells refined per sweep
  double inner_tolerance = 1e-3;  // tolerance of the guiding inpainting runs
  int max_sweeps = 100;
  RunOptions solve;               // guide solver (multilevel ORAS); tolerance := inner_tolerance
};

struct DensifyResult {
  InpaintingMask mask;
  int sweeps = 0;
  bool reached_target = false;
};

inline DensifyResult voronoi_densify(const ImageBuffer& f, double target_density, uint64_t seed,
                                     const DensifyOptions& options = {},
                                     Context& ctx = Context::thread_default()) {
  si_densify_options d;
  si_default_densify_options(&d);
  d.initial_density = options.initial_density;
  d.cell_fraction = options.cell_fraction;
  d.inner_tolerance = options.inner_tolerance;
  d.max_sweeps = options.max_sweeps;
  d.solve = options.solve.to_c();
  DensifyResult r;
  r.mask = InpaintingMask(f.width, f.height);
  int reached = 0;
  detail::throw_status(si_voronoi_densify(ctx.get(), f.data.data(), f.width, f.height, f.channels,
                                          target_density, seed, &d, r.mask.known.data(),
                                          &r.sweeps, &reached));
  r.reached_target = reached != 0;
  return r;
}

inline double psnr(const ImageBuffer& u, const ImageBuffer& f) {
  detail::check_arg(u.width == f.width && u.height == f.height && u.channels == f.channels,
                    "mse_per_channel: image dimensions differ");
  double q = 0.0;
  detail::throw_status(si_psnr(u.data.data(), f.data.data(), u.width, u.height, u.channels, &q));
  return q;
}

}  // namespace schwarz_b200
