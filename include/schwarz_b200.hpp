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
//   * the lower seams: multilevel_solve + MultilevelSolveOptions /
//     LevelSolver (multilevel.hpp:130-310), solve_schwarz + SchwarzOptions /
//     SchwarzSolveOptions (schwarz.hpp:20-45, 325-389), run_schwarz_level +
//     LevelRunStats (schwarz.hpp:252-323), canonical_r0 (schwarz.hpp:333-345)
// Errors: SI_ERR_INVALID_ARGUMENT -> std::invalid_argument (same message the
// reference throws); other failures -> std::runtime_error.  Non-convergence
// is reported in SolveReport, never thrown.
// C++17 or later (the reference itself is C++20; under C++20 channel()
// returns std::span like image.hpp:44-52).  Link with libschwarz_b200.so.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <optional>
#include <type_traits>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>
#if __cplusplus >= 202002L && __has_include(<span>)
#include <span>
#define SCHWARZ_B200_HAS_SPAN 1
#endif

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

using ChannelVector = std::vector<double>;  // image.hpp:14

#ifdef SCHWARZ_B200_HAS_SPAN
template <typename T>
using Span = std::span<T>;
#else
// Minimal contiguous view for C++17 callers (std::span under C++20).
template <typename T>
struct Span {
  T* ptr = nullptr;
  std::size_t n = 0;
  Span(T* p, std::size_t count) : ptr(p), n(count) {}
  T* data() const { return ptr; }
  std::size_t size() const { return n; }
  T& operator[](std::size_t i) const { return ptr[i]; }
  T* begin() const { return ptr; }
  T* end() const { return ptr + n; }
};
#endif

// Planar image, channel c at [c*w*h, (c+1)*w*h) row-major (image.hpp:24-63).
struct ImageBuffer {
  int width = 0, height = 0, channels = 1;
  std::vector<double> data;
  ImageBuffer() = default;
  ImageBuffer(int w, int h, int ch, double fill = 0.0) : width(w), height(h), channels(ch) {
    detail::check_arg(w > 0 && h > 0 && ch > 0, "ImageBuffer: dimensions must be positive");
    data.assign(static_cast<size_t>(w) * h * ch, fill);
  }
  size_t pixel_count() const { return static_cast<size_t>(width) * height; }
  Span<double> channel(int c) {
    detail::check_arg(c >= 0 && c < channels, "ImageBuffer::channel: index out of range");
    return {data.data() + static_cast<size_t>(c) * pixel_count(), pixel_count()};
  }
  Span<const double> channel(int c) const {
    detail::check_arg(c >= 0 && c < channels, "ImageBuffer::channel: index out of range");
    return {data.data() + static_cast<size_t>(c) * pixel_count(), pixel_count()};
  }
  double& at(int x, int y, int c = 0) { return data[c * pixel_count() + static_cast<size_t>(y) * width + x]; }
  double at(int x, int y, int c = 0) const { return data[c * pixel_count() + static_cast<size_t>(y) * width + x]; }
};

// uint8 per pixel, nonzero = known (image.hpp:67-94).
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
  size_t known_count() const {
    size_t n = 0;
    for (uint8_t k : known) n += k != 0;
    return n;
  }
  double density() const {
    return size() == 0 ? 0.0 : static_cast<double>(known_count()) / static_cast<double>(size());
  }
};

// image.hpp:96-99
inline void require_same_grid(const ImageBuffer& image, const InpaintingMask& mask) {
  detail::check_arg(image.width == mask.width && image.height == mask.height,
                    "image and mask dimensions differ");
}

enum class Method { Cg = 0, MultilevelCg = 1, Ras = 2, Oras = 3, MultilevelOras = 4 };
enum class CoarseAveraging { KnownOnly = 0, AllPixels = 1 };
enum class ResidualNormalizer { InitialGuess = 0, RhsNorm = 1 };
enum class SchwarzFlavour { Ras = 0, Oras = 1 };   // schwarz.hpp:29
enum class LevelSolver { Cg, Ras, Oras };          // multilevel.hpp:130

// methods.hpp:15-40
inline const char* method_name(Method m) {
  switch (m) {
    case Method::Cg: return "cg";
    case Method::MultilevelCg: return "mlcg";
    case Method::Ras: return "ras";
    case Method::Oras: return "oras";
    case Method::MultilevelOras: return "mloras";
  }
  return "?";
}
inline Method parse_method(const std::string& name) {
  if (name == "cg") return Method::Cg;
  if (name == "mlcg") return Method::MultilevelCg;
  if (name == "ras") return Method::Ras;
  if (name == "oras") return Method::Oras;
  if (name == "mloras") return Method::MultilevelOras;
  throw std::invalid_argument("unknown method '" + name +
                              "' (expected cg, mlcg, ras, oras or mloras)");
}
inline bool is_multilevel(Method m) {
  return m == Method::MultilevelCg || m == Method::MultilevelOras;
}
enum class Precision { FP64 = 0, FP32 = 1, MIXED = 2 };  // MIXED: float local CG, double outer iteration

inline constexpr double kDefaultOrasAlpha = 0.25;

struct SolverConfig {
  double tolerance = 1e-6;
  int max_iterations = 10000;
  int residual_check_interval = 1;
};

// schwarz.hpp:38-45
struct SchwarzOptions {
  SchwarzFlavour flavour = SchwarzFlavour::Oras;
  double alpha = kDefaultOrasAlpha;
  SolverConfig local{1e-2, 30, 30};
  int max_outer_iterations = 1000;
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

// schwarz.hpp:325-329 (+ device precision)
struct SchwarzSolveOptions {
  SchwarzOptions schwarz;
  double tolerance = 1e-3;
  ResidualNormalizer normalizer = ResidualNormalizer::InitialGuess;
  Precision precision = Precision::FP64;
};

// multilevel.hpp:132-142 (+ device precision)
struct MultilevelSolveOptions {
  int levels = 3;
  double tolerance = 1e-3;         // finest level
  double coarse_tolerance = 1e-2;  // every level above the finest
  CoarseAveraging averaging = CoarseAveraging::KnownOnly;
  int block_size = 32;
  int overlap = 6;
  SchwarzOptions schwarz;              // flavour is overridden by the solver choice
  SolverConfig cg{1e-3, 100000, 4};    // tolerance field is overridden per level
  ResidualNormalizer normalizer = ResidualNormalizer::InitialGuess;
  Precision precision = Precision::FP64;
};

// run_schwarz_level's statistics (schwarz.hpp:254-260).
struct LevelRunStats {
  int iterations = 0;
  double final_rel = 0.0;
  bool converged = false;
  long long local_solves = 0;
  long long local_failures = 0;
};

struct TraceRow {
  int iteration = 0;
  double time_ms = 0.0;
  double rel_residual = 0.0;
  std::optional<double> psnr;
};

// metrics.hpp:67-97
struct ConvergenceTrace {
  static constexpr const char* kCsvHeader = "iter,time_ms,rel_residual,psnr";
  std::vector<TraceRow> rows;
  void append(int it, double ms, double rel, std::optional<double> q = std::nullopt) {
    rows.push_back({it, ms, rel, q});
  }
  void write_csv(std::ostream& os) const {
    os << kCsvHeader << '\n';
    char buf[160];
    for (const auto& row : rows) {
      std::snprintf(buf, sizeof buf, "%d,%.3f,%.9e", row.iteration, row.time_ms,
                    row.rel_residual);
      os << buf;
      if (row.psnr) {
        if (std::isinf(*row.psnr)) {
          os << ",inf";
        } else {
          std::snprintf(buf, sizeof buf, ",%.4f", *row.psnr);
          os << buf;
        }
      } else {
        os << ',';
      }
      os << '\n';
    }
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
  require_same_grid(f, mask);
  if (reference)  // mse_per_channel's check (metrics.hpp:30-35), before any copy
    detail::check_arg(reference->width == f.width && reference->height == f.height &&
                          reference->channels == f.channels,
                      "mse_per_channel: image dimensions differ");
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

// ---- one image over G ranks in horizontal stripes (configs[4]) ----
// A communicator of the ranks: NCCL (one process per GPU; rank 0 makes the id
// and the caller broadcasts it) or local (G ranks as threads of one process).
class StripeComm {
 public:
  using NcclId = std::array<unsigned char, SI_NCCL_ID_BYTES>;
  static NcclId nccl_unique_id() {
    NcclId id{};
    detail::throw_status(si_nccl_unique_id(id.data()));
    return id;
  }
  static StripeComm nccl(Context& ctx, int world, int rank, const NcclId& id) {
    si_stripe_comm* h = nullptr;
    detail::throw_status(si_stripe_comm_init_nccl(ctx.get(), world, rank, id.data(), &h));
    return StripeComm(h, world, rank);
  }
  // comms[r] for rank r, driven on contexts[r]
  static std::vector<StripeComm> local(const std::vector<Context*>& contexts) {
    const int world = static_cast<int>(contexts.size());
    std::vector<si_ctx*> ctxs;
    for (Context* c : contexts) ctxs.push_back(c->get());
    std::vector<si_stripe_comm*> hs(contexts.size(), nullptr);
    detail::throw_status(si_stripe_comm_init_local(ctxs.data(), world, hs.data()));
    std::vector<StripeComm> out;
    for (int r = 0; r < world; ++r) out.push_back(StripeComm(hs[r], world, r));
    return out;
  }
  StripeComm(StripeComm&& o) noexcept : h_(o.h_), world_(o.world_), rank_(o.rank_) {
    o.h_ = nullptr;
  }
  StripeComm& operator=(StripeComm&& o) noexcept {
    std::swap(h_, o.h_);
    world_ = o.world_;
    rank_ = o.rank_;
    return *this;
  }
  StripeComm(const StripeComm&) = delete;
  StripeComm& operator=(const StripeComm&) = delete;
  ~StripeComm() {
    if (h_) si_stripe_comm_destroy(h_);
  }
  // repeated solves issue their outer iterations without host round trips
  // (default on; every rank must agree)
  void set_speculation(bool on) { detail::throw_status(si_stripe_comm_set_speculation(h_, on)); }
  si_stripe_comm* get() const { return h_; }
  int world() const { return world_; }
  int rank() const { return rank_; }

 private:
  StripeComm(si_stripe_comm* h, int world, int rank) : h_(h), world_(world), rank_(rank) {}
  si_stripe_comm* h_ = nullptr;
  int world_ = 1, rank_ = 0;
};

// run_method over the ranks of `comm` (collective: every rank calls it with
// the full image).  The result image holds this rank's own finest rows
// (zeros elsewhere); the report and trace are the global ones.
inline SolveResult run_method_striped(Method method, const ImageBuffer& f,
                                      const InpaintingMask& mask, const RunOptions& options,
                                      StripeComm& comm, Context& ctx) {
  require_same_grid(f, mask);
  SolveResult res;
  res.image = ImageBuffer(f.width, f.height, f.channels);
  si_report rep;
  const si_options o = options.to_c();
  detail::throw_status(si_run_method_striped(ctx.get(), comm.get(), static_cast<int>(method),
                                             f.data.data(), mask.known.data(), f.width, f.height,
                                             f.channels, &o, res.image.data.data(), &rep,
                                             &detail::trace_sink, &res.trace));
  res.report = detail::to_report(rep);
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

// random_mask (masks.hpp:25-43), with the reference's checks and messages.
inline InpaintingMask random_mask(int w, int h, double density, uint64_t seed) {
  detail::check_arg(w > 0 && h > 0, "random_mask: dimensions must be positive");
  detail::check_arg(density > 0.0 && density <= 1.0, "random_mask: density must lie in (0, 1]");
  const size_t n = static_cast<size_t>(w) * h;
  detail::check_arg(std::llround(density * static_cast<double>(n)) >= 1,
                    "random_mask: density rounds to zero known pixels");
  InpaintingMask m(w, h);
  detail::throw_status(si_random_mask(w, h, density, seed, m.known.data()));
  return m;
}

// clamped_partition (multilevel.hpp:146-150).
inline SubdomainPartition clamped_partition(int w, int h, int block, int overlap) {
  const int be = std::min(block, std::min(w, h));
  const int oe = std::max(0, std::min(overlap, be - 1));
  return partition_domain(w, h, be, oe);
}

// multilevel_solve (multilevel.hpp:239-310).  LevelSolver::Ras on a pyramid
// runs the ORAS kernels with alpha = 1, whose Robin diagonal is exactly the
// RAS one (deg + 0 * cut, schwarz.hpp:12-15, 106-108).
inline SolveResult multilevel_solve(const ImageBuffer& f, const InpaintingMask& mask,
                                    LevelSolver solver, const MultilevelSolveOptions& options,
                                    const ImageBuffer* reference = nullptr,
                                    Context& ctx = Context::thread_default()) {
  RunOptions ro;
  ro.tolerance = options.tolerance;
  ro.levels = options.levels;
  ro.block_size = options.block_size;
  ro.overlap = options.overlap;
  ro.alpha = options.schwarz.alpha;
  ro.coarse_tolerance = options.coarse_tolerance;
  ro.averaging = options.averaging;
  ro.local = options.schwarz.local;
  ro.max_outer_iterations = options.schwarz.max_outer_iterations;
  ro.cg_max_iterations = options.cg.max_iterations;
  ro.cg_check_interval = options.cg.residual_check_interval;
  ro.normalizer = options.normalizer;
  ro.precision = options.precision;
  Method m = Method::MultilevelOras;
  if (solver == LevelSolver::Cg) {
    m = Method::MultilevelCg;
  } else if (solver == LevelSolver::Ras) {
    if (options.levels == 1) {
      m = Method::Ras;
    } else {
      ro.alpha = 1.0;
    }
  }
  return run_method(m, f, mask, ro, reference, ctx);
}

// solve_schwarz (schwarz.hpp:349-389): single level on an explicit partition.
inline SolveResult solve_schwarz(const ImageBuffer& f, const InpaintingMask& mask,
                                 const SubdomainPartition& partition,
                                 const SchwarzSolveOptions& options,
                                 const ImageBuffer* reference = nullptr,
                                 Context& ctx = Context::thread_default()) {
  require_same_grid(f, mask);
  if (reference)
    detail::check_arg(reference->width == f.width && reference->height == f.height &&
                          reference->channels == f.channels,
                      "mse_per_channel: image dimensions differ");
  RunOptions ro;
  ro.tolerance = options.tolerance;
  ro.levels = 1;
  ro.alpha = options.schwarz.alpha;
  ro.local = options.schwarz.local;
  ro.max_outer_iterations = options.schwarz.max_outer_iterations;
  ro.normalizer = options.normalizer;
  ro.precision = options.precision;
  const si_options o = ro.to_c();
  SolveResult res;
  res.image = ImageBuffer(f.width, f.height, f.channels);
  si_report rep;
  detail::throw_status(si_solve_schwarz(
      ctx.get(), f.data.data(), mask.known.data(), f.width, f.height, f.channels,
      partition.block_size, partition.overlap, static_cast<int>(options.schwarz.flavour), &o,
      reference ? reference->data.data() : nullptr, res.image.data.data(), &rep,
      &detail::trace_sink, &res.trace));
  res.report = detail::to_report(rep);
  return res;
}

// InpaintingOperator (operators.hpp:21-97), constructed from the mask as the
// reference does (InpaintingOperator op(mask)); the device applies it.
class InpaintingOperator {
 public:
  explicit InpaintingOperator(const InpaintingMask& mask) : mask_(&mask) {}
  int width() const { return mask_->width; }
  int height() const { return mask_->height; }
  const InpaintingMask& mask() const { return *mask_; }

 private:
  const InpaintingMask* mask_;
};

namespace detail {
// vector<ChannelVector> <-> planar buffer
inline std::vector<double> planar(const std::vector<ChannelVector>& v, size_t n) {
  std::vector<double> out;
  out.reserve(v.size() * n);
  for (const auto& c : v) {
    check_arg(c.size() == n, "run_schwarz_level: vector length mismatch");
    out.insert(out.end(), c.begin(), c.end());
  }
  return out;
}
template <class Sink>
void row_thunk(int it, double, double rel, double, void* user) {
  (*static_cast<Sink*>(user))(it, rel);
}
}  // namespace detail

// canonical_r0 (schwarz.hpp:333-345): ||b - A b|| (u0 = b) or ||b||.
inline double canonical_r0(const InpaintingOperator& op, const std::vector<ChannelVector>& b,
                           ResidualNormalizer normalizer,
                           Context& ctx = Context::thread_default()) {
  const size_t n = static_cast<size_t>(op.width()) * op.height();
  const std::vector<double> bp = detail::planar(b, n);
  double r0 = 0.0;
  detail::throw_status(si_canonical_r0(ctx.get(), op.mask().known.data(), op.width(),
                                       op.height(), static_cast<int>(b.size()), bp.data(),
                                       static_cast<int>(normalizer), &r0));
  return r0;
}

// run_schwarz_level (schwarz.hpp:266-323): the outer ORAS/RAS loop of one
// level, u updated in place; row(iteration, rel) is called for every outer
// iteration, iteration 0 included.
template <class RowSink>
LevelRunStats run_schwarz_level(const InpaintingOperator& op, const SubdomainPartition& part,
                                const std::vector<ChannelVector>& b,
                                std::vector<ChannelVector>& u, double r0_norm, double tolerance,
                                const SchwarzOptions& opt, RowSink&& row,
                                Context& ctx = Context::thread_default()) {
  detail::check_arg(part.image_width == op.width() && part.image_height == op.height(),
                    "run_schwarz_level: partition and operator dimensions differ");
  detail::check_arg(!b.empty() && b.size() == u.size(),
                    "run_schwarz_level: channel count mismatch");
  const size_t n = static_cast<size_t>(op.width()) * op.height();
  const std::vector<double> bp = detail::planar(b, n);
  std::vector<double> up = detail::planar(u, n);
  RunOptions ro;
  ro.alpha = opt.alpha;
  ro.local = opt.local;
  ro.max_outer_iterations = opt.max_outer_iterations;
  const si_options o = ro.to_c();
  si_report rep;
  using Sink = std::remove_reference_t<RowSink>;
  detail::throw_status(si_run_schwarz_level(
      ctx.get(), op.mask().known.data(), op.width(), op.height(), static_cast<int>(b.size()),
      bp.data(), up.data(), part.block_size, part.overlap, r0_norm, tolerance,
      static_cast<int>(opt.flavour), &o, &rep, &detail::row_thunk<Sink>,
      const_cast<void*>(static_cast<const void*>(&row))));
  for (size_t c = 0; c < u.size(); ++c)
    std::copy(up.begin() + static_cast<std::ptrdiff_t>(c * n),
              up.begin() + static_cast<std::ptrdiff_t>((c + 1) * n), u[c].begin());
  LevelRunStats st;
  st.iterations = rep.iterations;
  st.final_rel = rep.final_relative_residual;
  st.converged = rep.converged != 0;
  st.local_solves = rep.local_solves;
  st.local_failures = rep.local_failures;
  return st;
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
