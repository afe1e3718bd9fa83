// Host orchestration of the multilevel ORAS solver + the C ABI
// (include/schwarz_b200.h).  Everything below the ABI runs on the device:
// the pyramid (K5 ingest, K3 restrict), per level the residual norms (K1)
// and fused sweeps (K2), and the prolongation (K4).  The host only keeps the
// outer loop's scalar decisions (rel <= tol, outer >= max_outer), exactly as
// run_schwarz_level (schwarz.hpp:288-320) and multilevel_solve
// (multilevel.hpp:239-310) take them.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <type_traits>
#include <vector>
#include <functional>
#include <future>
#include <memory>

#include "../../include/schwarz_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "sweep.cuh"
#include "sweep_generic.cuh"
#include "cg_level.cuh"
#include "densify.cuh"
#include "host_copy.h"

#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost ~ns without a tool attached

using namespace sib;

namespace {

thread_local std::string g_last_error;

struct Failure {
  si_status status;
  std::string message;
};

[[noreturn]] void fail(si_status s, const std::string& msg) { throw Failure{s, msg}; }

void check_arg(bool ok, const std::string& msg) {
  if (!ok) fail(SI_ERR_INVALID_ARGUMENT, msg);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) fail(SI_ERR_OOM, std::string(what) + ": out of device memory");
  fail(SI_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(x) cuda_check((x), #x)

// NVTX range for the enclosing scope (solve, level, outer iteration, sweep):
// visible in Nsight Systems / ncu --nvtx timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, int a) {
    char buf[64];
    std::snprintf(buf, sizeof buf, fmt, a);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// ---------------------------------------------------------------- buffers
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  // returns true when (re)allocated; the new memory is zero-filled
  bool ensure(size_t want) {
    if (want <= bytes) return false;
    release();
    CK(cudaMalloc(&ptr, want));
    // cudaMemset runs on the legacy stream, which does not order against the
    // non-blocking solve streams: finish it before any of them can write here
    // (else a late zero-fill can overwrite an upload or a kernel's output)
    CK(cudaMemset(ptr, 0, want));
    CK(cudaStreamSynchronize(cudaStreamLegacy));
    bytes = want;
    return true;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

struct LevelBuf {
  DevBuf mask, b, u0, u1;
};

// Voronoi densification work arrays (masks.hpp:45-215).
struct VoronoiBufs {
  DevBuf f, mask, u, flag, rank, sites, bin_start, bin_cursor, members, site_of;
  DevBuf key, key2, pix, pix2, err, area, area2, seg, bits, bits2, worst, order, order2, tmp, small;
  void release() {
    for (DevBuf* b : {&f, &mask, &u, &flag, &rank, &sites, &bin_start, &bin_cursor, &members,
                      &site_of, &key, &key2, &pix, &pix2, &err, &area, &area2, &seg, &bits,
                      &bits2, &worst, &order, &order2, &tmp, &small})
      b->release();
  }
};

constexpr int kFlavourCg = -1;  // level solver = multilevel CG (LevelSolver::Cg)

enum Kind {
  K_RESIDUAL = 0, K_SWEEP = 1, K_RESTRICT = 2, K_PROLONG = 3, K_INGEST = 4, K_METRIC = 5,
  K_VORONOI = 6
};

struct PendingEvent {
  int kind;
  double bytes;
  cudaEvent_t start, stop;
};

}  // namespace

// A batch frame whose device-driven levels are queued but not yet read back.
struct GraphCounts {
  long long fixed, per_sweep;  // kernels per level-graph launch / per sweep
};
struct PendingFrame {
  bool active = false;
  int slot = 0, depth = 0, fixed_block = -1;
  bool known_checked = false;
  int graph_level[SI_MAX_LEVELS] = {};
  GraphCounts counts[SI_MAX_LEVELS] = {};
  long long blocks[SI_MAX_LEVELS] = {};
  si_report* rep = nullptr;
};
constexpr int kFrameWords = SI_MAX_LEVELS * 4 + 4;  // LevelStates + counters

struct si_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  std::vector<LevelBuf> levels;
  DevBuf in_f, in_mask, in_ref, out_img, aux;   // host-API staging
  DevBuf red_partials, red_out, counters, scratch;
  DevBuf cg_rhs, cg_x, cg_r, cg_p, cg_q;        // multilevel-CG level vectors
  DevBuf ticket;
  // Scalars cross PCIe through mapped (zero-copy) pinned memory written by
  // the kernels themselves: no copy-engine transfer that could queue behind a
  // batch's 200 MB image copies on the same engine.
  double* host_red = nullptr;                   // mapped host memory
  double* dev_red = nullptr;                    // device alias of host_red
  size_t host_red_cap = 0;                      // doubles in host_red
  unsigned long long* host_cnt = nullptr;       // mapped host memory
  unsigned long long* dev_cnt = nullptr;        // device alias of host_cnt
  int profiling = 0;
  std::vector<PendingEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  si_kernel_stats stats{};
  int sweep_nw64 = 2, sweep_nw32 = 2;           // warps per sweep CTA (measured best)
  long long launch_count = 0;                   // kernels launched (always counted)
  int local_fp32 = 0;                           // MIXED precision: float local CG (set per call)
  // batch pipeline: two staging slots, one stream per copy direction
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  DevBuf slot_f[2], slot_mask[2], slot_out[2];
  VoronoiBufs vz;                               // densification
  std::unique_ptr<sib::Stager> stager;          // pageable host <-> device copies
  std::unique_ptr<sib::Stager> drain_stager;    // batch: pageable result copies (helper thread)
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_solved[2] = {nullptr, nullptr},
              ev_d2h[2] = {nullptr, nullptr};
  // known-sample upload of the batch entry (host_copy.h): pinned packs
  // [tile offsets | values] per slot, packed by pack_pool
  std::unique_ptr<sib::CopyPool> pack_pool;
  void* pack_buf[2] = {nullptr, nullptr};
  size_t pack_cap[2] = {0, 0};
  // device-driven outer iterations (batch entry): one cached CUDA graph per
  // level geometry and buffer set, conditional WHILE/IF nodes around the sweeps
  struct LevelGraph {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
    long long fixed = 0, per_sweep = 0;  // kernels per launch / per sweep
    unsigned long long stamp = 0;
  };
  std::vector<LevelGraph> graphs;
  unsigned long long graph_clock = 0;
  int graph_mode = 0;
  si_report batch_scratch_report[2];            // batch frames without a caller report
  int counters_fresh = 0;                       // host_cnt current (graph-mode frame)
  cudaStream_t cap_stream[2] = {nullptr, nullptr};
  DevBuf lvl_state, lvl_sums;
  // striped solves (stripes.cuh): per-level storage rows, comm scratch
  std::vector<LevelBuf> stripe_levels;
  DevBuf stripe_send, stripe_recv, stripe_in_f, stripe_in_mask, stripe_out;
  DevBuf stripe_state;                          // StripeState per level + counter snapshots
  void* stripe_host = nullptr;                  // mapped mirror of the StripeStates
  void* stripe_hdev = nullptr;                  // device alias of stripe_host
  const void* stripe_result = nullptr;          // finest own rows of the last striped solve
  size_t stripe_result_stride = 0;              // elements between channel planes
  int stripe_result_rows = 0, stripe_result_f64 = 0;
  void* stripe_log = nullptr;                   // mapped: finest-level trace rows
  size_t stripe_log_cap = 0;
  unsigned long long* host_state = nullptr;     // mapped: LevelState[SI_MAX_LEVELS]
  unsigned long long* dev_state = nullptr;      // device alias of host_state
  // batch pipelining: a graph-mode frame's outcome lands in frame_host[slot]
  // and is read while the next frame is already queued
  struct PendingFrame* defer_to = nullptr;
  unsigned long long* frame_host[2] = {nullptr, nullptr};  // mapped
  unsigned long long* frame_dev[2] = {nullptr, nullptr};
  cudaEvent_t frame_done[2] = {nullptr, nullptr};
};

namespace {

struct Ctx {
  si_ctx& c;
  cudaStream_t s;
};

cudaEvent_t take_event(si_ctx& c) {
  if (!c.event_pool.empty()) {
    cudaEvent_t e = c.event_pool.back();
    c.event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

// Brackets one kernel launch with CUDA events on the launching stream when
// profiling is enabled; resolved after the next synchronisation.
struct Timed {
  Ctx& x;
  int kind;
  double bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  Timed(Ctx& x_, int k, double by) : x(x_), kind(k), bytes(by) {
    if (x.c.profiling) {
      a = take_event(x.c);
      b = take_event(x.c);
      CK(cudaEventRecord(a, x.s));
    }
  }
  ~Timed() noexcept(false) {
    if (a) {
      CK(cudaEventRecord(b, x.s));
      x.c.pending.push_back({kind, bytes, a, b});
    }
  }
};

void resolve_events(si_ctx& c) {
  for (auto& p : c.pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.stop) == cudaSuccess && cudaEventElapsedTime(&ms, p.start, p.stop) == cudaSuccess) {
      c.stats.launches[p.kind] += 1;
      c.stats.device_ms[p.kind] += ms;
      c.stats.algorithmic_bytes[p.kind] += p.bytes;
    }
    c.event_pool.push_back(p.start);
    c.event_pool.push_back(p.stop);
  }
  c.pending.clear();
}

void sync(Ctx& x) {
  CK(cudaStreamSynchronize(x.s));
  if (!x.c.pending.empty()) resolve_events(x.c);
}

// Caller host buffers (pageable or pinned) <-> device, see host_copy.h.
sib::Stager& stager(si_ctx& c) {
  if (!c.stager)
    c.stager = std::make_unique<sib::Stager>([](cudaError_t e, const char* what) {
      cuda_check(e, what);
    });
  return *c.stager;
}
void h2d(Ctx& x, void* dst, const void* src, size_t n) { stager(x.c).h2d(dst, src, n, x.s); }
// returns with the data in dst (everything queued on x.s before has finished)
void d2h(Ctx& x, void* dst, const void* src, size_t n) {
  stager(x.c).d2h(dst, src, n, x.s);
  if (!x.c.pending.empty()) resolve_events(x.c);
}

int grid_for(size_t n, int threads, int cap) {
  size_t g = (n + threads - 1) / threads;
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(g, cap)));
}

// ---------------------------------------------------------------- launches
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// SI_NO_INGEST_FUSION=1: separate K5 ingest and K3 restriction (A/B).
bool ingest_fusion_disabled() {
  static const bool off = std::getenv("SI_NO_INGEST_FUSION") != nullptr;
  return off;
}

// SI_NO_PAIR_DERIVE=1: the pair pass reads b instead of deriving it (A/B).
bool pair_derive_disabled() {
  static const bool off = std::getenv("SI_NO_PAIR_DERIVE") != nullptr;
  return off;
}

// SI_NO_TMA=1 forces the cooperative / cp.async staging paths (A/B runs).
bool tma_disabled() {
  static const bool off = std::getenv("SI_NO_TMA") != nullptr;
  return off;
}

// 3-D map over a planar [C][H][W] buffer with a (box_w, box_h, 1) box; false
// when TMA cannot address it (row pitch or base not 16-byte aligned).
bool make_plane_map(CUtensorMap* m, const void* base, int W, int H, int C, int elem, int box_w,
                    int box_h) {
  auto enc = tensor_map_encoder();
  if (!enc || (static_cast<size_t>(W) * elem) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(base) % 16 != 0 || (box_w * elem) % 16 != 0 || box_w > 256 ||
      box_h > 256)
    return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(C)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(W) * elem,
                                 static_cast<cuuint64_t>(W) * H * elem};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D u8 map over a [H][W] mask with a (box_w, box_h) box.
bool make_mask_map(CUtensorMap* m, const void* base, int W, int H, int box_w, int box_h) {
  auto enc = tensor_map_encoder();
  if (!enc || tma_disabled() || W % 16 != 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0 ||
      box_w % 16 != 0 || box_w > 256 || box_h > 256)
    return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(W)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Kernel launch with programmatic stream serialization (PDL, see pdl_wait in
// common.cuh): the kernel must pdl_wait() before touching its predecessor's
// data.  SI_NO_PDL=1 launches normally (the waits are then no-ops).
bool pdl_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("SI_NO_PDL");
    return e && e[0] == '1';
  }();
  return off;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_disabled() ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// Stripe storage (srow_lo/srow_hi, see SweepArgs): mask/u/b hold image rows
// [srow_lo, srow_hi) and are pre-offset by -srow_lo rows; whole image: 0, H.
template <typename T>
void launch_residual(Ctx& x, const uint8_t* mask, const T* u, const T* b, int W, int H, int C,
                     int mode, double* out, bool known_invariant = true, int row0 = 0,
                     int row1 = -1, int srow_lo = 0, int srow_hi = -1,
                     const int* skip = nullptr) {
  if (row1 < 0) row1 = H;
  if (srow_hi < 0) srow_hi = H;
  const int HS = srow_hi - srow_lo;
  const size_t N = static_cast<size_t>(W) * HS;
  const size_t off = static_cast<size_t>(srow_lo) * W;  // storage start = pointer + off
  const int rows = std::max(1, row1 - row0);
  const int gx = (W + kRedThreads - 1) / kRedThreads;
  const int gy = (rows + kResBand - 1) / kResBand;
  x.c.red_partials.ensure(sizeof(double) * static_cast<size_t>(gx) * gy * C);
  x.c.ticket.ensure(sizeof(unsigned int) * 4);
  // algorithmic bytes: u (or b) once per pixel per channel + the mask
  Timed t(x, K_RESIDUAL,
          static_cast<double>(W) * std::max(0, row1 - row0) * (C * sizeof(T) + (mode == 1 ? 0 : 1)));
  CUtensorMap map;
  if (mode != 1 && !tma_disabled() &&
      make_plane_map(&map, u + off, W, HS, C, sizeof(T), res_tma_box_w<T>(), kResTmaBand + 2)) {
    const int tx = (W + kResTmaThreads - 1) / kResTmaThreads;
    const int gy = (rows + kResTmaBand - 1) / kResTmaBand;
    x.c.red_partials.ensure(sizeof(double) * static_cast<size_t>(tx) * gy * C);
    // the mask band rides on the same barrier when its rows are 16-byte aligned
    CUtensorMap mmap{};
    const bool mtma = make_mask_map(&mmap, mask + off, W, HS, kResTmaThreads, kResTmaBand);
    auto launch = [&](auto inv, auto mt) {
      constexpr bool INV = decltype(inv)::value, MT = decltype(mt)::value;
      ++x.c.launch_count;
      launch_pdl(residual_sumsq_tma_kernel<T, INV, MT>, dim3(tx, gy, C), kResTmaThreads, x.s,
                 map, mmap, mask, b, W, H, N, row0, row1, srow_lo, x.c.red_partials.as<double>(),
                 skip);
    };
    if (known_invariant) {
      if (mtma) launch(std::true_type{}, std::true_type{});
      else launch(std::true_type{}, std::false_type{});
    } else {
      if (mtma) launch(std::false_type{}, std::true_type{});
      else launch(std::false_type{}, std::false_type{});
    }
    CK(cudaGetLastError());
    ++x.c.launch_count;
    launch_pdl(finish_partials_kernel, dim3(C), kRedThreads, x.s,
               static_cast<const double*>(x.c.red_partials.as<double>()), tx * gy, out);
  } else if (known_invariant) {
    ++x.c.launch_count;
    residual_sumsq_kernel<T, true><<<dim3(gx, gy, C), kRedThreads, 0, x.s>>>(
        mask, u, b, W, H, N, mode, row0, row1, srow_lo, srow_hi, x.c.red_partials.as<double>(),
        out, x.c.ticket.as<unsigned int>(), skip);
  } else {
    ++x.c.launch_count;
    residual_sumsq_kernel<T, false><<<dim3(gx, gy, C), kRedThreads, 0, x.s>>>(
        mask, u, b, W, H, N, mode, row0, row1, srow_lo, srow_hi, x.c.red_partials.as<double>(),
        out, x.c.ticket.as<unsigned int>(), skip);
  }
  CK(cudaGetLastError());
}

// launch_residual_pair derives b from u on these buffers (whole level).
template <typename T>
bool pair_derivable(const uint8_t* mask, const T* u, int W, int H, int C) {
  CUtensorMap umap, mmap;
  return !pair_derive_disabled() && !tma_disabled() &&
         make_plane_map(&umap, u, W, H, C, sizeof(T), res_tma_box_w<T>(), kResPairBand + 2) &&
         make_mask_map(&mmap, mask, W, H, kResTmaThreads + 32, kResPairBand + 2);
}

// The start of a level: sums of u0 -> out[0..C) and canonical_r0's sums of
// u = b -> out[C..2C) (normalizer InitialGuess, multilevel invariant), in one
// K1 pass when TMA can address the buffers, else as two K1 launches.
template <typename T>
void launch_residual_pair(Ctx& x, const uint8_t* mask, const T* u, const T* b, int W, int H,
                          int C, double* out, int row0 = 0, int row1 = -1, int srow_lo = 0,
                          int srow_hi = -1) {
  if (row1 < 0) row1 = H;
  if (srow_hi < 0) srow_hi = H;
  const int HS = srow_hi - srow_lo;
  const size_t off = static_cast<size_t>(srow_lo) * W;
  CUtensorMap umap, bmap, mmap{};
  // b derived from u (every caller runs the pair on a level's start iterate
  // after prolongation + snap: u = b at known pixels, b = 0 elsewhere)
  if (!pair_derive_disabled() && !tma_disabled() &&
      make_plane_map(&umap, u + off, W, HS, C, sizeof(T), res_tma_box_w<T>(), kResPairBand + 2) &&
      make_mask_map(&mmap, mask + off, W, HS, kResTmaThreads + 32, kResPairBand + 2)) {
    const int rows = std::max(1, row1 - row0);
    const int tx = (W + kResTmaThreads - 1) / kResTmaThreads;
    const int gy = (rows + kResPairBand - 1) / kResPairBand;
    x.c.red_partials.ensure(sizeof(double) * static_cast<size_t>(tx) * gy * 2 * C);
    Timed t(x, K_RESIDUAL, static_cast<double>(W) * std::max(0, row1 - row0) * (C * sizeof(T) + 1));
    ++x.c.launch_count;
    launch_pdl(residual_pair_derived_kernel<T>, dim3(tx, gy, C), kResTmaThreads, x.s, umap, mmap,
               W, H, row0, row1, srow_lo, x.c.red_partials.as<double>());
    CK(cudaGetLastError());
    ++x.c.launch_count;
    launch_pdl(finish_partials_kernel, dim3(2 * C), kRedThreads, x.s,
               static_cast<const double*>(x.c.red_partials.as<double>()), tx * gy, out);
    CK(cudaGetLastError());
    return;
  }
  if (!tma_disabled() &&
      make_plane_map(&umap, u + off, W, HS, C, sizeof(T), res_tma_box_w<T>(), kResPairBand + 2) &&
      make_plane_map(&bmap, b + off, W, HS, C, sizeof(T), res_tma_box_w<T>(), kResPairBand + 2)) {
    const int rows = std::max(1, row1 - row0);
    const int tx = (W + kResTmaThreads - 1) / kResTmaThreads;
    const int gy = (rows + kResPairBand - 1) / kResPairBand;
    x.c.red_partials.ensure(sizeof(double) * static_cast<size_t>(tx) * gy * 2 * C);
    const bool mtma = make_mask_map(&mmap, mask + off, W, HS, kResTmaThreads, kResPairBand);
    Timed t(x, K_RESIDUAL,
            static_cast<double>(W) * std::max(0, row1 - row0) * (2.0 * C * sizeof(T) + 1));
    ++x.c.launch_count;
    if (mtma)
      launch_pdl(residual_pair_tma_kernel<T, true>, dim3(tx, gy, C), kResTmaThreads, x.s, umap,
                 bmap, mmap, mask, W, H, row0, row1, srow_lo, x.c.red_partials.as<double>());
    else
      launch_pdl(residual_pair_tma_kernel<T, false>, dim3(tx, gy, C), kResTmaThreads, x.s, umap,
                 bmap, mmap, mask, W, H, row0, row1, srow_lo, x.c.red_partials.as<double>());
    CK(cudaGetLastError());
    ++x.c.launch_count;
    launch_pdl(finish_partials_kernel, dim3(2 * C), kRedThreads, x.s,
               static_cast<const double*>(x.c.red_partials.as<double>()), tx * gy, out);
    CK(cudaGetLastError());
    return;
  }
  launch_residual<T>(x, mask, u, b, W, H, C, 0, out, true, row0, row1, srow_lo, srow_hi);
  launch_residual<T>(x, mask, b, b, W, H, C, 0, out + C, true, row0, row1, srow_lo, srow_hi);
}

template <typename T>
void launch_sq_error(Ctx& x, const T* u, const double* f, size_t N, int C, double* out) {
  const int g = grid_for(N, kRedThreads, kRedBlocksMax);
  x.c.red_partials.ensure(sizeof(double) * static_cast<size_t>(g) * C);
  x.c.ticket.ensure(sizeof(unsigned int) * 4);
  Timed t(x, K_METRIC, static_cast<double>(N) * C * (sizeof(T) + 8.0));
  ++x.c.launch_count;
  sq_error_kernel<T><<<dim3(g, C), kRedThreads, 0, x.s>>>(
      u, f, N, x.c.red_partials.as<double>(), out, x.c.ticket.as<unsigned int>());
  CK(cudaGetLastError());
}

// Coarse rows [cy_lo, cy_hi) (stripe mode; -1: all); fn / cn: storage planes
// of the pre-offset fine / coarse buffers (0: whole-image planes).
template <typename T>
void launch_restrict(Ctx& x, const uint8_t* fmask, const T* fval, int fw, int fh, int C,
                     int averaging, uint8_t* cmask, T* cval, int cy_lo = 0, int cy_hi = -1,
                     size_t fn = 0, size_t cn = 0) {
  const int cw = (fw + 1) / 2, ch = (fh + 1) / 2;
  if (cy_hi < 0) cy_hi = ch;
  if (fn == 0) fn = static_cast<size_t>(fw) * fh;
  if (cn == 0) cn = static_cast<size_t>(cw) * ch;
  if (cy_hi <= cy_lo) return;
  const dim3 grid((cw + 127) / 128, cy_hi - cy_lo);
  // the vector path needs 16-byte aligned fine rows and planes
  const bool vec = fw % 2 == 0 && fn % 2 == 0 && reinterpret_cast<uintptr_t>(fval) % 16 == 0;
  ++x.c.launch_count;
  if (vec)
    launch_pdl(restrict_kernel<T, true>, grid, 128, x.s, fmask, fval, fw, fh, C, averaging, cmask,
               cval, cy_lo, fn, cn);
  else
    launch_pdl(restrict_kernel<T, false>, grid, 128, x.s, fmask, fval, fw, fh, C, averaging, cmask,
               cval, cy_lo, fn, cn);
  CK(cudaGetLastError());
}

// Fine rows [fy_lo, fy_hi); coarse storage rows [cs_lo, cs_hi); fn / cn
// storage planes; fine storage starts at row fs_lo_arg (stripe mode;
// defaults: the whole image).
template <typename T>
void launch_prolong(Ctx& x, const T* coarse, int cw, int ch, int fw, int fh, int C,
                    const uint8_t* fmask, const T* fval, T* fine, int fy_lo = 0, int fy_hi = -1,
                    int cs_lo = 0, int cs_hi = -1, size_t fn = 0, size_t cn = 0,
                    int fs_lo_arg = 0) {
  if (fy_hi < 0) fy_hi = fh;
  if (cs_hi < 0) cs_hi = ch;
  if (fn == 0) fn = static_cast<size_t>(fw) * fh;
  if (cn == 0) cn = static_cast<size_t>(cw) * ch;
  if (fy_hi <= fy_lo) return;
  const int tiles_x = (fw + kProX - 1) / kProX, tiles_y = (fy_hi - fy_lo + kProY - 1) / kProY;
  CUtensorMap cmap;
  if (C <= kProMaxC && !tma_disabled() &&
      make_plane_map(&cmap, coarse + static_cast<size_t>(cs_lo) * cw, cw, cs_hi - cs_lo, C,
                     sizeof(T), pro_box_w<T>(), kProCY) &&
      reinterpret_cast<uintptr_t>(coarse + static_cast<size_t>(cs_lo) * cw) % 16 == 0 &&
      (cn * sizeof(T)) % 16 == 0) {
    // persistent CTAs (kProTmaOcc per SM), each walking tiles with a 2-stage TMA ring
    static int sms = [] {
      int d = 0, n = 148;
      if (cudaGetDevice(&d) == cudaSuccess)
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
      return n;
    }();
    const int ntiles = tiles_x * tiles_y;
    const int grid = std::min(ntiles, sms * kProTmaOcc);
    // the fine mask tile by TMA too when its rows are 16-byte aligned (the
    // map covers the fine storage rows [fs_lo, fs_lo + fn / fw))
    const int fs_lo = fs_lo_arg;
    CUtensorMap mmap{};
    const bool mt = fmask != nullptr &&
                    make_mask_map(&mmap, fmask + static_cast<size_t>(fs_lo) * fw, fw,
                                  static_cast<int>(fn / fw), kProX, kProY);
    ++x.c.launch_count;
    if (mt)
      launch_pdl(prolong_snap_tma_kernel<T, true>, dim3(grid), 256, x.s, cmap, mmap, cw, ch, fw, C,
                 fmask, fval, fine, fy_lo, fy_hi, cs_lo, fs_lo, fn, tiles_x, ntiles);
    else
      launch_pdl(prolong_snap_tma_kernel<T, false>, dim3(grid), 256, x.s, cmap, mmap, cw, ch, fw,
                 C, fmask, fval, fine, fy_lo, fy_hi, cs_lo, fs_lo, fn, tiles_x, ntiles);
    CK(cudaGetLastError());
    return;
  }
  const dim3 grid(tiles_x, tiles_y);
  ++x.c.launch_count;
  launch_pdl(prolong_snap_kernel<T>, grid, 256, x.s, coarse, cw, ch, fw, fh, C, fmask, fval, fine,
             fy_lo, fy_hi, cs_lo, cs_hi, fn, cn);
  CK(cudaGetLastError());
}

struct LocalCfg {
  double tol;
  int max_it;
  int check;
};

template <typename T, int NW>
void launch_sweep_nw(Ctx& x, const SweepArgs<T>& a, int nblocks, int C) {
  if (a.skip != nullptr) {  // stripes (speculative iterations): the 2-warp sweeps only
    if constexpr (NW == 2) {
      ++x.c.launch_count;
      const dim3 grid(nblocks, C);
      const bool full = a.ax.block == kMaxBlock;
      if constexpr (sizeof(T) == 8) {
        if (x.c.local_fp32) {
          if (full) oras_sweep_kernel<T, 2, true, float, true><<<grid, 64, 0, x.s>>>(a);
          else oras_sweep_kernel<T, 2, false, float, true><<<grid, 64, 0, x.s>>>(a);
          CK(cudaGetLastError());
          return;
        }
      }
      if (full) oras_sweep_kernel<T, 2, true, T, true><<<grid, 64, 0, x.s>>>(a);
      else oras_sweep_kernel<T, 2, false, T, true><<<grid, 64, 0, x.s>>>(a);
      CK(cudaGetLastError());
      return;
    } else {
      fail(SI_ERR_RUNTIME, "skippable sweeps need 2 warps per CTA");
    }
  }
  if constexpr (sizeof(T) == 8) {
    if (x.c.local_fp32) {  // MIXED: double image / outer iteration, float local CG
      ++x.c.launch_count;
      if (a.ax.block == kMaxBlock)
        oras_sweep_kernel<T, NW, true, float><<<dim3(nblocks, C), NW * 32, 0, x.s>>>(a);
      else
        oras_sweep_kernel<T, NW, false, float><<<dim3(nblocks, C), NW * 32, 0, x.s>>>(a);
      CK(cudaGetLastError());
      return;
    }
  }
  if (a.ax.block == kMaxBlock) {
    ++x.c.launch_count;
    oras_sweep_kernel<T, NW, true><<<dim3(nblocks, C), NW * 32, 0, x.s>>>(a);
  } else {
    ++x.c.launch_count;
    oras_sweep_kernel<T, NW, false><<<dim3(nblocks, C), NW * 32, 0, x.s>>>(a);
  }
  CK(cudaGetLastError());
}

template <typename T>
void launch_sweep(Ctx& x, const uint8_t* mask, const T* b, const T* u_old, T* u_new, int W, int H,
                  int C, int block, int overlap, int flavour, double alpha, const LocalCfg& lc,
                  bool known_invariant, unsigned long long* counters, int by0 = 0, int by1 = -1,
                  int srow_lo = 0, int srow_hi = -1, const int* skip = nullptr) {
  if (srow_hi < 0) srow_hi = H;
  SweepArgs<T> a{};
  a.skip = skip;
  a.srow_lo = srow_lo;
  a.srow_hi = srow_hi;
  a.mask = mask;
  a.b = b;
  a.u_old = u_old;
  a.u_new = u_new;
  a.W = W;
  a.H = H;
  a.N = static_cast<size_t>(W) * (srow_hi - srow_lo);
  a.ax = Axis::make(W, block, overlap);
  a.ay = Axis::make(H, block, overlap);
  a.am1 = static_cast<T>(alpha - 1.0);
  a.ras = flavour == SI_FLAVOUR_RAS;
  a.ltol = static_cast<T>(lc.tol);
  a.lmax = lc.max_it;
  a.lcheck = lc.check;
  a.known_invariant = known_invariant;
  a.counters = counters;
  if (by1 < 0) by1 = a.ay.count;
  a.by0 = by0;
  if (block > kMaxBlock) {  // K2g: blocks beyond 32x32, CG vectors in global scratch
    if (by1 <= by0) return;
    const double bytes = static_cast<double>(W) * H * (2.0 * C * sizeof(T) + 1.0) * (by1 - by0) /
                         a.ay.count;
    Timed t(x, K_SWEEP, bytes);
    const size_t per_row = sizeof(T) * 5 * static_cast<size_t>(block) * block * a.ax.count * C;
    const int rows = static_cast<int>(std::max<size_t>(1, (size_t(1) << 30) / per_row));
    x.c.scratch.ensure(per_row * std::min(rows, by1 - by0));
    a.scratch = x.c.scratch.as<T>();
    for (int r0 = by0; r0 < by1; r0 += rows) {
      a.by0 = r0;
      const int n = a.ax.count * (std::min(by1, r0 + rows) - r0);
      ++x.c.launch_count;
      oras_sweep_generic_kernel<T><<<dim3(n, C), kGenThreads, 0, x.s>>>(a);
      CK(cudaGetLastError());
    }
    return;
  }
  // TMA tile loads: the box starts at the 16-byte aligned column left of each
  // block (tile_lead), so any anchor works; the row pitch must be a multiple
  // of 16 bytes (checked by make_plane_map)
  a.use_tma = !tma_disabled() &&
              make_plane_map(&a.umap, u_old + static_cast<size_t>(srow_lo) * W, W,
                             srow_hi - srow_lo, C, sizeof(T), tile_w<T>(), kTileH);
  const int nblocks = a.ax.count * (by1 - by0);
  if (nblocks <= 0) return;
  const double bytes = static_cast<double>(W) * H * (2.0 * C * sizeof(T) + 1.0) * (by1 - by0) /
                       a.ay.count;
  Timed t(x, K_SWEEP, bytes);
  const int nw = sizeof(T) == 8 ? x.c.sweep_nw64 : x.c.sweep_nw32;
  if constexpr (sizeof(T) == 8) {
    if (nw == 2) launch_sweep_nw<T, 2>(x, a, nblocks, C);
    else launch_sweep_nw<T, 4>(x, a, nblocks, C);
  } else {
    if (nw == 1) launch_sweep_nw<T, 1>(x, a, nblocks, C);
    else if (nw == 2) launch_sweep_nw<T, 2>(x, a, nblocks, C);
    else launch_sweep_nw<T, 4>(x, a, nblocks, C);
  }
}

// MIXED precision for the duration of one ABI call.
struct LocalPrecision {
  si_ctx& c;
  LocalPrecision(si_ctx& ctx, int precision) : c(ctx) {
    c.local_fp32 = precision == SI_PRECISION_MIXED;
  }
  ~LocalPrecision() { c.local_fp32 = 0; }
};

// ---------------------------------------------------------------- options
void validate_options_common(const si_options& o) {
  check_arg(o.tolerance > 0.0 && o.coarse_tolerance > 0.0,
            "multilevel_solve: tolerances must be positive");
  check_arg(o.averaging == 0 || o.averaging == 1, "averaging must be KnownOnly or AllPixels");
  check_arg(o.normalizer == 0 || o.normalizer == 1, "normalizer must be InitialGuess or RhsNorm");
  check_arg(o.precision == SI_PRECISION_FP64 || o.precision == SI_PRECISION_FP32 ||
                o.precision == SI_PRECISION_MIXED,
            "precision must be FP64, FP32 or MIXED");
}

// cg_solve's validate_solver_config (cg.hpp:75-80), applied to the local
// configuration before the first sweep that runs local solves.
void validate_local(const si_options& o) {
  check_arg(o.local_tolerance > 0.0, "SolverConfig: tolerance must be positive");
  check_arg(o.local_max_iterations >= 0, "SolverConfig: max_iterations must be non-negative");
  check_arg(o.local_check_interval >= 1, "SolverConfig: residual_check_interval must be >= 1");
}

void validate_partition(int w, int h, int block, int overlap) {
  // partition_domain (partition.hpp:68-73)
  check_arg(w > 0 && h > 0, "partition_domain: image dimensions must be positive");
  check_arg(block > 0, "partition_domain: block_size must be positive");
  check_arg(overlap >= 0, "partition_domain: overlap must be non-negative");
  check_arg(overlap < block, "partition_domain: overlap must be smaller than block_size");
  check_arg(block <= w && block <= h, "partition_domain: block_size exceeds image dimensions");
}

struct Clamped {
  int block, overlap;
};

// clamped_partition (multilevel.hpp:146-150)
Clamped clamp_partition(int w, int h, int block, int overlap) {
  const int be = std::min(block, std::min(w, h));
  const int oe = std::max(0, std::min(overlap, be - 1));
  validate_partition(w, h, be, oe);
  return {be, oe};
}

double psnr_from_sq(const std::vector<double>& sq, size_t N) {
  // psnr (metrics.hpp:51-57): mean of per-channel MSE, +inf when identical
  double mean = 0.0;
  for (double s : sq) mean += s / static_cast<double>(N);
  mean /= static_cast<double>(sq.size());
  if (mean == 0.0) return std::numeric_limits<double>::infinity();
  return 10.0 * std::log10(255.0 * 255.0 / mean);
}

// ---------------------------------------------------------------- the solve
struct Trace {
  si_trace_fn fn;
  void* user;
  Clock::time_point t0;
};

struct LevelOutcome {
  int iterations = 0;
  double final_rel = 0.0;
  bool converged = false;
};

template <typename T>
struct LevelView {
  int w, h;
  const uint8_t* mask;
  const T* b;
  T* u[2];
  int cur;
};

// Per-channel sums -> joint norm with the reference's sqrt-then-square
// (schwarz.hpp:290-295; the accumulate is an fma in the gcc build).
double joint_norm(const double* sums, int C) {
  double joint = 0.0;
  for (int k = 0; k < C; ++k) {
    const double nrm = std::sqrt(sums[k]);
    joint = std::fma(nrm, nrm, joint);
  }
  return std::sqrt(joint);
}

// run_schwarz_level (schwarz.hpp:266-323) on device buffers.  When
// r0_slot_pending, the r0 reduction was already launched into host_red[C..2C)
// and is read at the first synchronisation.
// r0_mode (how the level's canonical r0 arrives at the first synchronisation):
enum R0Mode {
  kR0Launched = 0,  // already launched into host_red[C..2C) (launch_r0)
  kR0Pair = 1,      // launched together with the first residual (launch_residual_pair)
  kR0Same = 2       // u0 is a copy of b (the coarsest level): r0's sums are the first
                    // residual's, bit for bit, so nothing extra runs
};

template <typename T>
LevelOutcome run_level(Ctx& x, LevelView<T>& L, int C, int block, int overlap, double* r0,
                       bool r0_pending, double tol, int flavour, const si_options& o,
                       bool known_invariant, bool sink, const Trace& tr, const double* d_ref,
                       si_report* rep, int r0_mode = kR0Launched, bool check_known = false) {
  LevelOutcome out;
  const size_t N = static_cast<size_t>(L.w) * L.h;
  double* d_out = x.c.dev_red;  // mapped: results land in host_red
  unsigned long long* d_cnt = x.c.counters.as<unsigned long long>();
  bool local_checked = false;
  const Axis ax = Axis::make(L.w, block, overlap), ay = Axis::make(L.h, block, overlap);
  const long long nblocks = static_cast<long long>(ax.count) * ay.count;
  for (int outer = 0;; ++outer) {
    NvtxRange nv_outer("outer %d", outer);
    if (outer == 0 && r0_mode == kR0Pair)
      launch_residual_pair<T>(x, L.mask, L.u[L.cur], L.b, L.w, L.h, C, d_out);
    else
      launch_residual<T>(x, L.mask, L.u[L.cur], L.b, L.w, L.h, C, 0, d_out, known_invariant);
    if (sink && d_ref) launch_sq_error<T>(x, L.u[L.cur], d_ref, N, C, d_out + 2 * C);
    sync(x);
    if (check_known && outer == 0)  // deferred build_rhs check (multilevel_device)
      check_arg(x.c.host_cnt[2] > 0, "build_rhs: mask has no known pixels");
    if (r0_pending) {
      *r0 = joint_norm(x.c.host_red + (r0_mode == kR0Same ? 0 : C), C);
      r0_pending = false;
    }
    const double rel = *r0 > 0.0 ? joint_norm(x.c.host_red, C) / *r0 : 0.0;
    if (sink && tr.fn) {
      double q = std::numeric_limits<double>::quiet_NaN();
      if (d_ref) q = psnr_from_sq(std::vector<double>(x.c.host_red + 2 * C, x.c.host_red + 3 * C), N);
      tr.fn(outer, ms_since(tr.t0), rel, q, tr.user);
    }
    out.iterations = outer;
    out.final_rel = rel;
    if (rel <= tol) {
      out.converged = true;
      break;
    }
    if (outer >= o.max_outer_iterations) break;
    if (!local_checked) {
      validate_local(o);
      local_checked = true;
    }
    const LocalCfg lc{o.local_tolerance, o.local_max_iterations, o.local_check_interval};
    NvtxRange nv_sweep("sweep");
    launch_sweep<T>(x, L.mask, L.b, L.u[L.cur], L.u[L.cur ^ 1], L.w, L.h, C, block, overlap,
                    flavour, o.alpha, lc, known_invariant, d_cnt);
    L.cur ^= 1;
    rep->local_solves += nblocks * C;
  }
  return out;
}

template <typename T>
void launch_r0(Ctx& x, const LevelView<T>& L, int C, int normalizer) {
  // canonical_r0 (schwarz.hpp:333-345): residual of u0 = b, or ||b||.
  double* d_out = x.c.dev_red;
  launch_residual<T>(x, L.mask, L.b, L.b, L.w, L.h, C, normalizer == 1 ? 1 : 0, d_out + C);
}

__global__ void copy_u64_kernel(const unsigned long long* src, unsigned long long* dst, int n,
                                bool zero_src) {
  const int i = threadIdx.x;
  if (i < n) {
    if (dst) dst[i] = src[i];
    if (zero_src) const_cast<unsigned long long*>(src)[i] = 0ull;
  }
}

void begin_counters(Ctx& x) {
  x.c.counters_fresh = 0;
  x.c.counters.ensure(sizeof(unsigned long long) * 8);
  ++x.c.launch_count;
  copy_u64_kernel<<<1, 32, 0, x.s>>>(x.c.counters.as<unsigned long long>(), nullptr, 8, true);
  CK(cudaGetLastError());
}

// device counters -> mapped host memory, then wait
void publish_counters(Ctx& x, int n) {
  ++x.c.launch_count;
  copy_u64_kernel<<<1, 32, 0, x.s>>>(x.c.counters.as<unsigned long long>(), x.c.dev_cnt, n, false);
  CK(cudaGetLastError());
  sync(x);
}

void end_counters(Ctx& x, si_report* rep) {
  // a graph-mode frame published them with its level states, nothing ran since
  if (!x.c.counters_fresh) publish_counters(x, 2);
  x.c.counters_fresh = 0;
  rep->local_failures += static_cast<long long>(x.c.host_cnt[0]);
  rep->local_cg_iterations += static_cast<long long>(x.c.host_cnt[1]);
}

// Mapped scalar slots for 4 values per channel (sums, r0, CG dots, PSNR).
void ensure_red(si_ctx& c, int C) {
  const size_t want = 4 * static_cast<size_t>(std::max(C, 1));
  if (c.host_red && c.host_red_cap >= want) return;
  if (c.host_red) {
    CK(cudaDeviceSynchronize());  // no kernel may still write the old slots
    CK(cudaFreeHost(c.host_red));
    c.host_red = nullptr;
  }
  const size_t cap = std::max<size_t>(want, 256);
  CK(cudaHostAlloc(&c.host_red, sizeof(double) * cap, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.dev_red), c.host_red, 0));
  c.host_red_cap = cap;
}

void prepare_red(Ctx& x, int C) {
  x.c.red_out.ensure(sizeof(double) * 4 * C);
  ensure_red(x.c, C);
}

// Diagnostics as multilevel_solve writes them (multilevel.hpp:284-293).
void write_diagnostic(si_report* rep, int depth, int fixed_block) {
  bool coarse_capped = false;
  for (int l = 1; l < depth; ++l) coarse_capped |= !rep->level_converged[l];
  if (!rep->converged)
    std::snprintf(rep->diagnostic, sizeof rep->diagnostic, "%s",
                  fixed_block >= 0 ? "schwarz: outer iteration cap reached"
                                   : "multilevel: finest level did not converge");
  else if (coarse_capped)
    std::snprintf(rep->diagnostic, sizeof rep->diagnostic, "%s",
                  "multilevel: a coarse level hit its iteration cap");
}

// Completes a deferred batch frame: waits for its publish, fills the report
// exactly as the synchronous path does.
void finish_frame(si_ctx& c, PendingFrame& P) {
  if (!P.active) return;
  P.active = false;
  CK(cudaEventSynchronize(c.frame_done[P.slot]));
  const unsigned long long* w = c.frame_host[P.slot];
  const unsigned long long* cnt = w + SI_MAX_LEVELS * 4;
  if (!P.known_checked) check_arg(cnt[2] > 0, "build_rhs: mask has no known pixels");
  si_report* rep = P.rep;
  const LevelState* hs = reinterpret_cast<const LevelState*>(w);
  for (int l = 0; l < P.depth; ++l) {
    const LevelState& S = hs[l];
    rep->level_iterations[l] = S.iterations;
    rep->level_final_rel[l] = S.final_rel;
    rep->level_converged[l] = S.converged != 0;
    rep->local_solves += static_cast<long long>(S.outer) * P.blocks[l];
    c.launch_count += P.counts[l].fixed + P.counts[l].per_sweep * S.outer;
    if (l == 0) {
      rep->iterations = S.iterations;
      rep->final_relative_residual = S.final_rel;
      rep->converged = S.converged != 0;
    }
  }
  rep->local_failures += static_cast<long long>(cnt[0]);
  rep->local_cg_iterations += static_cast<long long>(cnt[1]);
  write_diagnostic(rep, P.depth, P.fixed_block);
}

// ---- device-driven level (graph mode) ---------------------------------------
// Adds a conditional node at the capture point of stream s; returns its body.
cudaGraph_t add_conditional(cudaStream_t s, cudaGraphConditionalHandle h,
                            cudaGraphConditionalNodeType type) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &p));
  CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  return p.conditional.phGraph_out[0];
}

cudaGraph_t capturing_graph(cudaStream_t s) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, nullptr, nullptr));
  return g;
}

// Graph mode applies when nothing needs the host between outer iterations:
// Schwarz levels without trace sink, reference image or kernel profiling,
// K2 blocks, valid local options (validated up front; the host loop checks
// them only before a sweep, so invalid ones take the host path).
bool graph_eligible(const Ctx& x, const si_options& o, const Trace& tr, const double* d_ref,
                    int flavour, int block) {
  if (!x.c.graph_mode || tr.fn || d_ref || x.c.profiling) return false;
  if (flavour == kFlavourCg || block > kMaxBlock) return false;
  return o.local_tolerance > 0.0 && o.local_max_iterations >= 0 && o.local_check_interval >= 1;
}

// One level's outer iteration as a cached graph:
//   r0 residual, residual(u0), decide -> WHILE { sweep u0->u1, residual(u1),
//   decide -> IF { sweep u1->u0, residual(u0), decide } }, parity fixup.
// Launched on x.s without any host synchronisation; the LevelState slot
// `level` holds the outcome.  Returns the cache entry (launch counts).
template <typename T>
GraphCounts launch_level_graph(Ctx& x, LevelView<T>& L, int C, int level, int block,
                                             int overlap, double tol, int flavour,
                                             const si_options& o, bool coarsest) {
  si_ctx& c = x.c;
  LevelState* st = c.lvl_state.as<LevelState>() + level;
  double* sums = c.lvl_sums.as<double>() + static_cast<size_t>(level) * 2 * C;
  double* r0s = sums + C;
  // every buffer the captured kernels touch must stay put: size the shared
  // partials for this level first (launch_residual never grows it then)
  const size_t parts = static_cast<size_t>((L.w + kResTmaThreads - 1) / kResTmaThreads + 1) *
                       ((L.h + kResBand - 1) / kResBand + 1) * 2 * C;  // x2: the pair pass
  c.red_partials.ensure(sizeof(double) * parts);
  c.ticket.ensure(sizeof(unsigned int) * 4);
  const double alpha = o.alpha;
  uint64_t a_bits, t_bits, lt_bits;
  std::memcpy(&a_bits, &alpha, 8);
  std::memcpy(&t_bits, &tol, 8);
  std::memcpy(&lt_bits, &o.local_tolerance, 8);
  std::vector<uint64_t> key = {
      sizeof(T), static_cast<uint64_t>(c.local_fp32), static_cast<uint64_t>(L.w),
      static_cast<uint64_t>(L.h), static_cast<uint64_t>(C), static_cast<uint64_t>(level),
      static_cast<uint64_t>(block), static_cast<uint64_t>(overlap),
      static_cast<uint64_t>(flavour), a_bits, t_bits, lt_bits,
      static_cast<uint64_t>(o.local_max_iterations), static_cast<uint64_t>(o.local_check_interval),
      static_cast<uint64_t>(o.max_outer_iterations), static_cast<uint64_t>(o.normalizer),
      reinterpret_cast<uint64_t>(L.mask), reinterpret_cast<uint64_t>(L.b),
      reinterpret_cast<uint64_t>(L.u[0]), reinterpret_cast<uint64_t>(L.u[1]),
      reinterpret_cast<uint64_t>(st), reinterpret_cast<uint64_t>(sums),
      reinterpret_cast<uint64_t>(c.red_partials.ptr), reinterpret_cast<uint64_t>(c.ticket.ptr),
      reinterpret_cast<uint64_t>(c.counters.ptr), static_cast<uint64_t>(tma_disabled()),
      static_cast<uint64_t>(sizeof(T) == 8 ? c.sweep_nw64 : c.sweep_nw32),
      static_cast<uint64_t>(coarsest)};
  for (auto& g : c.graphs)
    if (g.key == key) {
      g.stamp = ++c.graph_clock;
      CK(cudaGraphLaunch(g.exec, x.s));
      return {g.fixed, g.per_sweep};
    }
  for (cudaStream_t& cs : c.cap_stream)
    if (!cs) CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  const LocalCfg lc{o.local_tolerance, o.local_max_iterations, o.local_check_interval};
  const size_t n = static_cast<size_t>(L.w) * L.h * C;
  const long long lc_before = c.launch_count;
  unsigned long long* cnt = c.counters.as<unsigned long long>();
  CK(cudaStreamBeginCapture(x.s, cudaStreamCaptureModeThreadLocal));
  // canonical r0 and the first residual (see R0Mode): one pair pass, or on
  // the coarsest level (u0 = b) one pass whose sums are both
  const double* first_r0 = r0s;
  if (o.normalizer == 1) {
    launch_residual<T>(x, L.mask, L.b, L.b, L.w, L.h, C, 1, r0s);
    launch_residual<T>(x, L.mask, L.u[0], L.b, L.w, L.h, C, 0, sums, true);
  } else if (coarsest) {
    launch_residual<T>(x, L.mask, L.u[0], L.b, L.w, L.h, C, 0, sums, true);
    first_r0 = sums;
  } else {
    launch_residual_pair<T>(x, L.mask, L.u[0], L.b, L.w, L.h, C, sums);  // r0s = sums + C
  }
  cudaGraphConditionalHandle hw;
  CK(cudaGraphConditionalHandleCreate(&hw, capturing_graph(x.s), 0, cudaGraphCondAssignDefault));
  ++c.launch_count;
  level_decide_kernel<<<1, 32, 0, x.s>>>(sums, first_r0, C, tol, o.max_outer_iterations, st, hw,
                                         0, 1, 0);
  CK(cudaGetLastError());
  const long long lc_loop = c.launch_count;
  {
    cudaGraph_t body = add_conditional(x.s, hw, cudaGraphCondTypeWhile);
    Ctx xb{c, c.cap_stream[0]};
    CK(cudaStreamBeginCaptureToGraph(xb.s, body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    cudaGraphConditionalHandle hi;
    CK(cudaGraphConditionalHandleCreate(&hi, body, 0, 0));
    launch_sweep<T>(xb, L.mask, L.b, L.u[0], L.u[1], L.w, L.h, C, block, overlap, flavour, alpha,
                    lc, true, cnt);
    launch_residual<T>(xb, L.mask, L.u[1], L.b, L.w, L.h, C, 0, sums, true);
    ++c.launch_count;
    level_decide_kernel<<<1, 32, 0, xb.s>>>(sums, r0s, C, tol, o.max_outer_iterations, st, hw,
                                            hi, 0, 1);
    CK(cudaGetLastError());
    {
      cudaGraph_t body2 = add_conditional(xb.s, hi, cudaGraphCondTypeIf);
      Ctx xc{c, c.cap_stream[1]};
      CK(cudaStreamBeginCaptureToGraph(xc.s, body2, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
      launch_sweep<T>(xc, L.mask, L.b, L.u[1], L.u[0], L.w, L.h, C, block, overlap, flavour,
                      alpha, lc, true, cnt);
      launch_residual<T>(xc, L.mask, L.u[0], L.b, L.w, L.h, C, 0, sums, true);
      ++c.launch_count;
      level_decide_kernel<<<1, 32, 0, xc.s>>>(sums, r0s, C, tol, o.max_outer_iterations, st, hw,
                                              0, 0, 0);
      CK(cudaGetLastError());
      cudaGraph_t tmp;
      CK(cudaStreamEndCapture(xc.s, &tmp));
    }
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(xb.s, &tmp));
  }
  const long long per_sweep = (c.launch_count - lc_loop) / 2;
  ++c.launch_count;
  parity_fixup_kernel<T><<<grid_for(n, 256, 148 * 8), 256, 0, x.s>>>(st, L.u[1], L.u[0], n);
  CK(cudaGetLastError());
  cudaGraph_t graph;
  CK(cudaStreamEndCapture(x.s, &graph));
  cudaGraphExec_t exec;
  CK(cudaGraphInstantiate(&exec, graph, 0));
  CK(cudaGraphDestroy(graph));
  const long long captured = c.launch_count - lc_before;
  c.launch_count = lc_before;  // counted when they run (finish_level_graphs)
  if (c.graphs.size() >= 16) {
    auto old = std::min_element(c.graphs.begin(), c.graphs.end(),
                                [](const si_ctx::LevelGraph& a, const si_ctx::LevelGraph& b) {
                                  return a.stamp < b.stamp;
                                });
    CK(cudaGraphExecDestroy(old->exec));
    c.graphs.erase(old);
  }
  si_ctx::LevelGraph g;
  g.key = std::move(key);
  g.exec = exec;
  g.per_sweep = per_sweep;
  g.fixed = captured - 2 * per_sweep;
  g.stamp = ++c.graph_clock;
  c.graphs.push_back(std::move(g));
  CK(cudaGraphLaunch(exec, x.s));
  return {captured - 2 * per_sweep, per_sweep};
}

// multilevel_solve (multilevel.hpp:239-310) for the Schwarz level solvers.
// run_cg_level (multilevel.hpp:162-209) on device buffers: the reduced
// system's lockstep CG (cg_solve_lockstep, cg.hpp:192-291) with every scalar
// decision on the host, every vector operation in cg_level.cuh.
template <typename T>
LevelOutcome run_cg_level(Ctx& x, LevelView<T>& V, int C, double tol, const si_options& o,
                          bool sink, const Trace& tr, const double* d_ref) {
  LevelOutcome out;
  check_arg(C <= kCgMaxChannels, "multilevel CG: at most 8 channels");
  const int W = V.w, H = V.h;
  const size_t N = static_cast<size_t>(W) * H;
  for (DevBuf* b : {&x.c.cg_rhs, &x.c.cg_x, &x.c.cg_r, &x.c.cg_p, &x.c.cg_q})
    b->ensure(N * C * sizeof(T));
  T *rhs = x.c.cg_rhs.as<T>(), *xv = x.c.cg_x.as<T>(), *r = x.c.cg_r.as<T>(),
    *p = x.c.cg_p.as<T>(), *q = x.c.cg_q.as<T>();
  const int gx = (W + kRedThreads - 1) / kRedThreads;
  const int gy = std::max(1, std::min(H, (2 * kRedBlocksMax + gx * C - 1) / (gx * C)));
  const dim3 grid(gx, gy, C);
  x.c.red_partials.ensure(sizeof(double) * 2 * static_cast<size_t>(gx) * gy * C);
  x.c.ticket.ensure(sizeof(unsigned int) * 4);
  double* red = x.c.dev_red;  // mapped host memory
  double* hred = x.c.host_red;
  auto P = [&] { return x.c.red_partials.as<double>(); };
  auto tk = [&] { return x.c.ticket.as<unsigned int>(); };
  const double vec_bytes = static_cast<double>(N) * C * sizeof(T);

  {
    Timed t(x, K_RESIDUAL, 6 * vec_bytes);
    ++x.c.launch_count;
    cg_init_kernel<T><<<grid, kRedThreads, 0, x.s>>>(V.mask, V.b, V.u[V.cur], rhs, xv, r, p, W, H,
                                                     N, P(), red, tk());
    CK(cudaGetLastError());
  }
  sync(x);
  // r0 from the reduced rhs, row 0 from the initial residual (multilevel.hpp:169-189)
  const double r0 = joint_norm(hred, C);
  const double rel0 = r0 > 0.0 ? joint_norm(hred + C, C) / r0 : 0.0;
  auto trace_row = [&](int it, double rel) {
    if (!sink || !tr.fn) return;
    double qv = std::numeric_limits<double>::quiet_NaN();
    if (d_ref) {
      ++x.c.launch_count;
      cg_embed_kernel<T><<<grid, kRedThreads, 0, x.s>>>(V.mask, V.b, xv, V.u[V.cur ^ 1], W, H, N);
      launch_sq_error<T>(x, V.u[V.cur ^ 1], d_ref, N, C, x.c.dev_red + 3 * C);
      sync(x);
      qv = psnr_from_sq(std::vector<double>(hred + 3 * C, hred + 4 * C), N);
    }
    tr.fn(it, ms_since(tr.t0), rel, qv, tr.user);
  };
  trace_row(0, rel0);

  // ---- cg_solve_lockstep
  std::vector<double> rr(hred + C, hred + 2 * C), rr_next(C), pAp(C);
  double joint0 = 0.0;
  for (int c = 0; c < C; ++c) joint0 += rr[c];
  const double rz = r0 > 0.0 ? r0 : std::sqrt(joint0);
  std::vector<char> frozen(C, 0);
  bool done = false;
  if (rz == 0.0 || std::sqrt(joint0) <= tol * rz) {
    out.converged = true;
    out.final_rel = rz == 0.0 ? 0.0 : std::sqrt(joint0) / rz;
    done = true;
  }
  if (!done) {
    check_arg(o.cg_max_iterations >= 0, "SolverConfig: max_iterations must be non-negative");
    check_arg(o.cg_check_interval >= 1, "SolverConfig: residual_check_interval must be >= 1");
    const double freeze_sq = 1e-4 * tol * tol * rz * rz;
    double rel = std::sqrt(joint0) / rz;
    out.final_rel = rel;
    const int maxit = o.cg_max_iterations;
    for (int iter = 1; iter <= maxit; ++iter) {
      unsigned active = 0;
      for (int c = 0; c < C; ++c) {
        if (frozen[c] || rr[c] <= freeze_sq) {
          frozen[c] = 1;
          rr_next[c] = rr[c];
        } else {
          active |= 1u << c;
        }
      }
      if (active) {
        Timed t(x, K_SWEEP, 2 * vec_bytes);
        ++x.c.launch_count;
        cg_apply_dot_kernel<T><<<grid, kRedThreads, 0, x.s>>>(V.mask, p, q, W, H, N, active, P(),
                                                              red, tk());
        CK(cudaGetLastError());
      }
      sync(x);
      CgCoef alpha{};
      unsigned upd = 0;
      int broke = -1;
      for (int c = 0; c < C; ++c) {
        if (!((active >> c) & 1u)) continue;
        const double pa = hred[c];
        if (!(pa > 0.0) || !std::isfinite(pa)) {  // breakdown (cg.hpp:243-250)
          broke = c;
          break;
        }
        alpha.v[c] = rr[c] / pa;
        upd |= 1u << c;
      }
      if (upd) {
        Timed t(x, K_SWEEP, 5 * vec_bytes);
        ++x.c.launch_count;
        cg_update_kernel<T><<<grid, kRedThreads, 0, x.s>>>(xv, p, r, q, W, H, N, upd, alpha, P(),
                                                           red, tk());
        CK(cudaGetLastError());
        sync(x);
      }
      if (broke >= 0) {
        // (multilevel_solve reports only converged / not converged for a level)
        out.iterations = iter - 1;
        out.final_rel = rel;
        done = true;
        break;  // partially updated channels stay as the reference leaves them
      }
      double joint_sq = 0.0;
      for (int c = 0; c < C; ++c) {
        if ((active >> c) & 1u) rr_next[c] = hred[c];
        joint_sq += rr_next[c];
      }
      const bool cadence = iter % o.cg_check_interval == 0 || iter == maxit;
      const bool maybe_done = std::sqrt(joint_sq) <= tol * rz;
      if (cadence || maybe_done) {
        unsigned replace = 0;
        for (int c = 0; c < C; ++c)
          if (!frozen[c]) replace |= 1u << c;
        {
          Timed t(x, K_RESIDUAL, 3 * vec_bytes);
          ++x.c.launch_count;
          cg_true_residual_kernel<T><<<grid, kRedThreads, 0, x.s>>>(V.mask, rhs, xv, r, W, H, N,
                                                                    replace, P(), red, tk());
          CK(cudaGetLastError());
        }
        sync(x);
        double true_sq = 0.0;
        for (int c = 0; c < C; ++c) {
          true_sq += hred[c];
          if (!frozen[c]) rr_next[c] = hred[c];
        }
        rel = std::sqrt(true_sq) / rz;
        out.final_rel = rel;
        trace_row(iter, rel);
        if (rel <= tol) {
          out.iterations = iter;
          out.converged = true;
          done = true;
          break;
        }
      }
      CgCoef beta{};
      unsigned pa = 0;
      for (int c = 0; c < C; ++c) {
        if (frozen[c]) continue;
        beta.v[c] = rr[c] > 0.0 ? rr_next[c] / rr[c] : 0.0;
        rr[c] = rr_next[c];
        pa |= 1u << c;
      }
      if (pa) {
        ++x.c.launch_count;
        cg_pupdate_kernel<T><<<grid, kRedThreads, 0, x.s>>>(p, r, W, H, N, pa, beta);
        CK(cudaGetLastError());
      }
    }
    if (!done) out.iterations = maxit;
  }
  // embed_solution (reduction.hpp:138-145) into the level's iterate
  ++x.c.launch_count;
  cg_embed_kernel<T><<<grid, kRedThreads, 0, x.s>>>(V.mask, V.b, xv, V.u[V.cur ^ 1], W, H, N);
  CK(cudaGetLastError());
  V.cur ^= 1;
  return out;
}

// Level-0 input as known samples (batch upload, host_copy.h) instead of f.
struct KnownSamples {
  const double* vals;        // [C][K]
  const uint32_t* tile_off;  // known count before each kScatterTile-pixel tile
  size_t K;
  size_t bytes;              // uploaded: offsets + values
};
static_assert(kScatterTile == sib::kKnownTile, "host and device tile sizes differ");

// fixed_block >= 0 selects solve_schwarz's explicit, unclamped partition
// (schwarz.hpp:349-389) instead of clamped_partition per level.
template <typename T>
void multilevel_device(Ctx& x, int levels_req, int flavour, const double* d_f,
                       const uint8_t* d_mask, int w, int h, int C, const si_options& o,
                       const double* d_ref, double* d_out, si_report* rep, const Trace& tr,
                       int fixed_block = -1, int fixed_overlap = 0,
                       const KnownSamples* ks = nullptr) {
  NvtxRange nv_solve("multilevel_solve");
  prepare_red(x, C);
  check_arg(levels_req >= 1, "build_pyramid: levels must be >= 1");
  // Level geometry: halve (ceil) until the requested depth or a level that
  // cannot be halved again (multilevel.hpp:90-93).
  std::vector<int> lw{w}, lh{h};
  while (static_cast<int>(lw.size()) < levels_req && static_cast<int>(lw.size()) < SI_MAX_LEVELS) {
    if (lw.back() < 2 || lh.back() < 2) break;
    lw.push_back((lw.back() + 1) / 2);
    lh.push_back((lh.back() + 1) / 2);
  }
  const int depth = static_cast<int>(lw.size());
  rep->depth = depth;
  if (static_cast<int>(x.c.levels.size()) < depth) x.c.levels.resize(depth);
  std::vector<LevelView<T>> L(depth);
  for (int l = 0; l < depth; ++l) {
    const size_t n = static_cast<size_t>(lw[l]) * lh[l];
    auto& lb = x.c.levels[l];
    lb.mask.ensure(n);
    lb.b.ensure(n * C * sizeof(T));
    lb.u0.ensure(n * C * sizeof(T));
    lb.u1.ensure(n * C * sizeof(T));
    T* u0 = lb.u0.as<T>();
    // fp64: the caller's output buffer is one of the finest level's ping-pong
    // iterates, so an even number of finest sweeps needs no export copy
    if constexpr (std::is_same<T, double>::value)
      if (l == 0 && d_out != nullptr && d_out != d_ref) u0 = d_out;
    L[l] = {lw[l], lh[l], l == 0 ? d_mask : lb.mask.as<uint8_t>(), lb.b.as<T>(), {u0, lb.u1.as<T>()},
            0};
  }
  // K5 ingest: level-0 values, known count for build_rhs's check.
  const size_t n0 = static_cast<size_t>(w) * h;
  bool fused_restrict = false;
  bool skip_b0 = false;  // level-0 b not materialised (the snap reads d_f)
  if (ks) {  // K5s: only the known samples came over
    Timed t(x, K_INGEST, static_cast<double>(n0) * (C * sizeof(T) + 1.0) + ks->K * C * 8.0);
    ++x.c.launch_count;
    known_scatter_kernel<T><<<static_cast<unsigned>((n0 + kScatterTile - 1) / kScatterTile),
                              kScatterWarps * 32, 0, x.s>>>(
        d_mask, n0, C, ks->vals, ks->K, ks->tile_off, x.c.levels[0].b.as<T>(),
        x.c.counters.as<unsigned long long>() + 2);
    CK(cudaGetLastError());
  } else if (depth > 1 && !ingest_fusion_disabled()) {
    // K5 + K3 fused: level-0 values and level 1 in one pass.  fp64 Schwarz
    // levels with the InitialGuess normaliser read level-0 b only where the
    // prolongation snaps (f itself there) once the pair pass derives b from
    // u0: then b0 is not written at all (199 MB per 4K RGB frame).
    skip_b0 = std::is_same<T, double>::value && flavour != kFlavourCg && o.normalizer != 1 &&
              pair_derivable(L[0].mask, L[0].u[0], w, h, C);
    Timed t(x, K_INGEST, static_cast<double>(n0) * (C * ((skip_b0 ? 0.0 : 8.0) + sizeof(T)) + 1.0) +
                             static_cast<double>(lw[1]) * lh[1] * (C * sizeof(T) + 1));
    const dim3 grid((lw[1] + 128 * kIrCells - 1) / (128 * kIrCells), lh[1]);
    T* b0 = skip_b0 ? nullptr : x.c.levels[0].b.as<T>();
    ++x.c.launch_count;
    if (w % 2 == 0)
      ingest_restrict_kernel<T, true><<<grid, 128, 0, x.s>>>(
          d_f, d_mask, w, h, C, o.averaging, b0, x.c.levels[1].mask.as<uint8_t>(),
          x.c.levels[1].b.as<T>(), x.c.counters.as<unsigned long long>() + 2);
    else
      ingest_restrict_kernel<T, false><<<grid, 128, 0, x.s>>>(
          d_f, d_mask, w, h, C, o.averaging, b0, x.c.levels[1].mask.as<uint8_t>(),
          x.c.levels[1].b.as<T>(), x.c.counters.as<unsigned long long>() + 2);
    CK(cudaGetLastError());
    fused_restrict = true;
  } else {
    Timed t(x, K_INGEST, static_cast<double>(n0) * (C * (8.0 + sizeof(T)) + 1.0));
    ++x.c.launch_count;
    ingest_kernel<T><<<ingest_grid(n0), 256, 0, x.s>>>(
        d_f, d_mask, n0, C, x.c.levels[0].b.as<T>(), x.c.counters.as<unsigned long long>() + 2);
    CK(cudaGetLastError());
  }
  // K3: restrict level by level (level 1 already made by the fused pass).
  for (int l = fused_restrict ? 2 : 1; l < depth; ++l) {
    const size_t cn = static_cast<size_t>(lw[l]) * lh[l];
    Timed t(x, K_RESTRICT, static_cast<double>(cn) * 4.0 * (C * sizeof(T) + 1) + cn * (C * sizeof(T) + 1));
    launch_restrict<T>(x, L[l - 1].mask, L[l - 1].b, lw[l - 1], lh[l - 1], C, o.averaging,
                       x.c.levels[l].mask.as<uint8_t>(), x.c.levels[l].b.as<T>());
    CK(cudaGetLastError());
  }
  bool known_checked = false;
  // graph-mode levels: outcome read after the frame's single synchronisation
  std::vector<int> graph_level(depth, 0);
  std::vector<GraphCounts> graph_counts(depth, GraphCounts{0, 0});
  std::vector<long long> graph_blocks(depth, 0);
  if (x.c.graph_mode) {
    x.c.lvl_state.ensure(sizeof(LevelState) * SI_MAX_LEVELS);
    x.c.lvl_sums.ensure(sizeof(double) * 2 * C * SI_MAX_LEVELS);
  }
  for (int level = depth - 1; level >= 0; --level) {
    NvtxRange nv_level("level %d", level);
    LevelView<T>& V = L[level];
    const size_t n = static_cast<size_t>(V.w) * V.h;
    if (level == depth - 1) {
      // canonical start u0 = b on the coarsest level (multilevel.hpp:267-273)
      ++x.c.launch_count;
      launch_pdl(convert_kernel<T, T>, dim3(grid_for(n * C, 256, 148 * 16)), 256, x.s,
                 static_cast<const T*>(V.b), V.u[0], n * C);
      CK(cudaGetLastError());
      V.cur = 0;
    }
    const bool finest = level == 0;
    const double tol = finest ? o.tolerance : o.coarse_tolerance;
    const bool cg_level = flavour == kFlavourCg;
    Clamped cp{fixed_block, fixed_overlap};
    if (!cg_level && fixed_block < 0) cp = clamp_partition(V.w, V.h, o.block_size, o.overlap);
    if (flavour == SI_FLAVOUR_ORAS)
      check_arg(std::isfinite(o.alpha), "run_schwarz_level: alpha must be finite");
    const bool by_graph = graph_eligible(x, o, tr, d_ref, flavour, cp.block);
    bool known_deferred = false;
    if (!known_checked && !by_graph && !cg_level) {
      // build_rhs rejects an empty mask (operators.hpp:83): the count taken by
      // the ingest kernel goes to mapped memory now and is checked at the
      // level's first synchronisation (no extra host round trip; an empty
      // mask gives r0 = 0 and the level returns at once)
      ++x.c.launch_count;
      copy_u64_kernel<<<1, 32, 0, x.s>>>(x.c.counters.as<unsigned long long>(), x.c.dev_cnt, 3,
                                         false);
      CK(cudaGetLastError());
      known_deferred = true;
    } else if (!known_checked && !by_graph) {
      publish_counters(x, 3);
      // reduce_structure's singularity check (reduction.hpp:84-112) can only
      // fail when no pixel is known (a component of the unknown region that
      // touches no known pixel is the whole grid); it runs before build_rhs.
      if (cg_level && x.c.host_cnt[2] == 0)
        fail(SI_ERR_RUNTIME,
             "reduce_structure: singular system (an unknown region touches no known pixel)");
      check_arg(x.c.host_cnt[2] > 0, "build_rhs: mask has no known pixels");
      known_checked = true;
    }
    LevelOutcome oc;
    if (by_graph) {
      graph_level[level] = 1;
      graph_counts[level] = launch_level_graph<T>(x, V, C, level, cp.block, cp.overlap, tol,
                                                  flavour, o, level == depth - 1);
      graph_blocks[level] = static_cast<long long>(Axis::make(V.w, cp.block, cp.overlap).count) *
                            Axis::make(V.h, cp.block, cp.overlap).count * C;
      V.cur = 0;  // the parity fixup leaves the level's iterate in u[0]
    } else if (cg_level) {
      oc = run_cg_level<T>(x, V, C, tol, o, finest, tr, finest ? d_ref : nullptr);
    } else {
      double r0 = 0.0;
      int r0_mode = kR0Launched;
      if (o.normalizer == 1)
        launch_r0<T>(x, V, C, o.normalizer);
      else
        r0_mode = level == depth - 1 ? kR0Same : kR0Pair;
      oc = run_level<T>(x, V, C, cp.block, cp.overlap, &r0, true, tol, flavour, o, true, finest,
                        tr, finest ? d_ref : nullptr, rep, r0_mode, known_deferred);
    }
    if (known_deferred) known_checked = true;
    rep->level_iterations[level] = oc.iterations;
    rep->level_final_rel[level] = oc.final_rel;
    rep->level_converged[level] = oc.converged;
    if (finest) {
      rep->iterations = oc.iterations;
      rep->final_relative_residual = oc.final_rel;
      rep->converged = oc.converged;
    } else {
      // K4: prolongate + snap into the next finer level's u.
      LevelView<T>& F = L[level - 1];
      const size_t fn = static_cast<size_t>(F.w) * F.h;
      Timed t(x, K_PROLONG, static_cast<double>(fn) * (2.0 * C * sizeof(T) + 1.0) + n * C * sizeof(T));
      // the snap's values: f itself when level-0 b was not kept (fp64: b0 == f
      // at known pixels bit for bit)
      const T* snap = F.b;
      if constexpr (std::is_same<T, double>::value)
        if (level == 1 && skip_b0) snap = d_f;
      launch_prolong<T>(x, V.u[V.cur], V.w, V.h, F.w, F.h, C, F.mask, snap, F.u[0]);
      CK(cudaGetLastError());
      F.cur = 0;
    }
  }
  const int n_graph = static_cast<int>(std::count(graph_level.begin(), graph_level.end(), 1));
  if (x.c.defer_to && n_graph == depth) {
    // batch pipelining: level states + counters to this slot's mapped words,
    // read by finish_frame once the next frame is queued
    PendingFrame& P = *x.c.defer_to;
    const int sl = P.slot;
    if (!x.c.frame_host[sl]) {
      CK(cudaHostAlloc(&x.c.frame_host[sl], sizeof(unsigned long long) * kFrameWords,
                       cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&x.c.frame_dev[sl]),
                                  x.c.frame_host[sl], 0));
      CK(cudaEventCreateWithFlags(&x.c.frame_done[sl], cudaEventDisableTiming));
    }
    const int words = static_cast<int>(sizeof(LevelState) / 8) * depth;
    ++x.c.launch_count;
    copy_bytes_kernel<<<1, 64, 0, x.s>>>(x.c.lvl_state.as<unsigned long long>(),
                                         x.c.frame_dev[sl], words);
    ++x.c.launch_count;
    copy_bytes_kernel<<<1, 64, 0, x.s>>>(x.c.counters.as<unsigned long long>(),
                                         x.c.frame_dev[sl] + SI_MAX_LEVELS * 4, 3);
    CK(cudaGetLastError());
    CK(cudaEventRecord(x.c.frame_done[sl], x.s));
    P.active = true;
    P.depth = depth;
    P.fixed_block = fixed_block;
    P.known_checked = known_checked;
    P.rep = rep;
    for (int l = 0; l < depth; ++l) {
      P.graph_level[l] = 1;
      P.counts[l] = graph_counts[l];
      P.blocks[l] = graph_blocks[l];
    }
  } else if (n_graph > 0) {
    // the frame's one synchronisation: level states and counters to the host
    if (!x.c.host_state) {
      CK(cudaHostAlloc(&x.c.host_state, sizeof(LevelState) * SI_MAX_LEVELS, cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&x.c.dev_state), x.c.host_state, 0));
    }
    const int words = static_cast<int>(sizeof(LevelState) / 8) * depth;
    ++x.c.launch_count;
    copy_bytes_kernel<<<1, 64, 0, x.s>>>(x.c.lvl_state.as<unsigned long long>(), x.c.dev_state,
                                         words);
    CK(cudaGetLastError());
    publish_counters(x, 3);
    if (!known_checked) check_arg(x.c.host_cnt[2] > 0, "build_rhs: mask has no known pixels");
    x.c.counters_fresh = 1;
    const LevelState* hs = reinterpret_cast<const LevelState*>(x.c.host_state);
    for (int l = 0; l < depth; ++l) {
      if (!graph_level[l]) continue;
      const LevelState& S = hs[l];
      rep->level_iterations[l] = S.iterations;
      rep->level_final_rel[l] = S.final_rel;
      rep->level_converged[l] = S.converged != 0;
      rep->local_solves += static_cast<long long>(S.outer) * graph_blocks[l];
      x.c.launch_count += graph_counts[l].fixed + graph_counts[l].per_sweep * S.outer;
      if (l == 0) {
        rep->iterations = S.iterations;
        rep->final_relative_residual = S.final_rel;
        rep->converged = S.converged != 0;
      }
    }
  }
  if (!(x.c.defer_to && x.c.defer_to->active)) write_diagnostic(rep, depth, fixed_block);
  // Export the finest u (T -> double) unless it already lives in d_out.
  if (static_cast<const void*>(L[0].u[L[0].cur]) != static_cast<const void*>(d_out)) {
    Timed t(x, K_INGEST, static_cast<double>(n0) * C * (8.0 + sizeof(T)));
    ++x.c.launch_count;
    convert_kernel<T, double><<<grid_for(n0 * C, 256, 148 * 16), 256, 0, x.s>>>(
        L[0].u[L[0].cur], d_out, n0 * C);
    CK(cudaGetLastError());
  }
}

}  // namespace

// ====================================================================== ABI
#include <functional>

namespace {
si_status guard(const std::function<void()>& fn) {
  try {
    fn();
    return SI_OK;
  } catch (const Failure& f) {
    g_last_error = f.message;
    return f.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return SI_ERR_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SI_ERR_CUDA;
  }
}

void set_device(si_ctx* c) { CK(cudaSetDevice(c->device)); }

cudaStream_t pick_stream(si_ctx* c, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
}

void clear_report(si_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
}

int levels_for(int method, const si_options& o) {
  return (method == SI_METHOD_MLORAS || method == SI_METHOD_MLCG) ? o.levels : 1;
}

int flavour_for(int method) {
  if (method == SI_METHOD_CG || method == SI_METHOD_MLCG) return kFlavourCg;
  return method == SI_METHOD_RAS ? SI_FLAVOUR_RAS : SI_FLAVOUR_ORAS;
}

void check_method(int method) {
  check_arg(method >= SI_METHOD_CG && method <= SI_METHOD_MLORAS,
            "unknown method (expected cg, mlcg, ras, oras or mloras)");

}

void check_dims(int w, int h, int c) {
  check_arg(w > 0 && h > 0 && c > 0, "ImageBuffer: dimensions must be positive");
}

void run_device(si_ctx* ctx, int method, const double* d_f, const uint8_t* d_mask, int w, int h,
                int c, const si_options& o, const double* d_ref, double* d_out, si_report* rep,
                si_trace_fn trace, void* user, cudaStream_t s, Clock::time_point t0,
                const KnownSamples* ks = nullptr) {
  check_method(method);
  check_dims(w, h, c);
  validate_options_common(o);
  Ctx x{*ctx, s};
  LocalPrecision lp(*ctx, o.precision);
  begin_counters(x);
  Trace tr{trace, user, t0};
  if (o.precision == SI_PRECISION_FP32)
    multilevel_device<float>(x, levels_for(method, o), flavour_for(method), d_f, d_mask, w, h, c,
                             o, d_ref, d_out, rep, tr, -1, 0, ks);
  else
    multilevel_device<double>(x, levels_for(method, o), flavour_for(method), d_f, d_mask, w, h, c,
                              o, d_ref, d_out, rep, tr, -1, 0, ks);
  if (!(ctx->defer_to && ctx->defer_to->active)) end_counters(x, rep);
}

// SI_NO_GRAPHS=1: batch frames keep the host-driven outer iteration.
bool graphs_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("SI_NO_GRAPHS");
    return e && e[0] == '1';
  }();
  return off;
}

// SI_NO_KNOWN_PACK=1: always upload the full f (A/B measurements).
// Host threads packing known samples (SI_PACK_THREADS; default half the
// hardware threads, at most 8: a 4K RGB frame packs in ~9 ms on one thread,
// memory-latency bound, and the thread driving the solves must keep a core;
// scripts/e2e_probe.py measures the settings).
int pack_threads() {
  static const int n = [] {
    const char* e = std::getenv("SI_PACK_THREADS");
    const int v = e ? std::atoi(e) : 0;
    const int hw = static_cast<int>(std::max(2u, std::thread::hardware_concurrency()));
    return v > 0 ? v : std::min(8, hw / 2);
  }();
  return n;
}

bool known_pack_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("SI_NO_KNOWN_PACK");
    return e && e[0] == '1';
  }();
  return off;
}

// Single-frame known-sample upload into ctx->in_f (host_copy.h): packs on the
// host pool into pack_buf[0] and queues the copy on x.s.  False (nothing
// queued) when more than 1/8 of the pixels are known.
bool upload_known(Ctx& x, const double* f, const uint8_t* mask, size_t n, int C,
                  KnownSamples* ks) {
  si_ctx& c = x.c;
  const size_t ntiles = (n + sib::kKnownTile - 1) / sib::kKnownTile;
  const size_t off_bytes = (ntiles * sizeof(uint32_t) + 15) / 16 * 16;
  if (n < (size_t(1) << 16) || known_pack_disabled()) return false;  // small: one plain copy
  if (!c.pack_pool) c.pack_pool = std::make_unique<sib::CopyPool>(pack_threads());
  if (c.ev_h2d[0]) CK(cudaEventSynchronize(c.ev_h2d[0]));  // a batch upload may still read it
  CK(cudaStreamSynchronize(x.s));                          // and so may this stream's last one
  auto grow = [&](size_t need, size_t keep) {
    if (c.pack_cap[0] >= need) return;
    void* nb = nullptr;
    const size_t cap = need + need / 4;
    CK(cudaMallocHost(&nb, cap));
    if (c.pack_buf[0]) {
      std::memcpy(nb, c.pack_buf[0], keep);
      CK(cudaFreeHost(c.pack_buf[0]));
    }
    c.pack_buf[0] = nb;
    c.pack_cap[0] = cap;
  };
  grow(off_bytes, 0);
  const size_t K = sib::count_known_tiles(*c.pack_pool, mask, n,
                                          static_cast<uint32_t*>(c.pack_buf[0]));
  if (K * 8 > n) return false;
  const size_t bytes = off_bytes + K * C * sizeof(double);
  grow(bytes, off_bytes);
  char* buf = static_cast<char*>(c.pack_buf[0]);
  sib::gather_known(*c.pack_pool, mask, f, n, C, reinterpret_cast<const uint32_t*>(buf), K,
                    reinterpret_cast<double*>(buf + off_bytes));
  CK(cudaMemcpyAsync(c.in_f.ptr, buf, bytes, cudaMemcpyHostToDevice, x.s));
  ks->tile_off = c.in_f.as<uint32_t>();
  ks->vals = reinterpret_cast<const double*>(c.in_f.as<uint8_t>() + off_bytes);
  ks->K = K;
  ks->bytes = bytes;
  return true;
}

// Batch pipeline shared by si_run_method_batch (f64 planar in/out) and
// si_run_pnm_batch (PNM/PBM payloads in/out): two staging slots, H2D of frame
// k+1 and D2H of frame k-1 on their own streams while frame k is solved.
void run_batch(si_ctx* ctx, int method, int n, const void* const* in, const uint8_t* const* mask,
               int w, int h, int c, const si_options* opt, void* const* out, si_report* reports,
               bool pnm) {
  check_dims(w, h, c);
  si_options o;
  if (opt) o = *opt; else si_default_options(&o);
  set_device(ctx);
  if (!ctx->h2d_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventCreateWithFlags(&ctx->ev_h2d[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_solved[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_d2h[k], cudaEventDisableTiming));
    }
  }
  const size_t n_px = static_cast<size_t>(w) * h, img = n_px * c * sizeof(double);
  const size_t row_bytes = (static_cast<size_t>(w) + 7) / 8;
  const size_t in_bytes = pnm ? n_px * c : img, mask_bytes = pnm ? row_bytes * h : n_px;
  const size_t out_bytes = pnm ? n_px * c : img;
  for (int k = 0; k < 2; ++k) {
    ctx->slot_f[k].ensure(img + (pnm ? in_bytes + 16 : 0));
    ctx->slot_mask[k].ensure(n_px + (pnm ? mask_bytes + 16 : 0));
    ctx->slot_out[k].ensure(img + (pnm ? out_bytes + 16 : 0));
  }
  // pnm: the raw payloads sit behind the decoded buffers in the same slot
  auto raw_in = [&](int s) { return ctx->slot_f[s].as<uint8_t>() + (pnm ? img : 0); };
  auto raw_mask = [&](int s) { return ctx->slot_mask[s].as<uint8_t>() + (pnm ? n_px : 0); };
  auto raw_out = [&](int s) { return ctx->slot_out[s].as<uint8_t>() + (pnm ? img : 0); };
  // Known-sample upload (f64 frames whose mask is at most 1/8 known): a
  // helper thread packs frame k+2 on the host pool while frame k is solved
  // and frame k+1 is in flight; pack_buf[s] = [tile offsets | C x K values].
  const size_t ntiles = (n_px + sib::kKnownTile - 1) / sib::kKnownTile;
  const size_t off_bytes = (ntiles * sizeof(uint32_t) + 15) / 16 * 16;
  struct Pack {
    size_t K = 0;
    bool sparse = false;
    long long h2d = 0;
  };
  std::vector<Pack> packs(n);
  const bool may_pack = !pnm && !known_pack_disabled();
  // outer iterations decided on the device (cached level graphs): no host
  // round trip per iteration while the result copies load the link
  struct GraphMode {
    si_ctx* c;
    explicit GraphMode(si_ctx* ctx) : c(ctx) { c->graph_mode = !graphs_disabled(); }
    ~GraphMode() { c->graph_mode = 0; }
  } graph_mode_guard(ctx);
  if (may_pack && !ctx->pack_pool) ctx->pack_pool = std::make_unique<sib::CopyPool>(pack_threads());
  // outgrown pack buffers are freed after the batch: cudaFreeHost may
  // synchronise the device, which must not happen on the packing thread while
  // the solving thread captures a level graph
  std::vector<void*> retired;
  std::mutex retired_m;
  struct RetiredFree {
    std::vector<void*>& v;
    ~RetiredFree() {
      for (void* p : v) cudaFreeHost(p);
    }
  } retired_free{retired};
  auto grow = [&](int s, size_t need, size_t keep) {
    if (ctx->pack_cap[s] >= need) return;
    void* nb = nullptr;
    const size_t cap = need + need / 4;
    CK(cudaMallocHost(&nb, cap));
    if (ctx->pack_buf[s]) {
      std::memcpy(nb, ctx->pack_buf[s], keep);
      std::lock_guard<std::mutex> g(retired_m);
      retired.push_back(ctx->pack_buf[s]);
    }
    ctx->pack_buf[s] = nb;
    ctx->pack_cap[s] = cap;
  };
  auto pack = [&](int k) {
    const int s = k & 1;
    CK(cudaEventSynchronize(ctx->ev_h2d[s]));  // frame k-2's upload left pack_buf[s]
    grow(s, off_bytes, 0);
    uint32_t* off = static_cast<uint32_t*>(ctx->pack_buf[s]);
    Pack& P = packs[k];
    P.K = sib::count_known_tiles(*ctx->pack_pool, mask[k], n_px, off);
    P.sparse = P.K * 8 <= n_px;
    if (!P.sparse) return;
    grow(s, off_bytes + P.K * c * sizeof(double), off_bytes);
    sib::gather_known(*ctx->pack_pool, mask[k], static_cast<const double*>(in[k]), n_px, c,
                      static_cast<const uint32_t*>(ctx->pack_buf[s]), P.K,
                      reinterpret_cast<double*>(static_cast<char*>(ctx->pack_buf[s]) + off_bytes));
  };
  auto h2d = [&](int k) {
    const int s = k & 1;
    Pack& P = packs[k];
    // slot s still feeds frame k-2 until its solve ends (frames are queued
    // ahead of their completion in graph mode)
    if (k >= 2) CK(cudaStreamWaitEvent(ctx->h2d_stream, ctx->ev_solved[s], 0));
    if (P.sparse) {
      const size_t bytes = off_bytes + P.K * c * sizeof(double);
      CK(cudaMemcpyAsync(raw_in(s), ctx->pack_buf[s], bytes, cudaMemcpyHostToDevice,
                         ctx->h2d_stream));
      P.h2d = static_cast<long long>(bytes + mask_bytes);
    } else {
      CK(cudaMemcpyAsync(raw_in(s), in[k], in_bytes, cudaMemcpyHostToDevice, ctx->h2d_stream));
      P.h2d = static_cast<long long>(in_bytes + mask_bytes);
    }
    CK(cudaMemcpyAsync(raw_mask(s), mask[k], mask_bytes, cudaMemcpyHostToDevice,
                       ctx->h2d_stream));
    CK(cudaEventRecord(ctx->ev_h2d[s], ctx->h2d_stream));
  };
  std::future<void> packing;
  auto pack_async = [&](int k) {
    if (may_pack && k < n) packing = std::async(std::launch::async, [&pack, k] { pack(k); });
  };
  cudaStream_t cs = ctx->own_stream;
  if (n > 0) {
    if (may_pack) pack(0);
    h2d(0);
    pack_async(1);
  }
  // graph-mode frames are read back one frame late: frame k is queued before
  // frame k-1's outcome is waited for, so the device never idles on the host
  PendingFrame pend[2];
  std::vector<Clock::time_point> t_start(n);
  // pageable result copies in flight (chained helper-thread jobs)
  std::vector<std::shared_future<void>> drains(n);
  struct DeferGuard {
    si_ctx* c;
    ~DeferGuard() { c->defer_to = nullptr; }
  } defer_guard{ctx};
  // An error part way through (e.g. an empty mask found by finish_frame)
  // unwinds through here: wait for the packing and drain helpers and the
  // three streams, so no copy into a caller buffer is still in flight when
  // the status is returned.
  struct Unwind {
    si_ctx* c;
    cudaStream_t cs;
    std::future<void>& packing;
    std::vector<std::shared_future<void>>& drains;
    bool armed = true;
    ~Unwind() {
      if (!armed) return;
      if (packing.valid()) packing.wait();
      for (auto& d : drains)
        if (d.valid()) d.wait();
      cudaStreamSynchronize(c->d2h_stream);
      cudaStreamSynchronize(c->h2d_stream);
      cudaStreamSynchronize(cs);
      cudaGetLastError();
    }
  } unwind{ctx, cs, packing, drains};
  auto finish = [&](int j) {
    PendingFrame& P = pend[j & 1];
    if (!P.active) return;
    finish_frame(*ctx, P);
    P.rep->elapsed_ms = ms_since(t_start[j]);
  };
  for (int k = 0; k < n; ++k) {
    NvtxRange nv_frame("batch frame %d", k);
    const int s = k & 1;
    // the other slot's input was consumed by frame k-1 (solved synchronously)
    if (k + 1 < n) {
      if (may_pack) packing.get();
      h2d(k + 1);
      pack_async(k + 2);
    }
    CK(cudaStreamWaitEvent(cs, ctx->ev_h2d[s], 0));
    if (k >= 2) {  // out slot free again
      if (drains[k - 2].valid())
        drains[k - 2].get();
      else
        CK(cudaStreamWaitEvent(cs, ctx->ev_d2h[s], 0));
    }
    si_report* rep = reports ? &reports[k] : &ctx->batch_scratch_report[s];
    clear_report(rep);
    const auto t0 = Clock::now();
    t_start[k] = t0;
    KnownSamples ks{};
    if (packs[k].sparse) {
      ks.tile_off = ctx->slot_f[s].as<uint32_t>();
      ks.vals = reinterpret_cast<const double*>(ctx->slot_f[s].as<uint8_t>() + off_bytes);
      ks.K = packs[k].K;
    }
    if (pnm) {
      // read_pnm / read_mask_pbm (pnm.hpp:98-188) on device
      ++ctx->launch_count;
      unpack_pnm_kernel<<<dim3((w + 255) / 256, std::min(h, 65535)), 256, 0, cs>>>(
          raw_in(s), raw_mask(s), w, h, c, ctx->slot_f[s].as<double>(),
          ctx->slot_mask[s].as<uint8_t>());
      CK(cudaGetLastError());
    }
    pend[s].slot = s;
    ctx->defer_to = ctx->graph_mode ? &pend[s] : nullptr;
    run_device(ctx, method, ctx->slot_f[s].as<double>(), ctx->slot_mask[s].as<uint8_t>(), w, h, c,
               o, nullptr, ctx->slot_out[s].as<double>(), rep, nullptr, nullptr, cs, t0,
               packs[k].sparse ? &ks : nullptr);
    ctx->defer_to = nullptr;
    if (pnm) {
      // write_pnm's quantise (pnm.hpp:82-85, 130-147)
      ++ctx->launch_count;
      quantise_kernel<<<grid_for(n_px, 256, 148 * 16), 256, 0, cs>>>(
          ctx->slot_out[s].as<double>(), n_px, c, raw_out(s));
      CK(cudaGetLastError());
    }
    rep->elapsed_ms = ms_since(t0);
    rep->h2d_bytes = packs[k].h2d;
    rep->d2h_bytes = static_cast<long long>(out_bytes);
    CK(cudaEventRecord(ctx->ev_solved[s], cs));
    CK(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev_solved[s], 0));
    if (out_bytes >= (size_t(1) << 20) && !sib::host_is_pinned(out[k])) {
      // pageable result: a plain async copy would block this thread for the
      // whole transfer; a helper thread drains it through pinned chunks
      // (host_copy.h Stager) while the next frame is queued
      if (!ctx->drain_stager)
        ctx->drain_stager = std::make_unique<sib::Stager>([](cudaError_t e, const char* what) {
          cuda_check(e, what);
        });
      std::shared_future<void> prev = k >= 1 ? drains[k - 1] : std::shared_future<void>();
      void* dst = out[k];
      const void* src = raw_out(s);
      drains[k] = std::async(std::launch::async, [ctx, prev, dst, src, out_bytes, s] {
                    if (prev.valid()) prev.wait();
                    CK(cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev_solved[s], 0));
                    ctx->drain_stager->d2h(dst, src, out_bytes, ctx->d2h_stream);
                  }).share();
    } else {
      CK(cudaMemcpyAsync(out[k], raw_out(s), out_bytes, cudaMemcpyDeviceToHost,
                         ctx->d2h_stream));
      CK(cudaEventRecord(ctx->ev_d2h[s], ctx->d2h_stream));
    }
    if (k >= 1) finish(k - 1);
  }
  if (n >= 1) finish(n - 1);
  for (auto& d : drains)
    if (d.valid()) d.get();
  unwind.armed = false;
  CK(cudaStreamSynchronize(ctx->d2h_stream));
  CK(cudaStreamSynchronize(ctx->h2d_stream));
  CK(cudaStreamSynchronize(cs));
}

// ---------------------------------------------------------------- densify
// CUB device-wide primitives with their temporary storage in vz.tmp.
template <typename F>
void cub_call(Ctx& x, F&& fn) {
  size_t bytes = 0;
  CK(fn(static_cast<void*>(nullptr), bytes));
  x.c.vz.tmp.ensure(std::max<size_t>(bytes, 256));
  CK(fn(x.c.vz.tmp.ptr, bytes));
}

// assign_nearest_site (masks.hpp:54-139) of a device mask into vz.sites /
// vz.site_of; returns the site count m.
int assign_device(Ctx& x, const uint8_t* d_mask, int W, int H) {
  auto& z = x.c.vz;
  const size_t n = static_cast<size_t>(W) * H;
  const int ni = static_cast<int>(n);
  z.flag.ensure(n * 4);
  z.rank.ensure(n * 4);
  z.sites.ensure(n * 4);
  z.site_of.ensure(n * 4);
  z.small.ensure(64);
  int32_t* flag = z.flag.as<int32_t>();
  int32_t* rank = z.rank.as<int32_t>();
  int m = 0;
  {
    Timed t(x, K_VORONOI, static_cast<double>(n) * 13.0);
    ++x.c.launch_count;
    site_flags_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, x.s>>>(d_mask, n, flag);
    CK(cudaGetLastError());
    cub_call(x, [&](void* tmp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tmp, b, flag, rank, ni, x.s);
    });
    ++x.c.launch_count;
    sites_scatter_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, x.s>>>(d_mask, rank, n,
                                                                     z.sites.as<int32_t>());
    CK(cudaGetLastError());
    int32_t tail[2];
    CK(cudaMemcpyAsync(&tail[0], rank + n - 1, 4, cudaMemcpyDeviceToHost, x.s));
    CK(cudaMemcpyAsync(&tail[1], flag + n - 1, 4, cudaMemcpyDeviceToHost, x.s));
    CK(cudaStreamSynchronize(x.s));
    m = tail[0] + tail[1];
  }
  check_arg(m > 0, "assign_nearest_site: mask has no known pixels");
  const int cell = std::max(1, static_cast<int>(std::sqrt(static_cast<double>(n) / m)));
  const int gw = (W + cell - 1) / cell, gh = (H + cell - 1) / cell;
  const size_t nb = static_cast<size_t>(gw) * gh;
  z.bin_start.ensure((nb + 1) * 4);
  z.bin_cursor.ensure((nb + 1) * 4);
  z.members.ensure(static_cast<size_t>(m) * 4);
  int32_t* start = z.bin_start.as<int32_t>();
  int32_t* cursor = z.bin_cursor.as<int32_t>();
  {
    Timed t(x, K_VORONOI, static_cast<double>(m) * 24.0 + nb * 12.0);
    CK(cudaMemsetAsync(cursor, 0, (nb + 1) * 4, x.s));
    ++x.c.launch_count;
    bucket_count_kernel<<<grid_for(m, 256, 148 * 8), 256, 0, x.s>>>(z.sites.as<int32_t>(), m, W,
                                                                    cell, gw, cursor);
    CK(cudaGetLastError());
    cub_call(x, [&](void* tmp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tmp, b, cursor, start, static_cast<int>(nb + 1), x.s);
    });
    CK(cudaMemcpyAsync(cursor, start, nb * 4, cudaMemcpyDeviceToDevice, x.s));
    ++x.c.launch_count;
    bucket_fill_kernel<<<grid_for(m, 256, 148 * 8), 256, 0, x.s>>>(
        z.sites.as<int32_t>(), m, W, cell, gw, cursor, z.members.as<int32_t>());
    CK(cudaGetLastError());
  }
  {
    Timed t(x, K_VORONOI, static_cast<double>(n) * 4.0);
    ++x.c.launch_count;
    assign_sites_kernel<<<dim3((W + 31) / 32, (H + 7) / 8), 256, 0, x.s>>>(
        z.sites.as<int32_t>(), start, z.members.as<int32_t>(), W, H, cell, gw, gh,
        z.site_of.as<int32_t>());
    CK(cudaGetLastError());
  }
  return m;
}

// One sweep's cell statistics and ranking (masks.hpp:175-203) from the guide
// solution d_u; plants the worst pixels of the first `quota` cells into
// d_mask and returns how many were planted.
long long densify_plant(Ctx& x, const uint8_t* mask_view, uint8_t* d_mask, const double* d_u,
                        const double* d_f, int W, int H, int C, int m, double cell_fraction,
                        long long remaining) {
  auto& z = x.c.vz;
  const size_t n = static_cast<size_t>(W) * H;
  const int ni = static_cast<int>(n);
  z.key.ensure(n * 4);
  z.key2.ensure(n * 4);
  z.pix.ensure(n * 4);
  z.pix2.ensure(n * 4);
  z.err.ensure(n * 8);
  z.area.ensure((static_cast<size_t>(m) + 1) * 4);
  z.area2.ensure((static_cast<size_t>(m) + 1) * 4);
  z.seg.ensure((static_cast<size_t>(m) + 1) * 4);
  z.bits.ensure(static_cast<size_t>(m) * 8);
  z.bits2.ensure(static_cast<size_t>(m) * 8);
  z.worst.ensure(static_cast<size_t>(m) * 4);
  z.order.ensure(static_cast<size_t>(m) * 4);
  z.order2.ensure(static_cast<size_t>(m) * 4);
  int32_t* area = z.area.as<int32_t>();
  int* nonempty = z.small.as<int>();
  int key_bits = 1;
  while ((1ll << key_bits) <= m) ++key_bits;
  {
    Timed t(x, K_VORONOI, static_cast<double>(n) * (C * 16.0 + 1 + 4 + 12));
    CK(cudaMemsetAsync(area, 0, (static_cast<size_t>(m) + 1) * 4, x.s));
    CK(cudaMemsetAsync(nonempty, 0, 4, x.s));
    ++x.c.launch_count;
    cell_keys_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, x.s>>>(
        mask_view, z.site_of.as<int32_t>(), d_u, d_f, n, C, m, z.key.as<int32_t>(),
        z.pix.as<int32_t>(), z.err.as<double>(), area);
    CK(cudaGetLastError());
  }
  {
    Timed t(x, K_VORONOI, static_cast<double>(n) * 16.0 * 2);
    cub_call(x, [&](void* tmp, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(tmp, b, z.key.as<int32_t>(), z.key2.as<int32_t>(),
                                             z.pix.as<int32_t>(), z.pix2.as<int32_t>(), ni, 0,
                                             key_bits, x.s);
    });
    cub_call(x, [&](void* tmp, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(tmp, b, area, z.seg.as<int32_t>(), m + 1, x.s);
    });
  }
  {
    Timed t(x, K_VORONOI, static_cast<double>(n) * 12.0 + m * 24.0);
    ++x.c.launch_count;
    cell_reduce_kernel<<<grid_for(m, 128, 148 * 16), 128, 0, x.s>>>(
        z.seg.as<int32_t>(), z.pix2.as<int32_t>(), z.err.as<double>(), m,
        z.bits.as<unsigned long long>(), z.worst.as<int32_t>(), z.order.as<int32_t>(), nonempty);
    CK(cudaGetLastError());
  }
  {
    Timed t(x, K_VORONOI, static_cast<double>(m) * 48.0);
    // stable: area desc, ties keep index asc; then error desc, ties keep (area desc, index asc)
    cub_call(x, [&](void* tmp, size_t& b) {
      return cub::DeviceRadixSort::SortPairsDescending(tmp, b, area, z.area2.as<int32_t>(),
                                                       z.order.as<int32_t>(),
                                                       z.order2.as<int32_t>(), m, 0, 32, x.s);
    });
    ++x.c.launch_count;
    gather_bits_kernel<<<grid_for(m, 256, 148 * 8), 256, 0, x.s>>>(
        z.bits.as<unsigned long long>(), z.order2.as<int32_t>(), m,
        z.bits2.as<unsigned long long>());
    CK(cudaGetLastError());
    cub_call(x, [&](void* tmp, size_t& b) {
      return cub::DeviceRadixSort::SortPairsDescending(
          tmp, b, z.bits2.as<unsigned long long>(), z.bits.as<unsigned long long>(),
          z.order2.as<int32_t>(), z.order.as<int32_t>(), m, 0, 64, x.s);
    });
  }
  int used = 0;
  CK(cudaMemcpyAsync(&used, nonempty, 4, cudaMemcpyDeviceToHost, x.s));
  CK(cudaStreamSynchronize(x.s));
  long long quota = std::max<long long>(1, static_cast<long long>(cell_fraction * static_cast<double>(m)));
  quota = std::min<long long>({quota, static_cast<long long>(used), remaining});
  if (quota > 0) {
    Timed t(x, K_VORONOI, static_cast<double>(quota) * 9.0);
    ++x.c.launch_count;
    plant_kernel<<<grid_for(quota, 256, 148 * 8), 256, 0, x.s>>>(
        z.order.as<int32_t>(), z.worst.as<int32_t>(), static_cast<int>(quota), d_mask);
    CK(cudaGetLastError());
  }
  return quota;
}

// voronoi_densify (masks.hpp:155-212).  f is host planar f64; the whole loop
// (guide solves, assignment, ranking, planting) stays on the device.
void voronoi_densify(si_ctx* ctx, const double* f, int w, int h, int c, double target,
                     uint64_t seed, const si_densify_options& d, uint8_t* mask_out, int* sweeps,
                     int* reached) {
  check_arg(target > 0.0 && target <= 1.0, "voronoi_densify: target density must lie in (0, 1]");
  check_arg(d.initial_density <= 0.0 || d.initial_density < target,
            "voronoi_densify: initial density must lie below the target");
  check_dims(w, h, c);
  check_arg(static_cast<double>(w) * h < 2147483647.0,
            "voronoi_densify: images beyond 2^31 pixels are not supported");
  const size_t n = static_cast<size_t>(w) * h;
  const long long target_k = std::max<long long>(
      1, std::min<long long>(static_cast<long long>(n),
                             std::llround(target * static_cast<double>(n))));
  double init = d.initial_density > 0.0 ? d.initial_density : target / 4.0;
  if (init * static_cast<double>(n) < 1.0) init = 1.5 / static_cast<double>(n);
  std::vector<uint8_t> seed_mask(n);
  check_arg(si_random_mask(w, h, init, seed, seed_mask.data()) == SI_OK,
            "random_mask: density rounds to zero known pixels");
  long long known = 0;
  for (uint8_t v : seed_mask) known += v != 0;

  si_options so = d.solve;
  so.tolerance = d.inner_tolerance;
  validate_options_common(so);
  Ctx x{*ctx, ctx->own_stream};
  auto& z = ctx->vz;
  z.f.ensure(n * c * 8);
  z.mask.ensure(n);
  z.u.ensure(n * c * 8);
  h2d(x, z.f.ptr, f, n * c * 8);
  h2d(x, z.mask.ptr, seed_mask.data(), n);
  int sw = 0;
  while (known < target_k && sw < d.max_sweeps) {
    si_report rep;
    clear_report(&rep);
    run_device(ctx, SI_METHOD_MLORAS, z.f.as<double>(), z.mask.as<uint8_t>(), w, h, c, so,
               nullptr, z.u.as<double>(), &rep, nullptr, nullptr, x.s, Clock::now());
    const int m = assign_device(x, z.mask.as<uint8_t>(), w, h);
    known += densify_plant(x, z.mask.as<uint8_t>(), z.mask.as<uint8_t>(), z.u.as<double>(),
                           z.f.as<double>(), w, h, c, m, d.cell_fraction, target_k - known);
    ++sw;
  }
  d2h(x, mask_out, z.mask.ptr, n);
  *sweeps = sw;
  *reached = known >= target_k;
}

}  // namespace

extern "C" {

int si_abi_version(void) { return SI_ABI_VERSION; }

const char* si_last_error(void) { return g_last_error.c_str(); }

const char* si_status_string(si_status s) {
  switch (s) {
    case SI_OK: return "ok";
    case SI_ERR_INVALID_ARGUMENT: return "invalid argument";
    case SI_ERR_CUDA: return "cuda error";
    case SI_ERR_OOM: return "out of memory";
    case SI_ERR_UNSUPPORTED: return "unsupported";
    case SI_ERR_NO_DEVICE: return "no device";
    case SI_ERR_RUNTIME: return "runtime error";
  }
  return "unknown";
}

void si_default_options(si_options* o) {
  o->tolerance = 1e-3;
  o->levels = 3;
  o->block_size = 32;
  o->overlap = 6;
  o->alpha = 0.25;
  o->coarse_tolerance = 1e-2;
  o->averaging = SI_AVERAGING_KNOWN_ONLY;
  o->local_tolerance = 1e-2;
  o->local_max_iterations = 30;
  o->local_check_interval = 30;
  o->max_outer_iterations = 1000;
  o->cg_max_iterations = 100000;
  o->cg_check_interval = 4;
  o->normalizer = SI_NORMALIZER_INITIAL_GUESS;
  o->precision = SI_PRECISION_FP64;
}

si_status si_validate_options(int method, const si_options* opt) {
  return guard([&] {
    check_arg(opt != nullptr, "options must not be null");
    check_method(method);
    validate_options_common(*opt);
    check_arg(levels_for(method, *opt) >= 1, "build_pyramid: levels must be >= 1");
    check_arg(opt->block_size > 0, "partition_domain: block_size must be positive");
    if (method != SI_METHOD_RAS)
      check_arg(std::isfinite(opt->alpha), "run_schwarz_level: alpha must be finite");
    validate_local(*opt);
  });
}

si_status si_create(int device, si_ctx** out) {
  return guard([&] {
    check_arg(out != nullptr, "si_create: out must not be null");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(SI_ERR_NO_DEVICE, "no CUDA device available");
    }
    check_arg(device >= 0 && device < n, "si_create: device index out of range");
    auto* c = new si_ctx();
    c->device = device;
    try {
      CK(cudaSetDevice(device));
      CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
      ensure_red(*c, 64);
      CK(cudaHostAlloc(&c->host_cnt, sizeof(unsigned long long) * 8, cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->dev_cnt), c->host_cnt, 0));
      if (const char* e = std::getenv("SI_SWEEP_WARPS64")) c->sweep_nw64 = std::atoi(e);
      if (const char* e = std::getenv("SI_SWEEP_WARPS32")) c->sweep_nw32 = std::atoi(e);
    } catch (...) {
      si_destroy(c);
      throw;
    }
    *out = c;
  });
}

void si_destroy(si_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->own_stream) cudaStreamSynchronize(c->own_stream);
  for (auto& l : c->levels) {
    l.mask.release();
    l.b.release();
    l.u0.release();
    l.u1.release();
  }
  for (DevBuf* b : {&c->in_f, &c->in_mask, &c->in_ref, &c->out_img, &c->aux, &c->red_partials,
                    &c->red_out, &c->counters, &c->ticket, &c->scratch, &c->cg_rhs, &c->cg_x,
                    &c->cg_r, &c->cg_p, &c->cg_q})
    b->release();
  c->vz.release();
  c->stager.reset();
  c->drain_stager.reset();
  c->pack_pool.reset();
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  for (cudaStream_t cs : c->cap_stream)
    if (cs) cudaStreamDestroy(cs);
  if (c->host_state) cudaFreeHost(c->host_state);
  if (c->stripe_host) cudaFreeHost(c->stripe_host);
  if (c->stripe_log) cudaFreeHost(c->stripe_log);
  for (int k = 0; k < 2; ++k) {
    if (c->frame_host[k]) cudaFreeHost(c->frame_host[k]);
    if (c->frame_done[k]) cudaEventDestroy(c->frame_done[k]);
  }
  c->lvl_state.release();
  c->lvl_sums.release();
  for (auto& l : c->stripe_levels)
    for (DevBuf* b : {&l.mask, &l.b, &l.u0, &l.u1}) b->release();
  for (DevBuf* b : {&c->stripe_send, &c->stripe_recv, &c->stripe_in_f, &c->stripe_in_mask,
                    &c->stripe_out, &c->stripe_state})
    b->release();
  for (void* b : c->pack_buf)
    if (b) cudaFreeHost(b);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.start);
    cudaEventDestroy(p.stop);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    c->slot_f[k].release();
    c->slot_mask[k].release();
    c->slot_out[k].release();
    for (cudaEvent_t e : {c->ev_h2d[k], c->ev_solved[k], c->ev_d2h[k]})
      if (e) cudaEventDestroy(e);
  }
  if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  if (c->host_red) cudaFreeHost(c->host_red);
  if (c->host_cnt) cudaFreeHost(c->host_cnt);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
}

si_status si_trim(si_ctx* c) {
  return guard([&] {
    check_arg(c != nullptr, "null context");
    set_device(c);
    CK(cudaStreamSynchronize(c->own_stream));
    for (auto& g : c->graphs)
      if (g.exec) CK(cudaGraphExecDestroy(g.exec));
    c->graphs.clear();
    for (auto& l : c->levels) {
      l.mask.release();
      l.b.release();
      l.u0.release();
      l.u1.release();
    }
    for (DevBuf* b : {&c->in_f, &c->in_mask, &c->in_ref, &c->out_img, &c->aux}) b->release();
    c->vz.release();
    for (auto& l : c->stripe_levels)
      for (DevBuf* b : {&l.mask, &l.b, &l.u0, &l.u1}) b->release();
    for (DevBuf* b : {&c->stripe_send, &c->stripe_recv, &c->stripe_in_f, &c->stripe_in_mask,
                      &c->stripe_out})
      b->release();
  });
}

si_status si_run_method_device(si_ctx* ctx, int method, const double* d_f, const uint8_t* d_mask,
                               int w, int h, int c, const si_options* opt,
                               const double* d_reference, double* d_out, si_report* report,
                               si_trace_fn trace, void* user, void* stream) {
  si_report local;
  si_report* rep = report ? report : &local;
  clear_report(rep);
  const auto t0 = Clock::now();
  si_status st = guard([&] {
    check_arg(ctx && d_f && d_mask && d_out, "null argument");
    si_options o;
    if (opt) o = *opt; else si_default_options(&o);
    set_device(ctx);
    run_device(ctx, method, d_f, d_mask, w, h, c, o, d_reference, d_out, rep, trace, user,
               pick_stream(ctx, stream), t0);
  });
  rep->elapsed_ms = ms_since(t0);
  return st;
}

si_status si_run_method(si_ctx* ctx, int method, const double* f, const uint8_t* mask, int w,
                        int h, int c, const si_options* opt, const double* reference, double* out,
                        si_report* report, si_trace_fn trace, void* user) {
  si_report local;
  si_report* rep = report ? report : &local;
  clear_report(rep);
  const auto t0 = Clock::now();
  si_status st = guard([&] {
    check_arg(ctx && f && mask && out, "null argument");
    check_dims(w, h, c);
    si_options o;
    if (opt) o = *opt; else si_default_options(&o);
    set_device(ctx);
    const size_t n = static_cast<size_t>(w) * h;
    Ctx x{*ctx, ctx->own_stream};
    ctx->in_f.ensure(n * c * sizeof(double));
    ctx->in_mask.ensure(n);
    ctx->out_img.ensure(n * c * sizeof(double));
    KnownSamples ks{};
    const bool sparse = upload_known(x, f, mask, n, c, &ks);
    if (!sparse) h2d(x, ctx->in_f.ptr, f, n * c * sizeof(double));
    h2d(x, ctx->in_mask.ptr, mask, n);
    long long up = static_cast<long long>(sparse ? ks.bytes : n * c * sizeof(double)) + n;
    const double* d_ref = nullptr;
    if (reference) {
      ctx->in_ref.ensure(n * c * sizeof(double));
      h2d(x, ctx->in_ref.ptr, reference, n * c * sizeof(double));
      d_ref = ctx->in_ref.as<double>();
      up += static_cast<long long>(n * c * sizeof(double));
    }
    // A fresh pageable output buffer costs a page fault per 4 KB on its first
    // write; take them on host threads while the device solves (every input
    // has been read by now), so the result copy-out runs at memcpy speed.
    std::future<void> prefault;
    const size_t out_bytes = n * c * sizeof(double);
    if (out_bytes >= (size_t(16) << 20) && !sib::host_is_pinned(out)) {
      if (!ctx->pack_pool) ctx->pack_pool = std::make_unique<sib::CopyPool>(pack_threads());
      prefault = std::async(std::launch::async, [ctx, out, out_bytes] {
        char* base = reinterpret_cast<char*>(out);
        const size_t pages = (out_bytes + 4095) / 4096;
        ctx->pack_pool->run([&](int k, int parts) {
          for (size_t pg = pages * k / parts; pg < pages * (k + 1) / parts; ++pg)
            *reinterpret_cast<volatile char*>(base + pg * 4096) = 0;
        });
      });
    }
    try {
      run_device(ctx, method, ctx->in_f.as<double>(), ctx->in_mask.as<uint8_t>(), w, h, c, o,
                 d_ref, ctx->out_img.as<double>(), rep, trace, user, x.s, t0,
                 sparse ? &ks : nullptr);
    } catch (...) {
      if (prefault.valid()) prefault.wait();
      throw;
    }
    if (prefault.valid()) prefault.get();
    d2h(x, out, ctx->out_img.ptr, out_bytes);
    rep->h2d_bytes = up;
    rep->d2h_bytes = static_cast<long long>(n * c * sizeof(double));
  });
  rep->elapsed_ms = ms_since(t0);
  return st;
}

si_status si_run_method_batch(si_ctx* ctx, int method, int n, const double* const* f,
                              const uint8_t* const* mask, int w, int h, int c,
                              const si_options* opt, double* const* out, si_report* reports) {
  return guard([&] {
    check_arg(ctx && f && mask && out && n >= 0, "null argument");
    run_batch(ctx, method, n, reinterpret_cast<const void* const*>(f), mask, w, h, c, opt,
              reinterpret_cast<void* const*>(out), reports, false);
  });
}

si_status si_run_pnm_batch(si_ctx* ctx, int method, int n, const uint8_t* const* pixels,
                           const uint8_t* const* mask_pbm, int w, int h, int c,
                           const si_options* opt, uint8_t* const* out_pixels, si_report* reports) {
  return guard([&] {
    check_arg(ctx && pixels && mask_pbm && out_pixels && n >= 0, "null argument");
    check_arg(c == 1 || c == 3, "write_pnm: only 1- or 3-channel images are supported");
    run_batch(ctx, method, n, reinterpret_cast<const void* const*>(pixels), mask_pbm, w, h, c,
              opt, reinterpret_cast<void* const*>(out_pixels), reports, true);
  });
}

}  // extern "C"

// ---------------------------------------------------------------- building blocks
namespace {

// splitmix64
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// div_by_recip(a, b, RN(1/b)) == a / b over random normal doubles/floats,
// including significands near all-ones; counts mismatches.
__global__ void selftest_division_kernel(long long n, unsigned long long seed,
                                         unsigned long long* bad) {
  unsigned long long local = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long ra = mix64(seed ^ (2 * i)), rb = mix64(seed ^ (2 * i + 1));
    // exponents in [2^-60, 2^60], random significands (every 8th b all-ones-ish)
    const unsigned long long ea = 1023 - 60 + (ra >> 57) % 121, eb = 1023 - 60 + (rb >> 57) % 121;
    unsigned long long mb = rb & 0xfffffffffffffull;
    if ((i & 7) == 0) mb |= 0xffffffffff000ull;
    const double a = __longlong_as_double((long long)((ea << 52) | (ra & 0xfffffffffffffull)));
    const double b = __longlong_as_double((long long)((eb << 52) | mb));
    if (div_by_recip(a, b, recip_rn(b)) != a / b) ++local;
    const float af = (float)a * 1e-3f, bf = (float)b * 1e-3f;
    if (bf != 0.0f && isfinite(af) && isfinite(bf) && div_by_recip(af, bf, recip_rn(bf)) != af / bf)
      ++local;
  }
  if (local) atomicAdd(bad, local);
}

// LocalOperator::apply on one block (schwarz.hpp:57-75) with the diagonal of
// build_local_operator (schwarz.hpp:115-130); one thread per block cell.
__global__ void local_operator_kernel(const uint8_t* mask, int W, int H, int x0, int y0, int B,
                                      int ras, double am1, const double* v, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * B) return;
  const int ly = i / B, lx = i % B;
  const int gx = x0 + lx, gy = y0 + ly;
  if (mask[static_cast<size_t>(gy) * W + gx]) {
    out[i] = v[i];
    return;
  }
  double acc = robin_diag<double>(gx, gy, lx, ly, B, W, H, am1, ras) * v[i];
  if (lx > 0) acc -= v[i - 1];
  if (lx + 1 < B) acc -= v[i + 1];
  if (ly > 0) acc -= v[i - B];
  if (ly + 1 < B) acc -= v[i + B];
  out[i] = acc;
}

template <typename T>
T* upload(Ctx& x, DevBuf& buf, const T* host, size_t count) {
  buf.ensure(count * sizeof(T) + 16);
  h2d(x, buf.ptr, host, count * sizeof(T));
  return buf.as<T>();
}

template <typename T>
void download(Ctx& x, T* host, const void* dev, size_t count) {
  d2h(x, host, dev, count * sizeof(T));
}

si_options opts_or_default(const si_options* opt) {
  si_options o;
  if (opt) o = *opt; else si_default_options(&o);
  return o;
}

}  // namespace

extern "C" {

si_status si_solve_schwarz(si_ctx* ctx, const double* f, const uint8_t* mask, int w, int h, int c,
                           int block_size, int overlap, int flavour, const si_options* opt,
                           const double* reference, double* out, si_report* report,
                           si_trace_fn trace, void* user) {
  si_report local;
  si_report* rep = report ? report : &local;
  clear_report(rep);
  const auto t0 = Clock::now();
  si_status st = guard([&] {
    check_arg(ctx && f && mask && out, "null argument");
    check_dims(w, h, c);
    const si_options o = opts_or_default(opt);
    check_arg(o.tolerance > 0.0, "solve_schwarz: tolerance must be positive");
    check_arg(flavour == SI_FLAVOUR_RAS || flavour == SI_FLAVOUR_ORAS, "unknown flavour");
    validate_partition(w, h, block_size, overlap);
    si_options oo = o;
    oo.coarse_tolerance = 1.0;  // single level: unused
    validate_options_common(oo);
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    const size_t n = static_cast<size_t>(w) * h;
    const double* d_f = upload(x, ctx->in_f, f, n * c);
    const uint8_t* d_m = upload(x, ctx->in_mask, mask, n);
    const double* d_ref = reference ? upload(x, ctx->in_ref, reference, n * c) : nullptr;
    ctx->out_img.ensure(n * c * sizeof(double));
    LocalPrecision lp(*ctx, oo.precision);
    begin_counters(x);
    Trace tr{trace, user, t0};
    if (oo.precision == SI_PRECISION_FP32)
      multilevel_device<float>(x, 1, flavour, d_f, d_m, w, h, c, oo, d_ref,
                               ctx->out_img.as<double>(), rep, tr, block_size, overlap);
    else
      multilevel_device<double>(x, 1, flavour, d_f, d_m, w, h, c, oo, d_ref,
                                ctx->out_img.as<double>(), rep, tr, block_size, overlap);
    end_counters(x, rep);
    download(x, out, ctx->out_img.ptr, n * c);
  });
  rep->elapsed_ms = ms_since(t0);
  return st;
}

si_status si_run_schwarz_level(si_ctx* ctx, const uint8_t* mask, int w, int h, int c,
                               const double* b, double* u, int block_size, int overlap,
                               double r0_norm, double tolerance, int flavour,
                               const si_options* opt, si_report* report, si_trace_fn trace,
                               void* user) {
  si_report local;
  si_report* rep = report ? report : &local;
  clear_report(rep);
  const auto t0 = Clock::now();
  si_status st = guard([&] {
    check_arg(ctx && mask && b && u, "null argument");
    check_arg(c > 0, "run_schwarz_level: channel count mismatch");
    validate_partition(w, h, block_size, overlap);
    check_arg(flavour == SI_FLAVOUR_RAS || std::isfinite(opt ? opt->alpha : 0.25),
              "run_schwarz_level: alpha must be finite");
    const si_options o = opts_or_default(opt);
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    prepare_red(x, c);
    const size_t n = static_cast<size_t>(w) * h;
    if (ctx->levels.empty()) ctx->levels.resize(1);
    auto& lb = ctx->levels[0];
    lb.u0.ensure(n * c * sizeof(double));
    lb.u1.ensure(n * c * sizeof(double));
    const uint8_t* d_m = upload(x, ctx->in_mask, mask, n);
    const double* d_b = upload(x, ctx->in_f, b, n * c);
    CK(cudaMemcpyAsync(lb.u0.ptr, u, n * c * sizeof(double), cudaMemcpyHostToDevice, x.s));
    LevelView<double> V{w, h, d_m, d_b, {lb.u0.as<double>(), lb.u1.as<double>()}, 0};
    begin_counters(x);
    Trace tr{trace, user, t0};
    double r0 = r0_norm;
    const LevelOutcome oc = run_level<double>(x, V, c, block_size, overlap, &r0, false, tolerance,
                                              flavour, o, false, true, tr, nullptr, rep);
    end_counters(x, rep);
    download(x, u, V.u[V.cur], n * c);
    rep->depth = 1;
    rep->iterations = rep->level_iterations[0] = oc.iterations;
    rep->final_relative_residual = rep->level_final_rel[0] = oc.final_rel;
    rep->converged = rep->level_converged[0] = oc.converged;
  });
  rep->elapsed_ms = ms_since(t0);
  return st;
}

si_status si_canonical_r0(si_ctx* ctx, const uint8_t* mask, int w, int h, int c, const double* b,
                          int normalizer, double* r0_norm) {
  return guard([&] {
    check_arg(ctx && mask && b && r0_norm, "null argument");
    check_dims(w, h, c);
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    prepare_red(x, c);
    const size_t n = static_cast<size_t>(w) * h;
    const uint8_t* d_m = upload(x, ctx->in_mask, mask, n);
    const double* d_b = upload(x, ctx->in_f, b, n * c);
    launch_residual<double>(x, d_m, d_b, d_b, w, h, c, normalizer == 1 ? 1 : 0, ctx->dev_red,
                            false);
    sync(x);
    *r0_norm = joint_norm(ctx->host_red, c);
  });
}

si_status si_schwarz_sweep(si_ctx* ctx, const uint8_t* mask, int w, int h, int c, const double* b,
                           const double* u, int block_size, int overlap, int flavour,
                           const si_options* opt, double* u_new, long long* failures,
                           long long* cg_iterations) {
  return guard([&] {
    check_arg(ctx && mask && b && u && u_new, "null argument");
    check_dims(w, h, c);
    validate_partition(w, h, block_size, overlap);
    const si_options o = opts_or_default(opt);
    validate_local(o);
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    const size_t n = static_cast<size_t>(w) * h;
    if (ctx->levels.empty()) ctx->levels.resize(1);
    auto& lb = ctx->levels[0];
    lb.u0.ensure(n * c * sizeof(double));
    lb.u1.ensure(n * c * sizeof(double));
    const uint8_t* d_m = upload(x, ctx->in_mask, mask, n);
    const double* d_b = upload(x, ctx->in_f, b, n * c);
    CK(cudaMemcpyAsync(lb.u0.ptr, u, n * c * sizeof(double), cudaMemcpyHostToDevice, x.s));
    begin_counters(x);
    const LocalCfg lc{o.local_tolerance, o.local_max_iterations, o.local_check_interval};
    launch_sweep<double>(x, d_m, d_b, lb.u0.as<double>(), lb.u1.as<double>(), w, h, c, block_size,
                         overlap, flavour, o.alpha, lc, false,
                         ctx->counters.as<unsigned long long>());
    download(x, u_new, lb.u1.ptr, n * c);
    publish_counters(x, 2);
    if (failures) *failures = static_cast<long long>(ctx->host_cnt[0]);
    if (cg_iterations) *cg_iterations = static_cast<long long>(ctx->host_cnt[1]);
  });
}

si_status si_residual_sumsq(si_ctx* ctx, const uint8_t* mask, int w, int h, int c,
                            const double* u, const double* b, double* sumsq) {
  return guard([&] {
    check_arg(ctx && mask && u && b && sumsq, "null argument");
    check_dims(w, h, c);
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    prepare_red(x, c);
    const size_t n = static_cast<size_t>(w) * h;
    const uint8_t* d_m = upload(x, ctx->in_mask, mask, n);
    const double* d_b = upload(x, ctx->in_f, b, n * c);
    const double* d_u = upload(x, ctx->aux, u, n * c);
    launch_residual<double>(x, d_m, d_u, d_b, w, h, c, 0, ctx->dev_red, false);
    sync(x);
    std::memcpy(sumsq, ctx->host_red, sizeof(double) * c);
  });
}

si_status si_restrict_level(si_ctx* ctx, const uint8_t* mask, const double* values, int w, int h,
                            int c, int averaging, uint8_t* coarse_mask, double* coarse_values) {
  return guard([&] {
    check_arg(ctx && mask && values && coarse_mask && coarse_values, "null argument");
    check_dims(w, h, c);
    check_arg(w >= 2 && h >= 2, "restrict_level: fine grid must be at least 2x2");
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    const size_t n = static_cast<size_t>(w) * h;
    const int cw = (w + 1) / 2, ch = (h + 1) / 2;
    const size_t cn = static_cast<size_t>(cw) * ch;
    const uint8_t* d_m = upload(x, ctx->in_mask, mask, n);
    const double* d_v = upload(x, ctx->in_f, values, n * c);
    ctx->out_img.ensure(cn * c * sizeof(double));
    ctx->aux.ensure(cn + 16);
    launch_restrict<double>(x, d_m, d_v, w, h, c, averaging, ctx->aux.as<uint8_t>(),
                            ctx->out_img.as<double>());
    CK(cudaGetLastError());
    download(x, coarse_mask, ctx->aux.ptr, cn);
    download(x, coarse_values, ctx->out_img.ptr, cn * c);
  });
}

si_status si_prolongate(si_ctx* ctx, const double* coarse, int cw, int ch, int fw, int fh,
                        double* fine) {
  return guard([&] {
    check_arg(ctx && coarse && fine, "null argument");
    check_arg(cw == (fw + 1) / 2 && ch == (fh + 1) / 2,
              "prolongate: coarse grid is not the dyadic parent of the fine grid");
    check_arg(cw > 0 && ch > 0, "prolongate: coarse vector length mismatch");
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    const size_t fn = static_cast<size_t>(fw) * fh;
    const double* d_c = upload(x, ctx->in_f, coarse, static_cast<size_t>(cw) * ch);
    ctx->out_img.ensure(fn * sizeof(double));
    launch_prolong<double>(x, d_c, cw, ch, fw, fh, 1, nullptr, nullptr, ctx->out_img.as<double>());
    CK(cudaGetLastError());
    download(x, fine, ctx->out_img.ptr, fn);
  });
}

si_status si_local_operator_apply(si_ctx* ctx, const uint8_t* mask, int w, int h, int block_size,
                                  int overlap, int index, int flavour, double alpha,
                                  const double* v, double* out) {
  return guard([&] {
    check_arg(ctx && mask && v && out, "null argument");
    validate_partition(w, h, block_size, overlap);
    const Axis ax = Axis::make(w, block_size, overlap), ay = Axis::make(h, block_size, overlap);
    check_arg(index >= 0 && index < ax.count * ay.count,
              "build_local_operator: subdomain index out of range");
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    const int B = block_size;
    const size_t cells = static_cast<size_t>(B) * B;
    const uint8_t* d_m = upload(x, ctx->in_mask, mask, static_cast<size_t>(w) * h);
    const double* d_v = upload(x, ctx->in_f, v, cells);
    ctx->out_img.ensure(cells * sizeof(double));
    const int bx = index % ax.count, by = index / ax.count;
    ++x.c.launch_count;
    local_operator_kernel<<<grid_for(cells, 256, 1 << 20), 256, 0, x.s>>>(
        d_m, w, h, ax.anchor(bx), ay.anchor(by), B, flavour == SI_FLAVOUR_RAS, alpha - 1.0, d_v,
        ctx->out_img.as<double>());
    CK(cudaGetLastError());
    download(x, out, ctx->out_img.ptr, cells);
  });
}

si_status si_pack_known_samples(const double* f, const uint8_t* mask, int w, int h, int c,
                                uint32_t* tile_off, double* vals, long long* K) {
  return guard([&] {
    check_arg(mask && tile_off && K && (f || !vals), "null argument");
    check_dims(w, h, c);
    static_assert(SI_KNOWN_TILE == sib::kKnownTile, "header and host tile sizes differ");
    static sib::CopyPool pool;
    static std::mutex m;
    std::lock_guard<std::mutex> g(m);
    const size_t n = static_cast<size_t>(w) * h;
    const size_t k = sib::count_known_tiles(pool, mask, n, tile_off);
    if (vals) sib::gather_known(pool, mask, f, n, c, tile_off, k, vals);
    *K = static_cast<long long>(k);
  });
}

si_status si_partition_domain(int w, int h, int block_size, int overlap, int* blocks_x,
                              int* blocks_y, int* rects, int rects_capacity) {
  return guard([&] {
    validate_partition(w, h, block_size, overlap);
    const Axis ax = Axis::make(w, block_size, overlap), ay = Axis::make(h, block_size, overlap);
    if (blocks_x) *blocks_x = ax.count;
    if (blocks_y) *blocks_y = ay.count;
    if (!rects) return;
    int k = 0;
    for (int by = 0; by < ay.count; ++by)
      for (int bx = 0; bx < ax.count; ++bx, ++k) {
        if (k >= rects_capacity) return;
        int* r = rects + 8 * k;
        r[0] = ax.anchor(bx);
        r[1] = ay.anchor(by);
        r[2] = block_size;
        r[3] = block_size;
        r[4] = ax.owned_begin(bx);
        r[5] = ay.owned_begin(by);
        r[6] = ax.owned_end(bx);
        r[7] = ay.owned_end(by);
      }
  });
}

double si_joint_norm(const double* sumsq, int c) { return joint_norm(sumsq, c); }

si_status si_selftest(si_ctx* ctx, int which, long long n, long long* failures) {
  return guard([&] {
    check_arg(ctx && failures && which == 0 && n >= 0, "invalid self-test");
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    begin_counters(x);
    ++x.c.launch_count;
    selftest_division_kernel<<<148 * 8, 256, 0, x.s>>>(n, 0x5eedull,
                                                      ctx->counters.as<unsigned long long>());
    CK(cudaGetLastError());
    publish_counters(x, 1);
    *failures = static_cast<long long>(ctx->host_cnt[0]);
  });
}

si_status si_psnr(const double* u, const double* f, int w, int h, int c, double* psnr_db) {
  return guard([&] {
    check_arg(u && f && psnr_db, "null argument");
    check_dims(w, h, c);
    const size_t n = static_cast<size_t>(w) * h;
    std::vector<double> mse(c);
    for (int k = 0; k < c; ++k) {
      double acc = 0.0;
      for (size_t i = 0; i < n; ++i) {
        const double d = 255.0 * (u[k * n + i] - f[k * n + i]);
        acc += d * d;
      }
      mse[k] = acc;
    }
    *psnr_db = psnr_from_sq(mse, n);
  });
}

si_status si_set_profiling(si_ctx* ctx, int enabled) {
  return guard([&] {
    check_arg(ctx != nullptr, "null context");
    ctx->profiling = enabled != 0;
  });
}

si_status si_get_kernel_stats(si_ctx* ctx, si_kernel_stats* out, int reset) {
  return guard([&] {
    check_arg(ctx && out, "null argument");
    set_device(ctx);
    if (!ctx->pending.empty()) resolve_events(*ctx);
    *out = ctx->stats;
    out->total_launches = ctx->launch_count;
    if (reset) {
      ctx->stats = si_kernel_stats{};
      ctx->launch_count = 0;
    }
  });
}

si_status si_host_alloc(size_t bytes, void** ptr) {
  return guard([&] {
    check_arg(ptr != nullptr, "null argument");
    CK(cudaMallocHost(ptr, bytes));
  });
}

si_status si_host_free(void* ptr) {
  return guard([&] { CK(cudaFreeHost(ptr)); });
}

}  // extern "C"

extern "C" {

void si_default_densify_options(si_densify_options* o) {
  if (!o) return;
  o->initial_density = 0.0;
  o->cell_fraction = 0.20;
  o->inner_tolerance = 1e-3;
  o->max_sweeps = 100;
  si_default_options(&o->solve);
}

si_status si_voronoi_densify(si_ctx* ctx, const double* f, int w, int h, int c,
                             double target_density, uint64_t seed, const si_densify_options* opt,
                             uint8_t* mask_out, int* sweeps, int* reached_target) {
  return guard([&] {
    check_arg(ctx && f && mask_out && sweeps && reached_target, "null argument");
    set_device(ctx);
    si_densify_options d;
    if (opt)
      d = *opt;
    else
      si_default_densify_options(&d);
    voronoi_densify(ctx, f, w, h, c, target_density, seed, d, mask_out, sweeps, reached_target);
  });
}

si_status si_assign_nearest_site(si_ctx* ctx, const uint8_t* mask, int w, int h, int32_t* sites,
                                 int32_t* site_of, int* num_sites) {
  return guard([&] {
    check_arg(ctx && mask && sites && site_of && num_sites, "null argument");
    check_arg(w > 0 && h > 0, "InpaintingMask: dimensions must be positive");
    set_device(ctx);
    Ctx x{*ctx, ctx->own_stream};
    const size_t n = static_cast<size_t>(w) * h;
    auto& z = ctx->vz;
    z.mask.ensure(n);
    CK(cudaMemcpyAsync(z.mask.ptr, mask, n, cudaMemcpyHostToDevice, x.s));
    const int m = assign_device(x, z.mask.as<uint8_t>(), w, h);
    CK(cudaMemcpyAsync(sites, z.sites.ptr, static_cast<size_t>(m) * 4, cudaMemcpyDeviceToHost, x.s));
    CK(cudaMemcpyAsync(site_of, z.site_of.ptr, n * 4, cudaMemcpyDeviceToHost, x.s));
    sync(x);
    *num_sites = m;
  });
}

}  // extern "C"

// ====================================================================== stripes
#include "stripes.cuh"

namespace {

StripeLayout checked_layout(int method, int w, int h, int c, const si_options& o, int world,
                            int rank) {
  check_method(method);
  check_dims(w, h, c);
  validate_options_common(o);
  check_arg(world >= 1 && rank >= 0 && rank < world, "stripes: invalid world/rank");
  if (method == SI_METHOD_CG || method == SI_METHOD_MLCG)
    fail(SI_ERR_UNSUPPORTED, "stripes: the CG level solver is not striped (Schwarz methods only)");
  check_arg(levels_for(method, o) >= 1, "build_pyramid: levels must be >= 1");
  return stripe_layout(w, h, o, levels_for(method, o), world, rank);
}

// One rank's solve on device rows (see si_run_method_striped_device).
void run_striped_device(si_ctx* ctx, si_stripe_comm* comm, int method, const double* d_f,
                        const uint8_t* d_mask, int w, int h, int c, const si_options& o,
                        double* d_out, si_report* rep, si_trace_fn trace, void* user,
                        cudaStream_t s) {
  const StripeLayout P = checked_layout(method, w, h, c, o, comm->world, comm->rank);
  Ctx x{*ctx, s};
  LocalPrecision lp(*ctx, o.precision);
  begin_counters(x);
  Trace tr{trace, user, Clock::now()};
  const int flavour = flavour_for(method);
  ctx->stripe_result = nullptr;
  ctx->stripe_result_rows = 0;
  check_arg(d_out != nullptr || o.precision != SI_PRECISION_FP32,
            "stripes: an FP32 solve needs an output buffer (its rows are float in place)");
  if (o.precision == SI_PRECISION_FP32)
    stripe_solve_device<float>(x, *comm, P, flavour, d_f, d_mask, c, o, d_out, rep, tr);
  else
    stripe_solve_device<double>(x, *comm, P, flavour, d_f, d_mask, c, o, d_out, rep, tr);
  sync(x);
}

// Host buffers: upload the level-0 store rows, solve, download the own rows.
void run_striped_host(si_ctx* ctx, si_stripe_comm* comm, int method, const double* f,
                      const uint8_t* mask, int w, int h, int c, const si_options& o, double* out,
                      si_report* rep, si_trace_fn trace, void* user) {
  const StripeLayout P = checked_layout(method, w, h, c, o, comm->world, comm->rank);
  const Span st = P.L[0].store[comm->rank], own = P.L[0].own[comm->rank];
  const size_t W = static_cast<size_t>(w), N = W * h;
  const size_t rows = std::max(0, st.hi - st.lo), orows = std::max(0, own.hi - own.lo);
  set_device(ctx);
  Ctx x{*ctx, ctx->own_stream};
  ctx->stripe_in_f.ensure(std::max<size_t>(1, rows * W * c) * sizeof(double));
  ctx->stripe_in_mask.ensure(std::max<size_t>(1, rows * W));
  // double storage: the own rows are copied to the host straight from the
  // level storage (no device output pass)
  const bool in_place = o.precision != SI_PRECISION_FP32;
  if (!in_place) ctx->stripe_out.ensure(std::max<size_t>(1, orows * W * c) * sizeof(double));
  const auto t0 = Clock::now();
  for (int k = 0; k < c && rows; ++k)
    h2d(x, ctx->stripe_in_f.as<double>() + k * rows * W, f + k * N + st.lo * W,
        rows * W * sizeof(double));
  if (rows) h2d(x, ctx->stripe_in_mask.ptr, mask + st.lo * W, rows * W);
  run_striped_device(ctx, comm, method, ctx->stripe_in_f.as<double>(),
                     ctx->stripe_in_mask.as<uint8_t>(), w, h, c, o,
                     in_place ? nullptr : ctx->stripe_out.as<double>(), rep, trace, user,
                     ctx->own_stream);
  const double* res = in_place ? static_cast<const double*>(ctx->stripe_result)
                               : ctx->stripe_out.as<double>();
  const size_t stride = in_place ? ctx->stripe_result_stride : orows * W;
  for (int k = 0; k < c && orows; ++k)
    d2h(x, out + k * N + own.lo * W, res + k * stride, orows * W * sizeof(double));
  rep->h2d_bytes = static_cast<long long>(rows * W * (c * sizeof(double) + 1));
  rep->d2h_bytes = static_cast<long long>(orows * W * c * sizeof(double));
  rep->elapsed_ms = ms_since(t0);
}

}  // namespace

extern "C" {

si_status si_stripe_level_plan(int method, int w, int h, int c, const si_options* opt, int world,
                               int rank, int* depth, int* out) {
  return guard([&] {
    check_arg(depth && out, "null argument");
    const si_options o = opts_or_default(opt);
    const StripeLayout P = checked_layout(method, w, h, c, o, world, rank);
    *depth = P.depth;
    for (int l = 0; l < P.depth; ++l) {
      const StripeLevel& S = P.L[l];
      const int v[SI_STRIPE_PLAN_INTS] = {S.k0, S.k1, S.own[rank].lo, S.own[rank].hi,
                                         S.win[rank].lo, S.win[rank].hi, S.need[rank].lo,
                                         S.need[rank].hi, S.store[rank].lo, S.store[rank].hi,
                                         S.block, S.overlap};
      std::memcpy(out + l * SI_STRIPE_PLAN_INTS, v, sizeof v);
    }
  });
}

si_status si_nccl_unique_id(unsigned char* id) {
  return guard([&] {
    check_arg(id != nullptr, "null argument");
    static_assert(sizeof(ncclUniqueId) == SI_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof u);
  });
}

si_status si_stripe_comm_init_nccl(si_ctx* ctx, int world, int rank, const unsigned char* id,
                                   si_stripe_comm** out) {
  return guard([&] {
    check_arg(ctx && id && out, "null argument");
    check_arg(world >= 1 && rank >= 0 && rank < world, "stripes: invalid world/rank");
    set_device(ctx);
    auto comm = std::make_unique<NcclComm>();
    comm->world = world;
    comm->rank = rank;
    comm->device = ctx->device;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    nccl_check(nccl().CommInitRank(&comm->comm, world, u, rank), "ncclCommInitRank");
    *out = comm.release();
  });
}

si_status si_stripe_comm_init_local(si_ctx* const* ctxs, int world, si_stripe_comm** out) {
  return guard([&] {
    check_arg(ctxs && out && world >= 1, "null argument");
    int caller_dev = 0;
    CK(cudaGetDevice(&caller_dev));
    auto grp = std::make_shared<LocalGroup>();
    grp->world = world;
    grp->ready.assign(world, nullptr);
    grp->done.assign(world, nullptr);
    grp->posted.resize(world);
    grp->posted_vals.assign(world, nullptr);
    grp->posted_sends.assign(world, nullptr);
    for (int r = 0; r < world; ++r) {
      check_arg(ctxs[r] != nullptr, "null context");
      set_device(ctxs[r]);
      CK(cudaEventCreateWithFlags(&grp->ready[r], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&grp->done[r], cudaEventDisableTiming));
    }
    // ranks on different GPUs of the process pull each other's rows over
    // NVLink: peer access both ways where the devices support it (the
    // caller's current device is restored)
    for (int r = 0; r < world; ++r)
      for (int q = 0; q < world; ++q) {
        const int a = ctxs[r]->device, b = ctxs[q]->device;
        if (a == b) continue;
        int can = 0;
        CK(cudaDeviceCanAccessPeer(&can, a, b));
        if (!can) continue;
        CK(cudaSetDevice(a));
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
        else CK(e);
      }
    CK(cudaSetDevice(caller_dev));
    for (int r = 0; r < world; ++r) {
      auto comm = new LocalComm();
      comm->world = world;
      comm->rank = r;
      comm->device = ctxs[r]->device;
      comm->g = grp;
      out[r] = comm;
    }
  });
}

void si_stripe_comm_destroy(si_stripe_comm* comm) { delete comm; }

si_status si_stripe_result_rows(si_ctx* ctx, const double** rows, size_t* plane_stride,
                                int* n_rows) {
  return guard([&] {
    check_arg(ctx && rows && plane_stride && n_rows, "null argument");
    check_arg(ctx->stripe_result == nullptr || ctx->stripe_result_f64,
              "stripes: the last solve kept float rows");
    *rows = static_cast<const double*>(ctx->stripe_result);
    *plane_stride = ctx->stripe_result_stride;
    *n_rows = ctx->stripe_result_rows;
  });
}

si_status si_stripe_comm_set_speculation(si_stripe_comm* comm, int enabled) {
  return guard([&] {
    check_arg(comm != nullptr, "null argument");
    comm->speculate = enabled ? 1 : 0;
  });
}

si_status si_stripe_comm_counters(const si_stripe_comm* comm, long long* out) {
  return guard([&] {
    check_arg(comm && out, "null argument");
    out[0] = comm->solves;
    out[1] = comm->speculative;
    out[2] = comm->resumes;
  });
}

si_status si_run_method_striped(si_ctx* ctx, si_stripe_comm* comm, int method, const double* f,
                                const uint8_t* mask, int w, int h, int c, const si_options* opt,
                                double* out, si_report* report, si_trace_fn trace, void* user) {
  si_report scratch;
  si_report* rep = report ? report : &scratch;
  clear_report(rep);
  const si_status st = guard([&] {
    check_arg(ctx && comm && f && mask && out, "null argument");
    run_striped_host(ctx, comm, method, f, mask, w, h, c, opts_or_default(opt), out, rep, trace,
                     user);
  });
  if (st != SI_OK)
    if (auto* lc = dynamic_cast<LocalComm*>(comm)) lc->g->abort();  // release waiting peers
  return st;
}

si_status si_run_method_striped_device(si_ctx* ctx, si_stripe_comm* comm, int method,
                                       const double* d_f_rows, const uint8_t* d_mask_rows, int w,
                                       int h, int c, const si_options* opt, double* d_out_rows,
                                       si_report* report, void* stream) {
  si_report scratch;
  si_report* rep = report ? report : &scratch;
  clear_report(rep);
  const si_status st = guard([&] {
    check_arg(ctx && comm && d_f_rows && d_mask_rows, "null argument");
    set_device(ctx);
    const auto t0 = Clock::now();
    run_striped_device(ctx, comm, method, d_f_rows, d_mask_rows, w, h, c, opts_or_default(opt),
                       d_out_rows, rep, nullptr, nullptr, pick_stream(ctx, stream));
    rep->elapsed_ms = ms_since(t0);
  });
  if (st != SI_OK)
    if (auto* lc = dynamic_cast<LocalComm*>(comm)) lc->g->abort();
  return st;
}

si_status si_run_method_striped_local_device(si_stripe_comm* const* comms, si_ctx* const* ctxs,
                                             int world, int method,
                                             const double* const* d_f_rows,
                                             const uint8_t* const* d_mask_rows, int w, int h,
                                             int c, const si_options* opt,
                                             double* const* d_out_rows, si_report* reports,
                                             void* const* streams) {
  std::vector<si_status> sts(std::max(world, 1), SI_OK);
  std::vector<std::string> errs(std::max(world, 1));
  const si_status st = guard([&] {
    check_arg(comms && ctxs && d_f_rows && d_mask_rows && world >= 1, "null argument");
    auto* l0 = dynamic_cast<LocalComm*>(comms[0]);
    check_arg(l0 != nullptr && l0->world == world,
              "stripes: a group call needs the world's local communicators");
    for (int r = 0; r < world; ++r) {
      auto* lr = dynamic_cast<LocalComm*>(comms[r]);
      check_arg(lr && lr->g == l0->g && lr->rank == r,
                "stripes: communicators of one local group, in rank order");
    }
    l0->g->run_all([&](int r) {
      sts[r] = si_run_method_striped_device(ctxs[r], comms[r], method, d_f_rows[r],
                                            d_mask_rows[r], w, h, c, opt,
                                            d_out_rows ? d_out_rows[r] : nullptr,
                                            reports ? &reports[r] : nullptr,
                                            streams ? streams[r] : nullptr);
      if (sts[r] != SI_OK) errs[r] = g_last_error;
    });
  });
  if (st != SI_OK) return st;
  for (int pass = 0; pass < 2; ++pass)  // a failing rank first, then aborted peers
    for (int r = 0; r < world; ++r)
      if (sts[r] != SI_OK &&
          (pass == 1 || errs[r].find("aborted by another rank") == std::string::npos)) {
        g_last_error = errs[r];
        return sts[r];
      }
  return SI_OK;
}

si_status si_run_method_striped_group(si_ctx* const* ctxs, int world, int method, const double* f,
                                      const uint8_t* mask, int w, int h, int c,
                                      const si_options* opt, double* out, si_report* reports) {
  std::vector<si_stripe_comm*> comms(std::max(world, 1), nullptr);
  si_status st = si_stripe_comm_init_local(ctxs, world, comms.data());
  if (st != SI_OK) return st;
  std::vector<si_status> sts(world, SI_OK);
  std::vector<std::string> errs(world);
  std::vector<si_report> reps(world);
  {
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r)
      th.emplace_back([&, r] {
        sts[r] = si_run_method_striped(ctxs[r], comms[r], method, f, mask, w, h, c, opt, out,
                                       &reps[r], nullptr, nullptr);
        if (sts[r] != SI_OK) errs[r] = g_last_error;
      });
    for (auto& t : th) t.join();
  }
  for (auto* cm : comms) si_stripe_comm_destroy(cm);
  if (reports)
    for (int r = 0; r < world; ++r) reports[r] = reps[r];
  // the first failing rank's status (an aborted peer reports SI_ERR_RUNTIME)
  for (int r = 0; r < world; ++r)
    if (sts[r] != SI_OK && errs[r].find("aborted by another rank") == std::string::npos) {
      g_last_error = errs[r];
      return sts[r];
    }
  for (int r = 0; r < world; ++r)
    if (sts[r] != SI_OK) {
      g_last_error = errs[r];
      return sts[r];
    }
  return SI_OK;
}

}  // extern "C"
