// One very large image over G ranks (BASELINE configs[4]):
// the multilevel ORAS solve (multilevel.hpp:239-310) with every pyramid level
// split into horizontal stripes of whole block rows.
//
// Included at the end of solver.cu (it drives that file's launchers).
//
// Decomposition.  Level l is partitioned exactly as the single-GPU solve
// partitions it (clamped_partition, multilevel.hpp:146-150; partition_domain,
// partition.hpp:46-106); rank g takes the block rows [k0, k1) =
// [g*nby/G, (g+1)*nby/G) and owns the pixel rows those blocks own.  Every
// block's arithmetic is therefore the single-GPU one, and the image is
// bit-identical to it whenever the stop decisions agree (only the order of
// the global residual sum differs: per-rank partials, then a fixed rank
// order).
//
// Rows a rank holds per level (all in global row coordinates):
//   own   rows its blocks own (the owned rows of all ranks tile the level)
//   win   rows its sweeps and residual stencil read: block windows + 1 ghost
//         row, own +- 1
//   need  (l >= 1) rows of level l its prolongation onto level l-1's window
//         reads (multilevel.hpp:101-128 coordinates)
//   store hull(win, need, rows restricted into level l+1's store): the only
//         rows the rank allocates, ingests and restricts -- device memory
//         scales as 1/G plus a few halo rows.
// Data movement: the rank uploads f and the mask for its level-0 store rows
// only, restricts and prolongs only its own rows, and per outer iteration
//   residual over own rows -> all-gather of the G x C partial sums (+ r0) ->
//   the same stop decision on every rank (fixed rank order) -> sweep of its
//   block rows -> halo exchange (win \ own rows from their owners).
// After a level, rows of `need` outside `win` come from their owners; the
// finest level's own rows are the rank's share of the result.
//
// Communicators: NcclComm (one process per GPU: ncclAllGather and grouped
// ncclSend/ncclRecv on the solve stream, NCCL loaded at run time) and
// LocalComm (G ranks as host threads of one process, e.g. on one device:
// each rank pulls peers' rows with device copies ordered by events; no
// kernel ever waits on another rank's kernel).
#pragma once

#include <dlfcn.h>

#include <condition_variable>
#include <mutex>
#include <thread>

#include <nccl.h>

namespace {

struct Span {
  int lo = 0, hi = 0;
  bool empty() const { return hi <= lo; }
};

Span span_inter(Span a, Span b) { return {std::max(a.lo, b.lo), std::min(a.hi, b.hi)}; }
Span span_hull(Span a, Span b) {
  if (a.empty()) return b;
  if (b.empty()) return a;
  return {std::min(a.lo, b.lo), std::max(a.hi, b.hi)};
}
// a \ b as up to two spans
void span_minus(Span a, Span b, std::vector<Span>& out) {
  if (a.empty()) return;
  const Span i = span_inter(a, b);
  if (i.empty()) {
    out.push_back(a);
    return;
  }
  if (a.lo < i.lo) out.push_back({a.lo, i.lo});
  if (i.hi < a.hi) out.push_back({i.hi, a.hi});
}

struct StripeLevel {
  int w = 0, h = 0, block = 0, overlap = 0;
  int k0 = 0, k1 = 0;            // this rank's block rows
  std::vector<Span> own, win, need, store;  // per rank
};

struct StripeLayout {
  int world = 1, rank = 0, depth = 0;
  std::vector<StripeLevel> L;   // index 0 = finest
};

// prolongate's coarse rows for fine rows [a, b) (multilevel.hpp:101-128):
// y0 = floor(clamp(0.5 f - 0.25, 0, ch - 1)), y1 = min(y0 + 1, ch - 1).
Span prolong_source(Span fine, int ch) {
  if (fine.empty()) return {};
  auto c0 = [&](int f) {
    const double c = std::min(std::max(0.5 * f - 0.25, 0.0), static_cast<double>(ch - 1));
    return static_cast<int>(c);
  };
  return {c0(fine.lo), std::min(c0(fine.hi - 1) + 1, ch - 1) + 1};
}

// The whole decomposition, identical on every rank (pure function of the
// shapes and options).
StripeLayout stripe_layout(int w, int h, const si_options& o, int levels_req, int world,
                           int rank) {
  StripeLayout P;
  P.world = world;
  P.rank = rank;
  std::vector<int> lw{w}, lh{h};
  while (static_cast<int>(lw.size()) < levels_req && static_cast<int>(lw.size()) < SI_MAX_LEVELS) {
    if (lw.back() < 2 || lh.back() < 2) break;
    lw.push_back((lw.back() + 1) / 2);
    lh.push_back((lh.back() + 1) / 2);
  }
  P.depth = static_cast<int>(lw.size());
  P.L.resize(P.depth);
  for (int l = 0; l < P.depth; ++l) {
    StripeLevel& S = P.L[l];
    S.w = lw[l];
    S.h = lh[l];
    const Clamped cp = clamp_partition(S.w, S.h, o.block_size, o.overlap);
    S.block = cp.block;
    S.overlap = cp.overlap;
    const Axis ay = Axis::make(S.h, S.block, S.overlap);
    S.own.resize(world);
    S.win.resize(world);
    S.need.resize(world);
    S.store.resize(world);
    for (int g = 0; g < world; ++g) {
      const int k0 = static_cast<int>(static_cast<long long>(g) * ay.count / world);
      const int k1 = static_cast<int>(static_cast<long long>(g + 1) * ay.count / world);
      if (g == rank) {
        S.k0 = k0;
        S.k1 = k1;
      }
      if (k0 == k1) continue;
      S.own[g] = {ay.owned_begin(k0), ay.owned_end(k1 - 1)};
      S.win[g] = {std::max(0, std::min(ay.anchor(k0) - 1, S.own[g].lo - 1)),
                  std::min(S.h, std::max(ay.anchor(k1 - 1) + S.block + 1, S.own[g].hi + 1))};
    }
  }
  for (int l = 1; l < P.depth; ++l)
    for (int g = 0; g < world; ++g)
      P.L[l].need[g] = prolong_source(P.L[l - 1].win[g], P.L[l].h);
  for (int g = 0; g < world; ++g) {
    for (int l = P.depth - 1; l >= 0; --l) {
      StripeLevel& S = P.L[l];
      Span st = span_hull(S.win[g], S.need[g]);
      if (l + 1 < P.depth) {
        const Span up = P.L[l + 1].store[g];
        if (!up.empty()) st = span_hull(st, {2 * up.lo, std::min(2 * up.hi, S.h)});
      }
      S.store[g] = st;
    }
  }
  return P;
}

// One row transfer of a level: rows [lo, hi) between this rank and `peer`.
struct RowXfer {
  int peer, lo, hi;
};

// A level buffer as the communicator sees it: planar, C channels, rows
// [lo, hi) of a w-wide level stored from `base`.
struct RowBuf {
  char* base = nullptr;
  size_t row_bytes = 0, plane_bytes = 0;
  int C = 0, lo = 0;
  char* row(int c, int y) const {
    return base + static_cast<size_t>(c) * plane_bytes + static_cast<size_t>(y - lo) * row_bytes;
  }
};

}  // namespace

// ---------------------------------------------------------------- comms
struct si_stripe_comm {
  int world = 1, rank = 0;
  int device = 0;
  // Level iteration counts of the last solve per (shape, options): the
  // number of outer iterations issued without a host round trip next time.
  // Every rank of a group makes the same calls, so every rank holds the same
  // history and issues the same collectives.
  struct Hist {
    std::vector<uint64_t> key;
    std::vector<int> iters;
  };
  std::vector<Hist> history;
  int speculate = 1;                 // 0: one host round trip per decision
  long long solves = 0, speculative = 0, resumes = 0;  // si_stripe_comm_counters
  virtual ~si_stripe_comm() = default;
  // n doubles from every rank -> recv[rank * n + i] on every rank (device)
  virtual void allgather(const double* d_send, double* d_recv, int n, cudaStream_t s) = 0;
  // rows: sends (my rows to peers) and recvs (peers' rows into mine)
  virtual void exchange(const std::vector<RowXfer>& sends, const std::vector<RowXfer>& recvs,
                        const RowBuf& buf, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
};

namespace {

// ---- NCCL, loaded at run time (the library has no link-time dependency) ----
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // An NCCL already in the process (e.g. torch's) is reused: a second copy
    // under the same soname would shadow the newer one torch links against.
    // SI_NCCL_LIBRARY names a specific build; else the loader's search path.
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
      if (a.h) break;
    }
    if (!a.h)
      if (const char* env = std::getenv("SI_NCCL_LIBRARY")) a.h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      if (a.h) break;
      a.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    }
    if (!a.h) return a;
    auto sym = [&](auto& fp, const char* n) { fp = reinterpret_cast<std::decay_t<decltype(fp)>>(dlsym(a.h, n)); };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.CommAbort, "ncclCommAbort");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.Send ||
      !api.Recv || !api.GroupStart || !api.GroupEnd)
    fail(SI_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  fail(SI_ERR_CUDA, std::string(what) + ": " +
                        (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error"));
}

struct NcclComm final : si_stripe_comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void allgather(const double* d_send, double* d_recv, int n, cudaStream_t s) override {
    nccl_check(nccl().AllGather(d_send, d_recv, static_cast<size_t>(n), ncclFloat64, comm, s),
               "ncclAllGather");
  }
  void exchange(const std::vector<RowXfer>& sends, const std::vector<RowXfer>& recvs,
                const RowBuf& buf, cudaStream_t s) override {
    if (sends.empty() && recvs.empty()) return;
    // point-to-point pairs match in issue order: both sides walk the same
    // (peer, span, channel) order derived from the shared layout
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (const RowXfer& x : sends)
      for (int c = 0; c < buf.C; ++c)
        nccl_check(nccl().Send(buf.row(c, x.lo), static_cast<size_t>(x.hi - x.lo) * buf.row_bytes,
                               ncclUint8, x.peer, comm, s),
                   "ncclSend");
    for (const RowXfer& x : recvs)
      for (int c = 0; c < buf.C; ++c)
        nccl_check(nccl().Recv(buf.row(c, x.lo), static_cast<size_t>(x.hi - x.lo) * buf.row_bytes,
                               ncclUint8, x.peer, comm, s),
                   "ncclRecv");
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }
  const char* kind() const override { return "nccl"; }
};

// ---- G ranks as host threads of one process ---------------------------------
struct LocalGroup {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  bool aborted = false;
  std::vector<cudaEvent_t> ready, done;
  std::vector<RowBuf> posted;
  std::vector<const double*> posted_vals;
  std::vector<const std::vector<RowXfer>*> posted_sends;

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) fail(SI_ERR_RUNTIME, "stripe group aborted by another rank");
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return generation != gen || aborted; });
    if (aborted && generation == gen) fail(SI_ERR_RUNTIME, "stripe group aborted by another rank");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }

  // Persistent host threads for ranks 1..world-1 of a one-call group solve
  // (si_run_method_striped_local_device); rank 0 runs on the caller's
  // thread.  Started on first use; one group call at a time.
  std::vector<std::thread> workers;
  std::mutex wm;
  std::condition_variable wcv, wdone;
  std::function<void(int)> job;
  long long job_gen = 0;
  int job_left = 0;
  bool quit = false;
  void run_all(const std::function<void(int)>& f) {
    if (world > 1 && workers.empty())
      for (int r = 1; r < world; ++r) workers.emplace_back([this, r] { worker(r); });
    {
      std::lock_guard<std::mutex> lk(wm);
      job = f;
      job_left = world - 1;
      ++job_gen;
    }
    wcv.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(wm);
    wdone.wait(lk, [&] { return job_left == 0; });
  }
  void worker(int r) {
    long long seen = 0;
    std::unique_lock<std::mutex> lk(wm);
    for (;;) {
      wcv.wait(lk, [&] { return quit || job_gen != seen; });
      if (quit) return;
      seen = job_gen;
      const std::function<void(int)> f = job;
      lk.unlock();
      f(r);
      lk.lock();
      if (--job_left == 0) wdone.notify_all();
    }
  }
  ~LocalGroup() {
    {
      std::lock_guard<std::mutex> lk(wm);
      quit = true;
    }
    wcv.notify_all();
    for (auto& t : workers) t.join();
    for (auto e : ready) if (e) cudaEventDestroy(e);
    for (auto e : done) if (e) cudaEventDestroy(e);
  }
};

struct LocalComm final : si_stripe_comm {
  std::shared_ptr<LocalGroup> g;

  // pull model: publish + ready event, barrier, pull what I need from the
  // owners (ordered after their ready events), done event, barrier, and
  // order my later writes after every peer's pulls (their done events)
  template <typename Pull>
  void round(cudaStream_t s, Pull&& pull) {
    CK(cudaEventRecord(g->ready[rank], s));
    g->barrier();
    pull();
    CK(cudaEventRecord(g->done[rank], s));
    g->barrier();
    for (int p = 0; p < world; ++p)
      if (p != rank) CK(cudaStreamWaitEvent(s, g->done[p], 0));
  }
  void allgather(const double* d_send, double* d_recv, int n, cudaStream_t s) override {
    g->posted_vals[rank] = d_send;
    round(s, [&] {
      for (int p = 0; p < world; ++p) {
        if (p != rank) CK(cudaStreamWaitEvent(s, g->ready[p], 0));
        CK(cudaMemcpyAsync(d_recv + static_cast<size_t>(p) * n, g->posted_vals[p],
                           sizeof(double) * n, cudaMemcpyDefault, s));
      }
    });
  }
  void exchange(const std::vector<RowXfer>& sends, const std::vector<RowXfer>& recvs,
                const RowBuf& buf, cudaStream_t s) override {
    g->posted[rank] = buf;
    g->posted_sends[rank] = &sends;
    round(s, [&] {
      // the pairing NCCL relies on (NcclComm::exchange): every peer's sends
      // to me, in order, are exactly my receives from it -- checked here on
      // every exchange, so the local-communicator tests cover the NCCL plan
      for (int p = 0; p < world; ++p) {
        if (p == rank) continue;
        size_t k = 0;
        for (const RowXfer& x : *g->posted_sends[p]) {
          if (x.peer != rank) continue;
          while (k < recvs.size() && recvs[k].peer != p) ++k;
          check_arg(k < recvs.size() && recvs[k].lo == x.lo && recvs[k].hi == x.hi,
                    "stripes: send/receive plans of two ranks disagree");
          ++k;
        }
        for (; k < recvs.size(); ++k)
          check_arg(recvs[k].peer != p, "stripes: a receive without a matching send");
      }
      int last = -1;
      for (const RowXfer& x : recvs) {
        if (x.peer != last) CK(cudaStreamWaitEvent(s, g->ready[x.peer], 0));
        last = x.peer;
        const RowBuf& src = g->posted[x.peer];
        for (int c = 0; c < buf.C; ++c)
          CK(cudaMemcpyAsync(buf.row(c, x.lo), src.row(c, x.lo),
                             static_cast<size_t>(x.hi - x.lo) * buf.row_bytes, cudaMemcpyDefault,
                             s));
      }
    });
  }
  const char* kind() const override { return "local"; }
};

// Transfers of one level: rows of `want[g]` outside own[g] from their owners
// (recvs), and rows I own inside the peers' `want` (sends); same (peer, span)
// order on both sides.
void plan_xfers(const StripeLevel& S, int rank, const std::vector<std::vector<Span>>& want,
                std::vector<RowXfer>& sends, std::vector<RowXfer>& recvs) {
  sends.clear();
  recvs.clear();
  const int world = static_cast<int>(S.own.size());
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    for (const Span& a : want[rank]) {
      const Span i = span_inter(a, S.own[p]);
      if (!i.empty()) recvs.push_back({p, i.lo, i.hi});
    }
    for (const Span& a : want[p]) {
      const Span i = span_inter(a, S.own[rank]);
      if (!i.empty()) sends.push_back({p, i.lo, i.hi});
    }
  }
}

// Outcome of one level's outer iterations, decided on the device.
struct StripeState {
  double r0, final_rel;
  int outer;       // sweeps executed on this level
  int iterations;  // outer count at the last decision (report.iterations)
  int converged;
  int stop;        // final: the level's later sweeps and residuals skip
  int fix_base;    // sweeps at the last parity fixup: the iterate is in u[(swept - fix_base) & 1]
  int known_ok;    // build_rhs: some known pixel (every decision carries the count)
};

// A finest-level trace row, written by the decision itself.
struct StripeTraceRow {
  unsigned long long t;  // %globaltimer (ns) at the decision
  double rel;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void stripe_clock_kernel(unsigned long long* out) {
  if (threadIdx.x == 0) *out = global_ns();
}

// One stop decision from the gathered G x NG rows [sums C | r0 C | known |
// failures | CG iterations | -], in the host path's arithmetic: per-channel
// sums in rank order from 0.0, joint_norm, rel = joint / r0 (schwarz.hpp:
// 288-320).  first: also r0 (from the sums at r0_off: C, or 0 when u0 = b
// bitwise) and a fresh level.  A stopped level keeps its outcome (the
// speculative iterations after it are no-ops).  The gathered rows and the
// state are mirrored into mapped host memory; on the finest level each
// decision is also a trace row (log, mapped, indexed by outer).  cnt (one
// rank): the counters are read directly instead of through the gather.
__global__ void stripe_decide_kernel(const double* __restrict__ g, int G, int C, double tol,
                                     int max_outer, StripeState* st, StripeState* mirror,
                                     double* host_copy, int first, int r0_off,
                                     StripeTraceRow* log, const unsigned long long* cnt) {
  const int NG = 2 * C + 4;
  for (int i = threadIdx.x; i < NG * G; i += blockDim.x) host_copy[i] = g[i];
  __syncthreads();  // the copy lands before thread 0 overwrites the counter slots
  if (threadIdx.x != 0) return;
  if (cnt != nullptr) {  // one rank: the local counters directly (no stats pass)
    host_copy[2 * C] = static_cast<double>(cnt[2]);
    host_copy[2 * C + 1] = static_cast<double>(cnt[0]);
    host_copy[2 * C + 2] = static_cast<double>(cnt[1]);
  }
  StripeState s = *st;
  auto joint = [&](int off) {
    double j = 0.0;
    for (int k = 0; k < C; ++k) {
      double sum = 0.0;
      for (int r = 0; r < G; ++r) sum += g[r * NG + off + k];
      const double nrm = sqrt(sum);
      j = fma(nrm, nrm, j);
    }
    return sqrt(j);
  };
  if (first) {
    s.r0 = joint(r0_off);
    s.outer = s.iterations = s.converged = s.stop = s.fix_base = 0;
    double known = 0.0;
    if (cnt != nullptr) known = static_cast<double>(cnt[2]);
    else
      for (int r = 0; r < G; ++r) known += g[r * NG + 2 * C];
    s.known_ok = known > 0.0;
  }
  if (!s.stop) {
    const double rel = s.r0 > 0.0 ? joint(0) / s.r0 : 0.0;
    s.iterations = s.outer;
    s.final_rel = rel;
    if (log != nullptr) log[s.outer] = {global_ns(), rel};  // finest level: the trace row
    if (rel <= tol) {
      s.converged = 1;
      s.stop = 1;
    } else if (s.outer >= max_outer) {
      s.stop = 1;
    } else {
      s.outer += 1;  // the next sweep runs
    }
  }
  *st = s;
  *mirror = s;
}

// Sweeps a level has executed: a live level's `outer` already counts the
// next one (the decision to continue increments it).
__device__ __forceinline__ int stripe_swept(const StripeState* st) {
  return st->stop ? st->outer : st->outer - 1;
}

// After a level: its iterate -> u0 when it sits in u1.
template <typename T>
__global__ void stripe_fixup_kernel(const StripeState* st, const T* __restrict__ u1,
                                    T* __restrict__ u0, size_t n) {
  if (((stripe_swept(st) - st->fix_base) & 1) == 0) return;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    u0[i] = u1[i];
}

// The finest level's own rows of every channel -> the compact output, from
// whichever buffer holds the iterate: plane c's own rows start `skip`
// elements into its `plane`-long storage plane.  VEC: 16-byte moves (the
// offsets are even and the buffers 16-byte aligned).
template <typename T, bool VEC>
__global__ void stripe_output_kernel(const StripeState* st, const T* __restrict__ u0,
                                     const T* __restrict__ u1, size_t plane, size_t skip,
                                     double* __restrict__ out, size_t n, int C) {
  const T* __restrict__ src = ((stripe_swept(st) - st->fix_base) & 1) ? u1 : u0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t t0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int c = 0; c < C; ++c) {
    const T* __restrict__ s = src + c * plane + skip;
    double* __restrict__ d = out + c * n;
    if constexpr (VEC && sizeof(T) == 8) {
      // four 16-byte loads in flight per thread
      const size_t m = n / 2;
      const double2* __restrict__ s2 = reinterpret_cast<const double2*>(s);
      double2* __restrict__ d2 = reinterpret_cast<double2*>(d);
      size_t i = t0;
      for (; i + 3 * stride < m; i += 4 * stride) {
        double2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldg(s2 + i + k * stride);
#pragma unroll
        for (int k = 0; k < 4; ++k) d2[i + k * stride] = v[k];
      }
      for (; i < m; i += stride) d2[i] = __ldg(s2 + i);
    } else {
      for (size_t i = t0; i < n; i += stride) d[i] = static_cast<double>(s[i]);
    }
  }
}

// A level resumed after its fixup: the iterate is in u0 again.
__global__ void stripe_rebase_kernel(StripeState* st) {
  if (threadIdx.x == 0) st->fix_base = stripe_swept(st);
}

// known pixels among n mask bytes -> *out: 16-byte loads over the aligned
// body, bytes at the ends
__global__ void count_known_rows_kernel(const uint8_t* __restrict__ mask, size_t n,
                                        unsigned long long* out) {
  const size_t lead = (16 - (reinterpret_cast<uintptr_t>(mask) & 15)) & 15;
  const size_t head = n < lead ? n : lead;
  const size_t body = (n - head) / 16;
  const uint4* __restrict__ v = reinterpret_cast<const uint4*>(mask + head);
  const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  auto nz = [](unsigned w) {  // nonzero bytes of a word
    const unsigned t = ((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w;
    return __popc(t & 0x80808080u);
  };
  unsigned cnt = 0;
  for (size_t i = tid; i < body; i += stride) {
    const uint4 q = __ldg(v + i);
    cnt += nz(q.x) + nz(q.y) + nz(q.z) + nz(q.w);
  }
  const size_t tail0 = head + body * 16;
  if (tid < head) cnt += mask[tid] != 0;
  if (tid < n - tail0) cnt += mask[tail0 + tid] != 0;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, static_cast<unsigned long long>(cnt));
}

// K5 for rows [lo, hi) of a stripe store (pre-offset pointers, planes
// `plane` apart): the rows the fused K5+K3 pass does not cover
template <typename T>
__global__ void ingest_rows_kernel(const double* __restrict__ f, const uint8_t* __restrict__ mask,
                                   int w, int lo, int hi, int C, size_t plane, T* __restrict__ b) {
  const size_t n = static_cast<size_t>(hi - lo) * w, base = static_cast<size_t>(lo) * w;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool kn = mask[base + i] != 0;
    for (int c = 0; c < C; ++c)
      b[c * plane + base + i] = kn ? static_cast<T>(f[c * plane + base + i]) : T(0);
  }
}

// counters [failures, CG iterations, known pixels of my own rows] -> the
// gather row's [known | failures | CG iterations] (exact below 2^53)
__global__ void stripe_stats_kernel(const unsigned long long* cnt, double* out) {
  if (threadIdx.x == 0) {
    out[0] = static_cast<double>(cnt[2]);
    out[1] = static_cast<double>(cnt[0]);
    out[2] = static_cast<double>(cnt[1]);
  }
}

template <typename T>
RowBuf row_buf(T* storage, int w, Span store, int C) {
  RowBuf b;
  b.base = reinterpret_cast<char*>(storage);
  b.row_bytes = sizeof(T) * static_cast<size_t>(w);
  b.plane_bytes = b.row_bytes * static_cast<size_t>(store.hi - store.lo);
  b.C = C;
  b.lo = store.lo;
  return b;
}

// The striped multilevel solve of one rank.  d_f / d_mask hold the level-0
// store rows (compact [C][rows][w] / [rows][w]); d_out receives the finest
// own rows (compact), or is null: the rows stay in the level storage
// (c.stripe_result, si_stripe_result_rows).  Everything is issued on x.s.
template <typename T>
void stripe_solve_device(Ctx& x, si_stripe_comm& comm, const StripeLayout& P, int flavour,
                         const double* d_f, const uint8_t* d_mask, int C, const si_options& o,
                         double* d_out, si_report* rep, const Trace& tr) {
  si_ctx& c = x.c;
  const int G = comm.world, me = comm.rank;
  const int depth = P.depth;
  rep->depth = depth;
  // storage per level: rows store[me] only
  if (static_cast<int>(c.stripe_levels.size()) < depth) c.stripe_levels.resize(depth);
  struct View {
    Span st;
    size_t rows_n;         // storage pixels
    uint8_t* mask;         // pre-offset: index with global rows
    T* b;
    T* u[2];
    T* base_b;             // storage starts
    T* base_u[2];
    uint8_t* base_mask;
  };
  std::vector<View> V(depth);
  for (int l = 0; l < depth; ++l) {
    const StripeLevel& S = P.L[l];
    View& v = V[l];
    v.st = S.store[me];
    const int rows = std::max(0, v.st.hi - v.st.lo);
    v.rows_n = static_cast<size_t>(rows) * S.w;
    auto& lb = c.stripe_levels[l];
    const size_t cells = std::max<size_t>(v.rows_n, 1);
    lb.mask.ensure(cells);
    lb.b.ensure(cells * C * sizeof(T));
    lb.u0.ensure(cells * C * sizeof(T));
    lb.u1.ensure(cells * C * sizeof(T));
    const ptrdiff_t off = static_cast<ptrdiff_t>(v.st.lo) * S.w;
    v.base_mask = l == 0 ? const_cast<uint8_t*>(d_mask) : lb.mask.as<uint8_t>();
    v.base_b = lb.b.as<T>();
    v.base_u[0] = lb.u0.as<T>();
    // fp64, finest level, store rows == own rows (one rank, or no halo): the
    // caller's output is one of the ping-pong iterates, as in the direct solve
    if constexpr (std::is_same<T, double>::value)
      if (l == 0 && d_out != nullptr && S.store[me].lo == S.own[me].lo &&
          S.store[me].hi == S.own[me].hi && rows > 0)
        v.base_u[0] = d_out;
    v.base_u[1] = lb.u1.as<T>();
    v.mask = v.base_mask - off;
    v.b = v.base_b - off;
    v.u[0] = v.base_u[0] - off;
    v.u[1] = v.base_u[1] - off;
  }
  // comm scratch: one row of NG = 2C + 4 doubles per rank (see gather below)
  c.stripe_send.ensure(sizeof(double) * (2 * C + 4));
  c.stripe_recv.ensure(sizeof(double) * (2 * C + 4) * G);
  double* d_send = c.stripe_send.as<double>();
  double* d_recv = c.stripe_recv.as<double>();
  prepare_red(x, ((2 * C + 4) * G + 3) / 4 + 1);  // mapped slots for the G x (2C+4) gathers

  // ---- K5 ingest of the store rows, K3 restriction store -> store; K5 and
  // the first K3 in one pass over the coarse store rows (as the direct path)
  // plus plain K5 for fine store rows outside twice them
  int restrict_from = 1;
  bool known_counted = false;  // counters[2] = known pixels of my own level-0 rows
  bool skip_b0 = false;        // level-0 b not written: the snap reads f (as the direct path)
  if (depth > 1 && !ingest_fusion_disabled() && !V[1].st.empty()) {
    const StripeLevel& F = P.L[0];
    const Span cs = V[1].st, fs = V[0].st;
    const Span pair{2 * cs.lo, std::min(2 * cs.hi, F.h)};
    Timed t(x, K_INGEST, static_cast<double>(V[0].rows_n) * (C * 8.0 + 1.0) +
                             static_cast<double>(V[1].rows_n) * (C * sizeof(T) + 1));
    const ptrdiff_t off0 = static_cast<ptrdiff_t>(fs.lo) * F.w;
    const double* f_pre = d_f - off0;
    const Span own0 = F.own[me];
    known_counted = own0.empty() || (pair.lo <= own0.lo && own0.hi <= pair.hi);
    const dim3 grid((P.L[1].w + 128 * kIrCells - 1) / (128 * kIrCells), cs.hi - cs.lo);
    skip_b0 = std::is_same<T, double>::value && o.normalizer != 1 &&
              pair_derivable(V[0].base_mask, V[0].base_u[0], F.w, fs.hi - fs.lo, C);
    T* b0 = skip_b0 ? nullptr : V[0].b;
    ++c.launch_count;
    auto fused = [&](auto vec) {
      ingest_restrict_kernel<T, decltype(vec)::value><<<grid, 128, 0, x.s>>>(
          f_pre, V[0].mask, F.w, F.h, C, o.averaging, b0, V[1].mask, V[1].b,
          c.counters.as<unsigned long long>() + (known_counted ? 2 : 3), cs.lo, V[0].rows_n,
          V[1].rows_n, own0.empty() ? 0 : own0.lo, own0.empty() ? 0 : own0.hi);
    };
    // the vector path moves cell pairs: even width (every offset even) and
    // 16-byte aligned f / 2-byte aligned mask
    if (F.w % 2 == 0 && (reinterpret_cast<uintptr_t>(d_f) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(d_mask) & 1) == 0)
      fused(std::true_type{});
    else fused(std::false_type{});
    CK(cudaGetLastError());
    std::vector<Span> rest;
    if (!skip_b0) span_minus(fs, pair, rest);
    for (const Span& r : rest) {
      ++c.launch_count;
      ingest_rows_kernel<T><<<grid_for(static_cast<size_t>(r.hi - r.lo) * F.w, 256, 148 * 4), 256,
                              0, x.s>>>(f_pre, V[0].mask, F.w, r.lo, r.hi, C, V[0].rows_n, V[0].b);
      CK(cudaGetLastError());
    }
    restrict_from = 2;
  } else {
    const size_t n0 = V[0].rows_n;
    if (n0) {
      Timed t(x, K_INGEST, static_cast<double>(n0) * (C * (8.0 + sizeof(T)) + 1.0));
      ++c.launch_count;
      ingest_kernel<T><<<ingest_grid(n0), 256, 0, x.s>>>(  // counts halo rows too: sink
          d_f, d_mask, n0, C, V[0].base_b, c.counters.as<unsigned long long>() + 3);
      CK(cudaGetLastError());
    }
  }
  for (int l = restrict_from; l < depth; ++l) {
    const StripeLevel& F = P.L[l - 1];
    const Span cs = V[l].st;
    if (cs.empty()) continue;
    Timed t(x, K_RESTRICT, static_cast<double>(V[l].rows_n) * 5.0 * (C * sizeof(T) + 1));
    launch_restrict<T>(x, V[l - 1].mask, V[l - 1].b, F.w, F.h, C, o.averaging, V[l].mask, V[l].b,
                       cs.lo, cs.hi, V[l - 1].rows_n, V[l].rows_n);
  }
  // One all-gather per outer iteration carries every rank's
  // [sums C | r0 C | known | failures | CG iterations | -]; the stop decision
  // is taken on the device from it (stripe_decide_kernel), identically on
  // every rank, so the host issues iterations without waiting for them.
  const int NG = 2 * C + 4;
  c.stripe_state.ensure(sizeof(StripeState) * SI_MAX_LEVELS +
                        sizeof(unsigned long long) * 2 * SI_MAX_LEVELS);
  StripeState* d_st = c.stripe_state.as<StripeState>();
  unsigned long long* d_snap = reinterpret_cast<unsigned long long*>(d_st + SI_MAX_LEVELS);
  if (!c.stripe_host) {
    CK(cudaHostAlloc(&c.stripe_host, sizeof(StripeState) * SI_MAX_LEVELS, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&c.stripe_hdev, c.stripe_host, 0));
  }
  const StripeState* h_st = static_cast<const StripeState*>(c.stripe_host);
  StripeState* m_st = static_cast<StripeState*>(c.stripe_hdev);
  unsigned long long* d_cnt = c.counters.as<unsigned long long>();
  // finest-level trace rows, written by the decisions (mapped host memory):
  // [0] = the solve's start stamp, then one row per outer iteration
  StripeTraceRow* log_dev = nullptr;
  const StripeTraceRow* log_host = nullptr;
  if (tr.fn) {
    const size_t rows = static_cast<size_t>(std::max(o.max_outer_iterations, 0)) + 2;
    if (c.stripe_log_cap < rows) {
      if (c.stripe_log) {
        CK(cudaStreamSynchronize(x.s));
        CK(cudaFreeHost(c.stripe_log));
        c.stripe_log = nullptr;
      }
      CK(cudaHostAlloc(&c.stripe_log, sizeof(StripeTraceRow) * rows, cudaHostAllocMapped));
      c.stripe_log_cap = rows;
    }
    void* d = nullptr;
    CK(cudaHostGetDevicePointer(&d, c.stripe_log, 0));
    log_dev = static_cast<StripeTraceRow*>(d);
    log_host = static_cast<const StripeTraceRow*>(c.stripe_log);
    ++c.launch_count;
    stripe_clock_kernel<<<1, 32, 0, x.s>>>(&log_dev[0].t);
    CK(cudaGetLastError());
  }
  auto gather = [&](int level, bool first, bool r0_same = false) {
    if (G > 1) {  // one rank: nothing to gather, the decision reads the counters
      ++c.launch_count;
      stripe_stats_kernel<<<1, 32, 0, x.s>>>(d_cnt, d_send + 2 * C);
      CK(cudaGetLastError());
      comm.allgather(d_send, d_recv, NG, x.s);
    }
    ++c.launch_count;
    stripe_decide_kernel<<<1, 128, 0, x.s>>>(G > 1 ? d_recv : d_send, G, C,
                                             level == 0 ? o.tolerance : o.coarse_tolerance,
                                             o.max_outer_iterations, d_st + level, m_st + level,
                                             c.dev_red, first ? 1 : 0, r0_same ? 0 : C,
                                             level == 0 && log_dev ? log_dev + 1 : nullptr,
                                             G > 1 ? nullptr : d_cnt);
    CK(cudaGetLastError());
  };
  // known count of the rows this rank owns at level 0 (own rows tile the
  // image; counted by the fused K5+K3 pass, else here): every gather
  // carries it, the first decision checks it (build_rhs, operators.hpp:83)
  CK(cudaMemsetAsync(d_send, 0, sizeof(double) * NG, x.s));
  if (!known_counted) {
    const StripeLevel& S = P.L[0];
    const Span own = S.own[me];
    if (!own.empty()) {
      ++c.launch_count;
      count_known_rows_kernel<<<grid_for(static_cast<size_t>(own.hi - own.lo) * S.w / 16, 256,
                                         148 * 8),
                                256, 0, x.s>>>(V[0].mask + static_cast<size_t>(own.lo) * S.w,
                                               static_cast<size_t>(own.hi - own.lo) * S.w,
                                               d_cnt + 2);
      CK(cudaGetLastError());
    }
  }
  bool known_checked = false;
  auto check_known = [&](const StripeState& st) {
    if (known_checked) return;
    check_arg(st.known_ok != 0, "build_rhs: mask has no known pixels");
    known_checked = true;
  };

  bool local_checked = false;  // cg_solve's config check before the first sweep (cg.hpp:75-80)
  if (flavour == SI_FLAVOUR_ORAS)
    check_arg(std::isfinite(o.alpha), "run_schwarz_level: alpha must be finite");
  const LocalCfg lc{o.local_tolerance, o.local_max_iterations, o.local_check_interval};
  std::vector<RowXfer> sends, recvs;
  std::vector<std::vector<Span>> want(G);
  struct Run {
    int cur = 0;  // host view of the ping-pong (issued sweeps)
    std::vector<RowXfer> hs, hr;  // halo plan
  };
  std::vector<Run> R(depth);

  // Speculation: the iteration counts of the last solve with this key (same
  // on every rank) are issued without a host round trip; a level that has
  // not stopped by then is found at the end and resumed, and the finer
  // levels after it are redone (results and counts identical to the
  // synchronous loop).  No history, or local options the sweep would
  // reject: one decision per host round trip.
  std::vector<uint64_t> key = {static_cast<uint64_t>(P.L[0].w), static_cast<uint64_t>(P.L[0].h),
                               static_cast<uint64_t>(C), static_cast<uint64_t>(flavour),
                               sizeof(T), static_cast<uint64_t>(c.local_fp32),
                               static_cast<uint64_t>(depth)};
  {
    auto bits = [&](double v) {
      uint64_t u;
      std::memcpy(&u, &v, 8);
      key.push_back(u);
    };
    bits(o.tolerance);
    bits(o.coarse_tolerance);
    bits(o.alpha);
    bits(o.local_tolerance);
    for (int v : {o.block_size, o.overlap, o.averaging, o.local_max_iterations,
                  o.local_check_interval, o.max_outer_iterations, o.normalizer})
      key.push_back(static_cast<uint64_t>(static_cast<int64_t>(v)));
  }
  std::vector<int> pred(depth, -1);  // -1: synchronous
  const bool local_ok = o.local_tolerance > 0.0 && o.local_max_iterations >= 0 &&
                        o.local_check_interval >= 1;
  // (the skippable sweeps are the 2-warp ones; K2g checks at run time).
  // Trace rows come from the device log after the solve.
  bool nw_ok = true;
  for (int l = 0; l < depth; ++l)
    if (P.L[l].block <= kMaxBlock) nw_ok &= (sizeof(T) == 8 ? c.sweep_nw64 : c.sweep_nw32) == 2;
  if (local_ok && nw_ok && comm.speculate)
    for (const auto& h : comm.history)
      if (h.key == key && static_cast<int>(h.iters.size()) == depth) pred = h.iters;

  auto begin_level = [&](int level) {
    const StripeLevel& S = P.L[level];
    View& v = V[level];
    const Span own = S.own[me];
    if (level == depth - 1 && v.rows_n) {
      // canonical start u0 = b (multilevel.hpp:267-273)
      ++c.launch_count;
      launch_pdl(convert_kernel<T, T>, dim3(grid_for(v.rows_n * C, 256, 148 * 16)), 256, x.s,
                 static_cast<const T*>(v.base_b), v.base_u[0], v.rows_n * C);
      CK(cudaGetLastError());
    }
    // halo want: window rows outside my own
    for (int g = 0; g < G; ++g) {
      want[g].clear();
      span_minus(S.win[g], S.own[g], want[g]);
    }
    plan_xfers(S, me, want, R[level].hs, R[level].hr);
    R[level].cur = 0;
    // residual of my own rows and r0 with u = b; on the coarsest level u0
    // is a bitwise copy of b, so one pass gives both (R0Mode kR0Same)
    const bool same = level == depth - 1 && o.normalizer != 1;
    if (own.empty()) {
      CK(cudaMemsetAsync(d_send, 0, sizeof(double) * 2 * C, x.s));
    } else if (same) {
      launch_residual<T>(x, v.mask, v.u[0], v.b, S.w, S.h, C, 0, d_send, true, own.lo, own.hi,
                         v.st.lo, v.st.hi);
    } else if (o.normalizer != 1) {  // u0 and r0 in one pass
      launch_residual_pair<T>(x, v.mask, v.u[0], v.b, S.w, S.h, C, d_send, own.lo, own.hi,
                              v.st.lo, v.st.hi);
    } else {
      launch_residual<T>(x, v.mask, v.u[0], v.b, S.w, S.h, C, 0, d_send, true, own.lo, own.hi,
                         v.st.lo, v.st.hi);
      launch_residual<T>(x, v.mask, v.b, v.b, S.w, S.h, C, 1, d_send + C, true, own.lo, own.hi,
                         v.st.lo, v.st.hi);
    }
    gather(level, true, same);
  };
  // one outer iteration, skipped on the device once the level has stopped:
  // sweep, halo exchange (an exchange after a skipped sweep copies rows
  // equal to the ones it overwrites), residual, gather + decision
  auto iterate = [&](int level) {
    NvtxRange nv_sweep("stripe sweep + halo");
    const StripeLevel& S = P.L[level];
    View& v = V[level];
    const Span own = S.own[me];
    // skippable launches only while speculating (else the level is known live)
    const int* skip = pred[level] >= 0 ? &d_st[level].stop : nullptr;
    if (!local_checked) {  // every rank takes the same decisions: all fail alike
      validate_local(o);
      local_checked = true;
    }
    int& cur = R[level].cur;
    if (S.k1 > S.k0)
      launch_sweep<T>(x, v.mask, v.b, v.u[cur], v.u[cur ^ 1], S.w, S.h, C, S.block, S.overlap,
                      flavour, o.alpha, lc, true, d_cnt, S.k0, S.k1, v.st.lo, v.st.hi, skip);
    cur ^= 1;
    comm.exchange(R[level].hs, R[level].hr, row_buf<T>(v.base_u[cur], S.w, v.st, C), x.s);
    if (own.empty())
      CK(cudaMemsetAsync(d_send, 0, sizeof(double) * 2 * C, x.s));
    else
      launch_residual<T>(x, v.mask, v.u[cur], v.b, S.w, S.h, C, 0, d_send, true, own.lo, own.hi,
                         v.st.lo, v.st.hi, skip);
    gather(level, false);
  };
  auto end_level = [&](int level, bool snapshot) {
    const StripeLevel& S = P.L[level];
    View& v = V[level];
    const Span own = S.own[me];
    if (level == 0) {
      if (own.empty() || d_out == nullptr) return;  // no output: the rows stay in place
      if (static_cast<const void*>(v.base_u[0]) == static_cast<const void*>(d_out)) {
        ++c.launch_count;
        stripe_fixup_kernel<T><<<grid_for(v.rows_n * C, 256, 148 * 8), 256, 0, x.s>>>(
            d_st, v.base_u[1], v.base_u[0], v.rows_n * C);
        CK(cudaGetLastError());
        return;
      }
      const size_t rows_px = static_cast<size_t>(own.hi - own.lo) * S.w;
      const size_t skip = static_cast<size_t>(own.lo - v.st.lo) * S.w;
      Timed t(x, K_INGEST, static_cast<double>(rows_px) * C * (8.0 + sizeof(T)));
      ++c.launch_count;
      const bool vec = sizeof(T) == 8 && rows_px % 2 == 0 && skip % 2 == 0 && v.rows_n % 2 == 0 &&
                       ((reinterpret_cast<uintptr_t>(d_out) | reinterpret_cast<uintptr_t>(v.base_u[0]) |
                         reinterpret_cast<uintptr_t>(v.base_u[1])) & 15) == 0;
      const unsigned grid = 148 * 4;
      if (vec)
        stripe_output_kernel<T, true><<<grid, 256, 0, x.s>>>(d_st, v.base_u[0], v.base_u[1],
                                                             v.rows_n, skip, d_out, rows_px, C);
      else
        stripe_output_kernel<T, false><<<grid, 256, 0, x.s>>>(d_st, v.base_u[0], v.base_u[1],
                                                              v.rows_n, skip, d_out, rows_px, C);
      CK(cudaGetLastError());
      return;
    }
    if (v.rows_n) {
      ++c.launch_count;
      stripe_fixup_kernel<T><<<grid_for(v.rows_n * C, 256, 148 * 8), 256, 0, x.s>>>(
          d_st + level, v.base_u[1], v.base_u[0], v.rows_n * C);
      CK(cudaGetLastError());
    }
    if (snapshot)  // the counters as of this level's end: restored if a finer level is redone
      CK(cudaMemcpyAsync(d_snap + 2 * level, d_cnt, 2 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToDevice, x.s));
    // rows my prolongation reads but my window does not hold: from owners
    for (int g = 0; g < G; ++g) {
      want[g].clear();
      span_minus(S.need[g], S.win[g], want[g]);
    }
    plan_xfers(S, me, want, sends, recvs);
    comm.exchange(sends, recvs, row_buf<T>(v.base_u[0], S.w, v.st, C), x.s);
    // K4 onto the finer level's window rows
    const StripeLevel& F = P.L[level - 1];
    View& fv = V[level - 1];
    const Span fw = F.win[me];
    if (!fw.empty()) {
      Timed t(x, K_PROLONG, static_cast<double>(fw.hi - fw.lo) * F.w * (2.0 * C * sizeof(T) + 1.0));
      const T* snap = fv.b;  // the snap's values (f itself when b0 was not kept)
      if constexpr (std::is_same<T, double>::value)
        if (level == 1 && skip_b0) snap = d_f - static_cast<ptrdiff_t>(fv.st.lo) * F.w;
      launch_prolong<T>(x, v.u[0], S.w, S.h, F.w, F.h, C, fv.mask, snap, fv.u[0], fw.lo, fw.hi,
                        v.st.lo, v.st.hi, fv.rows_n, v.rows_n, fv.st.lo);
    }
  };
  // synchronous: one host round trip per decision
  auto run_sync = [&](int level) {
    for (;;) {
      sync(x);
      const StripeState st = h_st[level];
      check_known(st);
      if (st.stop) return;
      iterate(level);
    }
  };
  auto run_level = [&](int level) {
    NvtxRange nv_level("stripe level %d", level);
    begin_level(level);
    if (pred[level] < 0) {
      run_sync(level);
    } else {
      for (int k = 0; k < pred[level] && k < o.max_outer_iterations; ++k) iterate(level);
    }
    end_level(level, pred[level] >= 0);
  };

  NvtxRange nv_solve("striped multilevel_solve");
  ++comm.solves;
  if (pred[0] >= 0) ++comm.speculative;
  for (int level = depth - 1; level >= 0; --level) run_level(level);
  sync(x);
  check_known(h_st[depth - 1]);
  for (;;) {  // levels that needed more iterations than were issued
    int bad = -1;
    for (int l = depth - 1; l >= 0 && bad < 0; --l)
      if (!h_st[l].stop) bad = l;
    if (bad < 0) break;
    ++comm.resumes;
    if (bad > 0)
      CK(cudaMemcpyAsync(d_cnt, d_snap + 2 * bad, 2 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToDevice, x.s));
    if (bad == 0 && V[0].rows_n) {  // the finest level's end wrote the output only
      ++c.launch_count;
      stripe_fixup_kernel<T><<<grid_for(V[0].rows_n * C, 256, 148 * 8), 256, 0, x.s>>>(
          d_st, V[0].base_u[1], V[0].base_u[0], V[0].rows_n * C);
      CK(cudaGetLastError());
    }
    ++c.launch_count;
    stripe_rebase_kernel<<<1, 32, 0, x.s>>>(d_st + bad);
    CK(cudaGetLastError());
    R[bad].cur = 0;
    pred[bad] = -1;
    {
      NvtxRange nv_level("stripe level %d (resumed)", bad);
      iterate(bad);
      run_sync(bad);
      end_level(bad, true);
    }
    for (int level = bad - 1; level >= 0; --level) run_level(level);
    sync(x);
  }

  rep->local_failures = rep->local_cg_iterations = rep->local_solves = 0;
  for (int l = 0; l < depth; ++l) {
    const StripeState& st = h_st[l];
    rep->level_iterations[l] = st.iterations;
    rep->level_final_rel[l] = st.final_rel;
    rep->level_converged[l] = st.converged;
    const StripeLevel& S = P.L[l];
    const Axis ax = Axis::make(S.w, S.block, S.overlap), ay = Axis::make(S.h, S.block, S.overlap);
    rep->local_solves += static_cast<long long>(st.outer) * ax.count * ay.count * C;
  }
  if (tr.fn)  // trace rows (multilevel.hpp:252-261), stamped on the device
    for (int i = 0; i <= h_st[0].iterations; ++i)
      tr.fn(i, static_cast<double>(log_host[1 + i].t - log_host[0].t) * 1e-6, log_host[1 + i].rel,
            std::numeric_limits<double>::quiet_NaN(), tr.user);
  {  // where my finest own rows ended (si_stripe_result_rows)
    const StripeState& st = h_st[0];
    const int par = ((st.stop ? st.outer : st.outer - 1) - st.fix_base) & 1;
    const Span own = P.L[0].own[me];
    c.stripe_result = own.empty() ? nullptr
                                  : V[0].base_u[par] + static_cast<size_t>(own.lo - V[0].st.lo) * P.L[0].w;
    c.stripe_result_stride = V[0].rows_n;
    c.stripe_result_rows = own.empty() ? 0 : own.hi - own.lo;
    c.stripe_result_f64 = sizeof(T) == 8;
  }
  rep->iterations = h_st[0].iterations;
  rep->final_relative_residual = h_st[0].final_rel;
  rep->converged = h_st[0].converged;
  // local statistics summed over ranks (the last gather came after the last
  // sweep): failures, CG iterations
  for (int g = 0; g < G; ++g) {
    rep->local_failures += static_cast<long long>(c.host_red[g * NG + 2 * C + 1]);
    rep->local_cg_iterations += static_cast<long long>(c.host_red[g * NG + 2 * C + 2]);
  }
  {  // remember this solve's counts for the next one with the same key
    std::vector<int> it(depth);
    for (int l = 0; l < depth; ++l) it[l] = h_st[l].iterations;
    auto hit = std::find_if(comm.history.begin(), comm.history.end(),
                            [&](const si_stripe_comm::Hist& h) { return h.key == key; });
    if (hit != comm.history.end()) {
      hit->iters = it;
    } else {
      if (comm.history.size() >= 16) comm.history.erase(comm.history.begin());
      comm.history.push_back({key, it});
    }
  }
  write_diagnostic(rep, depth, -1);
}

}  // namespace
