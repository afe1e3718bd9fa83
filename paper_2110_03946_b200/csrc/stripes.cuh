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
  ~LocalGroup() {
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

__global__ void stripe_decide_copy_kernel(const double* __restrict__ src, double* dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// known pixels among n mask bytes -> *out (a double; exact below 2^53)
__global__ void count_known_rows_kernel(const uint8_t* __restrict__ mask, size_t n, double* out) {
  unsigned long long cnt = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    cnt += mask[i] != 0;
  cnt = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(cnt));
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, static_cast<double>(cnt));
}

__global__ void stripe_stats_kernel(const unsigned long long* cnt, double solves, double* out) {
  if (threadIdx.x == 0) {
    out[0] = static_cast<double>(cnt[0]);
    out[1] = static_cast<double>(cnt[1]);
    out[2] = solves;
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
// own rows (compact).  Everything is issued on x.s.
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

  // ---- K5 ingest of the store rows, K3 restriction store -> store
  {
    const size_t n0 = V[0].rows_n;
    if (n0) {
      Timed t(x, K_INGEST, static_cast<double>(n0) * (C * (8.0 + sizeof(T)) + 1.0));
      ++c.launch_count;
      ingest_kernel<T><<<ingest_grid(n0), 256, 0, x.s>>>(
          d_f, d_mask, n0, C, V[0].base_b, c.counters.as<unsigned long long>() + 2);
      CK(cudaGetLastError());
    }
  }
  for (int l = 1; l < depth; ++l) {
    const StripeLevel& F = P.L[l - 1];
    const Span cs = V[l].st;
    if (cs.empty()) continue;
    Timed t(x, K_RESTRICT, static_cast<double>(V[l].rows_n) * 5.0 * (C * sizeof(T) + 1));
    launch_restrict<T>(x, V[l - 1].mask, V[l - 1].b, F.w, F.h, C, o.averaging, V[l].mask, V[l].b,
                       cs.lo, cs.hi, V[l - 1].rows_n, V[l].rows_n);
  }
  // One all-gather per outer iteration carries everything the host needs,
  // per rank: [sums C | r0 C | known | failures | CG iterations | solves].
  const int NG = 2 * C + 4;
  auto gather = [&](double solves) {
    ++c.launch_count;
    stripe_stats_kernel<<<1, 32, 0, x.s>>>(c.counters.as<unsigned long long>(), solves,
                                           d_send + 2 * C + 1);
    CK(cudaGetLastError());
    if (G > 1) comm.allgather(d_send, d_recv, NG, x.s);  // one rank: nothing to gather
    ++c.launch_count;
    stripe_decide_copy_kernel<<<1, 256, 0, x.s>>>(G > 1 ? d_recv : d_send, c.dev_red, NG * G);
    CK(cudaGetLastError());
    sync(x);
  };
  // known count of the rows this rank owns at level 0 (own rows tile the
  // image), checked at the first gather (build_rhs, operators.hpp:83)
  CK(cudaMemsetAsync(d_send, 0, sizeof(double) * NG, x.s));
  {
    const StripeLevel& S = P.L[0];
    const Span own = S.own[me];
    if (!own.empty()) {
      ++c.launch_count;
      count_known_rows_kernel<<<grid_for(static_cast<size_t>(own.hi - own.lo) * S.w, 256, 148 * 8),
                                256, 0, x.s>>>(V[0].mask + static_cast<size_t>(own.lo) * S.w,
                                               static_cast<size_t>(own.hi - own.lo) * S.w,
                                               d_send + 2 * C);
      CK(cudaGetLastError());
    }
  }
  bool known_checked = false;

  bool local_checked = false;  // cg_solve's config check before the first sweep (cg.hpp:75-80)
  if (flavour == SI_FLAVOUR_ORAS)
    check_arg(std::isfinite(o.alpha), "run_schwarz_level: alpha must be finite");
  const LocalCfg lc{o.local_tolerance, o.local_max_iterations, o.local_check_interval};
  unsigned long long* d_cnt = c.counters.as<unsigned long long>();
  std::vector<RowXfer> sends, recvs;
  std::vector<std::vector<Span>> want(G);

  NvtxRange nv_solve("striped multilevel_solve");
  for (int level = depth - 1; level >= 0; --level) {
    NvtxRange nv_level("stripe level %d", level);
    const StripeLevel& S = P.L[level];
    View& v = V[level];
    const Span own = S.own[me];
    int cur = 0;
    if (level == depth - 1 && v.rows_n) {
      // canonical start u0 = b (multilevel.hpp:267-273)
      ++c.launch_count;
      launch_pdl(convert_kernel<T, T>, dim3(grid_for(v.rows_n * C, 256, 148 * 16)), 256, x.s,
                 static_cast<const T*>(v.base_b), v.base_u[0], v.rows_n * C);
      CK(cudaGetLastError());
    }
    const bool finest = level == 0;
    const double tol = finest ? o.tolerance : o.coarse_tolerance;
    // halo want: window rows outside my own
    for (int g = 0; g < G; ++g) {
      want[g].clear();
      span_minus(S.win[g], S.own[g], want[g]);
    }
    plan_xfers(S, me, want, sends, recvs);
    const std::vector<RowXfer> halo_sends = sends, halo_recvs = recvs;
    double r0 = 0.0;
    bool r0_pending = true;
    const Axis ax = Axis::make(S.w, S.block, S.overlap);
    LevelOutcome oc;
    for (int outer = 0;; ++outer) {
      // residual of my own rows (+ r0 with u = b the first time)
      if (own.empty()) {
        CK(cudaMemsetAsync(d_send, 0, sizeof(double) * 2 * C, x.s));
      } else if (r0_pending && o.normalizer != 1) {  // u0 and r0 in one pass
        launch_residual_pair<T>(x, v.mask, v.u[cur], v.b, S.w, S.h, C, d_send, own.lo, own.hi,
                                v.st.lo, v.st.hi);
      } else {
        launch_residual<T>(x, v.mask, v.u[cur], v.b, S.w, S.h, C, 0, d_send, true, own.lo, own.hi,
                           v.st.lo, v.st.hi);
        if (r0_pending)
          launch_residual<T>(x, v.mask, v.b, v.b, S.w, S.h, C, 1, d_send + C, true, own.lo,
                             own.hi, v.st.lo, v.st.hi);
      }
      gather(static_cast<double>(rep->local_solves));
      if (!known_checked) {
        double known = 0.0;
        for (int g = 0; g < G; ++g) known += c.host_red[g * NG + 2 * C];
        check_arg(known > 0.0, "build_rhs: mask has no known pixels");
        known_checked = true;
      }
      // fixed rank order: identical sums (and decisions) on every rank
      std::vector<double> sums(C, 0.0), r0s(C, 0.0);
      for (int g = 0; g < G; ++g)
        for (int k = 0; k < C; ++k) {
          sums[k] += c.host_red[g * NG + k];
          r0s[k] += c.host_red[g * NG + C + k];
        }
      if (r0_pending) {
        r0 = joint_norm(r0s.data(), C);
        r0_pending = false;
      }
      const double rel = r0 > 0.0 ? joint_norm(sums.data(), C) / r0 : 0.0;
      if (finest && tr.fn) tr.fn(outer, ms_since(tr.t0), rel, std::numeric_limits<double>::quiet_NaN(), tr.user);
      oc.iterations = outer;
      oc.final_rel = rel;
      if (rel <= tol) {
        oc.converged = true;
        break;
      }
      if (outer >= o.max_outer_iterations) break;
      NvtxRange nv_sweep("stripe sweep + halo");
      if (!local_checked) {  // every rank takes the same decisions: all fail alike
        validate_local(o);
        local_checked = true;
      }
      if (S.k1 > S.k0)
        launch_sweep<T>(x, v.mask, v.b, v.u[cur], v.u[cur ^ 1], S.w, S.h, C, S.block, S.overlap,
                        flavour, o.alpha, lc, true, d_cnt, S.k0, S.k1, v.st.lo, v.st.hi);
      cur ^= 1;
      rep->local_solves += static_cast<long long>(ax.count) * (S.k1 - S.k0) * C;
      comm.exchange(halo_sends, halo_recvs, row_buf<T>(v.base_u[cur], S.w, v.st, C), x.s);
    }
    rep->level_iterations[level] = oc.iterations;
    rep->level_final_rel[level] = oc.final_rel;
    rep->level_converged[level] = oc.converged;
    if (finest) {
      rep->iterations = oc.iterations;
      rep->final_relative_residual = oc.final_rel;
      rep->converged = oc.converged;
      if (!own.empty() && static_cast<const void*>(v.base_u[cur]) != static_cast<const void*>(d_out)) {
        const size_t rows_px = static_cast<size_t>(own.hi - own.lo) * S.w;
        Timed t(x, K_INGEST, static_cast<double>(rows_px) * C * (8.0 + sizeof(T)));
        for (int k = 0; k < C; ++k) {  // own rows of each plane -> compact output
          ++c.launch_count;
          convert_kernel<T, double><<<grid_for(rows_px, 256, 148 * 16), 256, 0, x.s>>>(
              v.u[cur] + static_cast<size_t>(k) * v.rows_n + static_cast<size_t>(own.lo) * S.w,
              d_out + static_cast<size_t>(k) * rows_px, rows_px);
          CK(cudaGetLastError());
        }
      }
    } else {
      // rows my prolongation reads but my window does not hold: from owners
      for (int g = 0; g < G; ++g) {
        want[g].clear();
        span_minus(S.need[g], S.win[g], want[g]);
      }
      plan_xfers(S, me, want, sends, recvs);
      comm.exchange(sends, recvs, row_buf<T>(v.base_u[cur], S.w, v.st, C), x.s);
      // K4 onto the finer level's window rows
      const StripeLevel& F = P.L[level - 1];
      View& fv = V[level - 1];
      const Span fw = F.win[me];
      if (!fw.empty()) {
        Timed t(x, K_PROLONG, static_cast<double>(fw.hi - fw.lo) * F.w * (2.0 * C * sizeof(T) + 1.0));
        launch_prolong<T>(x, v.u[cur], S.w, S.h, F.w, F.h, C, fv.mask, fv.b, fv.u[0], fw.lo,
                          fw.hi, v.st.lo, v.st.hi, fv.rows_n, v.rows_n, fv.st.lo);
      }
    }
  }
  // local statistics summed over ranks (the finest level's last gather came
  // after the last sweep): failures, CG iterations, solves
  rep->local_failures = rep->local_cg_iterations = rep->local_solves = 0;
  for (int g = 0; g < G; ++g) {
    rep->local_failures += static_cast<long long>(c.host_red[g * NG + 2 * C + 1]);
    rep->local_cg_iterations += static_cast<long long>(c.host_red[g * NG + 2 * C + 2]);
    rep->local_solves += static_cast<long long>(c.host_red[g * NG + 2 * C + 3]);
  }
  write_diagnostic(rep, depth, -1);
}

}  // namespace
