// Host <-> device copies of caller buffers at pinned-memory speed.
//
// The reference API hands images over as ordinary (pageable) host memory.
// A plain cudaMemcpy from pageable memory runs at ~11 GB/s H2D / ~20 GB/s D2H
// on the B200 box (scripts/micro/pageable.cu: 18.3 / 10 ms for a 199 MB 4K
// RGB f64 frame), pinning the caller's buffer costs more than it saves
// (cudaHostRegister 17.5 ms).  Instead the copy runs through two pinned
// chunks: a small pool of host threads copies chunk k while the DMA engine
// moves chunk k-1 (≈ 46 GB/s for the host copies with 16 threads).  Pinned
// caller buffers go straight to cudaMemcpyAsync.  Host code only.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace sib {

// Work split over a persistent pool of worker threads (the caller takes a
// share too): run(fn) calls fn(k, parts) once for every k in [0, parts).
class CopyPool {
 public:
  // threads = 0: min(hardware threads, 16)
  explicit CopyPool(int threads = 0) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int t = threads > 0 ? threads : static_cast<int>(std::min(hw, 16u));
    nworkers_ = std::max(1, t) - 1;
    for (int k = 0; k < nworkers_; ++k) workers_.emplace_back([this, k] { loop(k); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;

  int parts() const { return nworkers_ + 1; }

  void run(const std::function<void(int, int)>& fn) {
    const int parts = nworkers_ + 1;
    if (parts == 1) {
      fn(0, 1);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &fn;
      pending_ = nworkers_;
      ++gen_;
    }
    cv_.notify_all();
    fn(parts - 1, parts);  // the caller's share
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

  void memcpy(void* dst, const void* src, size_t n) {
    if (n < (size_t(1) << 20) || nworkers_ == 0) {
      std::memcpy(dst, src, n);
      return;
    }
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    run([&](int k, int parts) {
      const size_t a = n * k / parts, b = n * (k + 1) / parts;
      std::memcpy(d + a, s + a, b - a);
    });
  }

 private:
  void loop(int k) {
    long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      const std::function<void(int, int)>* job = job_;
      lk.unlock();
      (*job)(k, nworkers_ + 1);
      lk.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }

  int nworkers_ = 0;
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int, int)>* job_ = nullptr;
  int pending_ = 0;
  long gen_ = 0;
  bool stop_ = false;
};

// Known-sample upload (batch entry): the solver reads f only where the mask
// is set (build_pyramid zeroes the rest, multilevel.hpp:84-88), so a frame
// crosses PCIe as its mask, the known values in pixel order per channel and
// the exclusive known-count of every kKnownTile-pixel tile (the device
// scatter's offsets).  Pass 1 counts per tile, pass 2 gathers.
constexpr int kKnownTile = 4096;

// high bit of every nonzero byte of w
inline uint64_t nonzero_bytes(uint64_t w) {
  constexpr uint64_t lo7 = 0x7F7F7F7F7F7F7F7Full;
  return (((w & lo7) + lo7) | w) & ~lo7;
}

inline uint64_t load_word(const uint8_t* p) {
  uint64_t w;
  std::memcpy(&w, p, 8);
  return w;
}

// Bit j of the result = (mask[a + j] != 0), j < min(64, b - a).  Branch-free
// over eight 8-byte words (the high bits of nonzero_bytes gathered by one
// multiply).
inline uint64_t known_bits64(const uint8_t* mask, size_t a, size_t b) {
  uint64_t bits = 0;
  if (b - a >= 64) {
    for (int k = 0; k < 8; ++k) {
      const uint64_t hi = nonzero_bytes(load_word(mask + a + 8 * k)) >> 7;  // bit 8j
      bits |= ((hi * 0x0102040810204080ull) >> 56) << (8 * k);
    }
  } else {
    for (size_t i = a; i < b; ++i) bits |= static_cast<uint64_t>(mask[i] != 0) << (i - a);
  }
  return bits;
}

// tile_off[t] <- known pixels in tiles [0, t); returns the total.
inline size_t count_known_tiles(CopyPool& pool, const uint8_t* mask, size_t n, uint32_t* tile_off) {
  const size_t ntiles = (n + kKnownTile - 1) / kKnownTile;
  pool.run([&](int k, int parts) {
    const size_t t0 = ntiles * k / parts, t1 = ntiles * (k + 1) / parts;
    for (size_t t = t0; t < t1; ++t) {
      const size_t a = t * kKnownTile, b = std::min(n, a + kKnownTile);
      uint32_t cnt = 0;
      for (size_t i = a; i < b; i += 64)
        cnt += __builtin_popcountll(known_bits64(mask, i, std::min(b, i + 64)));
      tile_off[t] = cnt;
    }
  });
  size_t run = 0;
  for (size_t t = 0; t < ntiles; ++t) {
    const uint32_t c = tile_off[t];
    tile_off[t] = static_cast<uint32_t>(run);
    run += c;
  }
  return run;
}

// vals[c*K + rank] = f[c*n + p] for the rank-th known pixel p.  Each part
// lists its known positions first (64 pixels per mask word, one tzcnt per
// known pixel), then gathers channel by channel with software prefetch: the
// loads are independent, so the part runs at memory-level parallelism
// instead of stalling on mispredicted mask branches.
inline void gather_known(CopyPool& pool, const uint8_t* mask, const double* f, size_t n, int C,
                         const uint32_t* tile_off, size_t K, double* vals) {
  const size_t ntiles = (n + kKnownTile - 1) / kKnownTile;
  pool.run([&](int k, int parts) {
    const size_t t0 = ntiles * k / parts, t1 = ntiles * (k + 1) / parts;
    if (t0 >= t1) return;
    const size_t o0 = tile_off[t0], o1 = t1 < ntiles ? tile_off[t1] : K;
    std::vector<size_t> pos(o1 - o0 + 1);
    size_t o = 0;
    const size_t a = t0 * kKnownTile, b = std::min(n, t1 * kKnownTile);
    for (size_t i = a; i < b; i += 64) {
      uint64_t bits = known_bits64(mask, i, std::min(b, i + 64));
      while (bits) {
        pos[o++] = i + __builtin_ctzll(bits);
        bits &= bits - 1;
      }
    }
    const size_t m = o;
    constexpr size_t kAhead = 24;
    for (int c = 0; c < C; ++c) {
      const double* fc = f + static_cast<size_t>(c) * n;
      double* vc = vals + static_cast<size_t>(c) * K + o0;
      for (size_t j = 0; j < m; ++j) {
        if (j + kAhead < m) __builtin_prefetch(fc + pos[j + kAhead]);
        vc[j] = fc[pos[j]];
      }
    }
  });
}

inline bool host_is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Two pinned chunks + events; errors are reported through the callback the
// owner passes (it throws).
class Stager {
 public:
  // a ring of kBufs pinned chunks: the DMA of the next chunks overlaps the
  // host copy of this one, and small chunks keep the unoverlapped first DMA
  // and last host copy short (was 2 x 32 MB)
  static constexpr size_t kChunk = size_t(8) << 20;
  static constexpr int kBufs = 4;

  explicit Stager(std::function<void(cudaError_t, const char*)> check) : check_(std::move(check)) {}
  ~Stager() { release(); }
  Stager(const Stager&) = delete;
  Stager& operator=(const Stager&) = delete;

  void release() {
    for (int b = 0; b < kBufs; ++b) {
      if (ev_[b]) cudaEventDestroy(ev_[b]);
      if (buf_[b]) cudaFreeHost(buf_[b]);
      ev_[b] = nullptr;
      buf_[b] = nullptr;
    }
  }

  // dst (device) <- src (host).  Returns once the caller's buffer has been
  // read; the last chunks' DMA may still be in flight on stream s.
  void h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
    if (n < (size_t(1) << 20) || host_is_pinned(src)) {
      check_(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync H2D");
      return;
    }
    ensure();
    size_t k = 0;
    for (size_t off = 0; off < n; off += kChunk, ++k) {
      const int b = static_cast<int>(k % kBufs);
      const size_t len = std::min(kChunk, n - off);
      check_(cudaEventSynchronize(ev_[b]), "cudaEventSynchronize");  // chunk free again
      pool_.memcpy(buf_[b], static_cast<const char*>(src) + off, len);
      check_(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf_[b], len, cudaMemcpyHostToDevice,
                             s),
             "cudaMemcpyAsync H2D");
      check_(cudaEventRecord(ev_[b], s), "cudaEventRecord");
    }
  }

  // dst (host) <- src (device), after all prior work on stream s; returns
  // with the data in dst.
  void d2h(void* dst, const void* src, size_t n, cudaStream_t s) {
    if (n < (size_t(1) << 20) || host_is_pinned(dst)) {
      check_(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync D2H");
      check_(cudaStreamSynchronize(s), "cudaStreamSynchronize");
      return;
    }
    ensure();
    const size_t chunks = (n + kChunk - 1) / kChunk;
    auto issue = [&](size_t k) {
      const size_t off = k * kChunk, len = std::min(kChunk, n - off);
      const int b = static_cast<int>(k % kBufs);
      check_(cudaMemcpyAsync(buf_[b], static_cast<const char*>(src) + off, len,
                             cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync D2H");
      check_(cudaEventRecord(ev_[b], s), "cudaEventRecord");
    };
    for (size_t k = 0; k < std::min<size_t>(kBufs - 1, chunks); ++k) issue(k);
    for (size_t k = 0; k < chunks; ++k) {
      const int b = static_cast<int>(k % kBufs);
      check_(cudaEventSynchronize(ev_[b]), "cudaEventSynchronize");
      if (k + kBufs - 1 < chunks) issue(k + kBufs - 1);  // keep kBufs - 1 DMAs ahead
      const size_t off = k * kChunk, len = std::min(kChunk, n - off);
      pool_.memcpy(static_cast<char*>(dst) + off, buf_[b], len);
    }
  }

 private:
  void ensure() {
    for (int b = 0; b < kBufs; ++b) {
      if (!buf_[b]) check_(cudaMallocHost(&buf_[b], kChunk), "cudaMallocHost");
      if (!ev_[b]) {
        check_(cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming), "cudaEventCreate");
      }
    }
  }

  std::function<void(cudaError_t, const char*)> check_;
  CopyPool pool_;
  void* buf_[kBufs] = {};
  cudaEvent_t ev_[kBufs] = {};
};

}  // namespace sib
