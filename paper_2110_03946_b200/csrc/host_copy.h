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
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace sib {

// memcpy split over a persistent pool of worker threads (the caller takes a
// share too).
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    nworkers_ = static_cast<int>(std::min(hw, 16u)) - 1;
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

  void memcpy(void* dst, const void* src, size_t n) {
    const int parts = nworkers_ + 1;
    if (n < (size_t(1) << 20) || parts == 1) {
      std::memcpy(dst, src, n);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      n_ = n;
      pending_ = nworkers_;
      ++gen_;
    }
    cv_.notify_all();
    slice(parts - 1, parts);  // the caller's share
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void slice(int k, int parts) {
    const size_t a = n_ * k / parts, b = n_ * (k + 1) / parts;
    std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void loop(int k) {
    long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      lk.unlock();
      slice(k, nworkers_ + 1);
      lk.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }

  int nworkers_ = 0;
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
  int pending_ = 0;
  long gen_ = 0;
  bool stop_ = false;
};

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
  static constexpr size_t kChunk = size_t(32) << 20;

  explicit Stager(std::function<void(cudaError_t, const char*)> check) : check_(std::move(check)) {}
  ~Stager() { release(); }
  Stager(const Stager&) = delete;
  Stager& operator=(const Stager&) = delete;

  void release() {
    for (int b = 0; b < 2; ++b) {
      if (ev_[b]) cudaEventDestroy(ev_[b]);
      if (buf_[b]) cudaFreeHost(buf_[b]);
      ev_[b] = nullptr;
      buf_[b] = nullptr;
    }
  }

  // dst (device) <- src (host).  Returns once the caller's buffer has been
  // read; the last chunk's DMA may still be in flight on stream s.
  void h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
    if (n < (size_t(1) << 20) || host_is_pinned(src)) {
      check_(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync H2D");
      return;
    }
    ensure();
    int b = 0;
    for (size_t off = 0; off < n; off += kChunk, b ^= 1) {
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
      const int b = static_cast<int>(k & 1);
      check_(cudaMemcpyAsync(buf_[b], static_cast<const char*>(src) + off, len,
                             cudaMemcpyDeviceToHost, s),
             "cudaMemcpyAsync D2H");
      check_(cudaEventRecord(ev_[b], s), "cudaEventRecord");
    };
    issue(0);
    for (size_t k = 0; k < chunks; ++k) {
      const int b = static_cast<int>(k & 1);
      check_(cudaEventSynchronize(ev_[b]), "cudaEventSynchronize");
      if (k + 1 < chunks) issue(k + 1);  // next chunk's DMA overlaps this copy-out
      const size_t off = k * kChunk, len = std::min(kChunk, n - off);
      pool_.memcpy(static_cast<char*>(dst) + off, buf_[b], len);
    }
  }

 private:
  void ensure() {
    for (int b = 0; b < 2; ++b) {
      if (!buf_[b]) check_(cudaMallocHost(&buf_[b], kChunk), "cudaMallocHost");
      if (!ev_[b]) {
        check_(cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming), "cudaEventCreate");
      }
    }
  }

  std::function<void(cudaError_t, const char*)> check_;
  CopyPool pool_;
  void* buf_[2] = {nullptr, nullptr};
  cudaEvent_t ev_[2] = {nullptr, nullptr};
};

}  // namespace sib
