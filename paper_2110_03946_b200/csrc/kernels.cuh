// Memory-bound kernels around the sweep: K1 residual norms, K3 pyramid
// restriction, K4 prolongation + snap, K5 ingest, export, K6 MSE.
#pragma once

#include "common.cuh"

namespace sib {

// Per-channel deterministic reduction: each CTA writes one partial per
// channel (blockIdx.y); the last CTA to finish (atomic ticket) sums the
// partials in a fixed order, so the result depends only on the launch shape.
constexpr int kRedThreads = 256;
constexpr int kRedBlocksMax = 1184;  // 148 SMs x 8

template <typename Term>
__device__ void reduce_epilogue(double v, double* partials, double* out, unsigned int* ticket,
                                int nblk, int nch) {
  __shared__ double wsum[kRedThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) wsum[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += wsum[w];
    partials[blockIdx.y * nblk + blockIdx.x] = s;
    __threadfence();
    const unsigned int total = gridDim.x * gridDim.y;
    last = atomicAdd(ticket, 1u) == total - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Fixed-order final sum per channel: strided partial sums + butterfly.
  for (int c = 0; c < nch; ++c) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nblk; i += kRedThreads)
      s += reinterpret_cast<volatile double*>(partials)[c * nblk + i];
    s = warp_sum(s);
    __syncthreads();
    if (lane == 0) wsum[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kRedThreads / 32; ++w) t += wsum[w];
      out[c] = t;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

struct NoTerm {};

// K1: per channel sum of (b - A u)^2 (residual_into + vec::norm^2,
// operators.hpp:38-66/91-97, cg.hpp:46-50).  mode 1: sum of b^2 (RhsNorm).
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    residual_sumsq_kernel(const uint8_t* __restrict__ mask, const T* __restrict__ u,
                          const T* __restrict__ b, int W, int H, size_t N, int mode,
                          double* partials, double* out, unsigned int* ticket) {
  const int c = blockIdx.y;
  const T* uc = u + c * N;
  const T* bc = b + c * N;
  double acc = 0.0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
    T r;
    if (mode == 1) {
      r = bc[i];
    } else if (mask[i]) {
      r = bc[i] - uc[i];
    } else {
      const int y = static_cast<int>(i / W), x = static_cast<int>(i - static_cast<size_t>(y) * W);
      T sum = T(0);
      int deg = 0;
      if (x > 0) { sum += uc[i - 1]; ++deg; }
      if (x + 1 < W) { sum += uc[i + 1]; ++deg; }
      if (y > 0) { sum += uc[i - W]; ++deg; }
      if (y + 1 < H) { sum += uc[i + W]; ++deg; }
      r = bc[i] - fma(T(deg), uc[i], -sum);
    }
    const double rd = static_cast<double>(r);
    acc = fma(rd, rd, acc);
  }
  reduce_epilogue<NoTerm>(acc, partials, out, ticket, gridDim.x, gridDim.y);
}

// K6: per channel sum of (255 u - 255 f)^2 (mse_per_channel, metrics.hpp:30-47).
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    sq_error_kernel(const T* __restrict__ u, const double* __restrict__ f, size_t N,
                    double* partials, double* out, unsigned int* ticket) {
  const int c = blockIdx.y;
  double acc = 0.0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
    const double d = 255.0 * (static_cast<double>(u[c * N + i]) - f[c * N + i]);
    acc = fma(d, d, acc);
  }
  reduce_epilogue<NoTerm>(acc, partials, out, ticket, gridDim.x, gridDim.y);
}

// K5: level-0 values = f at known pixels, 0 elsewhere (build_pyramid,
// multilevel.hpp:84-88); also counts known pixels for build_rhs's check.
template <typename T>
__global__ void ingest_kernel(const double* __restrict__ f, const uint8_t* __restrict__ mask,
                              size_t N, int C, T* __restrict__ b, unsigned long long* known) {
  unsigned int cnt = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride) {
    const bool k = mask[i] != 0;
    cnt += k;
    for (int c = 0; c < C; ++c) b[c * N + i] = k ? static_cast<T>(f[c * N + i]) : T(0);
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(known, static_cast<unsigned long long>(cnt));
}

// K3: restrict_level (multilevel.hpp:33-70): coarse pixel = clipped 2x2 fine
// cell; known = OR; value = mean of known fine values (KnownOnly) or of all
// of them (AllPixels), accumulated in row-major order like the reference.
template <typename T>
__global__ void restrict_kernel(const uint8_t* __restrict__ fmask, const T* __restrict__ fval,
                                int fw, int fh, int C, int averaging, uint8_t* __restrict__ cmask,
                                T* __restrict__ cval) {
  const int cw = (fw + 1) / 2, ch = (fh + 1) / 2;
  const size_t fn = static_cast<size_t>(fw) * fh, cn = static_cast<size_t>(cw) * ch;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cn; j += stride) {
    const int cy = static_cast<int>(j / cw), cx = static_cast<int>(j - static_cast<size_t>(cy) * cw);
    const int fx0 = 2 * cx, fy0 = 2 * cy;
    const int fx1 = min(fx0 + 2, fw), fy1 = min(fy0 + 2, fh);
    int known = 0, total = 0;
    for (int y = fy0; y < fy1; ++y)
      for (int x = fx0; x < fx1; ++x) {
        known += fmask[static_cast<size_t>(y) * fw + x] != 0;
        ++total;
      }
    cmask[j] = known ? 1 : 0;
    for (int c = 0; c < C; ++c) {
      T acc = T(0);
      if (known) {
        for (int y = fy0; y < fy1; ++y)
          for (int x = fx0; x < fx1; ++x) {
            const size_t i = static_cast<size_t>(y) * fw + x;
            if (averaging == 0 && !fmask[i]) continue;
            acc += fval[c * fn + i];
          }
        acc = acc / T(averaging == 0 ? known : total);
      }
      cval[c * cn + j] = acc;
    }
  }
}

// K4: prolongate (multilevel.hpp:101-128) + snap known fine pixels to their
// data (multilevel.hpp:294-303): cell-centred bilinear, coordinate
// 0.5*f - 0.25 clamped to the coarse grid.
template <typename T>
__global__ void prolong_snap_kernel(const T* __restrict__ coarse, int cw, int ch, int fw, int fh,
                                    int C, const uint8_t* __restrict__ fmask,
                                    const T* __restrict__ fval, T* __restrict__ fine) {
  const size_t fn = static_cast<size_t>(fw) * fh, cn = static_cast<size_t>(cw) * ch;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < fn; i += stride) {
    const int fy = static_cast<int>(i / fw), fx = static_cast<int>(i - static_cast<size_t>(fy) * fw);
    const bool snap = fmask != nullptr && fmask[i] != 0;
    double yc = fmin(fmax(0.5 * fy - 0.25, 0.0), static_cast<double>(ch - 1));
    double xc = fmin(fmax(0.5 * fx - 0.25, 0.0), static_cast<double>(cw - 1));
    const int y0 = static_cast<int>(yc), x0 = static_cast<int>(xc);
    const int y1 = min(y0 + 1, ch - 1), x1 = min(x0 + 1, cw - 1);
    const T ty = static_cast<T>(yc - y0), tx = static_cast<T>(xc - x0);
    for (int c = 0; c < C; ++c) {
      T v;
      if (snap) {
        v = fval[c * fn + i];
      } else {
        const T* cc = coarse + c * cn;
        const T v00 = cc[static_cast<size_t>(y0) * cw + x0];
        const T v01 = cc[static_cast<size_t>(y0) * cw + x1];
        const T v10 = cc[static_cast<size_t>(y1) * cw + x0];
        const T v11 = cc[static_cast<size_t>(y1) * cw + x1];
        // (1-ty)*((1-tx)*v00 + tx*v01) + ty*((1-tx)*v10 + tx*v11), with the
        // contraction gcc -O3 applies to the reference expression
        // (p*q + r*s -> fma(p, q, r*s); checked bitwise in the tests).
        const T a0 = fma(T(1) - tx, v00, tx * v01);
        const T a1 = fma(T(1) - tx, v10, tx * v11);
        v = fma(T(1) - ty, a0, ty * a1);
      }
      fine[c * fn + i] = v;
    }
  }
}

template <typename Tin, typename Tout>
__global__ void convert_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<Tout>(in[i]);
}

}  // namespace sib
