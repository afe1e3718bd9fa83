// Multilevel CG level solver (the paper's baseline):
// run_cg_level (multilevel.hpp:162-209) = reduce_structure + reduced_rhs
// (reduction.hpp:64-145) + cg_solve_lockstep (cg.hpp:192-291).
//
// The reduced system (unknown pixels only) is applied to full-grid vectors
// holding exactly 0 at known pixels: A_red x at an unknown pixel is
// deg*x - (its in-image unknown neighbours), in the reference's order, so
// every value equals the reference's; only the dot products are summed in a
// different (tree) order.  Channels advance in lockstep; per-channel alpha,
// beta and the frozen set come from the host, which takes every scalar
// decision exactly as cg_solve_lockstep does.  Grid: (x segments of 256
// pixels, row groups, channel); no per-pixel integer division.
#pragma once

#include "kernels.cuh"

namespace sib {

constexpr int kCgMaxChannels = 8;

struct CgCoef {
  double v[kCgMaxChannels];  // alpha or beta per channel
};

template <typename T>
__device__ __forceinline__ T reduced_apply(const uint8_t* __restrict__ mask,
                                           const T* __restrict__ v, size_t i, int x, int y, int W,
                                           int H) {
  // ReducedSystem::apply (reduction.hpp:41-50): diag*x, then the unknown
  // neighbours W, E, N, S in that order.
  const int deg = (x > 0) + (x + 1 < W) + (y > 0) + (y + 1 < H);
  T acc = T(deg) * v[i];
  if (x > 0 && !mask[i - 1]) acc -= v[i - 1];
  if (x + 1 < W && !mask[i + 1]) acc -= v[i + 1];
  if (y > 0 && !mask[i - W]) acc -= v[i - W];
  if (y + 1 < H && !mask[i + W]) acc -= v[i + W];
  return acc;
}

// reduced_rhs (reduction.hpp:119-134) + x = u at unknowns + r = rhs - A x,
// p = r.  Sums: [0,C) rhs.rhs (-> r0), [C,2C) r.r (-> rr, init_sq).
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    cg_init_kernel(const uint8_t* __restrict__ mask, const T* __restrict__ b,
                   const T* __restrict__ u, T* rhs, T* xv, T* r, T* p, int W, int H, size_t N,
                   double* partials, double* out, unsigned int* ticket) {
  const int c = blockIdx.z, x = blockIdx.x * kRedThreads + threadIdx.x;
  const T* bc = b + c * N;
  const T* uc = u + c * N;
  double s[2] = {0.0, 0.0};
  if (x < W) {
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
      const size_t i = static_cast<size_t>(y) * W + x;
      T hv = T(0), xx = T(0), rv = T(0);
      if (!mask[i]) {
        T h = bc[i];
        if (x > 0 && mask[i - 1]) h += bc[i - 1];
        if (x + 1 < W && mask[i + 1]) h += bc[i + 1];
        if (y > 0 && mask[i - W]) h += bc[i - W];
        if (y + 1 < H && mask[i + W]) h += bc[i + W];
        hv = h;
        xx = uc[i];
        // A_red x with x = u at unknown pixels only
        const int deg = (x > 0) + (x + 1 < W) + (y > 0) + (y + 1 < H);
        T ax = T(deg) * xx;
        if (x > 0 && !mask[i - 1]) ax -= uc[i - 1];
        if (x + 1 < W && !mask[i + 1]) ax -= uc[i + 1];
        if (y > 0 && !mask[i - W]) ax -= uc[i - W];
        if (y + 1 < H && !mask[i + W]) ax -= uc[i + W];
        rv = h - ax;
      }
      const size_t o = c * N + i;
      rhs[o] = hv;
      xv[o] = xx;
      r[o] = rv;
      p[o] = rv;
      s[0] = fma(static_cast<double>(hv), static_cast<double>(hv), s[0]);
      s[1] = fma(static_cast<double>(rv), static_cast<double>(rv), s[1]);
    }
  }
  reduce_epilogue_k<2>(s, partials, out, ticket, blockIdx.y * gridDim.x + blockIdx.x,
                       gridDim.x * gridDim.y, c, gridDim.z);
}

// q = A_red p for active channels; sum p.q.
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    cg_apply_dot_kernel(const uint8_t* __restrict__ mask, const T* __restrict__ p, T* q, int W,
                        int H, size_t N, unsigned active, double* partials, double* out,
                        unsigned int* ticket) {
  const int c = blockIdx.z, x = blockIdx.x * kRedThreads + threadIdx.x;
  double s = 0.0;
  if (x < W && ((active >> c) & 1u)) {
    const T* pc = p + c * N;
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
      const size_t i = static_cast<size_t>(y) * W + x;
      const T t = mask[i] ? T(0) : reduced_apply(mask, pc, i, x, y, W, H);
      q[c * N + i] = t;
      s = fma(static_cast<double>(pc[i]), static_cast<double>(t), s);
    }
  }
  reduce_epilogue(s, partials, out, ticket, blockIdx.y * gridDim.x + blockIdx.x,
                  gridDim.x * gridDim.y, c, gridDim.z);
}

// x += alpha p, r -= alpha q (vec::axpy, cg.hpp:52-54) on active channels; sum r.r.
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    cg_update_kernel(T* xv, const T* __restrict__ p, T* r, const T* __restrict__ q, int W, int H,
                     size_t N, unsigned active, CgCoef alpha, double* partials, double* out,
                     unsigned int* ticket) {
  const int c = blockIdx.z, x = blockIdx.x * kRedThreads + threadIdx.x;
  double s = 0.0;
  if (x < W && ((active >> c) & 1u)) {
    const T a = static_cast<T>(alpha.v[c]);
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
      const size_t o = c * N + static_cast<size_t>(y) * W + x;
      xv[o] = fma(a, p[o], xv[o]);
      const T rv = fma(-a, q[o], r[o]);
      r[o] = rv;
      s = fma(static_cast<double>(rv), static_cast<double>(rv), s);
    }
  }
  reduce_epilogue(s, partials, out, ticket, blockIdx.y * gridDim.x + blockIdx.x,
                  gridDim.x * gridDim.y, c, gridDim.z);
}

// true residual t = rhs - A_red x for every channel; r = t where not frozen
// (residual replacement, cg.hpp:260-271); sum t.t.
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    cg_true_residual_kernel(const uint8_t* __restrict__ mask, const T* __restrict__ rhs,
                            const T* __restrict__ xv, T* r, int W, int H, size_t N,
                            unsigned replace, double* partials, double* out,
                            unsigned int* ticket) {
  const int c = blockIdx.z, x = blockIdx.x * kRedThreads + threadIdx.x;
  double s = 0.0;
  if (x < W) {
    const T* xc = xv + c * N;
    const bool rep = (replace >> c) & 1u;
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
      const size_t i = static_cast<size_t>(y) * W + x, o = c * N + i;
      const T t = mask[i] ? T(0) : rhs[o] - reduced_apply(mask, xc, i, x, y, W, H);
      if (rep) r[o] = t;
      s = fma(static_cast<double>(t), static_cast<double>(t), s);
    }
  }
  reduce_epilogue(s, partials, out, ticket, blockIdx.y * gridDim.x + blockIdx.x,
                  gridDim.x * gridDim.y, c, gridDim.z);
}

// p = r + beta p (vec::xpay, cg.hpp:57-59) on active channels.
template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    cg_pupdate_kernel(T* p, const T* __restrict__ r, int W, int H, size_t N, unsigned active,
                      CgCoef beta) {
  const int c = blockIdx.z, x = blockIdx.x * kRedThreads + threadIdx.x;
  if (x >= W || !((active >> c) & 1u)) return;
  const T bt = static_cast<T>(beta.v[c]);
  for (int y = blockIdx.y; y < H; y += gridDim.y) {
    const size_t o = c * N + static_cast<size_t>(y) * W + x;
    p[o] = fma(bt, p[o], r[o]);
  }
}

// embed_solution (reduction.hpp:138-145): u = b at known pixels, x elsewhere.
template <typename T>
__global__ void cg_embed_kernel(const uint8_t* __restrict__ mask, const T* __restrict__ b,
                                const T* __restrict__ xv, T* u, int W, int H, size_t N) {
  const int c = blockIdx.z, x = blockIdx.x * kRedThreads + threadIdx.x;
  if (x >= W) return;
  for (int y = blockIdx.y; y < H; y += gridDim.y) {
    const size_t i = static_cast<size_t>(y) * W + x, o = c * N + i;
    u[o] = mask[i] ? b[o] : xv[o];
  }
}

}  // namespace sib
