// K2g: the sweep for subdomains larger than 32x32 (block_size up to any
// value the partition allows).  Same algorithm and control flow as K2
// (schwarz.hpp:202-250, cg.hpp:90-154), organised for generality instead of
// speed: one CTA of 256 threads per (block, channel), threads striding over
// the block's cells, the CG vectors in a per-CTA global scratch (L1/L2
// resident), CTA-wide reductions in a fixed order.  The default block size
// (32) never takes this path.
#pragma once

#include "sweep.cuh"

namespace sib {

constexpr int kGenThreads = 256;

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // previous readers of red are done
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = red[0];
#pragma unroll
  for (int w = 1; w < kGenThreads / 32; ++w) s += red[w];
  return s;
}

// scratch: 5 vectors of B*B values per (block, channel): r/rhs, x, p, q, b-tilde.
template <typename T>
__global__ void __launch_bounds__(kGenThreads) oras_sweep_generic_kernel(SweepArgs<T> a) {
  __shared__ T red[kGenThreads / 32];
  __shared__ int any_unk;
  if (a.skip != nullptr && *a.skip) return;
  const int nb = a.ax.count;
  const int bx = blockIdx.x % nb, by = a.by0 + static_cast<int>(blockIdx.x) / nb;
  const int ch = blockIdx.y;
  const int B = a.ax.block, NB = B * B;
  const int x0 = a.ax.anchor(bx), y0 = a.ay.anchor(by);
  const size_t plane = static_cast<size_t>(ch) * a.N, W = static_cast<size_t>(a.W);
  const T* __restrict__ u = a.u_old + plane;
  const T* __restrict__ b = a.b + plane;
  T* base = a.scratch + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 5 * NB;
  T *rv = base, *xv = base + NB, *pv = base + 2 * NB, *qv = base + 3 * NB, *bt = base + 4 * NB;
  auto known = [&](int lx, int ly) {
    return a.mask[static_cast<size_t>(y0 + ly) * W + x0 + lx] != 0;
  };
  // residual r = b - A u of every block cell (operators.hpp:38-66, 91-97)
  for (int i = threadIdx.x; i < NB; i += kGenThreads) {
    const int ly = i / B, lx = i - ly * B, gx = x0 + lx, gy = y0 + ly;
    const size_t p = static_cast<size_t>(gy) * W + gx;
    const T uc = u[p];
    T r;
    if (known(lx, ly)) {
      r = a.known_invariant ? T(0) : b[p] - uc;
    } else {
      const T nW = gx > 0 ? u[p - 1] : T(0), nE = gx + 1 < a.W ? u[p + 1] : T(0);
      const T nN = gy > 0 ? u[p - W] : T(0), nS = gy + 1 < a.H ? u[p + W] : T(0);
      const int deg = (gx > 0) + (gx + 1 < a.W) + (gy > 0) + (gy + 1 < a.H);
      const T sum = ((nW + nE) + nN) + nS;
      r = (a.known_invariant ? T(0) : b[p]) - fma(T(deg), uc, -sum);
    }
    rv[i] = r;
  }
  if (threadIdx.x == 0) any_unk = 0;
  __syncthreads();
  // local right-hand side (schwarz.hpp:219-230); x = 0, p = rhs
  int my_unk = 0;
  for (int i = threadIdx.x; i < NB; i += kGenThreads) {
    const int ly = i / B, lx = i - ly * B;
    T t = T(0);
    if (!known(lx, ly)) {
      my_unk = 1;
      t = rv[i];
      if (lx > 0 && known(lx - 1, ly)) t += rv[i - 1];
      if (lx + 1 < B && known(lx + 1, ly)) t += rv[i + 1];
      if (ly > 0 && known(lx, ly - 1)) t += rv[i - B];
      if (ly + 1 < B && known(lx, ly + 1)) t += rv[i + B];
    }
    bt[i] = t;
    xv[i] = T(0);
    pv[i] = t;
  }
  if (my_unk) any_unk = 1;
  __syncthreads();
  // r := rhs (kept in rv), after every thread has read the residual above
  for (int i = threadIdx.x; i < NB; i += kGenThreads) rv[i] = bt[i];
  __syncthreads();
  const int unk_any = any_unk;
  // o = A v on unknown cells (LocalStencilOperator::apply, schwarz.hpp:146-159)
  auto apply = [&](const T* v, T* o) {
    for (int i = threadIdx.x; i < NB; i += kGenThreads) {
      const int ly = i / B, lx = i - ly * B;
      T t = T(0);
      if (!known(lx, ly)) {
        const T d = robin_diag<T>(x0 + lx, y0 + ly, lx, ly, B, a.W, a.H, a.am1, a.ras);
        const T vW = lx > 0 ? v[i - 1] : T(0), vE = lx + 1 < B ? v[i + 1] : T(0);
        const T vN = ly > 0 ? v[i - B] : T(0), vS = ly + 1 < B ? v[i + B] : T(0);
        t = fma(d, v[i], -(vW + vE)) - (vN + vS);
      }
      o[i] = t;
    }
  };
  int iters = 0;
  bool converged = true;
  if (unk_any) {
    T part = T(0);
    for (int i = threadIdx.x; i < NB; i += kGenThreads) part = fma(rv[i], rv[i], part);
    T rr = block_sum(part, red);
    const T r0 = sqrt(rr);
    converged = false;
    if (r0 == T(0)) {
      converged = true;
    } else {
      for (int iter = 1; iter <= a.lmax; ++iter) {
        apply(pv, qv);
        part = T(0);
        for (int i = threadIdx.x; i < NB; i += kGenThreads) part = fma(pv[i], qv[i], part);
        const T pAp = block_sum(part, red);
        if (!(pAp > T(0)) || !isfinite(pAp)) {  // breakdown (cg.hpp:120-125)
          iters = iter - 1;
          break;
        }
        const T alpha = rr / pAp;
        part = T(0);
        for (int i = threadIdx.x; i < NB; i += kGenThreads) {
          xv[i] = fma(alpha, pv[i], xv[i]);
          rv[i] = fma(-alpha, qv[i], rv[i]);
          part = fma(rv[i], rv[i], part);
        }
        T rr_new = block_sum(part, red);  // also orders the x writes
        const bool cadence = iter % a.lcheck == 0 || iter == a.lmax;
        const bool maybe_done = sqrt(rr_new) <= a.ltol * r0;
        if (cadence || maybe_done) {
          // true residual b~ - A x, then confirm or replace (cg.hpp:131-146)
          apply(xv, qv);
          part = T(0);
          for (int i = threadIdx.x; i < NB; i += kGenThreads) {
            const T t = bt[i] - qv[i];
            qv[i] = t;
            part = fma(t, t, part);
          }
          const T tt = block_sum(part, red);
          if (sqrt(tt) / r0 <= a.ltol) {
            iters = iter;
            converged = true;
            break;
          }
          for (int i = threadIdx.x; i < NB; i += kGenThreads) rv[i] = qv[i];
          rr_new = tt;
        }
        const T beta = rr_new / rr;
        for (int i = threadIdx.x; i < NB; i += kGenThreads) pv[i] = fma(beta, pv[i], rv[i]);
        rr = rr_new;
        if (iter == a.lmax) iters = a.lmax;
        __syncthreads();  // p complete before the next apply
      }
    }
  }
  __syncthreads();
  // accumulate_owned (partition.hpp:148-156): u_new = u_old + v on the owned
  // rectangle; v = x at unknown cells, b - u at known cells
  const int ox0 = a.ax.owned_begin(bx), ox1 = a.ax.owned_end(bx);
  const int oy0 = a.ay.owned_begin(by), oy1 = a.ay.owned_end(by);
  T* __restrict__ un = a.u_new + plane;
  for (int i = threadIdx.x; i < NB; i += kGenThreads) {
    const int ly = i / B, lx = i - ly * B, gx = x0 + lx, gy = y0 + ly;
    if (gx < ox0 || gx >= ox1 || gy < oy0 || gy >= oy1) continue;
    const size_t p = static_cast<size_t>(gy) * W + gx;
    const T uo = u[p];
    const T v = known(lx, ly) ? (a.known_invariant ? T(0) : b[p] - uo) : xv[i];
    un[p] = uo + v;
  }
  if (threadIdx.x == 0 && a.counters && unk_any) {
    if (!converged) atomicAdd(&a.counters[0], 1ull);
    atomicAdd(&a.counters[1], static_cast<unsigned long long>(iters));
  }
}

}  // namespace sib
