// K2 (warp variant): one WARP per (32x32 subdomain, channel).
//
// Same contract as oras_sweep_kernel (sweep.cuh) — one outer ORAS sweep,
// residual gather, Robin local system, local CG, restricted write-back —
// specialised for full 32x32 blocks (every level of any image >= 32 pixels
// per side with the default block size).  One warp owns the whole local
// problem, so the CG needs no CTA barrier at all: dot products are a single
// butterfly, and the scalar recurrences run once per block instead of once
// per warp.  Layout: lane l owns columns 2*(l%16), 2*(l%16)+1 of rows
// 16*(l/16) .. 16*(l/16)+15 (32 cells), so
//   * one shuffle pair per row serves two cells (E/W across lanes), the
//     neighbour inside the pair and the N/S neighbours are own registers,
//     and the row pair 15/16 crosses half-warps with a 16-lane shuffle;
//   * r, p and Ap (q) live in registers; the iterate x lives in shared memory
//     (updated in place with 16-byte accesses), as does the local right-hand
//     side for the rare true-residual checks.
// Arithmetic per cell is identical to the CTA variant (same fma order).
#pragma once

#include "sweep.cuh"

namespace sib {

template <typename T>
struct WarpSweepSmem {
  T xt[kMaxBlock][kMaxBlock];  // CG iterate x
  T qt[kMaxBlock][kMaxBlock];  // A p of the current iteration
};

#ifndef SI_WOCC64
#define SI_WOCC64 12
#endif
#ifndef SI_WOCC32
#define SI_WOCC32 14
#endif

template <typename T>
struct WarpOcc {
  static constexpr int value = sizeof(T) == 8 ? SI_WOCC64 : SI_WOCC32;
};

template <typename T>
__device__ __forceinline__ void load2(const T* __restrict__ p, T& a, T& b) {
  if constexpr (sizeof(T) == 8) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    a = v.x;
    b = v.y;
  } else {
    const float2 v = *reinterpret_cast<const float2*>(p);
    a = v.x;
    b = v.y;
  }
}

template <typename T>
__device__ __forceinline__ void store2(T* p, T a, T b) {
  if constexpr (sizeof(T) == 8) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
  } else {
    *reinterpret_cast<float2*>(p) = make_float2(a, b);
  }
}

// u at (gy, gx), (gy, gx+1); zero outside the image.  gx is even relative to
// the block origin but not necessarily aligned globally: scalar loads.
template <typename T>
__device__ __forceinline__ void load_u2(const T* __restrict__ u, int W, int H, int gy, int gx, T& a,
                                        T& b) {
  a = b = T(0);
  if (gy < 0 || gy >= H) return;
  const T* row = u + static_cast<size_t>(gy) * W;
  a = row[gx];
  b = row[gx + 1];
}

template <typename T>
__global__ void __launch_bounds__(32, (WarpOcc<T>::value)) oras_sweep_warp_kernel(SweepArgs<T> a) {
  constexpr int R = 16;  // rows per lane
  __shared__ WarpSweepSmem<T> S;
  const int lane = threadIdx.x;
  const int cp = lane & 15, half = lane >> 4;
  const int c0 = 2 * cp, row0 = R * half;
  const int bx = blockIdx.x % a.ax.count, by = a.by0 + static_cast<int>(blockIdx.x) / a.ax.count;
  const int x0 = a.ax.anchor(bx), y0 = a.ay.anchor(by);
  const int W = a.W, H = a.H;
  const int gx = x0 + c0;  // my columns gx, gx+1
  const size_t plane = static_cast<size_t>(blockIdx.y) * a.N;
  const T* __restrict__ u = a.u_old + plane;
  const T* __restrict__ bb = a.b + plane;
  const uint8_t* __restrict__ mask = a.mask;
  constexpr unsigned FULLM = 0xffffffffu;

  T r[R][2], p[R][2];
  // local right-hand side of this (block, channel), kept for the rare
  // true-residual checks in a global scratch tile (L2/HBM, not registers)
  T* __restrict__ bt = a.scratch + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) *
                                       (kMaxBlock * kMaxBlock);
  uint32_t unk = 0;  // bit 2*i+k: cell (row0+i, c0+k) unknown

  // ---- setup: residual of block rows row0-1 .. row0+R (index j), ghosts 0 --
  {
    T ra[R + 2], rb[R + 2];
    uint64_t kb = 0;  // bit 2*j+k: known
    T ua_prev, ub_prev, ua_cur, ub_cur, ua_next, ub_next;
    load_u2(u, W, H, y0 + row0 - 2, gx, ua_prev, ub_prev);
    load_u2(u, W, H, y0 + row0 - 1, gx, ua_cur, ub_cur);
#pragma unroll
    for (int j = 0; j < R + 2; ++j) {
      const int ly = row0 - 1 + j, gy = y0 + ly;
      load_u2(u, W, H, gy + 1, gx, ua_next, ub_next);
      T uw = __shfl_up_sync(FULLM, ub_cur, 1);
      T ue = __shfl_down_sync(FULLM, ua_cur, 1);
      const bool row_img = gy >= 0 && gy < H;
      if (cp == 0) uw = (row_img && gx > 0) ? u[static_cast<size_t>(gy) * W + gx - 1] : T(0);
      if (cp == 15) ue = (row_img && gx + 2 < W) ? u[static_cast<size_t>(gy) * W + gx + 2] : T(0);
      T r0v = T(0), r1v = T(0);
      if (ly >= 0 && ly < kMaxBlock) {
        const size_t pix = static_cast<size_t>(gy) * W + gx;
        const bool k0 = mask[pix] != 0, k1 = mask[pix + 1] != 0;
        kb |= (uint64_t(k0) << (2 * j)) | (uint64_t(k1) << (2 * j + 1));
        // r = b - A u (operators.hpp:44-58); known rows: b - u (+0 under the invariant)
        if (k0) {
          r0v = a.known_invariant ? T(0) : bb[pix] - ua_cur;
        } else {
          T sum = T(0);
          int deg = 0;
          if (gx > 0) { sum += uw; ++deg; }
          sum += ub_cur; ++deg;  // gx + 1 < W inside a full block
          if (gy > 0) { sum += ua_prev; ++deg; }
          if (gy + 1 < H) { sum += ua_next; ++deg; }
          r0v = (a.known_invariant ? T(0) : bb[pix]) - fmaT(T(deg), ua_cur, -sum);
        }
        if (k1) {
          r1v = a.known_invariant ? T(0) : bb[pix + 1] - ub_cur;
        } else {
          T sum = T(0);
          int deg = 0;
          sum += ua_cur; ++deg;  // gx + 1 > 0
          if (gx + 2 < W) { sum += ue; ++deg; }
          if (gy > 0) { sum += ub_prev; ++deg; }
          if (gy + 1 < H) { sum += ub_next; ++deg; }
          r1v = (a.known_invariant ? T(0) : bb[pix + 1]) - fmaT(T(deg), ub_cur, -sum);
        }
      }
      ra[j] = r0v;
      rb[j] = r1v;
      ua_prev = ua_cur;
      ub_prev = ub_cur;
      ua_cur = ua_next;
      ub_cur = ub_next;
    }
    // rhs = unk*(pv + knw_W pv_W + knw_E pv_E + knw_N pv_N + knw_S pv_S)
    // over in-block neighbours (schwarz.hpp:219-230).
    const uint64_t kbW = __shfl_up_sync(FULLM, kb, 1), kbE = __shfl_down_sync(FULLM, kb, 1);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int j = i + 1, ly = row0 + i;
      const T rW = __shfl_up_sync(FULLM, rb[j], 1);   // column c0-1
      const T rE = __shfl_down_sync(FULLM, ra[j], 1); // column c0+2
      const bool k0 = (kb >> (2 * j)) & 1, k1 = (kb >> (2 * j + 1)) & 1;
      T t0 = T(0), t1 = T(0);
      if (!k0) {
        unk |= 1u << (2 * i);
        t0 = ra[j];
        if (cp > 0 && ((kbW >> (2 * j + 1)) & 1)) t0 += rW;
        if (k1) t0 += rb[j];
        if (ly > 0 && ((kb >> (2 * (j - 1))) & 1)) t0 += ra[j - 1];
        if (ly + 1 < kMaxBlock && ((kb >> (2 * (j + 1))) & 1)) t0 += ra[j + 1];
      }
      if (!k1) {
        unk |= 1u << (2 * i + 1);
        t1 = rb[j];
        if (k0) t1 += ra[j];
        if (cp < 15 && ((kbE >> (2 * j)) & 1)) t1 += rE;
        if (ly > 0 && ((kb >> (2 * (j - 1) + 1)) & 1)) t1 += rb[j - 1];
        if (ly + 1 < kMaxBlock && ((kb >> (2 * (j + 1) + 1)) & 1)) t1 += rb[j + 1];
      }
      r[i][0] = t0;
      r[i][1] = t1;
      store2(&bt[ly * kMaxBlock + c0], t0, t1);
      store2(&S.xt[ly][c0], T(0), T(0));
    }
  }

  // Robin diagonals of my two columns (fill_local_structure, schwarz.hpp:100-108)
  T dI[2], dF[2], dL[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    dI[k] = robin_diag(gx + k, y0 + 1, c0 + k, 1, kMaxBlock, W, H, a.am1, a.ras);
    const T dT = robin_diag(gx + k, y0, c0 + k, 0, kMaxBlock, W, H, a.am1, a.ras);
    const T dB = robin_diag(gx + k, y0 + kMaxBlock - 1, c0 + k, kMaxBlock - 1, kMaxBlock, W, H,
                            a.am1, a.ras);
    dF[k] = half == 0 ? dT : dI[k];  // row i = 0 is block row 0 only in the upper half
    dL[k] = half == 1 ? dB : dI[k];  // row i = R-1 is block row 31 only in the lower half
  }

  // q = A v on my cells (LocalStencilOperator::apply, schwarz.hpp:146-159),
  // stored to the q tile; returns my part of v.q.
  auto apply = [&](const T(&v)[R][2]) {
    T acc0 = T(0), acc1 = T(0);
    // N neighbour of my row 0 / S neighbour of my row R-1 across the halves
    const T n0 = __shfl_up_sync(FULLM, v[R - 1][0], 16), n1 = __shfl_up_sync(FULLM, v[R - 1][1], 16);
    const T s0 = __shfl_down_sync(FULLM, v[0][0], 16), s1 = __shfl_down_sync(FULLM, v[0][1], 16);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      T w = __shfl_up_sync(FULLM, v[i][1], 1);
      T e = __shfl_down_sync(FULLM, v[i][0], 1);
      if (cp == 0) w = T(0);
      if (cp == 15) e = T(0);
      const T vn0 = i > 0 ? v[i - 1][0] : (half ? n0 : T(0));
      const T vn1 = i > 0 ? v[i - 1][1] : (half ? n1 : T(0));
      const T vs0 = i + 1 < R ? v[i + 1][0] : (half ? T(0) : s0);
      const T vs1 = i + 1 < R ? v[i + 1][1] : (half ? T(0) : s1);
      const T d0 = i == 0 ? dF[0] : (i == R - 1 ? dL[0] : dI[0]);
      const T d1 = i == 0 ? dF[1] : (i == R - 1 ? dL[1] : dI[1]);
      T t0 = fmaT(d0, v[i][0], -w);
      t0 = t0 - v[i][1];
      t0 = t0 - vn0;
      t0 = t0 - vs0;
      T t1 = fmaT(d1, v[i][1], -v[i][0]);
      t1 = t1 - e;
      t1 = t1 - vn1;
      t1 = t1 - vs1;
      const T o0 = ((unk >> (2 * i)) & 1u) ? t0 : T(0);
      const T o1 = ((unk >> (2 * i + 1)) & 1u) ? t1 : T(0);
      store2(&S.qt[row0 + i][c0], o0, o1);
      acc0 = fmaT(v[i][0], o0, acc0);
      acc1 = fmaT(v[i][1], o1, acc1);
    }
    return acc0 + acc1;
  };
  auto dot = [&](const T(&va)[R][2], const T(&vb)[R][2]) {
    T s0 = T(0), s1 = T(0);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      s0 = fmaT(va[i][0], vb[i][0], s0);
      s1 = fmaT(va[i][1], vb[i][1], s1);
    }
    return warp_sum(s0 + s1);
  };

  int iters = 0;
  bool converged = true;
  if (__any_sync(FULLM, unk != 0)) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      p[i][0] = r[i][0];  // r = b - A*0 = b exactly
      p[i][1] = r[i][1];
    }
    T rr = dot(r, r);
    T rr_rcp = recip_rn(rr);
    const T r0 = sqrt(rr);
    const T thr = a.ltol * r0;
    const T thr2 = thr * thr;
    const T thr2_lo = thr2 * T(1.0 - 1e-6), thr2_hi = thr2 * T(1.0 + 1e-6);
    converged = false;
    if (r0 == T(0)) {
      converged = true;
    } else {
      int until_check = a.lcheck;
      for (int iter = 1; iter <= a.lmax; ++iter) {
        const T pAp = warp_sum(apply(p));
        if (!(pAp > T(0)) || !isfinite(pAp)) {  // breakdown (cg.hpp:120-125)
          iters = iter - 1;
          break;
        }
        const T alpha = rr / pAp;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          T xa, xb, qa, qb;
          load2(&S.xt[row0 + i][c0], xa, xb);
          load2(&S.qt[row0 + i][c0], qa, qb);  // my own cells: no barrier needed
          store2(&S.xt[row0 + i][c0], fmaT(alpha, p[i][0], xa), fmaT(alpha, p[i][1], xb));
          r[i][0] = fmaT(-alpha, qa, r[i][0]);
          r[i][1] = fmaT(-alpha, qb, r[i][1]);
        }
        T rr_new = dot(r, r);
        if (--until_check == 0) until_check = a.lcheck;
        const bool cadence = until_check == a.lcheck || iter == a.lmax;
        bool maybe_done = rr_new < thr2_lo;
        if (rr_new >= thr2_lo && rr_new <= thr2_hi) maybe_done = band_sqrt_le(rr_new, thr);
        if (cadence || maybe_done) {
          // True residual b - A x from the x tile (cg.hpp:131-146).
          __syncwarp();
#pragma unroll
          for (int i = 0; i < R; ++i) {
            const int ly = row0 + i;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int lx = c0 + k;
              const T xc = S.xt[ly][lx];
              const T xw = lx > 0 ? S.xt[ly][lx - 1] : T(0);
              const T xe = lx + 1 < kMaxBlock ? S.xt[ly][lx + 1] : T(0);
              const T xn = ly > 0 ? S.xt[ly - 1][lx] : T(0);
              const T xs = ly + 1 < kMaxBlock ? S.xt[ly + 1][lx] : T(0);
              const T d = i == 0 ? dF[k] : (i == R - 1 ? dL[k] : dI[k]);
              T t = fmaT(d, xc, -xw);
              t = t - xe;
              t = t - xn;
              t = t - xs;
              t = ((unk >> (2 * i + k)) & 1u) ? t : T(0);
              // residual replacement target (r is not needed if this converges)
              r[i][k] = bt[ly * kMaxBlock + lx] - t;
            }
          }
          const T tt = dot(r, r);
          const T rel = sqrt(tt) / r0;
          if (rel <= a.ltol) {
            iters = iter;
            converged = true;
            break;
          }
          rr_new = tt;
          __syncwarp();  // x tile reads done before the next in-place update
        }
        const T beta = div_by_recip(rr_new, rr, rr_rcp);  // == rr_new / rr
#pragma unroll
        for (int i = 0; i < R; ++i) {
          p[i][0] = fmaT(beta, p[i][0], r[i][0]);
          p[i][1] = fmaT(beta, p[i][1], r[i][1]);
        }
        rr = rr_new;
        rr_rcp = recip_rn(rr);
        if (iter == a.lmax) iters = a.lmax;
      }
    }
  }
  __syncwarp();

  // ---- accumulate_owned: u_new = u_old + v on the owned rectangle ----------
  const int ox0 = a.ax.owned_begin(bx), ox1 = a.ax.owned_end(bx);
  const int oy0 = a.ay.owned_begin(by), oy1 = a.ay.owned_end(by);
  T* __restrict__ un = a.u_new + plane;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int gy = y0 + row0 + i;
    if (gy < oy0 || gy >= oy1) continue;
    const size_t pix = static_cast<size_t>(gy) * W + gx;
    T xa, xb;
    load2(&S.xt[row0 + i][c0], xa, xb);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (gx + k < ox0 || gx + k >= ox1) continue;
      const T uo = u[pix + k];
      // unknown cells take the CG solution, known cells the residual b - u
      const T v = ((unk >> (2 * i + k)) & 1u) ? (k ? xb : xa)
                                              : (a.known_invariant ? T(0) : bb[pix + k] - uo);
      un[pix + k] = uo + v;
    }
  }
  const bool any = __any_sync(FULLM, unk != 0);
  if (lane == 0 && a.counters && any) {
    if (!converged) atomicAdd(&a.counters[0], 1ull);
    atomicAdd(&a.counters[1], static_cast<unsigned long long>(iters));
  }
}

}  // namespace sib
