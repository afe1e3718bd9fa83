// K2 oras_sweep: one outer ORAS/RAS sweep, fused end to end.
//
// Replaces the whole block loop of run_schwarz_level (schwarz.hpp:305-318):
//   restrict_block_into (partition.hpp:109-121) of r = b - A u,
//   prepare_local_block / fill_local_structure (schwarz.hpp:84-111, 179-198),
//   solve_local_block + cg_solve (schwarz.hpp:202-250, cg.hpp:90-154),
//   accumulate_owned (partition.hpp:148-156).
//
// One CTA = one (subdomain, channel).  The residual slice is computed on chip
// from the (B+2)^2 window of u_old (so no global residual image is ever
// written), and the local CG runs entirely in registers:
//   * lane = block column, each warp owns R = 32/NW consecutive rows, so
//     horizontal stencil neighbours come from __shfl_up/down and vertical
//     ones from the thread's own registers;
//   * rows at warp boundaries are exchanged through shared memory, but never
//     with a dedicated barrier: before each reduction barrier every warp
//     publishes the *components* of its boundary rows (r, old p, x), and its
//     neighbours rebuild p_new = r + beta*p with the identical fma after the
//     barrier.  A CG iteration therefore costs exactly 2 CTA barriers (3 on
//     a true-residual check), and 0 when NW == 1;
//   * dot products: warp butterfly + fixed-order cross-warp sum, so every
//     thread holds the same value and all control flow stays CTA-uniform.
// The result u_new = u_old + v is written only on the block's owned
// rectangle into a separate buffer (ping-pong): owned rectangles tile the
// image, so every pixel is written exactly once and no CTA reads what
// another writes.
#pragma once

#include "common.cuh"

namespace sib {

template <typename T>
struct SweepArgs {
  const uint8_t* mask;
  const T* b;
  const T* u_old;
  T* u_new;
  int W, H;
  size_t N;            // W*H, channel plane stride
  Axis ax, ay;         // partition of x and y (square blocks)
  T am1;               // alpha - 1 (ORAS); unused for RAS
  int ras;             // 1: diag = deg (RAS)
  T ltol;              // local CG tolerance
  int lmax;            // local CG max iterations
  int lcheck;          // true-residual cadence
  int b_known_only;    // b is zero at unknown pixels: skip those loads
  unsigned long long* counters;  // [0] failures, [1] CG iterations (may be null)
};

template <typename T>
__device__ __forceinline__ T fmaT(T a, T b, T c) {
  return fma(a, b, c);
}

// Residual of the global operator at an interior-of-window cell whose u
// neighbours sit in the shared tile (operators.hpp:38-66, 91-97):
//   known:   r = b - u
//   unknown: r = b - (deg*u - (((W + E) + N) + S)) over in-image neighbours.
template <typename T>
__device__ __forceinline__ T residual_cell(T u, T uW, T uE, T uN, T uS, bool known, T bv, int gx,
                                           int gy, int W, int H) {
  if (known) return bv - u;
  T sum = T(0);
  int deg = 0;
  if (gx > 0) { sum += uW; ++deg; }
  if (gx + 1 < W) { sum += uE; ++deg; }
  if (gy > 0) { sum += uN; ++deg; }
  if (gy + 1 < H) { sum += uS; ++deg; }
  return bv - fmaT(T(deg), u, -sum);
}

// Robin diagonal of an unknown cell (fill_local_structure, schwarz.hpp:100-108):
//   diag = deg_global + (alpha - 1) * cut, cut = in-image neighbours outside the block.
template <typename T>
__device__ __forceinline__ T robin_diag(int gx, int gy, int lx, int ly, int B, int W, int H, T am1,
                                        int ras) {
  const int deg = (gx > 0) + (gx + 1 < W) + (gy > 0) + (gy + 1 < H);
  if (ras) return T(deg);
  const int cut = (gx > 0 && lx == 0) + (gx + 1 < W && lx + 1 == B) + (gy > 0 && ly == 0) +
                  (gy + 1 < H && ly + 1 == B);
  return T(deg) + am1 * T(cut);
}

template <typename T, int NW>
struct SweepSmem {
  T us[kTile][kTile];          // u_old window, rows/cols -1..B
  T rs[kTile][kTile];          // residual slice with a zero ghost ring
  T bs[kMaxBlock][kMaxBlock];  // local right-hand side (for true residuals)
  uint8_t ms[kTile][kTile + 2];
  T pub[NW > 1 ? NW : 1][2][3][32];   // [warp][top/bottom][r,p,x][col]
  T pubt[NW > 1 ? NW : 1][2][32];     // true-residual boundary rows
  T red[3][NW];
};

// CTA-wide sum; identical value in every thread.  slot selects the buffer so
// consecutive reductions never race (see the header comment).
template <typename T, int NW>
__device__ __forceinline__ T cta_sum(T v, T (*red)[NW], int slot, int warp, int lane) {
  v = warp_sum(v);
  if (NW == 1) return v;
  if (lane == 0) red[slot][warp] = v;
  __syncthreads();
  T s = red[slot][0];
#pragma unroll
  for (int w = 1; w < NW; ++w) s += red[slot][w];
  return s;
}

template <typename T, int NW>
__global__ void __launch_bounds__(NW * 32) oras_sweep_kernel(SweepArgs<T> a) {
  constexpr int R = 32 / NW;  // rows per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SweepSmem<T, NW>& S = *reinterpret_cast<SweepSmem<T, NW>*>(smem_raw);

  const int bx = blockIdx.x % a.ax.count;
  const int by = blockIdx.x / a.ax.count;
  const int c = blockIdx.y;
  const int B = a.ax.block;
  const int x0 = a.ax.anchor(bx), y0 = a.ay.anchor(by);
  const int W = a.W, H = a.H;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t plane = static_cast<size_t>(c) * a.N;
  const T* __restrict__ uo = a.u_old + plane;
  const T* __restrict__ bb = a.b + plane;

  // ---- 1. stage the u window and mask (coalesced along rows) ----------
  const int TW = B + 2;
  for (int i = tid; i < TW * TW; i += NW * 32) {
    const int ly = i / TW - 1, lx = i % TW - 1;
    const int gy = y0 + ly, gx = x0 + lx;
    T uv = T(0);
    uint8_t mk = 0;
    if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
      const size_t p = static_cast<size_t>(gy) * W + gx;
      uv = uo[p];
      mk = a.mask[p];
    }
    S.us[ly + 1][lx + 1] = uv;
    S.ms[ly + 1][lx + 1] = mk;
  }
  __syncthreads();

  // ---- 2. residual slice (restrict_block_into of r = b - A u) ----------
  int any_unknown = 0;
  for (int i = tid; i < TW * TW; i += NW * 32) {
    const int ly = i / TW - 1, lx = i % TW - 1;
    T rv = T(0);
    if (lx >= 0 && lx < B && ly >= 0 && ly < B) {
      const int gy = y0 + ly, gx = x0 + lx;
      const bool known = S.ms[ly + 1][lx + 1] != 0;
      any_unknown |= !known;
      const size_t p = static_cast<size_t>(gy) * W + gx;
      const T bv = (known || !a.b_known_only) ? bb[p] : T(0);
      rv = residual_cell(S.us[ly + 1][lx + 1], S.us[ly + 1][lx], S.us[ly + 1][lx + 2],
                         S.us[ly][lx + 1], S.us[ly + 2][lx + 1], known, bv, gx, gy, W, H);
    }
    S.rs[ly + 1][lx + 1] = rv;
  }
  any_unknown = __syncthreads_or(any_unknown);

  // ---- 3. local system in registers: lane = column, rows warp*R + i -----
  const int lx = lane;
  const int gx = x0 + lx;
  const bool col_ok = lx < B;
  const int row0 = warp * R;
  uint32_t unk = 0;  // bit i: cell (row0+i, lx) is an unknown block cell
  T x[R], r[R], p[R], q[R];
  T dI = T(0), dT = T(0), dB = T(0);  // Robin diagonals: interior / first / last row
  if (col_ok) {
    dI = robin_diag(gx, y0 + 1, lx, 1, B, W, H, a.am1, a.ras);
    dT = robin_diag(gx, y0, lx, 0, B, W, H, a.am1, a.ras);
    dB = robin_diag(gx, y0 + B - 1, lx, B - 1, B, W, H, a.am1, a.ras);
  }
  const int iT = -row0;             // local row index of ly == 0 (if in range)
  const int iB = (B - 1) - row0;    // local row index of ly == B-1
  int iters = 0;
  bool converged = true;

  if (any_unknown) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int ly = row0 + i;
      T rhs = T(0);
      if (col_ok && ly < B && !S.ms[ly + 1][lx + 1]) {
        unk |= 1u << i;
        // rhs = unk*(pv + sum_{in-block nbrs} knw*pv) (schwarz.hpp:219-230)
        T t = S.rs[ly + 1][lx + 1];
        if (lx > 0 && S.ms[ly + 1][lx]) t += S.rs[ly + 1][lx];
        if (lx + 1 < B && S.ms[ly + 1][lx + 2]) t += S.rs[ly + 1][lx + 2];
        if (ly > 0 && S.ms[ly][lx + 1]) t += S.rs[ly][lx + 1];
        if (ly + 1 < B && S.ms[ly + 2][lx + 1]) t += S.rs[ly + 2][lx + 1];
        rhs = t;
      }
      if (ly < kMaxBlock) S.bs[ly][lx] = rhs;
      x[i] = T(0);
      r[i] = rhs;  // r = b - A*0 = b exactly
      p[i] = rhs;
    }

    // Neighbour rows of my tile (vertical boundary): p, r, x of the row
    // above (index 0) and below (index 1).
    T nb_p[2] = {T(0), T(0)}, nb_r[2] = {T(0), T(0)}, nb_x[2] = {T(0), T(0)};

    auto publish = [&](void) {
      if (NW > 1) {
        S.pub[warp][0][0][lane] = r[0];
        S.pub[warp][0][1][lane] = p[0];
        S.pub[warp][0][2][lane] = x[0];
        S.pub[warp][1][0][lane] = r[R - 1];
        S.pub[warp][1][1][lane] = p[R - 1];
        S.pub[warp][1][2][lane] = x[R - 1];
      }
    };
    auto collect = [&](void) {
      if (NW > 1) {
        if (warp > 0) {
          nb_r[0] = S.pub[warp - 1][1][0][lane];
          nb_p[0] = S.pub[warp - 1][1][1][lane];
          nb_x[0] = S.pub[warp - 1][1][2][lane];
        }
        if (warp + 1 < NW) {
          nb_r[1] = S.pub[warp + 1][0][0][lane];
          nb_p[1] = S.pub[warp + 1][0][1][lane];
          nb_x[1] = S.pub[warp + 1][0][2][lane];
        }
      }
    };
    // q = A v on my cells (LocalStencilOperator::apply, schwarz.hpp:146-159):
    // o = unk * (d*v - vW - vE - vN - vS); neighbours outside the block are
    // ghost zeros, which every CG vector already holds there.
    auto apply = [&](const T* v, T vN0, T vS1, T* o) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        T vW = __shfl_up_sync(0xffffffffu, v[i], 1);
        T vE = __shfl_down_sync(0xffffffffu, v[i], 1);
        if (lane == 0) vW = T(0);
        if (lane == 31) vE = T(0);
        const T vN = i > 0 ? v[i - 1] : vN0;
        const T vS = i + 1 < R ? v[i + 1] : vS1;
        const T d = (i == iT) ? dT : ((i == iB) ? dB : dI);
        T t = fmaT(d, v[i], -vW);
        t = t - vE;
        t = t - vN;
        t = t - vS;
        o[i] = (unk >> i) & 1u ? t : T(0);
      }
    };

    publish();
    T part = T(0);
#pragma unroll
    for (int i = 0; i < R; ++i) part = fmaT(r[i], r[i], part);
    T rr = cta_sum<T, NW>(part, S.red, 1, warp, lane);
    collect();
    nb_p[0] = nb_r[0];  // p = r initially
    nb_p[1] = nb_r[1];
    const T r0 = sqrt(rr);
    converged = false;
    if (r0 == T(0)) {
      converged = true;
    } else {
      for (int iter = 1; iter <= a.lmax; ++iter) {
        apply(p, nb_p[0], nb_p[1], q);
        part = T(0);
#pragma unroll
        for (int i = 0; i < R; ++i) part = fmaT(p[i], q[i], part);
        const T pAp = cta_sum<T, NW>(part, S.red, 0, warp, lane);
        if (!(pAp > T(0)) || !isfinite(pAp)) {  // breakdown (cg.hpp:120-125)
          iters = iter - 1;
          break;
        }
        const T alpha = rr / pAp;
        part = T(0);
#pragma unroll
        for (int i = 0; i < R; ++i) {
          x[i] = fmaT(alpha, p[i], x[i]);
          r[i] = fmaT(-alpha, q[i], r[i]);
          part = fmaT(r[i], r[i], part);
        }
        publish();
        T rr_new = cta_sum<T, NW>(part, S.red, 1, warp, lane);
        collect();
        const bool cadence = iter % a.lcheck == 0 || iter == a.lmax;
        const bool maybe_done = sqrt(rr_new) <= a.ltol * r0;
        if (cadence || maybe_done) {
          // True residual b - A x, then confirm or replace (cg.hpp:131-146).
          apply(x, nb_x[0], nb_x[1], q);
          part = T(0);
#pragma unroll
          for (int i = 0; i < R; ++i) {
            const int ly = row0 + i;
            const T bv = (col_ok && ly < B) ? S.bs[ly][lx] : T(0);
            q[i] = bv - q[i];
            part = fmaT(q[i], q[i], part);
          }
          if (NW > 1) {
            S.pubt[warp][0][lane] = q[0];
            S.pubt[warp][1][lane] = q[R - 1];
          }
          const T tt = cta_sum<T, NW>(part, S.red, 2, warp, lane);
          const T rel = sqrt(tt) / r0;
          if (rel <= a.ltol) {
            iters = iter;
            converged = true;
            break;
          }
#pragma unroll
          for (int i = 0; i < R; ++i) r[i] = q[i];
          if (NW > 1) {
            if (warp > 0) nb_r[0] = S.pubt[warp - 1][1][lane];
            if (warp + 1 < NW) nb_r[1] = S.pubt[warp + 1][0][lane];
          }
          rr_new = tt;
        }
        const T beta = rr_new / rr;
#pragma unroll
        for (int i = 0; i < R; ++i) p[i] = fmaT(beta, p[i], r[i]);
        nb_p[0] = fmaT(beta, nb_p[0], nb_r[0]);
        nb_p[1] = fmaT(beta, nb_p[1], nb_r[1]);
        rr = rr_new;
        if (iter == a.lmax) iters = a.lmax;
      }
    }
  }

  // ---- 4. accumulate_owned: u_new = u_old + v on the owned rectangle ----
  const int ox0 = a.ax.owned_begin(bx), ox1 = a.ax.owned_end(bx);
  const int oy0 = a.ay.owned_begin(by), oy1 = a.ay.owned_end(by);
  T* __restrict__ un = a.u_new + plane;
  if (col_ok && gx >= ox0 && gx < ox1) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int ly = row0 + i;
      const int gy = y0 + ly;
      if (ly < B && gy >= oy0 && gy < oy1) {
        // unknown cells take the CG solution, known cells keep the residual
        const T v = ((unk >> i) & 1u) ? x[i] : S.rs[ly + 1][lx + 1];
        un[static_cast<size_t>(gy) * W + gx] = S.us[ly + 1][lx + 1] + v;
      }
    }
  }
  if (tid == 0 && a.counters && any_unknown) {
    if (!converged) atomicAdd(&a.counters[0], 1ull);
    atomicAdd(&a.counters[1], static_cast<unsigned long long>(iters));
  }
}

}  // namespace sib
