// K2 oras_sweep: one outer ORAS/RAS sweep, fused end to end.
//
// Replaces the whole block loop of run_schwarz_level (schwarz.hpp:305-318):
//   restrict_block_into (partition.hpp:109-121) of r = b - A u,
//   prepare_local_block / fill_local_structure (schwarz.hpp:84-111, 179-198),
//   solve_local_block + cg_solve (schwarz.hpp:202-250, cg.hpp:90-154),
//   accumulate_owned (partition.hpp:148-156).
//
// One CTA = one (subdomain, channel), NW warps (2 by default, chosen by
// measurement).  Layout: lane = block column, warp w owns rows
// [w*R, (w+1)*R), R = 32/NW, so every CG vector lives in registers (R values
// per thread per vector):
//   * setup: the block's u_old with a 2-pixel halo arrives in shared memory by
//     one TMA box copy (zero fill outside the image) where the box start is
//     16-byte aligned, else by one cooperative all-loads-first pass; the mask
//     bits of the thread's rows are loaded while the tile is in flight; the
//     residual slice and the local right-hand side are then evaluated
//     branch-free from the tile;
//   * stencil: W/E neighbours from the adjacent lanes by shuffle (no shared
//     memory traffic: the staged-row variant kept the LSU data pipe 73% busy),
//     N/S from the thread's registers;
//   * rows at warp boundaries are exchanged with no dedicated barrier: before
//     each reduction barrier every warp publishes the *components* of its
//     boundary rows (r, old p, x) and its neighbours rebuild p_new = r + beta*p
//     with the identical fma afterwards.  One CG iteration costs 2 CTA
//     barriers (3 on a true-residual check);
//   * dot products: 4-accumulator tree per thread, warp total on the FP64
//     tensor core (DMMA), pairwise tree over the warps, so every thread holds
//     the same value and all control flow is CTA-uniform.
// u_new = u_old + v is written only on the block's owned rectangle into a
// separate buffer (ping-pong): owned rectangles tile the image, so every
// pixel is written exactly once and no CTA reads what another writes.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "tma.cuh"

namespace sib {

// u_old tile of a block: rows y0-2 .. y0+B+1, columns x0-1 .. x0+B.
// Column j of the tile is x = x0 - lead + j: the block's columns are
// j = lead .. lead+B-1, the ring columns lead-1 and lead+B.  The cooperative
// copy uses lead 2; the TMA box starts at the 16-byte aligned column
// x0 - lead with lead = ((x0 - 1) mod q) + 1, q = 16 / sizeof(T), so the
// tile is 32 + q + 2 columns rounded to a 16-byte row (fp64 36, fp32 40).
constexpr int kTileH = kMaxBlock + 4;
template <typename T>
__host__ __device__ constexpr int tile_w() {
  return sizeof(T) == 8 ? kMaxBlock + 4 : kMaxBlock + 8;
}
template <typename T>
__host__ __device__ inline int tile_lead(int x0) {
  constexpr int q = 16 / static_cast<int>(sizeof(T));
  return ((x0 - 1) % q + q) % q + 1;
}

template <typename T>
struct SweepArgs {
  CUtensorMap umap;    // TMA map of u_old ([C][H][W], box tile_w x kTileH) when use_tma
  int use_tma;
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
  int known_invariant;    // multilevel invariant: b = 0 at unknown pixels and u = b at
                       // known pixels (so r = 0 there); b is never read
  unsigned long long* counters;  // [0] failures, [1] CG iterations (may be null)
  int by0;             // first block row of this launch (stripe mode; 0 otherwise)
  // Stripe storage: the buffers hold only image rows [srow_lo, srow_hi) (the
  // pointers above are pre-offset by -srow_lo rows, N is the storage plane);
  // the TMA map covers the storage, so tile rows outside it read as zeros --
  // only the discarded ghost-row residuals (tile rows 0 and B+3) can fall
  // there.  Whole-image solves: 0 and H.
  int srow_lo, srow_hi;
  T* scratch;          // K2g (blocks > 32): per-CTA CG vectors in global memory
  const int* skip;     // stripes: nonzero = the level has stopped, the sweep does nothing
};

template <typename T>
__device__ __forceinline__ T fmaT(T a, T b, T c) {
  return fma(a, b, c);
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

// W/E stencil neighbours by warp shuffle for a double local CG (the staged
// shared-memory row kept the L1 data pipe 73% busy: 3.135 -> 3.079 ms per
// frame's sweeps); a float CG keeps the staged row (one 4-byte shuffle per
// neighbour does not pay there: 437 -> 414 frames/s with shuffles).
template <typename L>
constexpr bool kShflWE = sizeof(L) == 8;

// T: storage / outer-iteration type of the image, L: type of the local CG
// (L = T, or float under double storage for the mixed-precision mode).
template <typename T, int NW, typename L = T>
struct SweepSmem {
  __align__(128) T ut[kTileH][tile_w<T>()];  // u_old tile with halo (TMA destination)
  uint64_t bar;                    // TMA completion
  // float local CG: stencil operand rows with zero ghost columns 0 and B+1
  // (double takes W/E by shuffle instead, see kShflWE)
  L pt[sizeof(L) == 8 ? 1 : kMaxBlock][sizeof(L) == 8 ? 1 : kMaxBlock + 2];
  L bt[kMaxBlock][kMaxBlock];      // local right-hand side (true-residual checks)
  L pub[NW][2][3][32];             // [warp][top/bottom][r,p,x][col]
  L pubt[NW][2][32];               // true-residual boundary rows
  L red[3][NW];
  uint32_t tslot;                  // TMEM base address (x in tensor memory)
};

// x (the CG iterate, touched once per iteration: x += alpha p) lives in TMEM
// for the full-block double CG with two warps: 32 registers per thread fewer
// in the loop, which removes the spills at the 168-register cap of 6 CTAs/SM.
// SI_NO_TMEM_X=1 at compile time keeps it in registers (A/B).
template <typename L, int NW, bool FULL>
constexpr bool kTmemX =
#ifdef SI_NO_TMEM_X
    false;
#else
    FULL && sizeof(L) == 8 && NW == 2;
#endif

// With x in TMEM, q = A p can follow it (columns 32..63): q leaves the
// registers four rows at a time as apply produces it and comes back for the
// r update, so the loop holds only r and p (64 registers of vectors) and
// the kernel fits 8 CTAs/SM (128 registers, no spill; 64 TMEM columns x 8
// CTAs = the SM's 512).  SI_NO_TMEM_Q=1 keeps q in registers (A/B).
// Full blocks: the W/E ghost zeros of lanes 0 and 31 are folded into the
// diagonal instead of selected: a shuffle past the warp edge returns the
// lane's own value v, and (d + 1) v - (v + vE) == d v - vE exactly in real
// arithmetic (rounding differs only in those two columns; the C3 frame keeps
// the reference's 1,716,457 local CG iterations).  Saves 4 selects per row:
// 2.79 -> 2.60 ms per frame's sweeps.  SI_NO_EDGE_FOLD=1 keeps the selects.
template <bool FULL>
constexpr bool kEdgeFold =
#ifdef SI_NO_EDGE_FOLD
    false;
#else
    FULL;
#endif

template <typename L, int NW, bool FULL>
constexpr bool kTmemQ =
#ifdef SI_NO_TMEM_Q
    false;
#else
    kTmemX<L, NW, FULL>;
#endif


// CTA-wide sum; identical value in every thread.  slot selects the buffer so
// consecutive reductions never race (see the header comment).  The warp part
// runs on the FP64 tensor core for double (warp_sum_mma), the cross-warp
// part is a pairwise tree over the NW warp totals.
template <typename T>
__device__ __forceinline__ T warp_total(T v) {
#ifdef SI_NO_DMMA
  return warp_sum(v);
#else
  if constexpr (sizeof(T) == 8)
    return warp_sum_mma(v);
  else
    return warp_sum(v);
#endif
}

template <typename T, int NW>
__device__ __forceinline__ T cta_sum(T v, T (*red)[NW], int slot, int warp, int lane) {
  v = warp_total(v);
  if (NW == 1) return v;
  if (lane == 0) red[slot][warp] = v;
  __syncthreads();
  T t[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) t[w] = red[slot][w];
#pragma unroll
  for (int h = 1; h < NW; h *= 2)
#pragma unroll
    for (int w = 0; w + h < NW; w += 2 * h) t[w] += t[w + h];
  return t[0];
}

// a / b, correctly rounded, from a precomputed rcp = RN(1/b): q0 = RN(a*rcp)
// is within an ulp of a/b, the residual a - b*q0 is exact under fma, and one
// correction q0 + rcp*(a - b*q0) rounds to RN(a/b) for normal operands
// (Markstein).  Lets beta = rr_new/rr take 1/rr computed an iteration early,
// off the critical path; si_selftest(0, ...) checks it bit for bit against
// the IEEE division.
__device__ __forceinline__ double recip_rn(double b) { return __drcp_rn(b); }
__device__ __forceinline__ float recip_rn(float b) { return __frcp_rn(b); }

template <typename T>
__device__ __forceinline__ T div_by_recip(T a, T b, T rcp) {
  const T q0 = a * rcp;
  const T e = fma(-b, q0, a);
  return fma(e, rcp, q0);
}

// Thread-local part of a dot product: four interleaved accumulators, then
// a pairwise tree (dependent depth R/4 + 2 instead of R).
template <typename T, int R>
__device__ __forceinline__ T dot2(const T (&a)[R], const T (&b)[R]) {
  constexpr int K = R >= 4 ? 4 : R;
  T s[K];
#pragma unroll
  for (int k = 0; k < K; ++k) s[k] = a[k] * b[k];
#pragma unroll
  for (int i = K; i < R; ++i) s[i % K] = fma(a[i], b[i], s[i % K]);
#pragma unroll
  for (int h = 1; h < K; h *= 2)
#pragma unroll
    for (int k = 0; k + h < K; k += 2 * h) s[k] += s[k + h];
  return s[0];
}

// sqrt(v) <= thr, evaluated out of line: the caller only needs it inside a
// narrow band around thr^2, everywhere else the squared test is exact.
template <typename T>
__device__ __noinline__ bool band_sqrt_le(T v, T thr) {
  return sqrt(v) <= thr;
}

// Per-thread view of the block: column lx, rows row0 .. row0+R-1.
template <typename T, int R>
struct Cell {
  int lx, gx, row0, x0, y0, B, W, H;
  int tl;  // tile column of pixel x0 (see tile_lead)
  bool col_ok;
  const uint8_t* __restrict__ mask;
  const T* __restrict__ u;
  const T* __restrict__ b;
  int known_invariant;
};

// u_old tile of the block with a 1-column / 2-row halo, rows y0-2 .. y0+B+1
// and columns x0-1 .. x0+B, zero outside the image.  Loaded cooperatively by
// the whole CTA (consecutive threads -> consecutive columns of a row: 272-byte
// coalesced row segments, every load independent and issued up front).
template <typename T, int NW>
__device__ __forceinline__ void stage_u_tile(T (*ut)[tile_w<T>()], const T* __restrict__ u, int x0,
                                             int y0, int B, int W, int row_lo, int row_hi) {
  // Warp w stages tile rows w, w+NW, ...: lanes 0..B load columns x0..x0+B
  // (one coalesced row segment), lanes 30/31 the ring columns x0-1 and x0+32.
  constexpr int kRows = (kTileH + NW - 1) / NW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx = x0 + lane;
  const bool col_ok = lane <= B && gx < W;
  const int ex = lane == 30 ? x0 - 1 : x0 + 32;
  const bool ecol_ok = (lane == 30 && x0 > 0) || (lane == 31 && B == 32 && x0 + 32 < W);
  const size_t Wz = static_cast<size_t>(W);
  T v[kRows], e[kRows];
#pragma unroll
  for (int i = 0; i < kRows; ++i) {
    const int tr = warp + i * NW;
    const int gy = y0 - 2 + tr;
    const bool row_ok = tr < kTileH && tr <= B + 3 && gy >= row_lo && gy < row_hi;
    const T* row = u + static_cast<size_t>(row_ok ? gy : row_lo) * Wz;  // a stored row
    v[i] = (row_ok && col_ok) ? row[gx] : T(0);
    e[i] = (row_ok && ecol_ok) ? row[ex] : T(0);
  }
#pragma unroll
  for (int i = 0; i < kRows; ++i) {
    const int tr = warp + i * NW;
    if (tr < kTileH) {
      ut[tr][lane + 2] = v[i];
      if (lane == 30) ut[tr][1] = e[i];
      if (lane == 31) ut[tr][kMaxBlock + 2] = e[i];
    }
  }
}

// Residual r = b - A u (operators.hpp:38-66, 91-97) of block rows
// row0-1 .. row0+R (index j = 0..R+1; rows outside the block are ghosts = 0)
// from the staged u tile, plus the in-block known bits of the same rows.
//   known:   r = b - u
//   unknown: r = b - (deg*u - (((W + E) + N) + S)) over in-image neighbours;
// out-of-image neighbours are zeros of the tile, i.e. the reference's skipped
// term (x + 0 == x), deg counts the in-image ones.  Branch-free, so the rows
// overlap.  INV: the multilevel invariant (b never read).
// Mask bits (and b where the invariant does not hold) of the rows
// row0-1 .. row0+R at my column: every load issued at once, before the u tile
// is waited for, so their latency overlaps the tile copy.
template <typename T, int R, bool INV>
__device__ __forceinline__ void load_rows(const Cell<T, R>& c, uint64_t& kbits, T (&bv)[R + 2]) {
  const size_t W = static_cast<size_t>(c.W);
  kbits = 0;
#pragma unroll
  for (int j = 0; j < R + 2; ++j) {
    const int ly = c.row0 - 1 + j;
    const int gy = c.y0 + ly;
    const bool in_blk = c.col_ok && ly >= 0 && ly < c.B;
    // lanes outside the block read the block's first pixel (always stored,
    // also under stripe storage), so every load is issued unconditionally
    const size_t p = in_blk ? static_cast<size_t>(gy) * W + c.gx : static_cast<size_t>(c.y0) * W + c.x0;
    const uint8_t mv = c.mask[p];
    kbits |= static_cast<uint64_t>(in_blk && mv != 0) << j;
    if (!INV) {
      const T bb = c.b[p];
      bv[j] = in_blk ? bb : T(0);
    }
  }
}

template <typename T, int R, bool INV>
__device__ __forceinline__ void residual_rows(const Cell<T, R>& c, const T (*ut)[tile_w<T>()],
                                              T (&r)[R + 2], uint64_t kbits,
                                              const T (&bv)[R + 2]) {
  const int lane = threadIdx.x & 31;
  const int deg_x = (c.gx > 0) + (c.gx + 1 < c.W);
#pragma unroll
  for (int j = 0; j < R + 2; ++j) {
    const int ly = c.row0 - 1 + j;
    const int gy = c.y0 + ly;
    const int tr = ly + 2;
    const int tc = lane + c.tl;
    const T uc = ut[tr][tc];
    const T sum = ((ut[tr][tc - 1] + ut[tr][tc + 1]) + ut[tr - 1][tc]) + ut[tr + 1][tc];
    const int deg = deg_x + (gy > 0) + (gy + 1 < c.H);
    const T bj = INV ? T(0) : bv[j];
    const T ru = bj - fmaT(T(deg), uc, -sum);
    const T rk = INV ? T(0) : bj - uc;
    const bool in_blk = c.col_ok && ly >= 0 && ly < c.B;
    r[j] = in_blk ? (((kbits >> j) & 1ull) ? rk : ru) : T(0);
  }
}

// Local right-hand side of my rows (solve_local_block, schwarz.hpp:219-230):
//   rhs = unk * (pv + knw_W pv_W + knw_E pv_E + knw_N pv_N + knw_S pv_S),
// knw counting only in-block neighbours (ghost ring = 0).  Returns unk bits.
template <typename T, int R, bool INV, typename L>
__device__ __forceinline__ uint32_t local_rhs(const Cell<T, R>& c, const T (*ut)[tile_w<T>()],
                                              L (&rhs)[R], uint64_t kb, const T (&bv)[R + 2]) {
  const int lane = threadIdx.x & 31;
  T r[R + 2];
  residual_rows<T, R, INV>(c, ut, r, kb, bv);
  const uint64_t kbW = __shfl_up_sync(0xffffffffu, kb, 1);
  const uint64_t kbE = __shfl_down_sync(0xffffffffu, kb, 1);
  uint32_t unk = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int j = i + 1;
    const int ly = c.row0 + i;
    const T rW = __shfl_up_sync(0xffffffffu, r[j], 1);
    const T rE = __shfl_down_sync(0xffffffffu, r[j], 1);
    const bool unk_i = c.col_ok && ly < c.B && !((kb >> j) & 1ull);
    if (unk_i) unk |= 1u << i;
    // known rows carry r = 0 under the multilevel invariant, so there the
    // neighbour terms vanish; otherwise add each known in-block neighbour's r
    // (+0 for the others: the reference's skipped term).
    T t = r[j];
    if (!INV) {
      t += (lane > 0 && ((kbW >> j) & 1ull)) ? rW : T(0);
      t += (lane + 1 < c.B && ((kbE >> j) & 1ull)) ? rE : T(0);
      t += (ly > 0 && ((kb >> (j - 1)) & 1ull)) ? r[j - 1] : T(0);
      t += (ly + 1 < c.B && ((kb >> (j + 1)) & 1ull)) ? r[j + 1] : T(0);
    }
    t = unk_i ? t : T(0);
    rhs[i] = static_cast<L>(t);
  }
  return unk;
}

// Resident CTAs per SM requested from ptxas (caps registers per thread):
// the CG vectors need 4*R values of T per thread.
#ifndef SI_OCC64
#define SI_OCC64 4
#endif
#ifndef SI_OCC32
#define SI_OCC32 6
#endif
#ifndef SI_OCC64_2
#define SI_OCC64_2 6
#endif
#ifndef SI_OCC32_2
#define SI_OCC32_2 8
#endif
#ifndef SI_OCC64_8
#define SI_OCC64_8 3
#endif
#ifndef SI_OCC32_8
#define SI_OCC32_8 4
#endif
template <typename T, int NW>
struct SweepOcc {
  static constexpr int value =
      sizeof(T) == 8 ? (NW == 8 ? SI_OCC64_8 : NW == 4 ? SI_OCC64 : (NW == 2 ? SI_OCC64_2 : 1))
                     : (NW == 8 ? SI_OCC32_8 : NW == 4 ? SI_OCC32 : (NW == 2 ? SI_OCC32_2 : 2));
};

// (8 CTAs/SM either way at 128 registers; the hint of 7 schedules the loop
// better: 2.81 vs 2.88 ms per frame's sweeps)
#ifndef SI_OCC64_QT
#define SI_OCC64_QT 7
#endif
template <typename L, int NW, bool FULL>
constexpr int kSweepMinBlocks = kTmemQ<L, NW, FULL> ? SI_OCC64_QT : SweepOcc<L, NW>::value;

// FULL: the block is exactly 32x32 (every level of any image >= 32 pixels
// wide and high with the default block size), so the Robin rows are
// compile-time positions.
// L: the local CG's type (T, or float under double storage: the outer
// iteration, residuals and the image stay in T).
// SKIP (stripes): a.skip nonzero = the level has stopped, the CTA exits at
// once.  A separate instantiation: the early exit costs the hot variant its
// zero-spill allocation.
template <typename T, int NW, bool FULL, typename L = T, bool SKIP = false>
__global__ void __launch_bounds__(NW * 32, (kSweepMinBlocks<L, NW, FULL>))
    oras_sweep_kernel(const __grid_constant__ SweepArgs<T> a) {
  constexpr int R = 32 / NW;  // rows per thread
  __shared__ SweepSmem<T, NW, L> S;

  constexpr bool XT = kTmemX<L, NW, FULL>;
  constexpr bool QT = kTmemQ<L, NW, FULL>;
  constexpr uint32_t kCols = QT ? 64 : 32;
  if constexpr (SKIP) {
    if (*a.skip) return;  // uniform: before any barrier or TMEM
  }
  const int bx = blockIdx.x % a.ax.count;
  const int by = a.by0 + static_cast<int>(blockIdx.x) / a.ax.count;
  const int ch = blockIdx.y;
  const int B = FULL ? kMaxBlock : a.ax.block;
  uint32_t tbase = 0, taddr = 0;
  if constexpr (XT) {
    tbase = tmem_alloc_cta<kCols>(&S.tslot);
    taddr = tmem_warp_addr(tbase);
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t plane = static_cast<size_t>(ch) * a.N;

  Cell<T, R> c;
  c.lx = lane;
  c.x0 = a.ax.anchor(bx);
  c.y0 = a.ay.anchor(by);
  c.gx = c.x0 + lane;
  c.row0 = warp * R;
  c.B = B;
  c.W = a.W;
  c.H = a.H;
  c.col_ok = lane < B;
  c.mask = a.mask;
  c.u = a.u_old + plane;
  c.b = a.b + plane;
  c.known_invariant = a.known_invariant;
  c.tl = a.use_tma ? tile_lead<T>(c.x0) : 2;

  L x[XT ? 1 : R], r[R], p[R], q[QT ? 1 : R];  // XT / QT: x / q in TMEM
  uint32_t unk;
  // u tile (TMA box or cooperative copy) and the mask bits of my rows, the
  // latter in flight while the tile arrives; then residual and right-hand side
  auto setup = [&](auto inv_tag) {
    constexpr bool INV = decltype(inv_tag)::value;
    uint64_t kb;
    T bv[R + 2];
    if (a.use_tma) {
      // one TMA box: rows y0-2 .. y0+33, columns x0-2 .. x0+33 of this
      // channel, zeros outside the image
      if (tid == 0) {
        mbar_init(&S.bar, 1);
        mbar_expect_tx(&S.bar, sizeof(S.ut));
        tma_load_3d(&S.ut[0][0], &a.umap, c.x0 - c.tl, c.y0 - 2 - a.srow_lo, ch, &S.bar);
      }
      load_rows<T, R, INV>(c, kb, bv);
      __syncthreads();
      mbar_wait(&S.bar, 0);
    } else {
      load_rows<T, R, INV>(c, kb, bv);
      stage_u_tile<T, NW>(S.ut, c.u, c.x0, c.y0, B, c.W, a.srow_lo, a.srow_hi);
      __syncthreads();
    }
    unk = local_rhs<T, R, INV, L>(c, S.ut, r, kb, bv);
  };
  if (a.known_invariant)
    setup(std::true_type{});
  else
    setup(std::false_type{});
  if constexpr (XT) {
    double z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0.0;
    tmem_store16(taddr, z);
  } else {
#pragma unroll
    for (int i = 0; i < R; ++i) x[i] = L(0);
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    S.bt[c.row0 + i][lane] = r[i];
    if constexpr (!kShflWE<L>) S.pt[c.row0 + i][lane + 1] = r[i];  // p = r initially
  }
  if constexpr (!kShflWE<L>) {
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) S.pt[c.row0 + i][0] = L(0);
    }
    if (lane == B - 1 || (!FULL && lane == 31)) {
#pragma unroll
      for (int i = 0; i < R; ++i) S.pt[c.row0 + i][B + 1] = L(0);
    }
  }
  const int any_unknown = __syncthreads_or(unk != 0);

  // Robin diagonals of my column: interior rows, block row 0, block row B-1.
  L dI = L(0), dT = L(0), dB = L(0);
  if (c.col_ok) {
    const L am1 = static_cast<L>(a.am1);
    dI = robin_diag<L>(c.gx, c.y0 + 1, lane, 1, B, c.W, c.H, am1, a.ras);
    dT = robin_diag<L>(c.gx, c.y0, lane, 0, B, c.W, c.H, am1, a.ras);
    dB = robin_diag<L>(c.gx, c.y0 + B - 1, lane, B - 1, B, c.W, c.H, am1, a.ras);
  }
  if constexpr (kShflWE<L> && kEdgeFold<FULL>) {
    if (lane == 0 || lane == 31) {  // see kEdgeFold
      dI += L(1);
      dT += L(1);
      dB += L(1);
    }
  }
  const L dFirst = (warp == 0) ? dT : dI;        // FULL: row i = 0
  const L dLast = (warp == NW - 1) ? dB : dI;    // FULL: row i = R-1
  const int iT = -c.row0;            // generic: local index of block row 0
  const int iB = (B - 1) - c.row0;   // generic: local index of block row B-1

  int iters = 0;
  bool converged = true;

  if (any_unknown) {
#pragma unroll
    for (int i = 0; i < R; ++i) p[i] = r[i];  // r = b - A*0 = b exactly
    L nb_p[2] = {L(0), L(0)}, nb_r[2] = {L(0), L(0)};

    auto publish = [&]() {
      if (NW > 1) {
        S.pub[warp][0][0][lane] = r[0];
        S.pub[warp][0][1][lane] = p[0];
        S.pub[warp][1][0][lane] = r[R - 1];
        S.pub[warp][1][1][lane] = p[R - 1];
        if constexpr (!XT) {  // XT: published by the x update itself
          S.pub[warp][0][2][lane] = x[0];
          S.pub[warp][1][2][lane] = x[R - 1];
        }
      }
    };
    if constexpr (XT) {  // x = 0 before the first iteration
      S.pub[warp][0][2][lane] = L(0);
      S.pub[warp][1][2][lane] = L(0);
    }
    auto collect = [&]() {
      if (NW > 1) {
        if (warp > 0) {
          nb_r[0] = S.pub[warp - 1][1][0][lane];
          nb_p[0] = S.pub[warp - 1][1][1][lane];
        }
        if (warp + 1 < NW) {
          nb_r[1] = S.pub[warp + 1][0][0][lane];
          nb_p[1] = S.pub[warp + 1][0][1][lane];
        }
      }
    };
    // float: stage my rows of v as stencil operand (the warp owns whole rows,
    // so a warp barrier suffices; the ghost columns stay zero)
    auto stage = [&](const L(&v)[R]) {
      if constexpr (!kShflWE<L>) {
        __syncwarp();
#pragma unroll
        for (int i = 0; i < R; ++i) S.pt[c.row0 + i][lane + 1] = v[i];
        __syncwarp();
      }
    };
    // o = A v on my cells (LocalStencilOperator::apply, schwarz.hpp:146-159):
    // o = unk * (d*v - vW - vE - vN - vS); block-external neighbours are
    // ghost zeros.  double: W/E come from the neighbouring lanes by shuffle
    // (lane 0's W and lane 31's E are the ghost zeros; columns >= B of a
    // partial block hold zeros); float: from the staged row.  N/S from my
    // registers or the neighbour warps' rows vN0/vS1.
    auto row_op = [&](const L(&v)[R], int i, L vN0, L vS1) -> L {
      L vW, vE;
      if constexpr (kShflWE<L> && kEdgeFold<FULL>) {
        // lanes 0 / 31 receive their own value; their diagonal carries +1
        vW = __shfl_up_sync(0xffffffffu, v[i], 1);
        vE = __shfl_down_sync(0xffffffffu, v[i], 1);
      } else if constexpr (kShflWE<L>) {
        const L sW = __shfl_up_sync(0xffffffffu, v[i], 1);
        const L sE = __shfl_down_sync(0xffffffffu, v[i], 1);
        vW = lane > 0 ? sW : L(0);
        vE = lane < 31 ? sE : L(0);
      } else {
        vW = S.pt[c.row0 + i][lane];
        vE = S.pt[c.row0 + i][lane + 2];
      }
      const L vN = i > 0 ? v[i - 1] : vN0;
      const L vS = i + 1 < R ? v[i + 1] : vS1;
      L d;
      if (FULL)
        d = (i == 0) ? dFirst : ((i == R - 1) ? dLast : dI);
      else
        d = (i == iT) ? dT : ((i == iB) ? dB : dI);
      // d*v - (vW + vE) - (vN + vS): dependent depth 3 (the reference's
      // left-to-right chain is 4; the values agree to rounding)
      const L t = fmaT(d, v[i], -(vW + vE)) - (vN + vS);
      return ((unk >> i) & 1u) ? t : L(0);
    };
    auto apply = [&](const L(&v)[R], L vN0, L vS1, L(&o)[R]) {
#pragma unroll
      for (int i = 0; i < R; ++i) o[i] = row_op(v, i, vN0, vS1);
    };
    // QT: q = A p streamed to TMEM four rows at a time with the thread part
    // of p.q accumulated on the way (dot2's exact order: s[k] = p_k q_k for
    // the first four rows, then s[i % 4] = fma(p_i, q_i, s[i % 4]), then the
    // pairwise tree)
    auto apply_pq_tmem = [&](L vN0, L vS1) -> L {
      if constexpr (QT) {
        double s4[4];
#pragma unroll
        for (int k = 0; k < R / 4; ++k) {
          double qc[4];
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            const int i = 4 * k + ii;
            qc[ii] = row_op(p, i, vN0, vS1);
            s4[ii] = k == 0 ? p[i] * qc[ii] : fma(p[i], qc[ii], s4[ii]);
          }
          tmem_store4(taddr + 32 + 8 * k, qc);
        }
        return (s4[0] + s4[1]) + (s4[2] + s4[3]);
      } else {
        return L(0);
      }
    };

    publish();
    L rr = cta_sum<L, NW>(dot2<L, R>(r, r), S.red, 1, warp, lane);  // also orders the pt staging
    L rr_rcp = recip_rn(rr);
    collect();
    nb_p[0] = nb_r[0];  // p = r initially
    nb_p[1] = nb_r[1];
    const L r0 = sqrt(rr);
    // maybe_done = sqrt(rr_new) <= tol*r0 (cg.hpp:132); the sqrt is only
    // evaluated inside a 1e-12 band around the threshold, outside it the
    // squared comparison decides identically.
    const L thr = a.ltol * r0;
    const L thr2 = thr * thr;
    const L thr2_lo = thr2 * L(1.0 - 1e-6), thr2_hi = thr2 * L(1.0 + 1e-6);
    converged = false;
    if (r0 == L(0)) {
      converged = true;
    } else {
      int until_check = a.lcheck;  // iter % lcheck == 0  <=>  countdown hits 0
      for (int iter = 1; iter <= a.lmax; ++iter) {
        L part_pq;
        if constexpr (QT) {
          part_pq = apply_pq_tmem(nb_p[0], nb_p[1]);
        } else {
          apply(p, nb_p[0], nb_p[1], q);
          part_pq = dot2<L, R>(p, q);
        }
        const L pAp = cta_sum<L, NW>(part_pq, S.red, 0, warp, lane);
        if (!(pAp > L(0)) || !isfinite(pAp)) {  // breakdown (cg.hpp:120-125)
          iters = iter - 1;
          break;
        }
        // alpha = rr / pAp through the correctly rounded reciprocal and one
        // Markstein step (== the IEEE quotient, si_selftest 0): 2.81 -> 2.78 ms
        // per frame's sweeps; SI_ALPHA_DIV=1 keeps the division (A/B)
#ifdef SI_ALPHA_DIV
        const L alpha = rr / pAp;
#else
        const L alpha = div_by_recip(rr, pAp, recip_rn(pAp));
#endif
        if constexpr (XT) {
          if constexpr (QT) {
            double qv[16];
            tmem_wait_st();
            tmem_load16(taddr + 32, qv);
#pragma unroll
            for (int i = 0; i < R; ++i) r[i] = fmaT(-alpha, qv[i], r[i]);
          } else {
#pragma unroll
            for (int i = 0; i < R; ++i) r[i] = fmaT(-alpha, q[i], r[i]);
          }
          // x += alpha p through TMEM (the previous store has long landed)
          double xv[16];
          tmem_wait_st();
          tmem_load16(taddr, xv);
#pragma unroll
          for (int i = 0; i < 16; ++i) xv[i] = fma(alpha, p[i], xv[i]);
          S.pub[warp][0][2][lane] = xv[0];
          S.pub[warp][1][2][lane] = xv[15];
          tmem_store16(taddr, xv);
        } else {
#pragma unroll
          for (int i = 0; i < R; ++i) {
            x[i] = fmaT(alpha, p[i], x[i]);
            r[i] = fmaT(-alpha, q[i], r[i]);
          }
        }
        publish();
        L rr_new = cta_sum<L, NW>(dot2<L, R>(r, r), S.red, 1, warp, lane);
        collect();
        if (--until_check == 0) until_check = a.lcheck;
        const bool cadence = until_check == a.lcheck || iter == a.lmax;
        bool maybe_done = rr_new < thr2_lo;
        if (rr_new >= thr2_lo && rr_new <= thr2_hi) maybe_done = band_sqrt_le(rr_new, thr);
        if (cadence || maybe_done) {
          // True residual b - A x, then confirm or replace (cg.hpp:131-146).
          // the neighbours' boundary rows of x were published before the rr
          // barrier of this iteration
          const L nx0 = (NW > 1 && warp > 0) ? S.pub[warp - 1][1][2][lane] : L(0);
          const L nx1 = (NW > 1 && warp + 1 < NW) ? S.pub[warp + 1][0][2][lane] : L(0);
          L tq[R];
          if constexpr (XT) {
            double xv[16];
            tmem_wait_st();
            tmem_load16(taddr, xv);
            apply(xv, nx0, nx1, tq);
          } else {
            stage(x);
            apply(x, nx0, nx1, tq);
          }
#pragma unroll
          for (int i = 0; i < R; ++i) tq[i] = S.bt[c.row0 + i][lane] - tq[i];
          const L part = dot2<L, R>(tq, tq);
          if (NW > 1) {
            S.pubt[warp][0][lane] = tq[0];
            S.pubt[warp][1][lane] = tq[R - 1];
          }
          const L tt = cta_sum<L, NW>(part, S.red, 2, warp, lane);
          const L rel = sqrt(tt) / r0;
          if (rel <= a.ltol) {
            iters = iter;
            converged = true;
            break;
          }
#pragma unroll
          for (int i = 0; i < R; ++i) r[i] = tq[i];
          if (NW > 1) {
            if (warp > 0) nb_r[0] = S.pubt[warp - 1][1][lane];
            if (warp + 1 < NW) nb_r[1] = S.pubt[warp + 1][0][lane];
          }
          rr_new = tt;
        }
        const L beta = div_by_recip(rr_new, rr, rr_rcp);  // == rr_new / rr
#pragma unroll
        for (int i = 0; i < R; ++i) p[i] = fmaT(beta, p[i], r[i]);
        stage(p);
        nb_p[0] = fmaT(beta, nb_p[0], nb_r[0]);
        nb_p[1] = fmaT(beta, nb_p[1], nb_r[1]);
        rr = rr_new;
        rr_rcp = recip_rn(rr);
        if (iter == a.lmax) iters = a.lmax;
      }
    }
  }

  // ---- accumulate_owned: u_new = u_old + v on the owned rectangle ----------
  // v = CG solution at unknown cells, the residual b - u at known cells.
  const int ox0 = a.ax.owned_begin(bx), ox1 = a.ax.owned_end(bx);
  const int oy0 = a.ay.owned_begin(by), oy1 = a.ay.owned_end(by);
  T* __restrict__ un = a.u_new + plane;
  const bool col_own = c.col_ok && c.gx >= ox0 && c.gx < ox1;
  L xf[R];  // the local solution of my cells
  if constexpr (XT) {
    double xv[16];
    tmem_wait_st();
    tmem_load16(taddr, xv);
#pragma unroll
    for (int i = 0; i < R; ++i) xf[i] = xv[i];
    // every warp has read its columns: free them
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    tmem_free_cta<kCols>(tbase);
  } else {
#pragma unroll
    for (int i = 0; i < R; ++i) xf[i] = x[i];
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int ly = c.row0 + i;
    const int gy = c.y0 + ly;
    const bool own = col_own && ly < B && gy >= oy0 && gy < oy1;
    const size_t pix = own ? static_cast<size_t>(gy) * c.W + c.gx
                           : static_cast<size_t>(c.y0) * c.W + c.x0;  // a stored pixel
    const T uo = S.ut[ly + 2][lane + c.tl];
    T v = static_cast<T>(xf[i]);
    if (!c.known_invariant) {
      const T bk = c.b[pix];
      if (!((unk >> i) & 1u)) v = bk - uo;
    } else if (!((unk >> i) & 1u)) {
      v = T(0);
    }
    if (own) un[pix] = uo + v;
  }
  pdl_trigger();  // the residual of u_new may start launching
  if (tid == 0 && a.counters && any_unknown) {
    if (!converged) atomicAdd(&a.counters[0], 1ull);
    atomicAdd(&a.counters[1], static_cast<unsigned long long>(iters));
  }
}

}  // namespace sib
