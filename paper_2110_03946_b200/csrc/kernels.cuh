// Memory-bound kernels around the sweep: K1 residual norms, K3 pyramid
// restriction, K4 prolongation + snap, K5 ingest, export, K6 MSE.
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace sib {

// Per-channel deterministic reduction: each CTA writes one partial per
// channel (blockIdx.y); the last CTA to finish (atomic ticket) sums the
// partials in a fixed order, so the result depends only on the launch shape.
constexpr int kRedThreads = 256;
constexpr int kRedBlocksMax = 1184;  // 148 SMs x 8

// K sums per CTA (v[k]); blk: this CTA's index among the nblk CTAs of its
// channel chn (of nch).  Final results: out[k*nch + c].
template <int K, int NT = kRedThreads>
__device__ void reduce_epilogue_k(const double (&vin)[K], double* partials, double* out,
                                  unsigned int* ticket, int blk, int nblk, int chn, int nch) {
  __shared__ double wsum[K][NT / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double v = warp_sum(vin[k]);
    if (lane == 0) wsum[k][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += wsum[k][w];
      partials[(k * nch + chn) * nblk + blk] = s;
    }
    __threadfence();
    const unsigned int total = gridDim.x * gridDim.y * gridDim.z;
    last = atomicAdd(ticket, 1u) == total - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Fixed-order final sum per (value, channel): strided partials + butterfly.
  for (int kc = 0; kc < K * nch; ++kc) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nblk; i += NT)
      s += reinterpret_cast<volatile double*>(partials)[kc * nblk + i];
    s = warp_sum(s);
    __syncthreads();
    if (lane == 0) wsum[0][warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < NT / 32; ++w) t += wsum[0][w];
      out[kc] = t;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

template <int NT = kRedThreads>
__device__ __forceinline__ void reduce_epilogue(double v, double* partials, double* out,
                                                unsigned int* ticket, int blk, int nblk, int chn,
                                                int nch) {
  const double vv[1] = {v};
  reduce_epilogue_k<1, NT>(vv, partials, out, ticket, blk, nblk, chn, nch);
}

// K1: per channel sum of (b - A u)^2 (residual_into + vec::norm^2,
// operators.hpp:38-66/91-97, cg.hpp:46-50); mode 1: sum of b^2 (RhsNorm).
// Grid (x segments of kRedThreads columns, bands of kResBand rows, channel).
// The CTA copies its band of u plus a one-pixel halo into shared memory with
// cp.async (every load in flight at once, zero fill outside the image, u read
// from memory once per pixel plus a 2-row halo per band), then each thread
// evaluates the stencil of its column from shared memory.  known_invariant:
// u == b at known pixels and b == 0 elsewhere (the multilevel data flow), so
// b is never read.
constexpr int kResBand = 16;
constexpr int kResTileW = kRedThreads + 2;
static_assert(kResBand + 2 <= 32, "halo loaders assume at most 32 band rows");

__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, int bytes, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src = ok ? bytes : 0;
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
}

template <typename T, bool INV>
__global__ void __launch_bounds__(kRedThreads)
    residual_sumsq_kernel(const uint8_t* __restrict__ mask, const T* __restrict__ u,
                          const T* __restrict__ b, int W, int H, size_t N, int mode, int row0,
                          int row1, int srow_lo, int srow_hi, double* partials, double* out,
                          unsigned int* ticket, const int* __restrict__ skip) {
  // rows [row0, row1) only (stripe mode); the stencil still sees rows
  // row0-1 and row1 as neighbours.  The buffers hold rows [srow_lo, srow_hi)
  // (pointers pre-offset, N = storage plane); whole image: 0 and H.
  __shared__ T tile[kResBand + 2][kResTileW];
  if (skip != nullptr && *skip) return;  // stripes: the level has stopped (every CTA alike)
  const int c = blockIdx.z;
  const T* __restrict__ uc = u + c * N;
  const T* __restrict__ bc = b + c * N;
  const int x0 = blockIdx.x * kRedThreads;
  const int x = x0 + threadIdx.x;
  const int y0 = row0 + static_cast<int>(blockIdx.y) * kResBand;
  const int ny = min(kResBand, row1 - y0);
  const bool xin = x < W;
  const size_t Wz = static_cast<size_t>(W);
  // inactive lanes address row0 (stored under stripe storage too)
  const T* ustored = uc + static_cast<size_t>(row0) * Wz;
  double acc = 0.0;
  if (mode == 1) {
    T v[kResBand];
#pragma unroll
    for (int k = 0; k < kResBand; ++k)
      v[k] = (xin && k < ny) ? __ldg(bc + static_cast<size_t>(y0 + k) * Wz + x) : T(0);
#pragma unroll
    for (int k = 0; k < kResBand; ++k) {
      const double d = static_cast<double>(v[k]);
      acc = fma(d, d, acc);
    }
  } else {
    // tile[k][1 + j] = u(y0 - 1 + k, x0 + j); column 0 / kResTileW-1 = the
    // halo columns x0 - 1 / x0 + kRedThreads.  Thread t copies column t of
    // every band row; threads 0..17 and 32..49 copy one halo element each.
    const int nrows = min(kResBand + 2, ny + 2);
    const T* col = uc + x;
#pragma unroll
    for (int k = 0; k < kResBand + 2; ++k) {
      const int gy = y0 - 1 + k;
      const bool ok = k < nrows && gy >= 0 && gy < H && gy >= srow_lo && gy < srow_hi && xin;
      cp_async_zfill(&tile[k][threadIdx.x + 1], ok ? col + static_cast<ptrdiff_t>(gy) * W : ustored,
                     sizeof(T), ok);
    }
    {
      const int t = threadIdx.x;
      const bool west = t < kResBand + 2, east = t >= 32 && t < 32 + kResBand + 2;
      if (west || east) {
        const int k = west ? t : t - 32;
        const int gy = y0 - 1 + k;
        const int gx = west ? x0 - 1 : x0 + kRedThreads;
        const bool ok = k < nrows && gy >= 0 && gy < H && gy >= srow_lo && gy < srow_hi &&
                        gx >= 0 && gx < W;
        cp_async_zfill(&tile[k][west ? 0 : kResTileW - 1],
                       ok ? uc + static_cast<size_t>(gy) * Wz + gx : ustored, sizeof(T), ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    // mask bytes (and b when the invariant does not hold) of my column,
    // loaded while the copies are in flight
    uint8_t mk[kResBand];
    T bv[kResBand];
    const size_t base = xin ? static_cast<size_t>(y0) * Wz + x : static_cast<size_t>(y0) * Wz;
#pragma unroll
    for (int k = 0; k < kResBand; ++k) {
      const bool in = xin && k < ny;
      const size_t i = in ? base + static_cast<size_t>(k) * Wz : static_cast<size_t>(y0) * Wz;
      const uint8_t m = __ldg(mask + i);
      mk[k] = in ? m : uint8_t(0);
      if (!INV) {
        const T bb = __ldg(bc + i);
        bv[k] = in ? bb : T(0);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    const int t = threadIdx.x + 1;
    const int deg_x = (x > 0) + (x + 1 < W);
    const T deg_in = T(deg_x + 2);  // rows with both vertical neighbours
    T up = tile[0][t], ctr = tile[1][t];
#pragma unroll
    for (int k = 0; k < kResBand; ++k) {
      const int y = y0 + k;
      const T dn = tile[k + 2][t];
      // operators.hpp:44-58: ((W + E) + N) + S over in-image neighbours; an
      // absent neighbour is a zero of the tile (x + 0 == x), deg counts the
      // present ones.  Known pixels: r = b - u (+0 under the invariant).
      const T sum = ((tile[k + 1][t - 1] + tile[k + 1][t + 1]) + up) + dn;
      const T deg = (y > 0 && y + 1 < H) ? deg_in : T(deg_x + (y > 0) + (y + 1 < H));
      const T au = fma(deg, ctr, -sum);
      T r;
      if (INV)
        r = mk[k] ? T(0) : au;  // (0 - au)^2 == au^2
      else
        r = mk[k] ? bv[k] - ctr : bv[k] - au;
      const double rd = (xin && k < ny) ? static_cast<double>(r) : 0.0;
      acc = fma(rd, rd, acc);
      up = ctr;
      ctr = dn;
    }
  }
  reduce_epilogue(acc, partials, out, ticket, blockIdx.y * gridDim.x + blockIdx.x,
                  gridDim.x * gridDim.y, blockIdx.z, gridDim.z);
}

// K1 with the band tile fetched by one TMA box copy (tensor map over the
// planar [C][H][W] iterate): 128 columns x kResBand rows per CTA, box
// (x0 - kLead .. x0 + 127 + kLead) x (y0 - 1 .. y0 + kResBand), zero
// outside the image.
// Used when the row pitch is a multiple of 16 bytes (every level of an even
// width in fp64); otherwise the cp.async kernel above runs.
constexpr int kResTmaThreads = 128;
#ifndef SI_RES_BAND
#define SI_RES_BAND 16
#endif
constexpr int kResTmaBand = SI_RES_BAND;  // rows per CTA of the TMA variant
// The box starts kLead = 16 / sizeof(T) columns left of the CTA's first
// column (TMA wants 16-byte aligned inner box starts) and is 128 + 2 kLead
// wide (a 16-byte multiple).
template <typename T>
__host__ __device__ constexpr int res_tma_lead() {
  return 16 / static_cast<int>(sizeof(T));
}
template <typename T>
__host__ __device__ constexpr int res_tma_box_w() {
  return kResTmaThreads + 2 * res_tma_lead<T>();
}

// MTMA: the mask band arrives by a second TMA box on the same barrier (row
// pitch a multiple of 16 bytes), else per-thread byte loads.  The CTA writes
// its partial sum; finish_partials_kernel adds them in a fixed order (no
// fence or ticket in this kernel: a last-CTA ticket finish measured 0.245 ->
// 0.306 ms of K1 per 4K frame, round 2, as in round 1).
template <typename T, bool INV, bool MTMA>
__global__ void __launch_bounds__(kResTmaThreads)
    residual_sumsq_tma_kernel(const __grid_constant__ CUtensorMap umap,
                              const __grid_constant__ CUtensorMap mmap,
                              const uint8_t* __restrict__ mask, const T* __restrict__ b, int W,
                              int H, size_t N, int row0, int row1, int srow_lo,
                              double* partials, const int* __restrict__ skip) {
  __shared__ __align__(128) T tile[kResTmaBand + 2][res_tma_box_w<T>()];
  __shared__ __align__(128) uint8_t mtile[kResTmaBand][kResTmaThreads];
  __shared__ uint64_t bar;
  const int c = blockIdx.z;
  const T* __restrict__ bc = b + c * N;
  const int x0 = blockIdx.x * kResTmaThreads;
  const int x = x0 + threadIdx.x;
  const int y0 = row0 + static_cast<int>(blockIdx.y) * kResTmaBand;
  const int ny = min(kResTmaBand, row1 - y0);
  const bool xin = x < W;
  const size_t Wz = static_cast<size_t>(W);
  pdl_wait();  // u is the predecessor's output
  if (skip != nullptr && *skip) return;  // stripes: the level has stopped (every CTA alike)
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, sizeof(tile) + (MTMA ? sizeof(mtile) : 0));
    // the maps cover the storage rows (stripe mode: [srow_lo, ...)): rows
    // outside it arrive as zeros and are never used for rows in [row0, row1)
    tma_load_3d(&tile[0][0], &umap, x0 - res_tma_lead<T>(), y0 - 1 - srow_lo, c, &bar);
    if (MTMA) tma_load_2d(&mtile[0][0], &mmap, x0, y0 - srow_lo, &bar);
  }
  uint8_t mk[kResTmaBand];
  T bv[kResTmaBand];
  // inactive lanes address row y0 (stored under stripe storage too)
  const size_t base = xin ? static_cast<size_t>(y0) * Wz + x : static_cast<size_t>(y0) * Wz;
#pragma unroll
  for (int k = 0; k < kResTmaBand; ++k) {
    const bool in = xin && k < ny;
    const size_t i = in ? base + static_cast<size_t>(k) * Wz : static_cast<size_t>(y0) * Wz;
    if (!MTMA) {
      const uint8_t m = __ldg(mask + i);
      mk[k] = in ? m : uint8_t(0);
    }
    if (!INV) {
      const T bb = __ldg(bc + i);
      bv[k] = in ? bb : T(0);
    }
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  mbar_wait(&bar, 0);
  if (MTMA) {
#pragma unroll
    for (int k = 0; k < kResTmaBand; ++k)
      mk[k] = (xin && k < ny) ? mtile[k][threadIdx.x] : uint8_t(0);
  }
  const int t = threadIdx.x + res_tma_lead<T>();
  const int deg_x = (x > 0) + (x + 1 < W);
  const T deg_in = T(deg_x + 2);
  T up = tile[0][t], ctr = tile[1][t];
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kResTmaBand; ++k) {
    const int y = y0 + k;
    const T dn = tile[k + 2][t];
    const T sum = ((tile[k + 1][t - 1] + tile[k + 1][t + 1]) + up) + dn;
    const T deg = (y > 0 && y + 1 < H) ? deg_in : T(deg_x + (y > 0) + (y + 1 < H));
    const T au = fma(deg, ctr, -sum);
    T r;
    if (INV)
      r = mk[k] ? T(0) : au;
    else
      r = mk[k] ? bv[k] - ctr : bv[k] - au;
    const double rd = (xin && k < ny) ? static_cast<double>(r) : 0.0;
    acc = fma(rd, rd, acc);
    up = ctr;
    ctr = dn;
  }
  // CTA partial: warp totals, then warp 0 adds them in order
  __shared__ double wsum[kResTmaThreads / 32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kResTmaThreads / 32; ++w) t += wsum[w];
    partials[static_cast<size_t>(blockIdx.z) * gridDim.x * gridDim.y + blockIdx.y * gridDim.x +
             blockIdx.x] = t;
  }
  pdl_trigger();
}

// K1 pair: the residual of the level's start iterate u0 AND canonical_r0's
// residual of u = b (schwarz.hpp:333-345) in one pass, under the multilevel
// invariant (b never read at unknown pixels, r = 0 at known ones): two TMA
// tiles (u0, b) and the mask band on one barrier; partials for u0 at
// [c][blk], for b at [C + c][blk] -- one finish over 2C "channels" leaves
// the sums at out[0..C) and r0's at out[C..2C).  Saves one launch pair and
// one mask pass per level against two separate K1 launches.
constexpr int kResPairBand = 16;  // rows per CTA of the pair pass (two tiles in smem)
template <typename T, bool MTMA>
__global__ void __launch_bounds__(kResTmaThreads)
    residual_pair_tma_kernel(const __grid_constant__ CUtensorMap umap,
                             const __grid_constant__ CUtensorMap bmap,
                             const __grid_constant__ CUtensorMap mmap,
                             const uint8_t* __restrict__ mask, int W, int H, int row0, int row1,
                             int srow_lo, double* partials) {
  // each TMA destination 128-byte aligned (a bare [2][18][w] array would put
  // the second tile at a 64-byte offset)
  struct __align__(128) Tile {
    T v[kResPairBand + 2][res_tma_box_w<T>()];
  };
  __shared__ Tile tiles[2];
  __shared__ __align__(128) uint8_t mtile[kResPairBand][kResTmaThreads];
  __shared__ uint64_t bar;
  const int c = blockIdx.z;
  const int x0 = blockIdx.x * kResTmaThreads;
  const int x = x0 + threadIdx.x;
  const int y0 = row0 + static_cast<int>(blockIdx.y) * kResPairBand;
  const int ny = min(kResPairBand, row1 - y0);
  const bool xin = x < W;
  const size_t Wz = static_cast<size_t>(W);
  pdl_wait();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, 2 * sizeof(tiles[0].v) + (MTMA ? sizeof(mtile) : 0));
    tma_load_3d(&tiles[0].v[0][0], &umap, x0 - res_tma_lead<T>(), y0 - 1 - srow_lo, c, &bar);
    tma_load_3d(&tiles[1].v[0][0], &bmap, x0 - res_tma_lead<T>(), y0 - 1 - srow_lo, c, &bar);
    if (MTMA) tma_load_2d(&mtile[0][0], &mmap, x0, y0 - srow_lo, &bar);
  }
  uint8_t mk[kResPairBand];
  if (!MTMA) {
    const size_t base = xin ? static_cast<size_t>(y0) * Wz + x : static_cast<size_t>(y0) * Wz;
#pragma unroll
    for (int k = 0; k < kResPairBand; ++k) {
      const bool in = xin && k < ny;
      const uint8_t m = __ldg(mask + (in ? base + static_cast<size_t>(k) * Wz
                                          : static_cast<size_t>(y0) * Wz));
      mk[k] = in ? m : uint8_t(0);
    }
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  if (MTMA) {
#pragma unroll
    for (int k = 0; k < kResPairBand; ++k)
      mk[k] = (xin && k < ny) ? mtile[k][threadIdx.x] : uint8_t(0);
  }
  const int t = threadIdx.x + res_tma_lead<T>();
  const int deg_x = (x > 0) + (x + 1 < W);
  const T deg_in = T(deg_x + 2);
  double acc[2] = {0.0, 0.0};
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    const auto& tile = tiles[v].v;
    T up = tile[0][t], ctr = tile[1][t];
#pragma unroll
    for (int k = 0; k < kResPairBand; ++k) {
      const int y = y0 + k;
      const T dn = tile[k + 2][t];
      const T sum = ((tile[k + 1][t - 1] + tile[k + 1][t + 1]) + up) + dn;
      const T deg = (y > 0 && y + 1 < H) ? deg_in : T(deg_x + (y > 0) + (y + 1 < H));
      const T au = fma(deg, ctr, -sum);
      const T r = mk[k] ? T(0) : au;
      const double rd = (xin && k < ny) ? static_cast<double>(r) : 0.0;
      acc[v] = fma(rd, rd, acc[v]);
      up = ctr;
      ctr = dn;
    }
  }
  __shared__ double wsum[2][kResTmaThreads / 32];
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    const double a = warp_sum(acc[v]);
    if ((threadIdx.x & 31) == 0) wsum[v][threadIdx.x >> 5] = a;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kResTmaThreads / 32; ++w) s += wsum[threadIdx.x][w];
    const size_t nblk = static_cast<size_t>(gridDim.x) * gridDim.y;
    partials[(threadIdx.x * gridDim.z + blockIdx.z) * nblk + blockIdx.y * gridDim.x +
             blockIdx.x] = s;
  }
  pdl_trigger();
}

// K1p with b derived from u: after prolongation + snap the level's start
// iterate equals b at known pixels and b is 0 elsewhere (the multilevel
// invariant), so b = (mask ? u : 0) pixel for pixel and the pair needs one
// TMA tile (u) plus the mask with a one-pixel halo (a 2-D box of
// (128 + 32) x (band + 2) bytes starting 16 columns left: TMA wants 16-byte
// aligned starts) instead of the u and b tiles: half the DRAM reads.  The
// per-pixel terms are residual_pair_tma_kernel's bit for bit.
template <typename T>
__global__ void __launch_bounds__(kResTmaThreads)
    residual_pair_derived_kernel(const __grid_constant__ CUtensorMap umap,
                                 const __grid_constant__ CUtensorMap mmap, int W, int H,
                                 int row0, int row1, int srow_lo, double* partials) {
  __shared__ __align__(128) T tile[kResPairBand + 2][res_tma_box_w<T>()];
  __shared__ __align__(128) uint8_t mt[kResPairBand + 2][kResTmaThreads + 32];
  __shared__ uint64_t bar;
  const int c = blockIdx.z;
  const int x0 = blockIdx.x * kResTmaThreads;
  const int x = x0 + threadIdx.x;
  const int y0 = row0 + static_cast<int>(blockIdx.y) * kResPairBand;
  const int ny = min(kResPairBand, row1 - y0);
  const bool xin = x < W;
  pdl_wait();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, sizeof(tile) + sizeof(mt));
    tma_load_3d(&tile[0][0], &umap, x0 - res_tma_lead<T>(), y0 - 1 - srow_lo, c, &bar);
    tma_load_2d(&mt[0][0], &mmap, x0 - 16, y0 - 1 - srow_lo, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int t = threadIdx.x + res_tma_lead<T>();  // tile column of x
  const int m = threadIdx.x + 16;                  // mask column of x
  const int deg_x = (x > 0) + (x + 1 < W);
  const T deg_in = T(deg_x + 2);
  double acc_u = 0.0, acc_b = 0.0;
  T up = tile[0][t], ctr = tile[1][t];
  bool mup = mt[0][m] != 0, mctr = mt[1][m] != 0;
#pragma unroll
  for (int k = 0; k < kResPairBand; ++k) {
    const int y = y0 + k;
    const T dn = tile[k + 2][t];
    const bool mdn = mt[k + 2][m] != 0;
    const T w = tile[k + 1][t - 1], e = tile[k + 1][t + 1];
    const T deg = (y > 0 && y + 1 < H) ? deg_in : T(deg_x + (y > 0) + (y + 1 < H));
    const bool in = xin && k < ny;
    // u0
    const T sum = ((w + e) + up) + dn;
    const T au = fma(deg, ctr, -sum);
    const double ru = (in && !mctr) ? static_cast<double>(au) : 0.0;
    acc_u = fma(ru, ru, acc_u);
    // b = (mask ? u : 0)
    const T bw = mt[k + 1][m - 1] ? w : T(0), be = mt[k + 1][m + 1] ? e : T(0);
    const T bn = mup ? up : T(0), bs = mdn ? dn : T(0);
    const T sumb = ((bw + be) + bn) + bs;
    const T ab = fma(deg, mctr ? ctr : T(0), -sumb);
    const double rb = (in && !mctr) ? static_cast<double>(ab) : 0.0;
    acc_b = fma(rb, rb, acc_b);
    up = ctr;
    ctr = dn;
    mup = mctr;
    mctr = mdn;
  }
  __shared__ double wsum[2][kResTmaThreads / 32];
  acc_u = warp_sum(acc_u);
  acc_b = warp_sum(acc_b);
  if ((threadIdx.x & 31) == 0) {
    wsum[0][threadIdx.x >> 5] = acc_u;
    wsum[1][threadIdx.x >> 5] = acc_b;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kResTmaThreads / 32; ++w) s += wsum[threadIdx.x][w];
    const size_t nblk = static_cast<size_t>(gridDim.x) * gridDim.y;
    partials[(threadIdx.x * gridDim.z + blockIdx.z) * nblk + blockIdx.y * gridDim.x +
             blockIdx.x] = s;
  }
  pdl_trigger();
}

// Fixed-order sum of nblk partials per channel (grid: one CTA per channel).
__global__ void __launch_bounds__(kRedThreads)
    finish_partials_kernel(const double* __restrict__ partials, int nblk, double* out) {
  __shared__ double wsum[kRedThreads / 32];
  const int c = blockIdx.x;
  pdl_wait();
  double s = 0.0;
  for (int i = threadIdx.x; i < nblk; i += kRedThreads) s += partials[static_cast<size_t>(c) * nblk + i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) t += wsum[w];
    out[c] = t;
  }
}

template <typename T>
struct Pair {
  T a, b;
};

// Two horizontally adjacent values of a row (vector load when aligned).
template <typename T, bool VEC>
__device__ __forceinline__ Pair<T> load_pair(const T* __restrict__ row, int x, int W) {
  if (VEC) {
    if (x + 1 < W) {
      if constexpr (sizeof(T) == 8) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(row + x));
        return {v.x, v.y};
      } else {
        const float2 v = __ldg(reinterpret_cast<const float2*>(row + x));
        return {v.x, v.y};
      }
    }
  }
  Pair<T> r{T(0), T(0)};
  if (x < W) r.a = row[x];
  if (x + 1 < W) r.b = row[x + 1];
  return r;
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
  reduce_epilogue(acc, partials, out, ticket, blockIdx.x, gridDim.x, blockIdx.y, gridDim.y);
}

// K5: level-0 values = f at known pixels, 0 elsewhere (build_pyramid,
// multilevel.hpp:84-88); also counts known pixels for build_rhs's check.
// f is read only where a pixel pair has a known pixel (at sparse masks most
// 32-byte sectors of f are never fetched).  Each thread takes kIngestPairs
// pixel pairs, one CTA-width apart (coalesced), and issues every mask load,
// then a channel's f loads for all of them, before storing: the dependent
// mask -> f chain of a pair overlaps the other pairs' (the one-pair-per-
// iteration loop ran at 3.9 TB/s, latency-bound).
constexpr int kIngestPairs = 4;
template <typename T>
__global__ void __launch_bounds__(256)
    ingest_kernel(const double* __restrict__ f, const uint8_t* __restrict__ mask, size_t N,
                  int C, T* __restrict__ b, unsigned long long* known) {
  unsigned int cnt = 0;
  if (N % 2 == 0) {
    const size_t pairs = N / 2;
    const size_t j0 = static_cast<size_t>(blockIdx.x) * blockDim.x * kIngestPairs + threadIdx.x;
    uchar2 m[kIngestPairs];
#pragma unroll
    for (int k = 0; k < kIngestPairs; ++k) {
      const size_t j = j0 + static_cast<size_t>(k) * blockDim.x;
      m[k] = j < pairs ? reinterpret_cast<const uchar2*>(mask)[j] : make_uchar2(0, 0);
      cnt += (m[k].x != 0) + (m[k].y != 0);
    }
    for (int c = 0; c < C; ++c) {
      double2 v[kIngestPairs];
#pragma unroll
      for (int k = 0; k < kIngestPairs; ++k) {
        const size_t j = j0 + static_cast<size_t>(k) * blockDim.x;
        v[k] = make_double2(0.0, 0.0);
        if (j < pairs && (m[k].x || m[k].y))
          v[k] = __ldg(reinterpret_cast<const double2*>(f + c * N) + j);
      }
#pragma unroll
      for (int k = 0; k < kIngestPairs; ++k) {
        const size_t j = j0 + static_cast<size_t>(k) * blockDim.x;
        if (j < pairs) {
          T* dst = b + c * N + 2 * j;
          dst[0] = m[k].x ? static_cast<T>(v[k].x) : T(0);
          dst[1] = m[k].y ? static_cast<T>(v[k].y) : T(0);
        }
      }
    }
  } else {
    const size_t i0 = static_cast<size_t>(blockIdx.x) * blockDim.x * kIngestPairs + threadIdx.x;
#pragma unroll
    for (int k = 0; k < kIngestPairs; ++k) {
      const size_t i = i0 + static_cast<size_t>(k) * blockDim.x;
      if (i >= N) break;
      const bool kn = mask[i] != 0;
      cnt += kn;
      for (int c = 0; c < C; ++c) b[c * N + i] = kn ? static_cast<T>(f[c * N + i]) : T(0);
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(known, static_cast<unsigned long long>(cnt));
}

// Grid of ingest_kernel for N pixels.
inline unsigned ingest_grid(size_t N) {
  const size_t units = N % 2 == 0 ? N / 2 : N;
  return static_cast<unsigned>((units + 256 * kIngestPairs - 1) / (256 * kIngestPairs));
}

// K5 + K3 in one pass (the whole-image device path): level-0 values
// b0 = f at known pixels, 0 elsewhere (multilevel.hpp:84-88), AND the first
// restriction (multilevel.hpp:33-70) from the values just made -- b0 is
// written once and never read back.  One thread per coarse pixel (a 2x2
// fine cell, clipped at odd edges); the accumulation order is
// restrict_kernel's (row-major over the cell, KnownOnly or AllPixels).
#ifndef SI_IR_CELLS
#define SI_IR_CELLS 2  // measured: 1 -> 0.092, 2 -> 0.077, 4 -> 0.106 ms per 4K frame
#endif
constexpr int kIrCells = SI_IR_CELLS;  // coarse cells per thread (kIrCells x 128 per CTA row)
template <typename T, bool VEC>
__global__ void __launch_bounds__(128)
    ingest_restrict_kernel(const double* __restrict__ f, const uint8_t* __restrict__ fmask,
                           int fw, int fh, int C, int averaging, T* __restrict__ b0,
                           uint8_t* __restrict__ cmask, T* __restrict__ cval,
                           unsigned long long* known_count, int cy0 = 0, size_t fn_s = 0,
                           size_t cn_s = 0, int klo = 0, int khi = 0x7fffffff) {
  // stripes: coarse rows cy0 + blockIdx.y; f / fmask / b0 / cmask / cval are
  // pre-offset storage pointers (index with global rows) whose planes are
  // fn_s / cn_s apart, and only fine rows [klo, khi) are counted as known
  // pixels (the rank's own rows); whole image: 0, 0, 0, all rows.  b0 null:
  // the level-0 values are not written.
  const int cw = (fw + 1) / 2;
  const int cy = cy0 + static_cast<int>(blockIdx.y);
  const size_t fn = fn_s ? fn_s : static_cast<size_t>(fw) * fh;
  const size_t cn = cn_s ? cn_s : static_cast<size_t>(cw) * ((fh + 1) / 2);
  const int fy0 = 2 * cy;
  const bool two_y = fy0 + 1 < fh;
  const bool all = averaging != 0;
  unsigned cnt = 0;
  // every cell's mask bits first (kIrCells cells, 128 apart: coalesced), then
  // a channel's f loads for all of them, then the stores
  unsigned kb[kIrCells];
#pragma unroll
  for (int q = 0; q < kIrCells; ++q) {
    const int cx = (blockIdx.x * kIrCells + q) * blockDim.x + threadIdx.x;
    kb[q] = 0;
    if (cx >= cw) continue;
    const int fx0 = 2 * cx;
    const bool two_x = fx0 + 1 < fw;
    const size_t r0 = static_cast<size_t>(fy0) * fw + fx0, r1 = r0 + fw;
    if (VEC) {  // fw even: both columns exist
      const uchar2 m0 = *reinterpret_cast<const uchar2*>(fmask + r0);
      kb[q] |= (m0.x != 0) | (m0.y != 0) << 1;
      if (two_y) {
        const uchar2 m1 = *reinterpret_cast<const uchar2*>(fmask + r1);
        kb[q] |= (m1.x != 0) << 2 | (m1.y != 0) << 3;
      }
    } else {
      kb[q] |= (fmask[r0] != 0) | (two_x && fmask[r0 + 1] != 0) << 1;
      if (two_y) kb[q] |= (fmask[r1] != 0) << 2 | (two_x && fmask[r1 + 1] != 0) << 3;
    }
    const int known = __popc(kb[q]);
    const unsigned rows = (fy0 >= klo && fy0 < khi ? 3u : 0u) |
                          (fy0 + 1 >= klo && fy0 + 1 < khi ? 12u : 0u);
    cnt += __popc(kb[q] & rows);
    cmask[static_cast<size_t>(cy) * cw + cx] = known ? 1 : 0;
  }
  for (int c = 0; c < C; ++c) {
    const double* fc = f + c * fn;
    T* bc = b0 + c * fn;
    Pair<T> a[kIrCells], bb[kIrCells];
#pragma unroll
    for (int q = 0; q < kIrCells; ++q) {  // f is read only where the cell has a known pixel
      const int cx = (blockIdx.x * kIrCells + q) * blockDim.x + threadIdx.x;
      a[q] = {T(0), T(0)};
      bb[q] = {T(0), T(0)};
      if (cx >= cw || !kb[q]) continue;
      const int fx0 = 2 * cx;
      const bool two_x = fx0 + 1 < fw;
      const size_t r0 = static_cast<size_t>(fy0) * fw + fx0, r1 = r0 + fw;
      if (VEC) {
        const double2 v0 = __ldg(reinterpret_cast<const double2*>(fc + r0));
        a[q] = {(kb[q] & 1) ? static_cast<T>(v0.x) : T(0), (kb[q] & 2) ? static_cast<T>(v0.y) : T(0)};
        if (two_y) {
          const double2 v1 = __ldg(reinterpret_cast<const double2*>(fc + r1));
          bb[q] = {(kb[q] & 4) ? static_cast<T>(v1.x) : T(0),
                   (kb[q] & 8) ? static_cast<T>(v1.y) : T(0)};
        }
      } else {
        a[q].a = (kb[q] & 1) ? static_cast<T>(fc[r0]) : T(0);
        if (two_x) a[q].b = (kb[q] & 2) ? static_cast<T>(fc[r0 + 1]) : T(0);
        if (two_y) {
          bb[q].a = (kb[q] & 4) ? static_cast<T>(fc[r1]) : T(0);
          if (two_x) bb[q].b = (kb[q] & 8) ? static_cast<T>(fc[r1 + 1]) : T(0);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kIrCells; ++q) {
      const int cx = (blockIdx.x * kIrCells + q) * blockDim.x + threadIdx.x;
      if (cx >= cw) continue;
      const int fx0 = 2 * cx;
      const bool two_x = fx0 + 1 < fw;
      const size_t r0 = static_cast<size_t>(fy0) * fw + fx0, r1 = r0 + fw;
      if (b0 == nullptr) {
        // level-0 values not kept (their only reader, the snap, takes f)
      } else if (VEC) {
        if constexpr (sizeof(T) == 8) {
          *reinterpret_cast<double2*>(bc + r0) = make_double2(a[q].a, a[q].b);
          if (two_y) *reinterpret_cast<double2*>(bc + r1) = make_double2(bb[q].a, bb[q].b);
        } else {
          *reinterpret_cast<float2*>(bc + r0) = make_float2(a[q].a, a[q].b);
          if (two_y) *reinterpret_cast<float2*>(bc + r1) = make_float2(bb[q].a, bb[q].b);
        }
      } else {
        bc[r0] = a[q].a;
        if (two_x) bc[r0 + 1] = a[q].b;
        if (two_y) {
          bc[r1] = bb[q].a;
          if (two_x) bc[r1 + 1] = bb[q].b;
        }
      }
      // restrict_kernel's accumulation order (row-major over the cell)
      const int known = __popc(kb[q]);
      const int total = (1 + two_x) * (1 + two_y);
      T acc = T(0);
      if (known) {
        if (all || (kb[q] & 1)) acc += a[q].a;
        if (two_x && (all || (kb[q] & 2))) acc += a[q].b;
        if (two_y && (all || (kb[q] & 4))) acc += bb[q].a;
        if (two_x && two_y && (all || (kb[q] & 8))) acc += bb[q].b;
        acc = acc / T(all ? total : known);
      }
      cval[c * cn + static_cast<size_t>(cy) * cw + cx] = acc;
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(known_count, static_cast<unsigned long long>(cnt));
  pdl_trigger();
}

// K5s: the same level-0 values from the known samples alone (the batch
// upload, host_copy.h): vals[c*K + rank] is the rank-th known pixel's value,
// tile_off[t] the known count before tile t (kKnownTile = 4096 pixels).
// One CTA per tile, warp w walks pixels w*512 .. w*512+511 of it in 16
// coalesced steps: the ballots of pass 1 give the warp totals, pass 2 the
// ranks (popc of the lower lanes' bits).
constexpr int kScatterTile = 4096, kScatterWarps = 8, kScatterSteps = kScatterTile / (32 * kScatterWarps);
template <typename T>
__global__ void __launch_bounds__(kScatterWarps * 32) known_scatter_kernel(
    const uint8_t* __restrict__ mask, size_t N, int C, const double* __restrict__ vals, size_t K,
    const uint32_t* __restrict__ tile_off, T* __restrict__ b, unsigned long long* known) {
  __shared__ uint32_t warp_cnt[kScatterWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t base = static_cast<size_t>(blockIdx.x) * kScatterTile + warp * (32 * kScatterSteps);
  uint32_t ballot[kScatterSteps];
  uint32_t cnt = 0;
#pragma unroll
  for (int s = 0; s < kScatterSteps; ++s) {
    const size_t p = base + s * 32 + lane;
    const bool k = p < N && mask[p] != 0;
    ballot[s] = __ballot_sync(0xffffffffu, k);
    cnt += __popc(ballot[s]);
  }
  if (lane == 0) warp_cnt[warp] = cnt;
  __syncthreads();
  size_t o = tile_off[blockIdx.x];
  for (int w = 0; w < warp; ++w) o += warp_cnt[w];
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < kScatterWarps; ++w) tot += warp_cnt[w];
    if (tot) atomicAdd(known, static_cast<unsigned long long>(tot));
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int s = 0; s < kScatterSteps; ++s) {
    const size_t p = base + s * 32 + lane;
    const bool k = (ballot[s] >> lane) & 1u;
    const size_t r = o + __popc(ballot[s] & lt);
    if (p < N)
      for (int c = 0; c < C; ++c)
        b[c * N + p] = k ? static_cast<T>(vals[c * K + r]) : T(0);
    o += __popc(ballot[s]);
  }
}

// K3: restrict_level (multilevel.hpp:33-70): coarse pixel = clipped 2x2 fine
// cell; known = OR; value = mean of known fine values (KnownOnly) or of all
// of them (AllPixels), accumulated in row-major order like the reference.
// One thread per coarse pixel; the two fine rows are read as pairs.
// Stripe mode: coarse rows cy0 + blockIdx.y only; fn / cn are the storage
// planes of the (pre-offset) fine and coarse buffers.
template <typename T, bool VEC>
__global__ void restrict_kernel(const uint8_t* __restrict__ fmask, const T* __restrict__ fval,
                                int fw, int fh, int C, int averaging, uint8_t* __restrict__ cmask,
                                T* __restrict__ cval, int cy0, size_t fn, size_t cn) {
  pdl_wait();
  const int cw = (fw + 1) / 2;
  const int cx = blockIdx.x * blockDim.x + threadIdx.x, cy = cy0 + static_cast<int>(blockIdx.y);
  if (cx >= cw) return;
  const int fx0 = 2 * cx, fy0 = 2 * cy;
  const bool two_x = fx0 + 1 < fw, two_y = fy0 + 1 < fh;
  const size_t r0 = static_cast<size_t>(fy0) * fw + fx0, r1 = r0 + fw;
  const bool k00 = fmask[r0] != 0, k01 = two_x && fmask[r0 + 1] != 0;
  const bool k10 = two_y && fmask[r1] != 0, k11 = two_x && two_y && fmask[r1 + 1] != 0;
  const int known = k00 + k01 + k10 + k11;
  const int total = (1 + two_x) * (1 + two_y);
  const size_t j = static_cast<size_t>(cy) * cw + cx;
  cmask[j] = known ? 1 : 0;
  for (int c = 0; c < C; ++c) {
    T acc = T(0);
    if (known) {
      const T* v = fval + c * fn;
      const Pair<T> a = load_pair<T, VEC>(v + static_cast<size_t>(fy0) * fw, fx0, fw);
      Pair<T> bb{T(0), T(0)};
      if (two_y) bb = load_pair<T, VEC>(v + static_cast<size_t>(fy0 + 1) * fw, fx0, fw);
      const bool all = averaging != 0;
      if (all || k00) acc += a.a;
      if (two_x && (all || k01)) acc += a.b;
      if (two_y && (all || k10)) acc += bb.a;
      if (two_x && two_y && (all || k11)) acc += bb.b;
      acc = acc / T(all ? total : known);
    }
    cval[c * cn + j] = acc;
  }
}

// K4: prolongate (multilevel.hpp:101-128) + snap known fine pixels to their
// data (multilevel.hpp:294-303): cell-centred bilinear, coordinate
// 0.5*f - 0.25 clamped to the coarse grid.
// Fine tile 64 x 16 per CTA (256 threads, a 2x2 quad each); the coarse
// window it samples (34 x 10 per channel) is staged in shared memory.
constexpr int kProX = 64, kProY = 16, kProCX = kProX / 2 + 2, kProCY = kProY / 2 + 2;

template <typename T>
__device__ __forceinline__ void prolong_axis(int f, int cn, double& t, int& i0, int& i1) {
  const double c = fmin(fmax(0.5 * f - 0.25, 0.0), static_cast<double>(cn - 1));
  i0 = static_cast<int>(c);
  i1 = min(i0 + 1, cn - 1);
  t = c - i0;
}

template <typename T>
#ifndef SI_PRO_OCC
#define SI_PRO_OCC 4
#endif
__global__ void __launch_bounds__(256, SI_PRO_OCC)
    prolong_snap_kernel(const T* __restrict__ coarse, int cw, int ch, int fw, int fh, int C,
                        const uint8_t* __restrict__ fmask, const T* __restrict__ fval,
                        T* __restrict__ fine, int fy_lo, int fy_hi, int cs_lo, int cs_hi,
                        size_t fn, size_t cn) {
  // Fine rows [fy_lo, fy_hi) only; the coarse buffer holds rows
  // [cs_lo, cs_hi) (stripe storage; pointers pre-offset, fn / cn the storage
  // planes).  Whole image: 0, fh, 0, ch, fw*fh, cw*ch.
  constexpr int kCh = 3;  // channels staged per pass
  __shared__ T tile[kCh][kProCY][kProCX];
  pdl_wait();
  const int fx0 = blockIdx.x * kProX, fy0 = fy_lo + static_cast<int>(blockIdx.y) * kProY;
  fh = fy_hi;  // rows at or beyond fy_hi are neither read nor written
  const int cx0 = fx0 / 2 - 1, cy0 = fy0 / 2 - 1;  // staged window origin
  const int qx = threadIdx.x & 31, qy = threadIdx.x >> 5;
  const int fxq = fx0 + 2 * qx, fyq = fy0 + 2 * qy;
  // snap bits of my quad, loaded before the staging barrier
  unsigned snap = 0;
  if (fmask != nullptr) {
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx)
        if (fyq + dy < fh && fxq + dx < fw && fmask[static_cast<size_t>(fyq + dy) * fw + fxq + dx])
          snap |= 1u << (2 * dy + dx);
  }
  for (int c0 = 0; c0 < C; c0 += kCh) {
    const int nc = min(kCh, C - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < nc * kProCY * kProCX; i += blockDim.x) {
      const int k = i / (kProCY * kProCX), rem = i - k * (kProCY * kProCX);
      const int ly = rem / kProCX, lx = rem - ly * kProCX;
      const int gy = min(max(cy0 + ly, cs_lo), cs_hi - 1), gx = min(max(cx0 + lx, 0), cw - 1);
      tile[k][ly][lx] = __ldg(coarse + (c0 + k) * cn + static_cast<size_t>(gy) * cw + gx);
    }
    // the known pixels' data of my quad, in flight across the barrier
    T sv[kCh][4];
#pragma unroll
    for (int k = 0; k < kCh; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool on = k < nc && ((snap >> q) & 1u);
        const size_t i = on ? static_cast<size_t>(fyq + (q >> 1)) * fw + fxq + (q & 1)
                            : static_cast<size_t>(fy_lo) * fw;  // a stored row
        sv[k][q] = on ? __ldg(fval + (c0 + k) * fn + i) : T(0);
      }
    __syncthreads();
    // the quad's two columns share the x interpolation across channels;
    // each row of the quad leaves as one 16-byte (fp64) / 8-byte (fp32) store
    double txd[2];
    int xb0[2], xb1[2];
#pragma unroll
    for (int dx = 0; dx < 2; ++dx) {
      int xa, xb;
      prolong_axis<T>(min(fxq + dx, fw - 1), cw, txd[dx], xa, xb);
      xb0[dx] = xa - cx0;
      xb1[dx] = xb - cx0;
    }
    const bool pair_store = (fw % 2 == 0) && fxq + 1 < fw;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const int fy = fyq + dy;
      if (fy >= fh || fxq >= fw) continue;
      double tyd;
      int ya, yb;
      prolong_axis<T>(fy, ch, tyd, ya, yb);
      const T ty = static_cast<T>(tyd);
      const int a0 = ya - cy0, a1 = yb - cy0;
      const size_t i = static_cast<size_t>(fy) * fw + fxq;
#pragma unroll
      for (int k = 0; k < kCh; ++k) {
        if (k >= nc) break;
        T v[2];
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const T tx = static_cast<T>(txd[dx]);
          const int b0 = xb0[dx], b1 = xb1[dx];
          const T v00 = tile[k][a0][b0], v01 = tile[k][a0][b1];
          const T v10 = tile[k][a1][b0], v11 = tile[k][a1][b1];
          // (1-ty)*((1-tx)*v00 + tx*v01) + ty*((1-tx)*v10 + tx*v11), with the
          // contraction gcc -O3 applies to the reference expression
          // (p*q + r*s -> fma(p, q, r*s); checked bitwise in the tests).
          const T p0 = fma(T(1) - tx, v00, tx * v01);
          const T p1 = fma(T(1) - tx, v10, tx * v11);
          v[dx] = fma(T(1) - ty, p0, ty * p1);
          if ((snap >> (2 * dy + dx)) & 1u) v[dx] = sv[k][2 * dy + dx];
        }
        T* dst = fine + (c0 + k) * fn + i;
        if (pair_store) {
          if constexpr (sizeof(T) == 8)
            *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[1]);
          else
            *reinterpret_cast<float2*>(dst) = make_float2(v[0], v[1]);
        } else {
          dst[0] = v[0];
          if (fxq + 1 < fw) dst[1] = v[1];
        }
      }
    }
  }
}

// K4 with the coarse windows fetched by TMA into a two-stage ring: a
// persistent CTA walks fine tiles of kProX x kProY; thread 0 issues the next
// tile's window (one box of kProBoxW x kProCY per channel; columns or rows
// outside the coarse level arrive as zeros and are never read: the sample
// coordinates are clamped to the level, multilevel.hpp:109-115) while the
// CTA computes the current one from shared memory.  The one-shot kernel
// above loaded its window with per-thread loads, then waited at a barrier
// (long-scoreboard bound, 3.0 TB/s on the finest 4K level).
// The box must start at a 16-byte aligned column (a misaligned start raises
// an illegal-instruction fault on B200, cf. tile_lead in sweep.cuh): it
// starts pro_lead columns left of the tile's first coarse column and is
// wide enough for its kProCX - 1 columns right of it.
template <typename T>
__host__ __device__ constexpr int pro_lead() {
  return 16 / static_cast<int>(sizeof(T));
}
template <typename T>
__host__ __device__ constexpr int pro_box_w() {
  return sizeof(T) == 8 ? kProCX + 2 : kProCX + 6;  // 36 x 8 B / 40 x 4 B rows
}
constexpr int kProMaxC = 4;  // channels per tile window (more: the one-shot kernel)
template <typename T>
struct __align__(128) ProSlice {  // one channel's window, a 128-byte multiple
  T v[kProCY][pro_box_w<T>()];
  char pad[(128 - (sizeof(T) * kProCY * pro_box_w<T>()) % 128) % 128];
};

// MT: the tile's fine mask bytes ride on the same barrier (a 2-D box of
// kProX x kProY; needs a 16-byte multiple mask row pitch), else byte loads.
#ifndef SI_PRO_TMA_OCC
#define SI_PRO_TMA_OCC 3
#endif
constexpr int kProTmaOcc = SI_PRO_TMA_OCC;  // resident CTAs per SM (persistent grid)
template <typename T, bool MT>
__global__ void __launch_bounds__(256, SI_PRO_TMA_OCC)
    prolong_snap_tma_kernel(const __grid_constant__ CUtensorMap cmap,
                            const __grid_constant__ CUtensorMap mmap, int cw, int ch, int fw,
                            int C, const uint8_t* __restrict__ fmask, const T* __restrict__ fval,
                            T* __restrict__ fine, int fy_lo, int fy_hi, int cs_lo, int fs_lo,
                            size_t fn, int tiles_x, int ntiles) {
  __shared__ ProSlice<T> ring[2][kProMaxC];
  __shared__ __align__(128) uint8_t mring[2][kProY][kProX];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  const int qx = tid & 31, qy = tid >> 5;
  const uint32_t box_bytes = static_cast<uint32_t>(sizeof(T) * kProCY * pro_box_w<T>()) * C +
                             (MT ? static_cast<uint32_t>(kProX * kProY) : 0u);
  pdl_wait();
  // (no lambda here: the tensor map must be addressed in parameter space;
  // a by-reference capture can make the compiler spill it to the stack)
#define SI_PRO_ISSUE(t_, stage_)                                                              \
  do {                                                                                        \
    const int ifx0 = ((t_) % tiles_x) * kProX, ify0 = fy_lo + ((t_) / tiles_x) * kProY;         \
    mbar_expect_tx(&bar[(stage_)], box_bytes);                                                \
    for (int kc = 0; kc < C; ++kc)                                                            \
      tma_load_3d(&ring[(stage_)][kc].v[0][0], &cmap, ifx0 / 2 - pro_lead<T>(),                \
                  ify0 / 2 - 1 - cs_lo, kc, &bar[(stage_)]);                                  \
    if (MT) tma_load_2d(&mring[(stage_)][0][0], &mmap, ifx0, ify0 - fs_lo, &bar[(stage_)]);    \
  } while (0)
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    if (static_cast<int>(blockIdx.x) < ntiles) SI_PRO_ISSUE(static_cast<int>(blockIdx.x), 0);
  }
  __syncthreads();
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int stage = k & 1;
    if (tid == 0 && t + static_cast<int>(gridDim.x) < ntiles)
      SI_PRO_ISSUE(t + static_cast<int>(gridDim.x), stage ^ 1);
    const int fx0 = (t % tiles_x) * kProX, fy0 = fy_lo + (t / tiles_x) * kProY;
    const int cx0 = fx0 / 2 - pro_lead<T>(), cy0 = fy0 / 2 - 1;  // window origin
    const int fxq = fx0 + 2 * qx, fyq = fy0 + 2 * qy;
    unsigned snap = 0;
    if (!MT && fmask != nullptr) {
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx)
          if (fyq + dy < fy_hi && fxq + dx < fw &&
              fmask[static_cast<size_t>(fyq + dy) * fw + fxq + dx])
            snap |= 1u << (2 * dy + dx);
    }
    double txd[2];
    int xb0[2], xb1[2];
#pragma unroll
    for (int dx = 0; dx < 2; ++dx) {
      int xa, xb;
      prolong_axis<T>(min(fxq + dx, fw - 1), cw, txd[dx], xa, xb);
      xb0[dx] = xa - cx0;
      xb1[dx] = xb - cx0;
    }
    const bool pair_store = (fw % 2 == 0) && fxq + 1 < fw;
    mbar_wait(&bar[stage], (k >> 1) & 1);
    if (MT) {  // rows / columns past the level arrive as zeros: no snap there
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx)
          if (fyq + dy < fy_hi && mring[stage][2 * qy + dy][2 * qx + dx])
            snap |= 1u << (2 * dy + dx);
    }
    // every snap value of the quad in flight before the interpolation (the
    // load-and-use inside it was the kernel's long-scoreboard stall:
    // 0.124 -> 0.108 ms per 4K frame with 3 CTAs/SM for the registers)
    T sv[kProMaxC][4];
#pragma unroll
    for (int c = 0; c < kProMaxC; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool on = c < C && ((snap >> q) & 1u);
        sv[c][q] = on ? __ldg(fval + c * fn + static_cast<size_t>(fyq + (q >> 1)) * fw + fxq +
                              (q & 1))
                      : T(0);
      }
    for (int c = 0; c < C; ++c) {
      const auto& tile = ring[stage][c].v;
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        const int fy = fyq + dy;
        if (fy >= fy_hi || fxq >= fw) continue;
        double tyd;
        int ya, yb;
        prolong_axis<T>(fy, ch, tyd, ya, yb);
        const T ty = static_cast<T>(tyd);
        const int a0 = ya - cy0, a1 = yb - cy0;
        const size_t i = static_cast<size_t>(fy) * fw + fxq;
        T v[2];
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const T tx = static_cast<T>(txd[dx]);
          const int b0 = xb0[dx], b1 = xb1[dx];
          const T v00 = tile[a0][b0], v01 = tile[a0][b1];
          const T v10 = tile[a1][b0], v11 = tile[a1][b1];
          // gcc -O3's contraction of the reference expression (see above)
          const T p0 = fma(T(1) - tx, v00, tx * v01);
          const T p1 = fma(T(1) - tx, v10, tx * v11);
          v[dx] = fma(T(1) - ty, p0, ty * p1);
          if ((snap >> (2 * dy + dx)) & 1u) {
            T sel = sv[0][2 * dy + dx];
#pragma unroll
            for (int cc = 1; cc < kProMaxC; ++cc)
              if (c == cc) sel = sv[cc][2 * dy + dx];
            v[dx] = sel;
          }
        }
        T* dst = fine + c * fn + i;
        if (pair_store) {
          if constexpr (sizeof(T) == 8)
            *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[1]);
          else
            *reinterpret_cast<float2*>(dst) = make_float2(v[0], v[1]);
        } else {
          dst[0] = v[0];
          if (fxq + 1 < fw) dst[1] = v[1];
        }
      }
    }
    __syncthreads();  // every thread is done with this stage before it is refilled
  }
#undef SI_PRO_ISSUE
}

// read_pnm / read_mask_pbm payloads (pnm.hpp:98-188): interleaved bytes ->
// planar f = byte / 255.0; P4 bits (MSB first, rows padded to bytes) -> mask.
__global__ void unpack_pnm_kernel(const uint8_t* __restrict__ pix, const uint8_t* __restrict__ pbm,
                                  int W, int H, int C, double* __restrict__ f,
                                  uint8_t* __restrict__ mask) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  const size_t N = static_cast<size_t>(W) * H, row_bytes = (static_cast<size_t>(W) + 7) / 8;
  for (int y = blockIdx.y; y < H; y += gridDim.y) {
    const size_t i = static_cast<size_t>(y) * W + x;
    for (int c = 0; c < C; ++c) f[c * N + i] = pix[i * C + c] / 255.0;
    mask[i] = (pbm[y * row_bytes + x / 8] >> (7 - x % 8)) & 1;
  }
}

// quantise (pnm.hpp:82-85): clamp to [0, 1], lround(255 v); planar -> interleaved.
__global__ void quantise_kernel(const double* __restrict__ u, size_t N, int C,
                                uint8_t* __restrict__ out) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += stride)
    for (int c = 0; c < C; ++c) {
      const double v = u[c * N + i];
      const double cl = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
      out[i * C + c] = static_cast<uint8_t>(llround(cl * 255.0));
    }
}

template <typename Tin, typename Tout>
__global__ void convert_kernel(const Tin* __restrict__ in, Tout* __restrict__ out, size_t n) {
  pdl_wait();
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<Tout>(in[i]);
}

}  // namespace sib

namespace sib {

// ---- device-driven outer iteration (CUDA graph with conditional nodes) ----
// run_schwarz_level's host loop (schwarz.hpp:266-323) moved to the device:
// level_decide_kernel evaluates the stopping test of one outer iteration
// with the host's arithmetic (joint norm sqrt-then-fma, IEEE division) and
// drives the WHILE / IF nodes that contain the next sweeps.
struct LevelState {
  double r0;         // canonical r0 (schwarz.hpp:333-345)
  double final_rel;  // last relative residual
  int outer;         // sweeps done
  int iterations;    // report.iterations
  int converged;
  int pad;
};

__device__ __forceinline__ double joint_norm_dev(const double* s, int C) {
  double joint = 0.0;
  for (int k = 0; k < C; ++k) {
    const double nrm = sqrt(s[k]);
    joint = fma(nrm, nrm, joint);
  }
  return sqrt(joint);
}

// first: also takes r0 from r0sums and resets the level.  Sets hw (loop
// continue) and, when set_i, hi (the second sweep of the body) to "sweep
// again".
__global__ void level_decide_kernel(const double* __restrict__ sums,
                                    const double* __restrict__ r0sums, int C, double tol,
                                    int max_outer, LevelState* st, cudaGraphConditionalHandle hw,
                                    cudaGraphConditionalHandle hi, int first, int set_i) {
  if (threadIdx.x != 0) return;
  if (first) {
    st->r0 = joint_norm_dev(r0sums, C);
    st->outer = 0;
    st->converged = 0;
  }
  const double r0 = st->r0;
  const double rel = r0 > 0.0 ? joint_norm_dev(sums, C) / r0 : 0.0;
  st->iterations = st->outer;
  st->final_rel = rel;
  unsigned cont = 0;
  if (rel <= tol)
    st->converged = 1;
  else if (st->outer < max_outer) {
    cont = 1;
    st->outer += 1;
  }
  cudaGraphSetConditional(hw, cont);
  if (set_i) cudaGraphSetConditional(hi, cont);
}

// After the loop the level's iterate is in u1 when the sweep count is odd:
// move it to u0 so the next stage reads a fixed buffer.
template <typename T>
__global__ void parity_fixup_kernel(const LevelState* st, const T* __restrict__ u1,
                                    T* __restrict__ u0, size_t n) {
  if ((st->outer & 1) == 0) return;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    u0[i] = u1[i];
}

__global__ void copy_bytes_kernel(const unsigned long long* __restrict__ src,
                                  unsigned long long* __restrict__ dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

}  // namespace sib
