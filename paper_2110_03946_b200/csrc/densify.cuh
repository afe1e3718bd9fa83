// Voronoi-guided mask densification (masks.hpp:45-215) on the device.
//
// One densify sweep = guide inpainting (the multilevel ORAS path) + these
// integer/byte kernels, all HBM- or latency-bound:
//   D1 site_flags / sites_scatter : known pixels -> ascending site list
//      (exclusive scan of the mask: site index = rank of the pixel);
//   D2 bucket_count / bucket_fill : sites binned on the reference's square
//      grid of side max(1, floor(sqrt(n/m))) (masks.hpp:66-81);
//   D3 assign_sites               : exact nearest site per pixel, one thread
//      per pixel, ring search over bins with the reference's pruning rules
//      (masks.hpp:83-127).  The answer is the lexicographic minimum of
//      (squared distance, site index) over all sites, so neither the order of
//      sites inside a bin nor the visiting order changes it: bins are filled
//      with atomics;
//   D4 cell_keys                  : per unknown pixel its cell and squared
//      error e = sum_c (u - f)^2 (fma per channel, as gcc contracts
//      masks.hpp:180-183), per cell the pixel count (area);
//   D5 cell_reduce                : one thread per cell walks the cell's
//      pixels in ascending pixel order (stable radix sort by cell), so the
//      error sum rounds exactly like the reference's serial loop
//      (masks.hpp:184-189); worst pixel = first maximum;
//   D6 rank + plant               : two stable descending radix sorts (area,
//      then error bits; errors are >= 0 so their IEEE bits order like the
//      values) give the reference's order (error desc, area desc, index asc,
//      masks.hpp:195-203); the first `quota` cells' worst pixels become known.
#pragma once

#include <cstdint>

namespace sib {

__global__ void site_flags_kernel(const uint8_t* __restrict__ mask, size_t n,
                                  int32_t* __restrict__ flag) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    flag[i] = mask[i] != 0;
}

__global__ void sites_scatter_kernel(const uint8_t* __restrict__ mask,
                                     const int32_t* __restrict__ rank, size_t n,
                                     int32_t* __restrict__ sites) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    if (mask[i]) sites[rank[i]] = static_cast<int32_t>(i);
}

__device__ __forceinline__ int bin_of(int32_t p, int W, int cell, int gw) {
  const int x = p % W, y = p / W;
  return (y / cell) * gw + x / cell;
}

__global__ void bucket_count_kernel(const int32_t* __restrict__ sites, int m, int W, int cell,
                                    int gw, int32_t* __restrict__ count) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x)
    atomicAdd(&count[bin_of(sites[s], W, cell, gw)], 1);
}

__global__ void bucket_fill_kernel(const int32_t* __restrict__ sites, int m, int W, int cell,
                                   int gw, int32_t* __restrict__ cursor,
                                   int32_t* __restrict__ members) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x)
    members[atomicAdd(&cursor[bin_of(sites[s], W, cell, gw)], 1)] = s;
}

// Squared distance from (px, py) to the clipped rectangle of bin (bx, by).
__device__ __forceinline__ long long bin_distance(int px, int py, int bx, int by, int cell, int W,
                                                  int H) {
  const int x0 = bx * cell, y0 = by * cell;
  const int x1 = min(W - 1, x0 + cell - 1), y1 = min(H - 1, y0 + cell - 1);
  const long long dx = px < x0 ? x0 - px : (px > x1 ? px - x1 : 0);
  const long long dy = py < y0 ? y0 - py : (py > y1 ? py - y1 : 0);
  return dx * dx + dy * dy;
}

__global__ void __launch_bounds__(256) assign_sites_kernel(
    const int32_t* __restrict__ sites, const int32_t* __restrict__ start,
    const int32_t* __restrict__ members, int W, int H, int cell, int gw, int gh,
    int32_t* __restrict__ site_of) {
  const int px = blockIdx.x * 32 + (threadIdx.x & 31);
  const int py = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (px >= W || py >= H) return;
  const int cx = px / cell, cy = py / cell;
  long long best_d = -1;
  int best = -1;
  const int rings = max(gw, gh);
  auto scan_bin = [&](int bx, int by) {
    if (bx < 0 || bx >= gw) return;
    if (best >= 0 && bin_distance(px, py, bx, by, cell, W, H) > best_d) return;
    const int b = by * gw + bx;
    for (int k = start[b], e = start[b + 1]; k < e; ++k) {
      const int s = members[k];
      const int sp = sites[s];
      const long long ex = sp % W - px, ey = sp / W - py;
      const long long d = ex * ex + ey * ey;
      if (best < 0 || d < best_d || (d == best_d && s < best)) {
        best_d = d;
        best = s;
      }
    }
  };
  for (int ring = 0; ring <= rings; ++ring) {
    if (best >= 0 && ring >= 1) {
      const long long reach = static_cast<long long>(ring - 1) * cell + 1;
      if (reach * reach > best_d) break;
    }
    for (int by = max(0, cy - ring); by <= min(gh - 1, cy + ring); ++by) {
      if (by == cy - ring || by == cy + ring) {
        for (int bx = cx - ring; bx <= cx + ring; ++bx) scan_bin(bx, by);
      } else {
        scan_bin(cx - ring, by);
        scan_bin(cx + ring, by);
      }
    }
  }
  site_of[static_cast<size_t>(py) * W + px] = best;
}

// Unknown pixels: key = cell, e = squared error, area[cell] += 1.  Known
// pixels get the sentinel key m (sorted past every cell).
__global__ void cell_keys_kernel(const uint8_t* __restrict__ mask, const int32_t* __restrict__ site_of,
                                 const double* __restrict__ u, const double* __restrict__ f,
                                 size_t n, int C, int m, int32_t* __restrict__ key,
                                 int32_t* __restrict__ pix, double* __restrict__ err,
                                 int32_t* __restrict__ area) {
  for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<size_t>(gridDim.x) * blockDim.x) {
    pix[p] = static_cast<int32_t>(p);
    if (mask[p]) {
      key[p] = m;
      continue;
    }
    const int s = site_of[p];
    double e = 0.0;
    for (int c = 0; c < C; ++c) {
      const double d = u[c * n + p] - f[c * n + p];
      e = fma(d, d, e);
    }
    err[p] = e;
    key[p] = s;
    atomicAdd(&area[s], 1);
  }
}

// One thread per cell: serial pixel-order sum (masks.hpp:184-189).
__global__ void cell_reduce_kernel(const int32_t* __restrict__ seg, const int32_t* __restrict__ pix,
                                   const double* __restrict__ err, int m,
                                   unsigned long long* __restrict__ err_bits,
                                   int32_t* __restrict__ worst, int32_t* __restrict__ order,
                                   int* __restrict__ nonempty) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    double sum = 0.0, best_e = -1.0;
    int best_p = -1;
    const int b = seg[s], e = seg[s + 1];
    for (int k = b; k < e; ++k) {
      const int p = pix[k];
      const double v = err[p];
      sum += v;
      if (v > best_e) {
        best_e = v;
        best_p = p;
      }
    }
    err_bits[s] = static_cast<unsigned long long>(__double_as_longlong(sum));
    worst[s] = best_p;
    order[s] = s;
    if (e > b) atomicAdd(nonempty, 1);
  }
}

__global__ void gather_bits_kernel(const unsigned long long* __restrict__ bits,
                                   const int32_t* __restrict__ idx, int m,
                                   unsigned long long* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    out[i] = bits[idx[i]];
}

__global__ void plant_kernel(const int32_t* __restrict__ order, const int32_t* __restrict__ worst,
                             int quota, uint8_t* __restrict__ mask) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < quota; i += gridDim.x * blockDim.x)
    mask[worst[order[i]]] = 1;
}

}  // namespace sib
