// Shared device/host helpers for the schwarz_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sib {

constexpr int kMaxBlock = 32;   // subdomain edge handled by the sweep kernel
constexpr int kTile = kMaxBlock + 2;

// Partition of one axis, computed arithmetically so no per-block tables are
// needed on device.  partition_axis / owned_end (partition.hpp:46-63):
// anchors k*(B-o), last block flush to the edge; block k owns pixels up to
// the midpoint between its centre and the next block's centre (ties low).
struct Axis {
  int extent, block, stride, count;

  __host__ __device__ static Axis make(int extent, int block, int overlap) {
    Axis a;
    a.extent = extent;
    a.block = block;
    a.stride = block - overlap;
    a.count = extent > block ? (extent - block + a.stride - 1) / a.stride + 1 : 1;
    return a;
  }
  __host__ __device__ int anchor(int k) const {
    return k + 1 == count ? extent - block : k * stride;
  }
  __host__ __device__ int owned_end(int k) const {
    return k + 1 == count ? extent : (anchor(k) + anchor(k + 1) + block - 1) / 2 + 1;
  }
  __host__ __device__ int owned_begin(int k) const { return k == 0 ? 0 : owned_end(k - 1); }
};

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Butterfly sum: every lane ends with the same, order-fixed warp total.
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += shfl_xor(v, m);
  return v;
}

}  // namespace sib
