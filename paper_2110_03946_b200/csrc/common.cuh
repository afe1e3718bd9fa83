// Shared device/host helpers for the schwarz_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sib {

constexpr int kMaxBlock = 32;   // subdomain edge handled by the sweep kernel

// Partition of one axis, computed arithmetically so no per-block tables are
// needed on device.  partition_axis / owned_end (partition.hpp:46-63):
// anchors k*(B-o), last block flush to the edge; block k owns pixels up to
// the midpoint between its centre and the next block's centre (ties low).
// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in the
// stream drains; pdl_wait() blocks until the predecessor grid has completed
// and its memory is visible (a no-op for an ordinary launch), pdl_trigger()
// lets this grid's dependents start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

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

// Warp total of one double per lane on the FP64 tensor core (DMMA m8n8k4):
// D = A * ones with A[i][k] = lane 4i+k gives the 8 row sums (lane l holds
// row l/4); two more MMAs with the row sums as B (k = 0..3, then 4..7) and
// ones as A fold them.  ~115 cycles of latency against ~170 for the 5-level
// shuffle butterfly; every lane ends with the same, order-fixed total.
// All 32 lanes must be converged.
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b, double c0,
                                            double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__device__ __forceinline__ double warp_sum_mma(double v) {
  const int k = threadIdx.x & 3;
  double r0, r1;
  dmma_m8n8k4(r0, r1, v, 1.0, 0.0, 0.0);
  const double lo = __shfl_sync(0xffffffffu, r0, 4 * k);
  const double hi = __shfl_sync(0xffffffffu, r0, 4 * (k + 4));
  double e0, e1, f0, f1;
  dmma_m8n8k4(e0, e1, 1.0, lo, 0.0, 0.0);
  dmma_m8n8k4(f0, f1, 1.0, hi, e0, e1);
  return f0;
}

}  // namespace sib
