// Latency of three simultaneous FP64 warp sums (the fused CG reduction).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2110_03946_b200/csrc/common.cuh"
using namespace sib;

template <int OP>
__global__ void k(double* out, long long* cyc, double bb) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 2.0 - threadIdx.x * 1e-3, c = 0.5 + threadIdx.x * 1e-4;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
    if (OP == 0) { a = warp_sum(a); b = warp_sum(b); c = warp_sum(c); }
    if (OP == 1) { a = warp_sum_mma(a); b = warp_sum_mma(b); c = warp_sum_mma(c); }
    if (OP == 2) { warp_sum3_mma(a, b, c); }
    if (OP == 3) { a = warp_sum_mma(a); }
    a = a * 1e-2 + bb; b = b * 1e-2 + bb; c = c * 1e-2 + bb;
  }
  long long t1 = clock64();
  out[threadIdx.x] = a + b + c;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 8 * 64); cudaMalloc(&c, 8);
  const char* names[] = {"3x butterfly", "3x dmma", "dmma3 fused", "1x dmma"};
  for (int op = 0; op < 4; ++op) {
    for (int r = 0; r < 2; ++r) {
      if (op == 0) k<0><<<1, 32>>>(o, c, 0.5);
      if (op == 1) k<1><<<1, 32>>>(o, c, 0.5);
      if (op == 2) k<2><<<1, 32>>>(o, c, 0.5);
      if (op == 3) k<3><<<1, 32>>>(o, c, 0.5);
    }
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-14s %.1f cycles per iteration (incl. one DFMA)\n", names[op], h / 64.0);
  }
  return 0;
}
