// Latency of a 32-lane FP64 warp sum: butterfly (5 x SHFL.64 + DADD) versus
// DMMA m8n8k4 (A = lane values, B = ones -> row sums; second pair of MMAs
// folds the 8 row sums), measured as a dependent chain.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double bfly(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// A[i][k] = value of lane 4i+k.  D = A * ones -> D[i][*] = sum of lanes 4i..4i+3;
// lane l holds D[l/4][2(l%4)], D[l/4][2(l%4)+1].  Then B2[k][n] = rowsum_k
// (k<4) via lane 4k, B3[k][n] = rowsum_{k+4}; D2 = ones*B2 + ones*B3.
__device__ __forceinline__ double mma_sum(double v) {
  const int lane = threadIdx.x & 31;
  double d0, d1;
  dmma(d0, d1, v, 1.0, 0.0, 0.0);
  // B fragment for m8n8k4 .col: lane l holds B[l%4][l/4]
  const int k = lane & 3;
  const double s_lo = __shfl_sync(0xffffffffu, d0, 4 * k);
  const double s_hi = __shfl_sync(0xffffffffu, d0, 4 * (k + 4));
  double e0, e1;
  dmma(e0, e1, 1.0, s_lo, 0.0, 0.0);
  double f0, f1;
  dmma(f0, f1, 1.0, s_hi, e0, e1);
  return f0;
}

template <int OP>
__global__ void k(double* out, long long* cyc, double b) {
  double x = 1.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
    double s = OP == 0 ? bfly(x) : mma_sum(x);
    x = s * 1e-2 + b;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* o; long long* c; long long h; double hv[32];
  cudaMalloc(&o, 8 * 64); cudaMalloc(&c, 8);
  for (int op = 0; op < 2; ++op) {
    for (int r = 0; r < 2; ++r) {
      if (op == 0) k<0><<<1, 32>>>(o, c, 0.5); else k<1><<<1, 32>>>(o, c, 0.5);
    }
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hv, o, 8 * 32, cudaMemcpyDeviceToHost);
    printf("%s: %.1f cycles per (sum + DFMA), lane0 %.17g lane31 %.17g\n", op ? "dmma" : "butterfly", h / 64.0, hv[0], hv[31]);
  }
  // correctness: sum of 1..32 style
  return 0;
}
