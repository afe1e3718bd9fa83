// Measured FP64 (DFMA) peak of this B200, the denominator for the sweep's
// informational "sweep_fp64_tflops" in bench.py's roofline object.
// 8 independent DFMA chains per thread, 148 x 8 CTAs of 256 threads, CUDA
// events, best of 10.  2 flops per DFMA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak scripts/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int iters = 1 << 16, threads = 256;
  for (int per_sm : {4, 8, 16}) {
    int blocks = sms * per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_chains<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * iters * double(blocks) * threads;
    printf("{\"ctas_per_sm\": %d, \"ms\": %.3f, \"fp64_tflops\": %.2f}\n", per_sm, best,
           flops / (best * 1e-3) / 1e12);
  }
  return cudaGetLastError() != cudaSuccess;
}
