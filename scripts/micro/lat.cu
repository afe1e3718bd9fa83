// Dependent-chain latency of the FP64 / shuffle / barrier operations the
// sweep's CG iteration is built from (clock64 around 256-long chains).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b) {
  double x = a + threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    if (OP == 0) x = fma(x, b, a);                        // DFMA
    if (OP == 1) x = x + b;                               // DADD
    if (OP == 2) x = __shfl_xor_sync(0xffffffffu, x, 1) + b;  // SHFL.64 + DADD
    if (OP == 3) x = __drcp_rn(x) + b;                    // rcp_rn
    if (OP == 4) x = a / x + b;                           // IEEE div
    if (OP == 5) { x = x + b; __syncthreads(); }          // DADD + BAR (128 thr)
    if (OP == 6) x = sqrt(x) + b;
    if (OP == 7) { __shared__ double s[256]; s[threadIdx.x] = x; __syncwarp(); x = s[threadIdx.x ^ 1] + b; __syncwarp(); }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads) {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
  chain<OP><<<1, threads>>>(o, c, 1.000001, 0.999999);
  chain<OP><<<1, threads>>>(o, c, 1.000001, 0.999999);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %6.1f cycles/op\n", name, h / 256.0);
  cudaFree(o); cudaFree(c);
}

int main() {
  run<0>("DFMA", 32);
  run<1>("DADD", 32);
  run<2>("SHFL.64 + DADD", 32);
  run<3>("__drcp_rn + DADD", 32);
  run<4>("IEEE div + DADD", 32);
  run<5>("DADD + __syncthreads(128)", 128);
  run<6>("sqrt + DADD", 32);
  run<7>("STS/LDS + syncwarp + DADD", 32);
  return 0;
}
