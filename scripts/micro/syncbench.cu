// Host round-trip latency: tiny kernel + cudaStreamSynchronize vs a kernel
// that writes a sequence number to mapped pinned memory the host spins on.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(double* x) { if (threadIdx.x == 0) x[0] += 1.0; }
__global__ void signal(volatile unsigned* flag, unsigned seq) {
  __threadfence_system();
  *flag = seq;
}

int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double* d; cudaMalloc(&d, 8);
  unsigned* hflag; cudaHostAlloc(&hflag, 64, cudaHostAllocMapped);
  unsigned* dflag; cudaHostGetDevicePointer((void**)&dflag, hflag, 0);
  *hflag = 0;
  const int n = 2000;
  for (int w = 0; w < 2; ++w) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) { tiny<<<1, 32, 0, s>>>(d); cudaStreamSynchronize(s); }
    auto t1 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) {
      tiny<<<1, 32, 0, s>>>(d);
      signal<<<1, 1, 0, s>>>(dflag, i + 1 + w * n);
      while (*(volatile unsigned*)hflag != (unsigned)(i + 1 + w * n)) {}
    }
    auto t2 = std::chrono::steady_clock::now();
    printf("stream sync %.2f us/round trip, mapped-flag spin %.2f us/round trip\n",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / n,
           std::chrono::duration<double, std::micro>(t2 - t1).count() / n);
  }
  cudaStreamSynchronize(s);
  return 0;
}
