// Host<->device of a 199 MB pageable buffer: plain cudaMemcpy vs
// cudaHostRegister + async copy + unregister vs a pinned buffer.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <thread>
#include <vector>
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

int main() {
  const size_t n = 3840ull * 2160 * 3 * 8;
  char* h = (char*)malloc(n);
  memset(h, 1, n);
  void* d; cudaMalloc(&d, n);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int rep = 0; rep < 2; ++rep) {
    auto t0 = clk::now();
    cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
    auto t1 = clk::now();
    cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost);
    auto t2 = clk::now();
    cudaHostRegister(h, n, cudaHostRegisterDefault);
    auto t3 = clk::now();
    cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    auto t4 = clk::now();
    cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    auto t5 = clk::now();
    cudaHostUnregister(h);
    auto t6 = clk::now();
    // chunked multi-threaded memcpy into pinned buffers
    char* pin; cudaMallocHost(&pin, n);
    auto t7 = clk::now();
    int T = std::thread::hardware_concurrency(); if (T > 16) T = 16;
    std::vector<std::thread> th;
    for (int k = 0; k < T; ++k) th.emplace_back([&, k] { size_t a = n * k / T, b = n * (k + 1) / T; memcpy(pin + a, h + a, b - a); });
    for (auto& x : th) x.join();
    auto t8 = clk::now();
    cudaFreeHost(pin);
    printf("pageable H2D %.1f ms, D2H %.1f ms | register %.1f ms, H2D %.1f, D2H %.1f, unregister %.1f | %d-thread memcpy to pinned %.1f ms\n",
           ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), ms(t5, t6), T, ms(t7, t8));
  }
  return 0;
}
