// Stand-alone check of the TMA residual kernel (fp32 / fp64) against a CPU loop.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include <cmath>
#include "../../paper_2110_03946_b200/csrc/kernels.cuh"
using namespace sib;

PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static int g_dtype = 0;
template <typename T>
int run(int W, int H, int C) {
  size_t N = (size_t)W * H;
  std::vector<T> u(N * C); std::vector<uint8_t> m(N);
  for (size_t i = 0; i < N * C; ++i) u[i] = T((i * 37 % 101) / 101.0);
  for (size_t i = 0; i < N; ++i) m[i] = (i * 7919 % 13) == 0;
  T* du; uint8_t* dm; double *part, *out; unsigned* tick;
  cudaMalloc(&du, N * C * sizeof(T)); cudaMalloc(&dm, N); cudaMalloc(&part, 1 << 22); cudaMalloc(&out, 64); cudaMalloc(&tick, 16);
  cudaMemset(tick, 0, 16);
  cudaMemcpy(du, u.data(), N * C * sizeof(T), cudaMemcpyHostToDevice);
  cudaMemcpy(dm, m.data(), N, cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C};
  cuuint64_t str[2] = {(cuuint64_t)W * sizeof(T), (cuuint64_t)N * sizeof(T)};
  cuuint32_t box[3] = {(cuuint32_t)res_tma_box_w<T>(), kResBand + 2, 1}, es[3] = {1, 1, 1};
  CUresult r = enc()(&map, g_dtype == 0 ? (sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32) : (sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32), 3, du, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int tx = (W + kResTmaThreads - 1) / kResTmaThreads, ty = (H + kResBand - 1) / kResBand;
  residual_sumsq_tma_kernel<T, true><<<dim3(tx, ty, C), kResTmaThreads>>>(map, dm, (const T*)du, W, H, N, 0, H, part, out, tick);
  cudaError_t e = cudaDeviceSynchronize();
  double g[8]; cudaMemcpy(g, out, 8 * C, cudaMemcpyDeviceToHost);
  for (int c = 0; c < C; ++c) {
    double ref = 0;
    for (int y = 0; y < H; ++y) for (int x = 0; x < W; ++x) {
      size_t i = (size_t)y * W + x; if (m[i]) continue;
      const T* uc = u.data() + c * N; double s = 0; int d = 0;
      if (x > 0) { s += uc[i - 1]; ++d; } if (x + 1 < W) { s += uc[i + 1]; ++d; }
      if (y > 0) { s += uc[i - W]; ++d; } if (y + 1 < H) { s += uc[i + W]; ++d; }
      double rr = d * (double)uc[i] - s; ref += rr * rr;
    }
    printf("%s W=%d H=%d c=%d enc=%d err=%s gpu=%.10g ref=%.10g rel=%.2e\n", sizeof(T) == 8 ? "f64" : "f32", W, H, c, (int)r,
           cudaGetErrorString(e), g[c], ref, std::fabs(g[c] - ref) / ref);
  }
  cudaFree(du); cudaFree(dm); cudaFree(part); cudaFree(out); cudaFree(tick);
  return e != cudaSuccess;
}

int main(int argc, char** argv) {
  if (argc > 1) g_dtype = atoi(argv[1]);
  if (run<double>(256, 256, 1)) return 1;
  if (run<float>(256, 256, 1)) return 1;
  if (run<float>(3840, 64, 3)) return 1;
  return 0;
}
