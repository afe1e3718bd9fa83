// Minimal TMA box copy (3-D map, zero fill) for fp32 and fp64.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_2110_03946_b200/csrc/tma.cuh"
using namespace sib;

template <typename T, int BW, int BH>
__global__ void copy_box(const __grid_constant__ CUtensorMap map, int x, int y, T* out) {
  __shared__ __align__(128) T tile[BH][BW];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, sizeof(tile));
    tma_load_3d(&tile[0][0], &map, x, y, 0, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < BW * BH; i += blockDim.x) out[i] = (&tile[0][0])[i];
}

template <typename T, int BW, int BH>
void run(int W, int H, int x, int y, CUtensorMapDataType dt) {
  void* p = nullptr; cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  std::vector<T> h((size_t)W * H);
  for (size_t i = 0; i < h.size(); ++i) h[i] = T(i);
  T *d, *o; cudaMalloc(&d, h.size() * sizeof(T)); cudaMalloc(&o, BW * BH * sizeof(T));
  cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
  cuuint64_t str[2] = {(cuuint64_t)W * sizeof(T), (cuuint64_t)W * H * sizeof(T)};
  cuuint32_t box[3] = {BW, BH, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, dt, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  copy_box<T, BW, BH><<<1, 128>>>(map, x, y, o);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<T> g(BW * BH);
  cudaMemcpy(g.data(), o, g.size() * sizeof(T), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int j = 0; j < BH; ++j) for (int i = 0; i < BW; ++i) {
    int gx = x + i, gy = y + j;
    T want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[(size_t)gy * W + gx] : T(0);
    bad += g[j * BW + i] != want;
  }
  printf("elem %zu box %dx%d at (%d,%d) W=%d dt=%d enc=%d err=%s bad=%d\n", sizeof(T), BW, BH, x, y, W, (int)dt, (int)r, cudaGetErrorString(e), bad);
  cudaFree(d); cudaFree(o);
}

int main(int argc, char** argv) {
  int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0) run<float, 144, 18>(256, 256, -2, -1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  if (which == 1) run<float, 128, 16>(256, 256, 0, 0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  if (which == 2) run<float, 32, 8>(256, 256, 0, 0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  if (which == 3) run<double, 136, 18>(256, 256, -2, -1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64);
  if (which == 4) run<float, 144, 18>(256, 256, -2, -1, CU_TENSOR_MAP_DATA_TYPE_UINT32);
  if (which == 5) run<float, 64, 18>(256, 256, -2, -1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  if (which == 6) run<float, 144, 18>(256, 256, 2, 0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  if (which == 7) run<float, 144, 18>(256, 256, -4, -1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  if (which == 8) run<double, 36, 36>(256, 256, 3, 5, CU_TENSOR_MAP_DATA_TYPE_FLOAT64);
  if (which == 9) run<double, 36, 36>(256, 256, -1, -2, CU_TENSOR_MAP_DATA_TYPE_FLOAT64);
  return 0;
}
