// Bisect: TMA into a 2-stage ring with parity waits.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2110_03946_b200/csrc/tma.cuh"
using namespace sib;
struct __align__(128) Slice { double v[10][BW]; };
__global__ void k3(const __grid_constant__ CUtensorMap m, int ntiles, double* out) {
  __shared__ Slice ring[2][4];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_expect_tx(&bar[0], 80 * BW);
    tma_load_3d(&ring[0][0].v[0][0], &m, 31, 7, 0, &bar[0]);
  }
  __syncthreads();
  mbar_wait(&bar[0], 0);
  out[blockIdx.x * blockDim.x + tid] = ring[0][0].v[tid % 10][tid % BW];
}
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap m, int ntiles, double* out) {
  __shared__ Slice ring[2][4];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
  __syncthreads();
  int kk = 0;
  double acc = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++kk) {
    const int stage = MODE == 2 ? 0 : (kk & 1);
    if (tid == 0) {
      mbar_expect_tx(&bar[stage], 80 * BW * (MODE == 1 ? 1 : 3));
      for (int c = 0; c < (MODE == 1 ? 1 : 3); ++c)
        tma_load_3d(&ring[stage][c].v[0][0], &m, (t % 16) * 32 - 1, (t / 16) * 8 - 1, c, &bar[stage]);
    }
    mbar_wait(&bar[stage], MODE == 2 ? (kk & 1) : ((kk >> 1) & 1));
    acc += ring[stage][0].v[tid % 10][tid % BW];
    __syncthreads();
  }
  out[blockIdx.x * blockDim.x + tid] = acc;
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  int cw = 512, ch = 128, C = 3;
  double *dc, *o; CK(cudaMalloc(&dc, (size_t)cw * ch * C * 8)); CK(cudaMemset(dc, 0, (size_t)cw*ch*C*8));
  CK(cudaMalloc(&o, 1 << 24));
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap m;
  const cuuint64_t dims[3] = {(cuuint64_t)cw, (cuuint64_t)ch, (cuuint64_t)C};
  const cuuint64_t strides[2] = {(cuuint64_t)cw * 8, (cuuint64_t)cw * ch * 8};
  const cuuint32_t box[3] = {BW, 10, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  printf("encode %d\n", (int)enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dc, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  if (mode == 0) k<0><<<8, 256>>>(m, 64, o);
  if (mode == 1) k<1><<<8, 256>>>(m, 64, o);
  if (mode == 2) k<2><<<8, 256>>>(m, 64, o);
  if (mode == 3) k3<<<8, 256>>>(m, 64, o);
  CK(cudaDeviceSynchronize());
  printf("mode %d ok\n", mode);
  return 0;
}
