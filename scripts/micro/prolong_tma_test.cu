// Standalone check of prolong_snap_tma_kernel against prolong_snap_kernel.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstring>
#include "../../paper_2110_03946_b200/csrc/kernels.cuh"
using namespace sib;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)
int main(int argc, char** argv) {
  int cw = argc > 1 ? atoi(argv[1]) : 960, ch = argc > 2 ? atoi(argv[2]) : 540, C = 3;
  int fw = 2 * cw, fh = 2 * ch;
  size_t cn = (size_t)cw * ch, fn = (size_t)fw * fh;
  std::vector<double> hc(cn * C);
  for (size_t i = 0; i < hc.size(); ++i) hc[i] = (i % 977) * 1e-3;
  double *dc, *d1, *d2; uint8_t* dm;
  CK(cudaMalloc(&dc, cn * C * 8)); CK(cudaMalloc(&d1, fn * C * 8)); CK(cudaMalloc(&d2, fn * C * 8));
  CK(cudaMalloc(&dm, fn)); CK(cudaMemset(dm, 0, fn));
  CK(cudaMemcpy(dc, hc.data(), cn * C * 8, cudaMemcpyHostToDevice));
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap m;
  const cuuint64_t dims[3] = {(cuuint64_t)cw, (cuuint64_t)ch, (cuuint64_t)C};
  const cuuint64_t strides[2] = {(cuuint64_t)cw * 8, (cuuint64_t)cn * 8};
  const cuuint32_t box[3] = {(cuuint32_t)pro_box_w<double>(), (cuuint32_t)kProCY, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dc, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int tx = (fw + kProX - 1) / kProX, ty = (fh + kProY - 1) / kProY;
  prolong_snap_kernel<double><<<dim3(tx, ty), 256>>>(dc, cw, ch, fw, fh, C, dm, (const double*)d1, d1, 0, fh, 0, ch, fn, cn);
  CK(cudaDeviceSynchronize());
  int grid = std::min(tx * ty, 148 * 4);
  prolong_snap_tma_kernel<double, false><<<grid, 256>>>(m, m, cw, ch, fw, C, dm, (const double*)d2, d2, 0, fh, 0, 0, fn, tx, tx * ty);
  CK(cudaDeviceSynchronize());
  std::vector<double> a(fn * C), b(fn * C);
  CK(cudaMemcpy(a.data(), d1, fn * C * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), d2, fn * C * 8, cudaMemcpyDeviceToHost));
  printf("identical %d\n", (int)(memcmp(a.data(), b.data(), fn * C * 8) == 0));
  return 0;
}
