// SPDX-License-Identifier: Apache-2.0
// Minimal TMA (cp.async.bulk.tensor.3d) probe: loads 68x12 / 66x10 fp64 boxes with
// negative / out-of-range coordinates and checks values and zero fill.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2008_01440_b200/csrc/cheb2.cuh"

using namespace pcgx;

__global__ void probe(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int n,
                      double* out) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* buf = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, n * 8);
    tma_load_3d(buf, &m, c0, c1, c2, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  // usage: tma_probe bx by c0 c1 c2   (one case per process: a fault poisons the context)
  const int nx = 64, ny = 16, nz = 4;
  std::vector<double> h(nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i + 1.0;
  double* d;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  double* o;
  cudaMalloc(&o, 8192 * 8);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<EncodeTiledFn>(f);
  int bad = 0;
  {
    const int bx = atoi(argv[1]), by = atoi(argv[2]);
    CUtensorMap m;
    const cuuint64_t dims[3] = {nx, ny, nz};
    const cuuint64_t strides[2] = {nx * 8, nx * ny * 8};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode box %dx%d -> %d\n", bx, by, (int)r);
    const int coords[1][3] = {{atoi(argv[3]), atoi(argv[4]), atoi(argv[5])}};
    for (auto& c : coords) {
      const int n = bx * by;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
      probe<<<1, 128, n * 8 + 128>>>(m, c[0], c[1], c[2], n, o);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("  coords (%d,%d,%d): %s\n", c[0], c[1], c[2], cudaGetErrorString(e));
        return 2;
      }
      std::vector<double> got(n);
      cudaMemcpy(got.data(), o, n * 8, cudaMemcpyDeviceToHost);
      int wrong = 0;
      for (int jj = 0; jj < by; ++jj)
        for (int ii = 0; ii < bx; ++ii) {
          const int gi = c[0] + ii, gj = c[1] + jj, gk = c[2];
          const double exp = (gi >= 0 && gi < nx && gj >= 0 && gj < ny && gk >= 0 && gk < nz)
                                 ? h[(size_t)gk * nx * ny + gj * nx + gi] : 0.0;
          if (got[jj * bx + ii] != exp) ++wrong;
        }
      printf("  coords (%d,%d,%d): %d wrong of %d\n", c[0], c[1], c[2], wrong, n);
      bad += wrong;
    }
  }
  return bad ? 1 : 0;
}
