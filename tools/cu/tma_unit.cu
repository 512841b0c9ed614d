// Stand-alone check of the TMA helpers (tma.cuh) on a 3-D double array:
// one CTA loads boxes with an mbarrier and compares them with the source.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2401_01745_b200/csrc/tma.cuh"

using namespace emrkc_dev;

struct Maps {
  CUtensorMap m3;
  CUtensorMap m4;
};

__global__ void k_test(const __grid_constant__ Maps mp, const CUtensorMap* gmap, const double* src,
                       int n0, int n1, int nz, int mode, int* bad) {
  extern __shared__ __align__(128) double sm[];
  double* buf = (double*)(((unsigned long long)sm + 127) & ~127ull);
  __shared__ __align__(8) unsigned long long bar;
  const int t = threadIdx.x;
  if (t == 0) {
    mbar_init(smem_u32(&bar), 1);
    if (mode != 4) mbar_fence_init();
  }
  __syncthreads();
  const int x0 = mode == 5 ? -2 : (mode == 6 ? 0 : -1), y0 = mode == 7 ? 0 : -1, z0 = 2;
  if (t == 0) {
    if (mode == 0 || mode >= 4) {
      mbar_expect_tx(smem_u32(&bar), 34 * 6 * 8);
      tma_load_3d(smem_u32(buf), &mp.m3, smem_u32(&bar), x0, y0, z0);
    } else if (mode == 3) {
      mbar_expect_tx(smem_u32(&bar), 34 * 6 * 8);
      tma_load_3d(smem_u32(buf), gmap, smem_u32(&bar), x0, y0, z0);
    } else if (mode == 2) {
      mbar_expect_tx(smem_u32(&bar), 34 * 6 * 8);
      tma_load_3d(smem_u32(buf), &mp.m3, smem_u32(&bar), 0, 0, z0);
    } else {
      mbar_expect_tx(smem_u32(&bar), 32 * 4 * 3 * 8);
      tma_load_4d(smem_u32(buf), &mp.m4, smem_u32(&bar), 0, 0, z0, 1);
    }
  }
  mbar_wait(smem_u32(&bar), 0);
  int nb = 0;
  if (mode != 1) {
    for (int i = t; i < 34 * 6; i += blockDim.x) {
      const int x = (mode == 2 ? 0 : x0) + i % 34, y = (mode == 2 ? 0 : y0) + i / 34;
      const double want = (x < 0 || y < 0 || x >= n0 || y >= n1) ? 0.0
                                                                 : src[x + n0 * (y + n1 * z0)];
      nb += buf[i] != want;
    }
  } else {
    const long long nn = (long long)n0 * n1 * nz;
    for (int i = t; i < 32 * 4 * 3; i += blockDim.x) {
      const int f = 1 + i / 128, x = i % 32, y = (i / 32) % 4;
      nb += buf[i] != src[f * nn + x + n0 * (y + n1 * z0)];
    }
  }
  atomicAdd(bad, nb);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int n0 = 64, n1 = 32, nz = 16;
  const long long nn = (long long)n0 * n1 * nz;
  std::vector<double> h(4 * nn);
  for (long long i = 0; i < 4 * nn; ++i) h[i] = 1.0 + i;
  double* d;
  int* bad;
  cudaMalloc(&d, 8 * 4 * nn);
  cudaMalloc(&bad, 4);
  cudaMemcpy(d, h.data(), 8 * 4 * nn, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  Maps mp;
  cuuint64_t dims[4] = {(cuuint64_t)n0, (cuuint64_t)n1, (cuuint64_t)nz, 4};
  cuuint64_t str[3] = {8ull * n0, 8ull * n0 * n1, 8ull * nn};
  cuuint32_t box3[3] = {34, 6, 1}, box4[4] = {32, 4, 1, 3}, es[4] = {1, 1, 1, 1};
  CUresult r1 = enc(&mp.m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box3, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&mp.m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box4, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &mp.m3, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  {
    cudaMemset(bad, 0, 4);
    k_test<<<1, 128, 8192>>>(mp, gm, d, n0, n1, nz, mode, bad);
    cudaError_t e = cudaDeviceSynchronize();
    int hb = -1;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("mode %d: %s, mismatches %d\n", mode, cudaGetErrorString(e), hb);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
