// TMA tile-load bandwidth with the pass kernel's access patterns, one CTA per
// SM, 8-deep ring of 16 KB stages:
//   G pattern: box 32 floats x 128 rows of a row-major [rows x n] fp32 matrix,
//              walking K (columns) within a 128-row tile
//   H pattern: four boxes of 32 x 32 (128 columns x 32 rows), walking rows
// over an L2-sized region (first 40 MB) or the whole 4 GB matrix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc
//        -o tools/tma_bench tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

constexpr int STAGES = 8, TILE = 16384;

template <int PAT, int PF>
__global__ void __launch_bounds__(64, 1)
bench(const __grid_constant__ CUtensorMap map, int rows, int n, int iters, unsigned long long *out,
      const void *map_base) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int nkb = n / 32, ntile = rows / 128;
  if (PF < 0 && threadIdx.x >= 32) {  // warp 1: LSU prefetch of the G tiles -PF K blocks ahead
    const int lane = threadIdx.x & 31;
    const float *base = (const float *)map_base;
    for (int k = -PF; k < iters - PF; ++k) {
      const int unit = k / nkb, kb = k % nkb;
      const int tile = (blockIdx.x + unit * gridDim.x) % ntile;
      for (int r = lane; r < 128; r += 32) {
        const float *p = base + (size_t)(tile * 128 + r) * n + kb * 32;
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
      }
      if ((k & 3) == 0) __nanosleep(200);
    }
    return;
  }
  if (threadIdx.x != 0) return;
  uint64_t g0 = ptx::globaltimer();
  for (int k = 0; k < iters + STAGES; ++k) {
    const int s = k % STAGES;
    if (k >= STAGES) ptx::mbar_wait(&full[s], ((k / STAGES) - 1) & 1);
    if (k >= iters) continue;
    ptx::mbar_arrive_expect_tx(&full[s], TILE);
    uint8_t *dst = smem + s * TILE;
    if (PAT == 0) {  // G: tile = CTA-strided, K walks
      const int unit = k / nkb, kb = k % nkb;
      const int tile = (blockIdx.x + unit * gridDim.x) % ntile;
      ptx::tma_load_2d(dst, &map, &full[s], kb * 32, tile * 128);
      if (PF > 0 && false) {
        const int kp = k + PF, up = kp / nkb, kbp = kp % nkb;
        ptx::tma_prefetch_2d(&map, kbp * 32, ((blockIdx.x + up * gridDim.x) % ntile) * 128);
      }
    } else {  // H: column tile = CTA-strided, rows walk
      const int rkb = rows / 32;
      const int unit = k / rkb, kb = k % rkb;
      const int x = (blockIdx.x + unit * gridDim.x) % (n / 128);
      if (PAT == 1)
        for (int j = 0; j < 4; ++j) ptx::tma_load_2d(dst + j * 4096, &map, &full[s], x * 128 + 32 * j, kb * 32);
      else  // one 128 x 32 box, no swizzle
        ptx::tma_load_2d(dst, &map, &full[s], x * 128, kb * 32);
    }
  }
  out[blockIdx.x] = ptx::globaltimer() - g0;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 10000;
  const size_t total_rows = 100000;
  float *a;
  cudaMalloc(&a, total_rows * n * 4);
  cudaMemset(a, 0, total_rows * n * 4);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  unsigned long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  for (int pat = 0; pat < 3; ++pat) {
    for (size_t rows : {(size_t)1024, total_rows}) {
      CUtensorMap map;
      cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)n * 4};
      cuuint32_t box[2] = {pat == 2 ? 128u : 32u, pat == 0 ? 128u : 32u};
      cuuint32_t es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          pat == 2 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int iters = 2048;
      for (int pf : {0, -8, -16, -32}) {
      if (pat != 0 && pf) continue;
      auto kern = pat == 0 ? (pf == 0 ? bench<0, 0> : pf == -8 ? bench<0, -8> : pf == -16 ? bench<0, -16> : bench<0, -32>)
                           : pat == 1 ? bench<1, 0> : bench<2, 0>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * TILE + 1024);
      kern<<<148, 64, STAGES * TILE + 1024>>>(map, (int)rows, n, iters, d, a);
      kern<<<148, 64, STAGES * TILE + 1024>>>(map, (int)rows, n, iters, d, a);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double tb = 148.0 * iters * TILE / (mx * 1e-9) / 1e12;
      printf("%s pattern pf %2d, %6zu rows (%5.0f MB): %s %.2f TB/s (%.1f GB/s per SM)\n", pat == 0 ? "G" : pat == 1 ? "H" : "H1", pf,
             rows, rows * n * 4 / 1e6, cudaGetErrorString(e), tb, tb * 1000 / 148);
      }
    }
  }
  return 0;
}
