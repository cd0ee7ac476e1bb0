// Does multicasting the shared B operand cut the L2 cost of the pass kernel's
// operand stream?  Each CTA streams, per iteration, a unique 16 KB A tile
// (box 32 x 128 rows, SW128, from an L2-resident 40 MB region) and a 12 KB B
// block (32 x 96 rows of an L2-resident W-like matrix, the same K block for
// every CTA).  G = number of CTAs that share one B block: G = 1 loads it
// unicast in every CTA; G = 2 / 4 splits it into G slices, each CTA loading one
// slice multicast to the G CTAs with the same pair parity (cluster = 2G CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc
//        -o tools/mc_bench tools/mc_bench.cu
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

constexpr int B_BYTES = 12288;

__device__ __forceinline__ void tma_load_mc(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(ptx::smem_u32(dst)),
      "l"(map), "r"(ptx::smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}

template <int G, int WITH_B, int STAGES, int ABOX>
__global__ void __launch_bounds__(32, 1)
bench(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int atiles, int nkb,
      int iters, unsigned long long *out) {
  constexpr int A_BYTES = 16384 * (ABOX == 1 ? 1 : 2), STAGE = A_BYTES + (WITH_B ? B_BYTES : 0);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const uint32_t rank = G > 1 ? ptx::cluster_rank() : 0;
  const uint32_t par = rank & 1, gi = rank >> 1;  // group = same parity
  uint16_t mask = 0;
  for (int j = 0; j < G; ++j) mask |= (uint16_t)(1u << (2 * j + par));
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], G);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (G > 1) ptx::cluster_sync();
  if (threadIdx.x == 0) {
  const uint32_t bytes = A_BYTES + (WITH_B ? B_BYTES : 0);
  constexpr int BROWS = 96 / G;
  uint64_t t0 = ptx::globaltimer();
  auto issue = [&](int k) {
    const int s = k % STAGES;
    if (k >= STAGES) ptx::mbar_wait_cluster(&empty[s], ((k / STAGES) - 1) & 1);
    ptx::mbar_arrive_expect_tx(&full[s], bytes);
    uint8_t *dst = smem + s * STAGE;
    const int kb = k % nkb, tile = (blockIdx.x + (k / nkb) * gridDim.x) % atiles;
    if (ABOX == 1)
      ptx::tma_load_2d(dst, &amap, &full[s], kb * 32, tile * 128);
    else if (ABOX == 4)
      ptx::tma_load_2d(dst, &amap, &full[s], kb * 32, (tile * 128) % (atiles * 128 - 128));
    else if (ABOX == 3)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
          ::"r"(ptx::smem_u32(dst)), "l"(&amap), "r"(ptx::smem_u32(&full[s])), "r"(0), "r"(tile * 128),
          "r"((kb * 2) % (nkb - 2)) : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
          ::"r"(ptx::smem_u32(dst)), "l"(&amap), "r"(ptx::smem_u32(&full[s])), "r"(0), "r"((kb * ABOX) % (nkb - ABOX)),
          "r"(tile * 128) : "memory");
    if (WITH_B) {
      if (G == 1)
        ptx::tma_load_2d(dst + A_BYTES, &bmap, &full[s], kb * 32, 0);
      else
        tma_load_mc(dst + A_BYTES + gi * BROWS * 128, &bmap, &full[s], kb * 32, gi * BROWS, mask);
    }
  };
  for (int k = 0; k < STAGES - 1 && k < iters; ++k) issue(k);
  for (int k = 0; k < iters; ++k) {
    if (k + STAGES - 1 < iters) issue(k + STAGES - 1);
    const int s = k % STAGES;
    // consume: wait for the stage, then release it to every CTA that writes it
    ptx::mbar_wait(&full[s], (k / STAGES) & 1);
    if (G == 1) {
      ptx::mbar_arrive(&empty[s]);
    } else {
      for (int j = 0; j < G; ++j) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&empty[s]), 2 * j + par));
    }
  }
  out[blockIdx.x] = ptx::globaltimer() - t0;
  }
  __syncwarp();
  if (G > 1) ptx::cluster_sync();
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int G, int WITH_B, int STAGES, int ABOX>
void run(EncodeFn enc, float *a, float *b, int n, int arows) {
  constexpr int A_BYTES = 16384 * (ABOX == 1 ? 1 : 2), STAGE = A_BYTES + (WITH_B ? B_BYTES : 0);
  CUtensorMap amap, bmap;
  cuuint32_t es[3] = {1, 1, 1};
  if (ABOX == 1) {
    cuuint64_t adims[2] = {(cuuint64_t)n, (cuuint64_t)arows}, astr[1] = {(cuuint64_t)n * 4};
    cuuint32_t abox[2] = {32, 128};
    enc(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, adims, astr, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (ABOX == 4) {
    cuuint64_t adims[2] = {(cuuint64_t)n, (cuuint64_t)arows}, astr[1] = {(cuuint64_t)n * 4};
    cuuint32_t abox[2] = {32, 256};
    enc(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, adims, astr, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (ABOX == 3) {
    cuuint64_t adims[3] = {32, (cuuint64_t)arows, (cuuint64_t)n / 32}, astr[2] = {(cuuint64_t)n * 4, 128};
    cuuint32_t abox[3] = {32, 128, 2};
    CUresult r = enc(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a, adims, astr, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode 3d (k-block outer) failed %d\n", (int)r);
  } else {
    cuuint64_t adims[3] = {32, (cuuint64_t)n / 32, (cuuint64_t)arows}, astr[2] = {128, (cuuint64_t)n * 4};
    cuuint32_t abox[3] = {32, ABOX, 128};
    CUresult r = enc(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a, adims, astr, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode 3d failed %d\n", (int)r);
  }
  // B: [96 rows x n] K-major (row = output column, 32-float K boxes)
  cuuint64_t bdims[2] = {(cuuint64_t)n, 96}, bstr[1] = {(cuuint64_t)n * 4};
  cuuint32_t bbox[2] = {32, (cuuint32_t)(96 / G)};
  enc(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b, bdims, bstr, bbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto kern = bench<G, WITH_B, STAGES, ABOX>;
  const int smem = STAGES * STAGE + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int cs = G > 1 ? 2 * G : 1;
  if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int maxc = 0;
  cfg.gridDim = dim3(cs);
  cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg);
  const int grid = (148 / cs < maxc ? 148 / cs : maxc) * cs;
  cfg.gridDim = dim3(grid);
  unsigned long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  const int iters = 4096, nkb = n / 32, atiles = arows / 128;
  cudaLaunchKernelEx(&cfg, kern, amap, bmap, atiles, nkb, iters, d);
  cudaLaunchKernelEx(&cfg, kern, amap, bmap, atiles, nkb, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per_sm_ingress = (double)iters * (A_BYTES + (WITH_B ? B_BYTES : 0)) / (mx * 1e-9) / 1e9;
  const double l2_reads = (double)grid * iters * (A_BYTES + (WITH_B ? B_BYTES / G : 0)) / (mx * 1e-9) / 1e12;
  printf("A %s box %dx16KB stages %2d G=%d B=%d cluster %2d grid %3d: %s  %.1f ns/iter, SM ingress %.1f GB/s"
         " per SM (%.2f TB/s chip), L2 reads %.2f TB/s\n",
         arows > 1024 ? "HBM" : "L2 ", ABOX, STAGES, G, WITH_B, cs, grid, cudaGetErrorString(e), mx / (double)iters,
         per_sm_ingress, per_sm_ingress * grid / 1e3, l2_reads);
  cudaFree(d);
}

int main(int argc, char **argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int which = argc > 1 ? atoi(argv[1]) : -1;
  const int n = 10000, arows = 1024, hrows = 65536;  // 40 MB L2 region / 2.6 GB
  float *a, *b;
  cudaMalloc(&a, (size_t)hrows * n * 4);
  cudaMalloc(&b, (size_t)96 * n * 4);
  cudaMemset(a, 0, (size_t)hrows * n * 4);
  cudaMemset(b, 0, (size_t)96 * n * 4);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  if (which < 0 || which == 0) run<1, 0, 6, 1>(enc, a, b, n, arows);
  if (which < 0 || which == 1) run<1, 1, 6, 1>(enc, a, b, n, arows);
  if (which < 0 || which == 2) run<2, 1, 6, 1>(enc, a, b, n, arows);
  if (which < 0 || which == 3) run<4, 1, 6, 1>(enc, a, b, n, arows);
  if (which < 0 || which == 4) run<1, 0, 4, 1>(enc, a, b, n, arows);
  if (which < 0 || which == 5) run<1, 0, 8, 1>(enc, a, b, n, arows);
  if (which < 0 || which == 6) run<1, 0, 12, 1>(enc, a, b, n, arows);
  if (which < 0 || which == 7) run<1, 0, 3, 2>(enc, a, b, n, arows);
  if (which < 0 || which == 8) run<1, 0, 6, 2>(enc, a, b, n, arows);
  if (which < 0 || which == 9) run<1, 0, 12, 1>(enc, a, b, n, hrows);
  if (which < 0 || which == 10) run<1, 0, 6, 1>(enc, a, b, n, hrows);
  if (which < 0 || which == 11) run<1, 0, 6, 2>(enc, a, b, n, hrows);
  if (which < 0 || which == 12) run<1, 1, 6, 1>(enc, a, b, n, hrows);
  if (which < 0 || which == 13) run<1, 0, 6, 3>(enc, a, b, n, arows);
  if (which < 0 || which == 14) run<1, 0, 6, 4>(enc, a, b, n, arows);
  if (which < 0 || which == 15) run<1, 1, 5, 2>(enc, a, b, n, arows);
  if (which < 0 || which == 16) run<1, 1, 5, 3>(enc, a, b, n, arows);
  if (which < 0 || which == 17) run<1, 0, 6, 3>(enc, a, b, n, hrows);
  return 0;
}
