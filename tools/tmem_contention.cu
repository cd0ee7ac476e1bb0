// Pair MMA (cta_group::2, M=256, N=64, A from TMEM) throughput while other
// warps store to TMEM (tcgen05.st 32x32b.x16) at full speed: cycles per MMA
// and store bandwidth per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/tmem_contention tools/tmem_contention.cu && tools/tmem_contention
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

template <int NBG, int N, int LDS = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) k2(int iters, unsigned long long *out,
                                                                           const char *gsrc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ uint64_t done;
  __shared__ volatile int stop;
  const uint32_t rank = ptx::cluster_rank();
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) ((float *)smem)[i] = 1.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
    stop = 0;
  }
  if (warp == 0) ptx::tmem_alloc2(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  unsigned long long stores = 0;
  float acc = 0.f;
  __shared__ uint64_t tbar[4];
  if (LDS == 2 && warp == 8) {  // background bulk copies global -> shared (4 x 16 KB ring)
    if (threadIdx.x == 256) {
      for (int i = 0; i < 4; ++i) ptx::mbar_init(&tbar[i], 1);
      ptx::fence_mbar_init();
      int it = 0;
      while (!stop) {
        const int sl = it & 3;
        if (it >= 4) ptx::mbar_wait(&tbar[sl], ((it >> 2) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&tbar[sl], 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         ptx::smem_u32(smem + 65536 + sl * 16384)),
                     "l"(gsrc + ((size_t)(it * 148 + blockIdx.x) % 2048) * 16384), "r"(16384), "r"(ptx::smem_u32(&tbar[sl]))
                     : "memory");
        ++it;
      }
      for (int k = it; k < it + 4; ++k)
        if (k >= 4) ptx::mbar_wait(&tbar[k & 3], ((k >> 2) - 1) & 1);
      stores = it;
    }
  }
  if (LDS == 1 && warp >= 8) {  // background shared loads (4 warps)
    const uint32_t sb = ptx::smem_u32(smem);
    int it = 0;
    while (!stop) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 x = ptx::lds128(sb + ((threadIdx.x * 16 + j * 512 + it * 64) & 32767));
        acc += x.x;
      }
      ++it;
    }
    stores = it;
    if (acc == 1234.f) out[3] = 1;
  }
  if (warp >= 4 && warp < 4 + NBG) {  // background TMEM stores into columns 384..511
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = 1.f;
    const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    int it = 0;
    while (!stop) {
      ptx::tmem_st16(lb + 384 + (it & 7) * 16, v);
      if ((it & 3) == 3) ptx::tmem_wait_st();
      ++it;
    }
    stores = it;
  }
  long long t0 = 0, t1 = 0;
  if (rank == 0 && warp == 1) {
    t0 = clock64();
    constexpr uint32_t idesc = ptx::idesc_tf32(256, N, 0, 0);
    const uint32_t sb = ptx::smem_u32(smem);
#pragma unroll 1
    for (int i0 = 0; i0 < iters; i0 += 12) {
      if (ptx::elect_one()) {
#pragma unroll
        for (int i = 0; i < 12; ++i)
          ptx::mma2_tf32_ts(tmem + (i0 / 12 & 1) * 64, tmem + 128 + (i & 7) * 8,
                            ptx::sdesc_sw128(sb + (i & 3) * 32, 16, 1024), idesc, 1);
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma2_commit_both(&done);
    __syncwarp();
  }
  if (warp == 1) ptx::mbar_wait(&done, 0);
  if (rank == 0 && warp == 1) t1 = clock64();
  if (warp == 1 && threadIdx.x == 32) stop = 1;
  __syncthreads();
  if (rank == 0 && threadIdx.x == 32) out[0] = (t1 - t0);
  if (rank == 0 && threadIdx.x == 128) out[1] = stores;
  if (rank == 0 && threadIdx.x == 256) out[2] = stores;
  if (LDS == 2 && rank == 0 && threadIdx.x == 256) out[3] = stores;
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 0) ptx::tmem_dealloc2(tmem, 512);
}

template <int NBG, int N, int LDS = 0>
void run(int iters) {
  unsigned long long *d, h[4];
  cudaMalloc(&d, 32);
  cudaMemset(d, 0, 32);
  static char *gsrc = nullptr;
  if (!gsrc) cudaMalloc(&gsrc, 2048 * 16384);
  cudaFuncSetAttribute(k2<NBG, N, LDS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k2<NBG, N, LDS><<<2, 384, 140 * 1024>>>(iters, d, gsrc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  if (LDS == 1) printf("   bg lds: %.1f B/clk per SM\n", (double)h[2] * 8 * 16 * 128 / h[0]);
  if (LDS == 2) printf("   bg bulk copies: %.1f B/clk per SM\n", (double)h[3] * 16384 / h[0]);
  // warp 4 stored h[1] x 16 cols x 32 lanes x 4 B; NBG warps in total
  const double bytes = (double)h[1] * 16 * 32 * 4 * NBG;
  printf("N=%3d bg store warps %d: %s  %.1f cycles/MMA, TMEM stores %.1f B/clk per SM\n", N, NBG,
         cudaGetErrorString(e), (double)h[0] / iters, bytes / h[0]);
}

int main() {
  for (int it = 0; it < 1; ++it) {
    run<0, 64>(12 * 512);
    run<4, 64>(12 * 512);
    run<8, 64>(12 * 512);
    run<0, 128>(12 * 512);
    run<8, 128>(12 * 512);
    run<0, 64, 1>(12 * 512);
    run<4, 64, 1>(12 * 512);
    run<0, 64, 2>(12 * 512);
    run<4, 64, 2>(12 * 512);
  }
  return 0;
}
