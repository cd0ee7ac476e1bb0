// The pass kernel's MMA-issue loop in isolation on a CTA pair: per K block,
// 12 pair MMAs (M=256, N=64, A from a rotating TMEM stage, B from a rotating
// SMEM stage, two alternating accumulators per 4-block period) and the
// commits, with optional per-block mbarrier waits on barriers that are
// already complete. Cycles per K block.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/mma_loop_bench tools/mma_loop_bench.cu && tools/mma_loop_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sketch_tc.cuh"

using namespace spca;
__device__ __forceinline__ bool lane0() { return (threadIdx.x & 31) == 0; }

template <int V, int BUSY = 0, int RND = 0, int MEM = 0, int STORES = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) kb(int nkb, unsigned long long *out,
                                                                    const char *gsrc = nullptr) {
  using C = TcCfg<64>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ uint64_t kb_empty[6], acc_full[2], ready, b_empty[8];
  const uint32_t rank = ptx::cluster_rank();
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (RND ? 12 : 6) * 8192 / 4; i += blockDim.x) {
    float x = 1.f;
    if (RND) {  // pseudo-random tf32-ish values
      uint32_t h = (i + 1) * 2654435761u ^ (blockIdx.x * 97u);
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      x = ((float)(h & 0xFFFFFF) / 16777216.f - 0.5f) * 3.f;
    }
    ((float *)smem)[i] = x;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) ptx::mbar_init(&kb_empty[i], 1);
    for (int i = 0; i < 2; ++i) ptx::mbar_init(&acc_full[i], 1);
    for (int i = 0; i < 8; ++i) ptx::mbar_init(&b_empty[i], 1);
    ptx::mbar_init(&ready, 1);
    ptx::mbar_arrive(&ready);  // phase 0 complete: waits on it return at once
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc2(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (RND && warp < 4) {  // random A operand stages in TMEM
    float v[16];
    for (int c = 128; c < 512; c += 16) {
      for (int i = 0; i < 16; ++i) {
        uint32_t h = (threadIdx.x * 512 + c + i + 7) * 2246822519u;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        v[i] = ((float)(h & 0xFFFFFF) / 16777216.f - 0.5f) * 3.f;
      }
      ptx::tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    }
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  __shared__ uint64_t tbar[4];
  if (MEM && warp == 15 && lane0()) {  // HBM -> SMEM bulk copies at full speed
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&tbar[i], 1);
    ptx::fence_mbar_init();
    int it = 0;
    uint8_t *dst = smem + 12 * 8192;
    while (!stop) {
      const int sl = it & 3;
      if (it >= 4) ptx::mbar_wait(&tbar[sl], ((it >> 2) - 1) & 1);
      ptx::mbar_arrive_expect_tx(&tbar[sl], 16384);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       ptx::smem_u32(dst + sl * 16384)),
                   "l"(gsrc + ((size_t)(it * 148 + blockIdx.x) % 65536) * 16384), "r"(16384),
                   "r"(ptx::smem_u32(&tbar[sl]))
                   : "memory");
      ++it;
    }
    for (int k = it; k < it + 4; ++k)
      if (k >= 4) ptx::mbar_wait(&tbar[k & 3], ((k >> 2) - 1) & 1);
  }
  if (STORES && warp >= 4 && warp < 12) {  // converter-like TMEM stores into the A stages
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = 0.5f + i;
    const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    int it = 0;
    while (!stop) {
      const uint32_t col = 256 + ((it + (warp >> 2)) & 3) * 64;
      ptx::tmem_st32(lb + col, v);
      ptx::tmem_st32(lb + col + 32, v);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ++it;
    }
  }
  if (BUSY && warp >= 4 && warp < 4 + BUSY) {  // ALU-bound warps sharing the schedulers
    float x = threadIdx.x, y = 1.0001f;
    while (!stop) {
#pragma unroll 16
      for (int i = 0; i < 64; ++i) { x = fmaf(x, y, 0.5f); y = fmaf(y, x, -0.25f); }
    }
    if (x == 1234.5f) out[15] = 1;
  }
  if (rank == 0 && warp == 1) {
    const uint64_t bdesc0 = ptx::sdesc_sw128(ptx::smem_u32(smem), 16, 1024);
    long long t0 = clock64();
#pragma unroll 1
    for (int gkb = 0; gkb < nkb; ++gkb) {
      const int ks = gkb % C::NS, kb = gkb & 3, q = gkb >> 2, buf = q & 1;
      if (V & 1) ptx::mbar_wait(&ready, 0);
      if ((V & 2) && kb == 0) ptx::mbar_wait(&ready, 0);
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        tc_mma_stage2<64>(tmem + C::A_TMEM + 64 * ks, tmem + buf * C::ACC_COLS,
                          bdesc0 + (uint64_t)((ks * C::B_STAGE) >> 4), kb == 0);
        ptx::mma2_commit_both(&kb_empty[ks]);
        if (V & 4) ptx::mma2_commit_both(&b_empty[gkb % 7]);
        if (kb == 3) ptx::mma2_commit_both(&acc_full[buf]);
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) out[V] = (t1 - t0) / nkb;
  }
  if (warp == 1) stop = 1;
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 1) ptx::tmem_dealloc2(tmem, 512);
}

int main() {
  unsigned long long *d, h[16] = {0};
  cudaMalloc(&d, 128);
  cudaMemset(d, 0, 128);
  cudaFuncSetAttribute(kb<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  cudaFuncSetAttribute(kb<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  cudaFuncSetAttribute(kb<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  kb<0><<<2, 128, 60 * 1024>>>(2048, d);
  kb<3><<<148, 128, 60 * 1024>>>(8192, d + 2);
  cudaFuncSetAttribute(kb<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  cudaFuncSetAttribute(kb<3, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  kb<3, 4><<<2, 512, 60 * 1024>>>(2048, d + 3);
  cudaFuncSetAttribute(kb<3, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kb<3, 0, 1><<<148, 512, 100 * 1024>>>(8192, d + 5);
  char *g;
  cudaMalloc(&g, (size_t)65536 * 16384);
  cudaMemset(g, 1, (size_t)65536 * 16384);
  cudaFuncSetAttribute(kb<3, 8, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  kb<3, 8, 1, 1><<<148, 512, 180 * 1024>>>(16384, d + 6, g);
  cudaFuncSetAttribute(kb<3, 0, 1, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kb<3, 0, 1, 0, 1><<<148, 512, 100 * 1024>>>(8192, d + 7);
  cudaFuncSetAttribute(kb<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  kb<7><<<2, 128, 60 * 1024>>>(2048, d + 1);
  kb<3, 12><<<2, 512, 60 * 1024>>>(2048, d + 4);
  kb<1><<<2, 128, 60 * 1024>>>(2048, d);
  kb<3><<<2, 128, 60 * 1024>>>(2048, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("%s: cycles per K block (ideal 384): no waits %llu, 1 wait %llu, 2 waits %llu, all SMs %llu,"
         " +4 busy warps %llu, +12 busy warps %llu, random data all SMs %llu, + HBM copies + ALU all SMs %llu,"
         " + TMEM stores into the A stages %llu, 3 commits %llu\n",
         cudaGetErrorString(e), h[0], h[1], h[3], h[2 + 3], h[3 + 3], h[4 + 3], h[5 + 3], h[6 + 3], h[7 + 3], h[1 + 7]);
  return 0;
}
