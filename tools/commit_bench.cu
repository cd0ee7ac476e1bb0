// Cost of the MMA warp's per-K-block bookkeeping on a CTA pair (no MMAs):
// tcgen05.commit (cta_group::2, multicast) and tcgen05.fence::after_thread_sync.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/commit_bench tools/commit_bench.cu && tools/commit_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

template <int V>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) kb(int iters, unsigned long long *out) {
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar[8];
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = ptx::cluster_rank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc2(&tbase, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  long long t0 = 0, t1 = 0;
  if (rank == 0 && warp == 1) {
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
      if (V & 1) ptx::tc_fence_after();
      if (ptx::elect_one()) {
        if (V & 2) ptx::mma2_commit_both(&bar[i & 7]);
        if (V & 4) ptx::mma_commit(&bar[i & 7]);
      }
      __syncwarp();
    }
    t1 = clock64();
    if (threadIdx.x == 32) out[V] = (t1 - t0) / iters;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 0) ptx::tmem_dealloc2(tbase, 512);
}

int main() {
  unsigned long long *d, h[8] = {0};
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  kb<0><<<2, 128>>>(4096, d);
  kb<1><<<2, 128>>>(4096, d);
  kb<2><<<2, 128>>>(4096, d);
  kb<3><<<2, 128>>>(4096, d);
  kb<4><<<2, 128>>>(4096, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("%s: loop %llu, fence %llu, commit2 multicast %llu, fence+commit2 %llu, commit1 %llu cycles/iter\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
