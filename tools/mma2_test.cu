// 2-CTA (cta_group::2) tf32 MMA check: M = 256 over a CTA pair, A from each
// CTA's TMEM, B halves in each CTA's SMEM, multicast commit, remote mbarrier
// arrive from the peer. Verifies the operand split and times the MMA rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/mma2_test tools/mma2_test.cu && tools/mma2_test
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k2(int iters, float *out, unsigned long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ uint64_t done, peer_ready;
  const uint32_t rank = cta_rank();
  const int warp = threadIdx.x >> 5;
  // B half: N/2 rows x 32 k (K-major, 128 B rows), value 1 (rank 0) or 2 (rank 1)
  for (int i = threadIdx.x; i < (N / 2) * 32; i += blockDim.x) ((float *)smem)[i] = rank == 0 ? 1.f : 2.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&done, 1);
    ptx::mbar_init(&peer_ready, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(&tbase)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  {  // A (this CTA's 128 rows): 1 (rank 0) or 3 (rank 1) in columns 256..287
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = rank == 0 ? 1.f : 3.f;
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    ptx::tmem_st16(lb + 256, v);
    ptx::tmem_st16(lb + 272, v);
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (rank == 1 && threadIdx.x == 0) arrive_remote(mapa(ptx::smem_u32(&peer_ready), 0));
  long long t0 = 0, t1 = 0;
  if (rank == 0 && warp == 1) {
    ptx::mbar_wait(&peer_ready, 0);
    ptx::tc_fence_after();
    t0 = clock64();
    constexpr uint32_t idesc = ptx::idesc_tf32(256, N, 0, 0);
    const uint32_t sb = ptx::smem_u32(smem);
#pragma unroll 1
    for (int i0 = 0; i0 < iters; i0 += 8) {
      if (ptx::elect_one()) {
#pragma unroll
       for (int i = i0; i < i0 + 8; ++i) {
        const int kk = i & 3;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(
                tmem),
            "r"(tmem + 256 + kk * 8), "l"(ptx::sdesc_sw128(sb + kk * 32, 16, 1024)), "r"(idesc), "r"(i > 0 ? 1 : 0),
            "r"(0)
            : "memory");
       }
      }
      __syncwarp();
    }
    if (ptx::elect_one())
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              ptx::smem_u32(&done)),
          "h"((uint16_t)3)
          : "memory");
    __syncwarp();
  }
  if (warp == 2) ptx::mbar_wait(&done, 0);  // both CTAs
  if (rank == 0 && warp == 1) t1 = clock64();
  __syncthreads();
  ptx::tc_fence_after();
  {  // D rows of this CTA: columns 0..N-1
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < N; c += 16) {
      float v[16];
      ptx::tmem_ld16(lb + c, v);
      for (int i = 0; i < 16; ++i) out[((size_t)rank * 128 + threadIdx.x) * N + c + i] = v[i];
    }
  }
  if (rank == 0 && threadIdx.x == 32) cyc[0] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N>
void run(int iters) {
  float *out;
  unsigned long long *cyc;
  cudaMalloc(&out, 256 * N * 4);
  cudaMalloc(&cyc, 8);
  cudaFuncSetAttribute(k2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20 * 1024);
  k2<N><<<2, 128, 20 * 1024>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  static float h[256 * 256];
  unsigned long long c = 0;
  cudaMemcpy(h, out, 256 * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("N=%d iters=%d: %s  %.1f cycles/MMA\n", N, iters, cudaGetErrorString(e), (double)c / iters);
  // expected D[r][n] = iters * 8 * A(r) * B(n): A = 1 (rows < 128) or 3; B = 1 (n < N/2) or 2
  int bad = 0;
  for (int r = 0; r < 256; ++r)
    for (int n = 0; n < N; ++n) {
      const float want = iters * 8.f * (r < 128 ? 1.f : 3.f) * (n < N / 2 ? 1.f : 2.f);
      if (h[r * N + n] != want && bad++ < 5) printf("  D[%d][%d] = %g want %g\n", r, n, h[r * N + n], want);
    }
  printf("  mismatches: %d; samples D[0][0]=%g D[0][%d]=%g D[200][0]=%g D[200][%d]=%g\n", bad, h[0], N - 1,
         h[N - 1], h[200 * N], N - 1, h[200 * N + N - 1]);
}

int main() {
  run<64>(4096);
  run<128>(8);
  run<128>(4096);
  run<256>(4096);
  return 0;
}
