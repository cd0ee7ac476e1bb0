// L2 / HBM -> SMEM bulk-copy bandwidth with one CTA per SM (cp.async.bulk,
// 16 KB pieces, 8-deep mbarrier ring), for an L2-resident and an HBM-sized
// source.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_1704_07669_b200/csrc -o tools/l2_bench tools/l2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

constexpr int PIECE = 16384, MAXST = 13;

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(64, 1) bench(const char *src, size_t bytes, int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t pieces = bytes / PIECE;
  long long t0 = clock64();
  uint64_t g0 = ptx::globaltimer();
  // piece p of iteration it: CTAs interleave over the buffer
  for (int k = 0; k < iters; ++k) {
    const int s = k % STAGES;
    if (k >= STAGES) ptx::mbar_wait(&full[s], ((k / STAGES) - 1) & 1);
    const size_t p = ((size_t)k * gridDim.x + blockIdx.x) % pieces;
    ptx::mbar_arrive_expect_tx(&full[s], PIECE);
    bulk_g2s(smem + s * PIECE, src + p * PIECE, PIECE, &full[s]);
  }
  for (int k = iters; k < iters + STAGES; ++k) {
    const int s = k % STAGES;
    if (k >= STAGES) ptx::mbar_wait(&full[s], ((k / STAGES) - 1) & 1);
  }
  uint64_t g1 = ptx::globaltimer();
  out[blockIdx.x] = g1 - g0;
  (void)t0;
}

template <int STAGES> void run(char *src, unsigned long long *d, unsigned long long *h);
int main() {
  const size_t big = 2048ull << 20;
  char *src;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  unsigned long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  run<2>(src, d, h);
  run<4>(src, d, h);
  run<8>(src, d, h);
  run<12>(src, d, h);
  return 0;
}
template <int STAGES>
void run(char *src, unsigned long long *d, unsigned long long *h) {
  cudaFuncSetAttribute(bench<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * PIECE);
  for (size_t mb : {32, 2048}) {
    const size_t bytes = mb << 20;
    const int iters = 4096;
    for (int grid : {148}) {
      printf("stages %2d ", STAGES);
      bench<STAGES><<<grid, 64, STAGES * PIECE>>>(src, bytes, iters, d);
      bench<STAGES><<<grid, 64, STAGES * PIECE>>>(src, bytes, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double tb = (double)grid * iters * PIECE / (mx * 1e-9) / 1e12;
      printf("buffer %5zu MB grid %3d: %s  %.2f TB/s (%.1f GB/s per CTA)\n", mb, grid, cudaGetErrorString(e),
             tb, tb * 1000 / grid);
    }
  }
}
