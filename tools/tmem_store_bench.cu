// tcgen05.st throughput per shape: 32x32b.x16 / .x32 / .x64 from N warps,
// one CTA per SM, bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/tmem_store_bench tools/tmem_store_bench.cu && tools/tmem_store_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

template <int X>
__device__ __forceinline__ void st(uint32_t taddr, const uint32_t *r);
template <>
__device__ __forceinline__ void st<16>(uint32_t a, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
               : "memory");
}
template <>
__device__ __forceinline__ void st<32>(uint32_t a, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

template <int X, int NW, int WAITEVERY>
__global__ void __launch_bounds__(512, 1) kb(int iters, unsigned long long *out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc(&tbase, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 32 + i;
  __syncthreads();
  long long t0 = clock64();
  if (warp < NW) {
    const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
      st<X>(lb + (i & 1) * 32, r);
      if ((i % WAITEVERY) == WAITEVERY - 1) ptx::tmem_wait_st();
    }
    ptx::tmem_wait_st();
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int X, int NW, int WE>
void run() {
  unsigned long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  const int iters = 2048;
  kb<X, NW, WE><<<148, 512>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double bytes = (double)iters * NW * 32 * X * 4;
  printf("32x32b.x%-2d warps %2d wait every %d: %s  %.1f B/clk per SM, %.0f cycles per warp-instruction\n", X, NW,
         WE, cudaGetErrorString(e), bytes / c, c / iters);
}

int main() {
  run<16, 4, 1>();
  run<16, 4, 4>();
  run<16, 8, 4>();
  run<16, 16, 4>();
  run<32, 4, 2>();
  run<32, 8, 2>();
  run<32, 16, 2>();
  return 0;
}
