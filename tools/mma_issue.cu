// MMA issue-overhead microbenchmark: a looped (not unrolled) issuer of 8
// tf32 N=128 MMAs per K block, like the sketch kernels, in several forms.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/mma_issue tools/mma_issue.cu && tools/mma_issue
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

constexpr int NKB = 512;  // K blocks (8 MMAs each)

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// 8 MMAs of one K block: A hi/lo from TMEM stage ts, B from smem stage bs
__device__ __forceinline__ void kblock(uint32_t tmem, uint32_t acc, uint32_t sb, int ts, int bs, bool first) {
  const uint32_t a_hi = tmem + 256 + 64 * ts, a_lo = a_hi + 32;
  const uint32_t w = sb + bs * 16384;
  constexpr uint32_t idesc = ptx::idesc_tf32(128, 128, 0, 0);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t dw = ptx::sdesc_sw128(w + kk * 32, 16, 1024);
    ptx::mma_tf32_ts(acc, a_hi + kk * 8, dw, idesc, (first && kk == 0) ? 0u : 1u);
    ptx::mma_tf32_ts(acc, a_lo + kk * 8, dw, idesc, 1u);
  }
}

// V: 0 thread-0 loop, commits only
//    1 warp-wide loop, one elect per K block
//    2 thread-0 loop, waits for the commit of K block kb-4 (ring of 4)
//    3 warp-wide loop, all lanes wait for kb-4, one elect per K block
//    4 warp-wide, waits kb-4, 2 accumulators alternating per 4 K blocks
template <int V>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar_done, ring[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 1.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_done, 1);
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&ring[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sb = ptx::smem_u32(smem);
  long long t0 = 0, t1 = 0;
  if (V == 0 || V == 2) {
    if (threadIdx.x == 0) {
      t0 = clock64();
#pragma unroll 1
      for (int kb = 0; kb < NKB; ++kb) {
        if (V == 2 && kb >= 4) ptx::mbar_wait(&ring[kb & 3], ((kb >> 2) - 1) & 1);
        ptx::tc_fence_after();
        kblock(tmem, tmem, sb, kb & 3, kb & 3, kb == 0);
        ptx::mma_commit(&ring[kb & 3]);
      }
      ptx::mma_commit(&bar_done);
      ptx::mbar_wait(&bar_done, 0);
      t1 = clock64();
    }
  } else if (warp == 0) {
    t0 = clock64();
#pragma unroll 1
    for (int kb = 0; kb < NKB; ++kb) {
      if (V >= 3 && kb >= 4) ptx::mbar_wait(&ring[kb & 3], ((kb >> 2) - 1) & 1);
      ptx::tc_fence_after();
      const uint32_t acc = V == 4 ? tmem + ((kb >> 2) & 1) * 128 : tmem;
      if (elect_one()) {
        kblock(tmem, acc, sb, kb & 3, kb & 3, V == 4 ? (kb & 3) == 0 : kb == 0);
        ptx::mma_commit(&ring[kb & 3]);
      }
      __syncwarp();
    }
    if (elect_one()) ptx::mma_commit(&bar_done);
    ptx::mbar_wait(&bar_done, 0);
    t1 = clock64();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int V>
void run(const char *name, unsigned long long *d, unsigned long long *h) {
  cudaFuncSetAttribute(bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  bench<V><<<148, 128, 70 * 1024>>>(d);
  bench<V><<<148, 128, 70 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-48s %s  %.1f cycles / MMA\n", name, cudaGetErrorString(e), s / 148 / (NKB * 8));
}

int main() {
  unsigned long long *d, h[148];
  cudaMalloc(&d, 148 * 8);
  run<0>("thread-0 loop, commits only", d, h);
  run<1>("warp loop + elect, commits only", d, h);
  run<2>("thread-0 loop, wait kb-4", d, h);
  run<3>("warp loop + elect, wait kb-4", d, h);
  run<4>("warp loop + elect, wait kb-4, 2 acc", d, h);
  return 0;
}
