// MMA issue-rate microbenchmark for tcgen05 kind::tf32 / kind::f16 on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/mma_bench tools/mma_bench.cu && tools/mma_bench
// One CTA per SM; one thread issues ITER MMAs into TMEM, commits, waits; the
// kernel reports cycles per MMA (clock64) for several shapes / operand forms.
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

constexpr int ITER = 2048;

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}

// BG: background load on warps 4..11 while warp 0 issues MMAs
//   0 none, 1 tcgen05.st into spare TMEM columns, 2 ld.shared of the B operand region,
//   3 tcgen05.ld of the accumulator columns, 4 ld.shared of a disjoint region,
//   5 = 1 + 4 (a converter-like mix)
__device__ __forceinline__ void mbar_wait_test(uint64_t *bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(a), "r"(parity)
                 : "memory");
  }
}

template <int VARIANT, int BG = 0>
__global__ void __launch_bounds__(384, 1) bench(unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  __shared__ uint64_t bars2[3];
  (void)0;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((float *)smem)[i] = 1.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    for (int i = 0; i < 3; ++i) ptx::mbar_init(&bars2[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp < 4) {
    float one[16];
    for (int i = 0; i < 16; ++i) one[i] = 1.f;
    for (int c = 256; c < 448; c += 16) ptx::tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + c, one);
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp >= 4 && BG != 0) {
    const uint32_t sb = ptx::smem_u32(smem);
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = (float)i;
    float acc = 0.f;
    int it = 0;
    while (!done) {
      if (BG == 1 || BG == 5) {
        ptx::tmem_st16(tmem + lane_off + 448 + ((warp >> 2) & 1) * 32 + (it & 1) * 16, v);
        ptx::tmem_wait_st();
      }
      if (BG == 2 || BG == 4 || BG == 5) {
        const uint32_t base = sb + (BG == 2 ? 0u : 65536u);
        for (int j = 0; j < 4; ++j) {
          float4 x = ptx::lds128(base + ((threadIdx.x * 16 + j * 6144 + it * 512) & 32767));
          acc += x.x + x.y + x.z + x.w;
        }
      }
      if (BG == 6) {  // spin on an mbarrier that never completes
        ptx::mbar_try_wait(ptx::smem_u32(&bars2[2]), 0);
      }
      if (BG == 7) {  // same, one lane per warp
        if ((threadIdx.x & 31) == 0) ptx::mbar_try_wait(ptx::smem_u32(&bars2[2]), 0);
        __syncwarp();
      }
      if (BG == 3) {
        ptx::tmem_ld16(tmem + lane_off + (it & 7) * 16, v);
        acc += v[0];
      }
      ++it;
    }
    if (acc == 12345.f) out[0] = 0;
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) atomicAdd(&out[300], (unsigned long long)it);
  }
  if (threadIdx.x == 0) {
    const uint32_t sb = ptx::smem_u32(smem);
    long long t0 = clock64();
    const uint64_t g0 = ptx::globaltimer();
    for (int i = 0; i < ITER; ++i) {
      const uint32_t kk = i & 3;
      if (VARIANT == 0) {  // TS tf32 N=128, one accumulator
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
      } else if (VARIANT == 1) {  // TS tf32 N=128, two accumulators alternating
        ptx::mma_tf32_ts(tmem + (i & 1) * 128, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 1);
      } else if (VARIANT == 2) {  // SS tf32 N=128
        ptx::mma_tf32(tmem, ptx::sdesc_sw128(sb + 32768 + kk * 32, 16, 1024),
                      ptx::sdesc_sw128(sb + kk * 32, 16, 1024), ptx::idesc_tf32(128, 128, 0, 0), i > 0);
      } else if (VARIANT == 3) {  // TS tf32 N=64
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 64, 0, 0), i > 0);
      } else if (VARIANT == 4) {  // TS tf32 N=256
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 256, 0, 0), i > 0);
      } else if (VARIANT == 5) {  // SS tf32 N=256
        ptx::mma_tf32(tmem, ptx::sdesc_sw128(sb + 65536 + kk * 32, 16, 1024),
                      ptx::sdesc_sw128(sb + kk * 32, 16, 1024), ptx::idesc_tf32(128, 256, 0, 0), i > 0);
      } else if (VARIANT == 6) {  // TS bf16 N=128 (kind::f16, K=16)
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        mma_f16_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024), idesc, i > 0);
      } else if (VARIANT == 8 || VARIANT == 9) {  // N128 + commits every 8 MMAs (like the kernel)
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
        if ((i & 7) == 7) {
          ptx::mma_commit(&bars2[0]);
          ptx::mma_commit(&bars2[1]);
          if (VARIANT == 9) ptx::mma_commit(&bars2[2]);
        }
      } else if (VARIANT == 10) {  // N128, wait for each 8-MMA group to complete (no overlap)
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
        if ((i & 7) == 7) {
          ptx::mma_commit(&bars2[0]);
          ptx::mbar_wait(&bars2[0], (i >> 3) & 1);
        }
      } else if (VARIANT >= 11 && VARIANT <= 15) {  // groups of 1,2,4,16,32 waited for
        constexpr int G = VARIANT == 11 ? 1 : VARIANT == 12 ? 2 : VARIANT == 13 ? 4 : VARIANT == 14 ? 16 : 32;
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
        if ((i % G) == G - 1) {
          ptx::mma_commit(&bars2[0]);
          ptx::mbar_wait(&bars2[0], (i / G) & 1);
        }
      } else if (VARIANT == 16) {  // N64 groups of 8 waited
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 64, 0, 0), i > 0);
        if ((i & 7) == 7) {
          ptx::mma_commit(&bars2[0]);
          ptx::mbar_wait(&bars2[0], (i >> 3) & 1);
        }
      } else if (VARIANT == 17 || VARIANT == 19) {  // groups of 32 serialized; 17: alternate acc, 19: fresh acc
        const uint32_t acc = VARIANT == 17 ? ((i >> 5) & 1) * 128 : 0;
        const bool accum = VARIANT == 17 ? (i > 63) : ((i & 31) != 0);
        ptx::mma_tf32_ts(tmem + acc, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), accum);
        if ((i & 31) == 31) {
          ptx::mma_commit(&bars2[0]);
          ptx::mbar_wait(&bars2[0], (i >> 5) & 1);
        }
      } else if (VARIANT == 18) {  // groups of 32, one group in flight (wait for g-1 after issuing g)
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
        if ((i & 31) == 31) {
          const int g = i >> 5;
          ptx::mma_commit(&bars2[g & 1]);
          if (g >= 1) ptx::mbar_wait(&bars2[(g - 1) & 1], ((g - 1) >> 1) & 1);
        }
      } else if (VARIANT == 20) {  // groups of 32, 1 in flight, test_wait polling
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
        if ((i & 31) == 31) {
          const int g = i >> 5;
          ptx::mma_commit(&bars2[g & 1]);
          if (g >= 1) mbar_wait_test(&bars2[(g - 1) & 1], ((g - 1) >> 1) & 1);
        }
      } else if (VARIANT == 21) {  // groups of 32 serialized, test_wait polling
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
        if ((i & 31) == 31) {
          ptx::mma_commit(&bars2[0]);
          mbar_wait_test(&bars2[0], (i >> 5) & 1);
        }
      } else if (VARIANT == 22) {  // groups of 32 serialized, waited by lane 1 of the warp? no: by warp 1 via flag
        ptx::mma_tf32_ts(tmem, tmem + 256 + kk * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 0);
        if ((i & 31) == 31) {
          ptx::mma_commit(&bars2[0]);
          ptx::mbar_wait(&bars2[0], (i >> 5) & 1);
          __nanosleep(0);
        }
      } else if (VARIANT == 7) {  // TS tf32 N=128, four accumulators round robin
        ptx::mma_tf32_ts(tmem + (i & 1) * 128, tmem + 256 + (i & 7) * 8, ptx::sdesc_sw128(sb + kk * 32, 16, 1024),
                         ptx::idesc_tf32(128, 128, 0, 0), i > 1);
      }
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    const uint64_t g1 = ptx::globaltimer();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
    out[148 + blockIdx.x] = g1 - g0;
    done = 1;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp < 4) {
    float v[16];
    ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
    if (threadIdx.x == 5 && blockIdx.x == 3) out[296] = (unsigned long long)v[7];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int V, int BG = 0>
void run(const char *name, unsigned long long *d, unsigned long long *h) {
  cudaFuncSetAttribute(bench<V, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  bench<V, BG><<<148, 384, 100 * 1024>>>(d);
  bench<V, BG><<<148, 384, 100 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  cudaMemcpy(h, d, 301 * 8, cudaMemcpyDeviceToHost);
  if (BG) printf("   bg warp-iterations (CTA 0): %llu  -> %.1f B/clk of lds (if lds mode)\n", h[300],
                 (double)h[300] * 32 * 64 / (s / 148));
  cudaMemset(d + 300, 0, 8);
  double ns = 0;
  for (int i = 148; i < 296; ++i) ns += h[i];
  printf("%-34s %s  %.1f cycles / MMA  %.2f ns / MMA  (%.0f MHz)  acc=%llu\n", name, cudaGetErrorString(e),
         s / 148 / ITER, ns / 148 / ITER, s / ns * 1000, h[296]);
}

int main() {
  unsigned long long *d, h[301];
  cudaMalloc(&d, 301 * 8);
  cudaMemset(d, 0, 301 * 8);
  run<0>("TS tf32 M128 N128 1 acc", d, h);
  run<1>("TS tf32 M128 N128 2 acc", d, h);
  run<2>("SS tf32 M128 N128", d, h);
  run<3>("TS tf32 M128 N64", d, h);
  run<4>("TS tf32 M128 N256", d, h);
  run<5>("SS tf32 M128 N256", d, h);
  run<6>("TS bf16 M128 N128 K16", d, h);
  run<7>("TS tf32 N128 2 acc, 8 A slices", d, h);
  run<8>("TS N128 + 2 commits / 8 MMA", d, h);
  run<9>("TS N128 + 3 commits / 8 MMA", d, h);
  run<10>("TS N128 serialized groups of 8", d, h);
  run<11>("TS N128 serialized groups of 1", d, h);
  run<12>("TS N128 serialized groups of 2", d, h);
  run<13>("TS N128 serialized groups of 4", d, h);
  run<14>("TS N128 serialized groups of 16", d, h);
  run<15>("TS N128 serialized groups of 32", d, h);
  run<16>("TS N64 serialized groups of 8", d, h);
  run<17>("groups of 32 serialized, alt acc", d, h);
  run<19>("groups of 32 serialized, fresh acc", d, h);
  run<18>("groups of 32, 1 group in flight", d, h);
  run<20>("groups of 32, 1 in flight, test_wait", d, h);
  run<21>("groups of 32 serialized, test_wait", d, h);
  run<0, 6>("TS N128 + bg try_wait spin (all lanes)", d, h);
  run<0, 7>("TS N128 + bg try_wait spin (lane 0)", d, h);
  run<0, 1>("TS N128 + bg tcgen05.st", d, h);
  run<0, 2>("TS N128 + bg lds on B region", d, h);
  run<0, 3>("TS N128 + bg tcgen05.ld acc", d, h);
  run<0, 4>("TS N128 + bg lds disjoint", d, h);
  run<0, 5>("TS N128 + bg st + lds", d, h);
  run<2, 4>("SS N128 + bg lds disjoint", d, h);
  run<2, 5>("SS N128 + bg st + lds", d, h);
  run<4, 5>("TS N256 + bg st + lds", d, h);
  return 0;
}
