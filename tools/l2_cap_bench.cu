// How much of a streamed region survives in L2 for a re-read, as a function of
// the region size W and of which SMs re-read it: phase 1 — all 148 CTAs read
// W (16 KB pieces, piece p by CTA p % 148, bulk copies); phase 2 — re-read W
// with the piece -> CTA assignment shifted by `shift` CTAs (shift 0: every
// piece re-read by the SM that loaded it). Reports the phase-2 rate; an L2 that
// keeps a copy of far-die lines next to the requesting SMs would hold less for
// shifted re-reads. Also phase 1 with the evict_last policy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/l2_cap_bench tools/l2_cap_bench.cu && tools/l2_cap_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

constexpr int PIECE = 16384, ST = 8;

__global__ void __launch_bounds__(32, 1) rd(const char *src, size_t bytes, int shift, int hint,
                                             unsigned long long *t) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[ST];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < ST; ++i) ptx::mbar_init(&full[i], 1);
  ptx::fence_mbar_init();
  const int nct = gridDim.x, me = (blockIdx.x + shift) % nct;
  const size_t pieces = bytes / PIECE;
  const size_t iters = (pieces + nct - 1) / nct;
  const uint64_t pol = hint == 1 ? ptx::policy_evict_last() : (hint == 2 ? ptx::policy_evict_first()
                                                                         : ptx::policy_evict_normal());
  uint64_t g0 = ptx::globaltimer();
  size_t issued = 0;
  for (size_t k = 0; k < iters + ST; ++k) {
    const int s = k % ST;
    if (k >= ST && (k - ST) < issued) ptx::mbar_wait(&full[s], ((k / ST) - 1) & 1);
    if (k >= iters) continue;
    const size_t p = k * nct + me;
    if (p >= pieces) continue;
    ptx::mbar_arrive_expect_tx(&full[s], PIECE);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            ptx::smem_u32(smem + s * PIECE)),
        "l"(src + p * PIECE), "r"(PIECE), "r"(ptx::smem_u32(&full[s])), "l"(pol)
        : "memory");
    issued = k + 1;
  }
  atomicMax(t, ptx::globaltimer() - g0);
}

int main() {
  const size_t maxw = 160ull << 20, flushb = 1024ull << 20;
  char *buf, *fl;
  cudaMalloc(&buf, maxw);
  cudaMalloc(&fl, flushb);
  cudaMemset(buf, 1, maxw);
  cudaMemset(fl, 2, flushb);
  unsigned long long *t, h;
  cudaMalloc(&t, 8);
  cudaFuncSetAttribute(rd, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * PIECE);
  auto run = [&](const char *src, size_t bytes, int shift, int hint) {
    cudaMemset(t, 0, 8);
    rd<<<148, 32, ST * PIECE>>>(src, bytes, shift, hint, t);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    return bytes / (h * 1e-9) / 1e9;
  };
  auto flush = [&]() { run(fl, flushb, 0, 0); };
  flush();
  printf("HBM cold read of 160 MB: %.0f GB/s\n", run(buf, maxw, 0, 0));
  const int sizes[] = {16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128};
  const int shifts[] = {0, 1, 37, 74};
  for (int hint = 0; hint < 2; ++hint) {
    printf("phase-1 policy %s\n", hint ? "evict_last" : "evict_normal");
    printf("   W MB |");
    for (int s : shifts) printf(" shift %3d |", s);
    printf("\n");
    for (int w : sizes) {
      const size_t b = (size_t)w << 20;
      printf("  %5d |", w);
      for (int s : shifts) {
        flush();
        run(buf, b, 0, hint);
        printf(" %9.0f |", run(buf, b, s, 0));
      }
      printf("\n");
    }
  }
  return 0;
}
