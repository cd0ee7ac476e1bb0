// Does an L2-resident region stay "hot" for SMs of the other half of the GPU?
// Phase 1: CTAs of group P read region R (bulk copies). Phase 2 (second
// launch): CTAs of group Q re-read R. Compare phase-2 bandwidth for Q = P,
// Q = the other half of the CTAs, and a cold region (HBM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/l2_die_bench tools/l2_die_bench.cu && tools/l2_die_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace spca;

constexpr int PIECE = 16384, ST = 8;

// active CTAs: blockIdx in [lo, hi); each reads its share of `bytes` at src
__global__ void __launch_bounds__(64, 1) rd(const char *src, size_t bytes, int lo, int hi,
                                             unsigned long long *t, unsigned *smid_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[ST];
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0 && smid_out) smid_out[blockIdx.x] = smid;
  if ((int)blockIdx.x < lo || (int)blockIdx.x >= hi || threadIdx.x != 0) return;
  for (int i = 0; i < ST; ++i) ptx::mbar_init(&full[i], 1);
  ptx::fence_mbar_init();
  const int nact = hi - lo, me = blockIdx.x - lo;
  const size_t pieces = bytes / PIECE;
  const int iters = (int)(pieces / nact);
  uint64_t g0 = ptx::globaltimer();
  for (int k = 0; k < iters + ST; ++k) {
    const int s = k % ST;
    if (k >= ST) ptx::mbar_wait(&full[s], ((k / ST) - 1) & 1);
    if (k >= iters) continue;
    ptx::mbar_arrive_expect_tx(&full[s], PIECE);
    const size_t p = (size_t)k * nact + me;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ptx::smem_u32(smem + s * PIECE)),
                 "l"(src + p * PIECE), "r"(PIECE), "r"(ptx::smem_u32(&full[s]))
                 : "memory");
  }
  atomicMax(t, ptx::globaltimer() - g0);
}

int main() {
  const size_t region = 40ull << 20;
  char *buf;
  cudaMalloc(&buf, 8 * region);
  cudaMemset(buf, 1, 8 * region);
  unsigned long long *t, h;
  unsigned *smid, hs[148];
  cudaMalloc(&t, 8);
  cudaMalloc(&smid, 148 * 4);
  cudaFuncSetAttribute(rd, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * PIECE);
  auto run = [&](const char *src, int lo, int hi) {
    cudaMemset(t, 0, 8);
    rd<<<148, 64, ST * PIECE>>>(src, region, lo, hi, t, smid);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    return region / (h * 1e-9) / 1e9;  // GB/s of the phase
  };
  // flush L2 with a big read
  auto flush = [&]() { run(buf + 3 * region, 0, 148); run(buf + 2 * region, 0, 148); };
  flush();
  double cold = run(buf, 0, 74);
  double warm_same = run(buf, 0, 74);
  flush();
  run(buf, 0, 74);
  double warm_other = run(buf, 74, 148);
  flush();
  run(buf, 0, 148);
  double warm_all = run(buf, 0, 148);
  // capacity: warm region 0, stream k more 40 MB regions, re-read region 0
  for (int k = 0; k <= 3; ++k) {
    flush();
    run(buf, 0, 148);
    for (int j = 1; j <= k; ++j) run(buf + (3 + j) * region, 0, 148);
    printf("re-read after %3d MB of other traffic: %.0f GB/s\n", 40 * k, run(buf, 0, 148));
  }
  cudaMemcpy(hs, smid, 148 * 4, cudaMemcpyDeviceToHost);
  printf("40 MB region re-read by 74 CTAs: cold %.0f GB/s, warmed by the same CTAs %.0f GB/s, warmed by the other "
         "74 CTAs %.0f GB/s; all 148 after all 148 %.0f GB/s\n", cold, warm_same, warm_other, warm_all);
  printf("smid of blockIdx 0..147:");
  for (int i = 0; i < 148; ++i) printf(" %u", hs[i]);
  printf("\n");
  return 0;
}
