// Minimal CTA-pair pipeline: a B producer streams the B operand with pair TMA
// loads (cta_group::2, completion on the leader's barrier) through an NB-deep
// ring; the leader's MMA warp consumes it (8 stacked MMAs per K block, A static
// in TMEM). Cycles per K block of the MMA warp -> is the B path the limiter?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_07669_b200/csrc \
//        -o tools/pipe_bench tools/pipe_bench.cu && tools/pipe_bench
#include <cuda.h>
#include <cstdio>
#include <cuda_runtime.h>

#include "sketch_tc.cuh"

using namespace spca;

constexpr int NB = 7;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
pipe(const __grid_constant__ CUtensorMap tW, const __grid_constant__ CUtensorMap tA, int nkb, int n,
     unsigned long long *out) {
  using C = TcCfg<64>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ uint64_t b_full[NB], b_empty[NB], done, kb_full[8], kb_empty[8], acc_full[2], acc_empty[2];
  __shared__ uint64_t a_full[6], a_empty[6];
  const uint32_t rank = ptx::cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) {
      ptx::mbar_init(&b_full[i], 1);
      ptx::mbar_init(&b_empty[i], 1);
    }
    ptx::mbar_init(&done, 1);
    for (int i = 0; i < C::NS; ++i) {
      ptx::mbar_init(&kb_full[i], 8);
      ptx::mbar_init(&kb_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_empty[i], 8);
    }
    for (int i = 0; i < 6; ++i) {
      ptx::mbar_init(&a_full[i], 1);
      ptx::mbar_init(&a_empty[i], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc2(&tbase, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  uint8_t *aring = smem + NB * C::B_STAGE + 16384;  // 6 x 16 KB A landing ring
  if (MODE >= 5 && warp == 0) {  // A producer: 128 rows x 32 k tiles from a large matrix (HBM)
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % 6;
      if (kb >= 6) ptx::mbar_wait(&a_empty[s], ((kb / 6) - 1) & 1);
      if (ptx::elect_one()) {
        ptx::mbar_arrive_expect_tx(&a_full[s], 16384);
        const int tile = MODE >= 7 ? (blockIdx.x % 8) : (blockIdx.x + (kb / (n / 32)) * gridDim.x) % 780;
        const int kk = kb % (n / 32);
        ptx::tma_load_2d(aring + s * 16384, &tA, &a_full[s], kk * 32, tile * 128);
      }
      __syncwarp();
    }
  }
  if (warp == 2) {  // B producer (both CTAs)
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % NB;
      if (kb >= NB) ptx::mbar_wait(&b_empty[s], ((kb / NB) - 1) & 1);
      if (ptx::elect_one()) {
        uint8_t *st = smem + s * C::B_STAGE;
        const uint32_t bar = ptx::mapa(ptx::smem_u32(&b_full[s]), 0);
        const int k = ((kb + blockIdx.x * 7) % (n / 32)) * 32;
        if (MODE != 1) {
          if (rank == 0) ptx::mbar_arrive_expect_tx(&b_full[s], 2 * C::B_STAGE);
          ptx::tma_load_2d_pair(st, &tW, bar, k, 0, 0);
          ptx::tma_load_2d_pair(st + C::BH_BYTES, &tW, bar, k, 32, 0);
          if (C::STACKED) ptx::tma_load_2d_pair(st + 2 * C::BH_BYTES, &tW, bar, k, 32 * (int)rank, 0);
        } else {
          if (rank == 0) ptx::mbar_arrive(&b_full[s]);
        }
      }
      __syncwarp();
    }
  } else if (MODE >= 3 && warp >= 12) {  // promoters: fold each period of the accumulator
    const int t = (threadIdx.x - 384) & 127;
    const uint32_t lane_base = tmem + ((uint32_t)(t & ~31) << 16);
    const uint32_t accempty_l = ptx::mapa(ptx::smem_u32(&acc_empty[0]), 0);
    float racc[64];
    for (int i = 0; i < 64; ++i) racc[i] = 0.f;
    for (int q = 0; q < nkb / 4; ++q) {
      const int buf = q & 1;
      ptx::mbar_wait(&acc_full[buf], (q >> 1) & 1);
      ptx::tc_fence_after();
      for (int c = 0; c < 64; c += 8) {
        float v8[8], w8[8];
        ptx::tmem_ld8(lane_base + buf * C::ACC_COLS + c, v8);
        if (C::STACKED) ptx::tmem_ld8(lane_base + buf * C::ACC_COLS + 64 + c, w8);
        else for (int i = 0; i < 8; ++i) w8[i] = 0.f;
        for (int i = 0; i < 8; ++i) racc[c + i] += v8[i] + w8[i];
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(accempty_l + 8 * buf);
    }
    if (racc[5] == 1234.f) out[7] = 1;
  } else if (MODE >= 2 && warp >= 4 && warp < 12) {  // converters: TMEM A stages with the handshakes
    const int ct = threadIdx.x - 128, t = ct & 127, grp = ct >> 7;
    const uint32_t lane_base = tmem + ((uint32_t)(t & ~31) << 16);
    const uint32_t kbfull_l = ptx::mapa(ptx::smem_u32(&kb_full[0]), 0);
    float v[32], hi[32];
    for (int i = 0; i < 32; ++i) { v[i] = 0.25f * i; hi[i] = 1.f; }
    const uint32_t arow = ptx::smem_u32(smem + NB * C::B_STAGE + t * 128);  // static A landing tile (16 KB)
    for (int kb = grp; kb < nkb; kb += 2) {
      const int ts = kb % C::NS;
      const int as = kb % 6;
      if (MODE >= 5) ptx::mbar_wait(&a_full[as], (kb / 6) & 1);
      const uint32_t srcrow = MODE >= 5 ? ptx::smem_u32(aring + as * 16384 + t * 128) : arow;
      if (MODE == 6) {  // H-style converter loads: column t, 32 x LDS.32 (A from HBM)
        const uint32_t raw = ptx::smem_u32(aring + as * 16384 + t * 4);
#pragma unroll
        for (int kq = 0; kq < 32; ++kq) v[kq] = ptx::lds32(raw + kq * 512);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          hi[i] = trunc_tf32(v[i]);
          v[i] -= hi[i];
        }
      } else if (MODE >= 4 && MODE != 8) {  // converter work: 8 x LDS.128 + split, like the pass kernel
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 x = ptx::lds128(srcrow + ((q4 ^ (t & 7)) << 4));
          v[4 * q4] = x.x; v[4 * q4 + 1] = x.y; v[4 * q4 + 2] = x.z; v[4 * q4 + 3] = x.w;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          hi[i] = trunc_tf32(v[i]);
          v[i] -= hi[i];
        }
      }
      if (MODE >= 5) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&a_empty[as]);
      }
      if (kb >= C::NS) ptx::mbar_wait(&kb_empty[ts], ((kb / C::NS) - 1) & 1);
      ptx::tc_fence_after();
      ptx::tmem_st32(lane_base + C::A_TMEM + 64 * ts, hi);
      ptx::tmem_st32(lane_base + C::A_TMEM + 64 * ts + 32, v);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(kbfull_l + 8 * ts);
    }
  } else if (warp == 1 && rank == 0) {  // MMA issuer
    const uint64_t bdesc0 = ptx::sdesc_sw128(ptx::smem_u32(smem), 16, 1024);
    long long t0 = clock64();
    for (int kb = 0; kb < nkb; ++kb) {
      const int bs = kb % NB, q = kb >> 2, buf = q & 1;
      unsigned long long *mt = (MODE == 8 && lane == 0) ? out + 16 + 4 * (kb & 1023) : nullptr;
      if (mt) mt[0] = clock64();
      if (mt) mt[1] = clock64();
      if (MODE >= 2) ptx::mbar_wait(&kb_full[kb % C::NS], (kb / C::NS) & 1);
      if (mt) mt[2] = clock64();
      if (MODE >= 3 && (kb & 3) == 0 && q >= 2) ptx::mbar_wait(&acc_empty[buf], ((q >> 1) - 1) & 1);
      ptx::mbar_wait(&b_full[bs], (kb / NB) & 1);
      if (mt) mt[3] = clock64();
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        tc_mma_stage2<64>(tmem + C::A_TMEM + 64 * (MODE == 9 ? 0 : kb % C::NS), tmem + buf * C::ACC_COLS,
                          bdesc0 + (uint64_t)((bs * C::B_STAGE) >> 4), (kb & 3) == 0);
        ptx::mma2_commit_both(&b_empty[bs]);
        if (MODE >= 2) ptx::mma2_commit_both(&kb_empty[kb % C::NS]);
        if (MODE >= 3 && (kb & 3) == 3) ptx::mma2_commit_both(&acc_full[buf]);
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma2_commit_both(&done);
    __syncwarp();
    ptx::mbar_wait(&done, 0);
    long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[MODE] = (t1 - t0) / nkb;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 1) ptx::tmem_dealloc2(tmem, 512);
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void fill_rand(float *p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)(i * 2654435761u) ^ (uint32_t)(i >> 32) ^ 0x9e3779b9u;
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    p[i] = ((float)(x & 0xffffff) / 16777216.f - 0.5f) * 3.4f;
  }
}

int main(int argc, char **argv) {
  const bool rnd = argc > 1;
  const int n = 10000;
  float *w;
  cudaMalloc(&w, (size_t)64 * n * 4);
  cudaMemset(w, 0, (size_t)64 * n * 4);
  if (rnd) fill_rand<<<1184, 256>>>(w, (size_t)64 * n);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)n, 64};
  cuuint64_t strides[1] = {(cuuint64_t)n * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  float *abuf;
  cudaMalloc(&abuf, (size_t)100000 * n * 4);
  cudaMemset(abuf, 0, (size_t)100000 * n * 4);
  if (rnd) fill_rand<<<1184, 256>>>(abuf, (size_t)100000 * n);
  CUtensorMap amap;
  cuuint64_t adims[2] = {(cuuint64_t)n, 100000};
  cuuint32_t abox[2] = {32, 128};
  ((EncodeFn)fn)(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, abuf, adims, strides, abox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long *d, h[10] = {0};
  cudaMalloc(&d, (16 + 4 * 1024) * 8);
  const int smem = NB * TcCfg<64>::B_STAGE + 16384 + 6 * 16384 + 1024;
  cudaFuncSetAttribute(pipe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pipe<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pipe<0><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<1><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<2><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<3><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<4><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<5><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<6><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<7><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<8><<<148, 512, smem>>>(map, amap, 4096, n, d);
  pipe<9><<<148, 512, smem>>>(map, amap, 4096, n, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
  printf("%s data %s: MMA cycles per K block: with pair-TMA B stream %llu, without B loads %llu, B stream + converter"
         " TMEM stages %llu, + promoters %llu, + converter loads/split %llu, + A TMA ring from HBM %llu,"
         " H-style column loads %llu, A TMA ring from L2 %llu, + per-block clock/STG trace %llu,"
         " MMA reads a fixed A stage %llu (ideal 384)\n",
         cudaGetErrorString(e), rnd ? "random" : "zero", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
  return 0;
}
