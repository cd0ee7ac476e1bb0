// sketch_tc.cuh — tcgen05 tensor-core sketch path (sm_100a), fp32 data.
//
// Split precision "3xTF32": every fp32 operand x is split on chip into
// x_hi = rna_tf32(x) and x_lo = rna_tf32(x - x_hi), and each contraction is
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in fp32 in TMEM (the
// dropped lo*lo term and the lo rounding are ~2^-22 relative): FFMA-class
// accuracy at tensor-core rate. Every operand the tensor
// core reads is an exact tf32 value, so the result does not depend on how
// the MMA unit treats the low 13 bits of an fp32 container.
//
// Per canonical chunk of R rows (sized so the chunk stays L2-resident):
//   tc_g_kernel    partial G (128-row tile x l) over a K (= n) split:
//                  TMA A tile {32 k x 128 rows} + Omega^T hi/lo tiles
//                  (K-major, SWIZZLE_128B) -> converter warps split A in
//                  shared memory and flag non-finite rows -> one thread
//                  issues tcgen05.mma kind::tf32 (M=128, N=l_pad, K=8) ->
//                  TMEM -> epilogue warps tcgen05.ld -> fp32 partials.
//   tc_g_finalize  fixed-order sum of the K-split partials -> G (output,
//                  fp32) and G^T hi / lo (K-major operands of the H pass).
//   tc_h_kernel    H tile (128 n x l) over a row split: TMA A tiles
//                  {32 n x 32 rows} (row-major as stored) -> converter
//                  thread t owns column n0+t: splits it, transposes it into
//                  a K-major row of the hi/lo operand tiles and accumulates
//                  the column sum -> tcgen05.mma (M=128 n, N=l_pad, K=8
//                  rows) with G^T hi/lo tiles -> TMEM -> Hpart (+)= fp32.
// The A chunk is read from HBM by tc_g_kernel and re-read by tc_h_kernel
// from L2.
#pragma once

#include <cuda.h>

#include "tc_ptx.cuh"

namespace spca {

constexpr int kTcThreads = 256;  // warp0 TMA, warp1 MMA (+TMEM alloc), warps4-7 convert+epilogue

template <int LPAD>
struct TcCfgG {
  static constexpr int STAGES = LPAD <= 64 ? 4 : (LPAD <= 128 ? 3 : 2);
  static constexpr uint32_t A_BYTES = 128 * 32 * 4;   // 128 rows x 32 k
  static constexpr uint32_t W_BYTES = LPAD * 32 * 4;  // Omega^T tile: l_pad x 32 k
  static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * W_BYTES;
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024;
};

template <int LPAD>
struct TcCfgH {
  static constexpr int STAGES = LPAD <= 64 ? 3 : 2;
  static constexpr uint32_t A_BYTES = 128 * 32 * 4;   // raw: 32 rows x 128 n; hi/lo: 128 n x 32 k
  static constexpr uint32_t W_BYTES = LPAD * 32 * 4;  // G^T tile: l_pad x 32 rows
  static constexpr uint32_t STAGE_BYTES = 3 * A_BYTES + 2 * W_BYTES;
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024;
};

__device__ __forceinline__ float4 tf32x4(float4 v) {
  return make_float4(ptx::to_tf32(v.x), ptx::to_tf32(v.y), ptx::to_tf32(v.z), ptx::to_tf32(v.w));
}

// ------------------------------------------------------------- G = A Omega
template <int LPAD>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_g_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tWhi,
            const __grid_constant__ CUtensorMap tWlo, int rows, int n, int kseg,
            float *__restrict__ gpart, int64_t split_stride, int64_t first_row,
            unsigned long long *__restrict__ bad_row, int dbg) {
  using C = TcCfgG<LPAD>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full_bar[STAGES], conv_bar[STAGES], empty_bar[STAGES], tmem_bar;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * 128;
  const int kbeg = blockIdx.y * kseg;
  const int kend = min(n, kbeg + kseg);
  const int nk = (kend - kbeg + 31) / 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&conv_bar[s], 128);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(&tmem_bar, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch(&tA);
    ptx::tma_prefetch(&tWhi);
    ptx::tma_prefetch(&tWlo);
  }
  if (warp == 1) ptx::tmem_alloc(&tmem_base, LPAD);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t it = kb / STAGES;
        if (kb >= STAGES) ptx::mbar_wait(&empty_bar[s], (it - 1) & 1);
        uint8_t *st = smem + s * C::STAGE_BYTES;
        const bool skip_w = (dbg & 4) && kb >= STAGES;  // debug: reuse Omega tiles
        ptx::mbar_arrive_expect_tx(&full_bar[s], C::A_BYTES + (skip_w ? 0 : 2 * C::W_BYTES));
        const int k = kbeg + kb * 32;
        ptx::tma_load_2d(st, &tA, &full_bar[s], k, row0);
        if (!skip_w) {
          ptx::tma_load_2d(st + 2 * C::A_BYTES, &tWhi, &full_bar[s], k, 0);
          ptx::tma_load_2d(st + 2 * C::A_BYTES + C::W_BYTES, &tWlo, &full_bar[s], k, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_tf32(128, LPAD, 0, 0);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t it = kb / STAGES;
        ptx::mbar_wait(&conv_bar[s], it & 1);
        ptx::tc_fence_after();
        const uint32_t base = ptx::smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t a_hi = base, a_lo = base + C::A_BYTES;
        const uint32_t w_hi = base + 2 * C::A_BYTES, w_lo = w_hi + C::W_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (dbg & 2) break;  // debug: no MMA
          const uint32_t off = kk * 32;  // 8 tf32 along K inside the 128-byte swizzled row
          const uint64_t dah = ptx::sdesc_sw128(a_hi + off, 16, 1024);
          const uint64_t dal = ptx::sdesc_sw128(a_lo + off, 16, 1024);
          const uint64_t dwh = ptx::sdesc_sw128(w_hi + off, 16, 1024);
          const uint64_t dwl = ptx::sdesc_sw128(w_lo + off, 16, 1024);
          ptx::mma_tf32(tmem, dah, dwh, idesc, (kb | kk) ? 1u : 0u);
          ptx::mma_tf32(tmem, dah, dwl, idesc, 1u);
          ptx::mma_tf32(tmem, dal, dwh, idesc, 1u);
        }
        ptx::mma_commit(&empty_bar[s]);
      }
      ptx::mma_commit(&tmem_bar);
    }
  } else if (warp >= 4) {
    const int t = threadIdx.x - 128;
    int bad = INT32_MAX;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t it = kb / STAGES;
      ptx::mbar_wait(&full_bar[s], it & 1);
      float4 *a4 = reinterpret_cast<float4 *>(smem + s * C::STAGE_BYTES);
      float4 *l4 = reinterpret_cast<float4 *>(smem + s * C::STAGE_BYTES + C::A_BYTES);
#pragma unroll
      for (int i = 0; i < (int)(C::A_BYTES / 16 / 128); ++i) {
        if (dbg & 1) break;  // debug: no conversion
        const int idx = t + i * 128;
        const float4 v = a4[idx];
        const float4 hi = tf32x4(v);
        a4[idx] = hi;
        l4[idx] = tf32x4(make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w));
        if (!(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w)))
          bad = min(bad, idx >> 3);  // 8 float4 per 128-byte row
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&conv_bar[s]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (lane == 0 && bad != INT32_MAX && row0 + bad < rows)
      report_bad_row(bad_row, first_row + row0 + bad);

    // epilogue: TMEM lanes = rows of the tile, columns = sketch columns
    ptx::mbar_wait(&tmem_bar, 0);
    ptx::tc_fence_after();
    const int q = warp - 4;
    const int r = row0 + q * 32 + lane;
    float *out = gpart + (int64_t)blockIdx.y * split_stride + (int64_t)r * LPAD;
#pragma unroll 1
    for (int c = 0; c < LPAD; c += 16) {
      float v[16];
      ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
      if (r < rows) {
        float4 *o4 = reinterpret_cast<float4 *>(out + c);
        o4[0] = make_float4(v[0], v[1], v[2], v[3]);
        o4[1] = make_float4(v[4], v[5], v[6], v[7]);
        o4[2] = make_float4(v[8], v[9], v[10], v[11]);
        o4[3] = make_float4(v[12], v[13], v[14], v[15]);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, LPAD);
  }
}

// G = sum_z partial_z (fixed order) -> G (rows x LPAD, output) and the split
// transposed operands G^T hi / lo (LPAD x ldt).
__global__ void tc_g_finalize(const float *__restrict__ gpart, int ksplit, int64_t split_stride,
                              int rows, int lpad, int ldt, float *__restrict__ g_out,
                              float *__restrict__ ghiT, float *__restrict__ gloT) {
  __shared__ float tile[8][33];
  // block: 8 rows x 32 columns, 32 x 8 threads; one output element per thread
  const int r0 = blockIdx.x * 8, c0 = blockIdx.y * 32;
  {
    const int r = r0 + threadIdx.y, c = c0 + threadIdx.x;
    float s = 0.f;
    if (r < rows) {
      const int64_t idx = (int64_t)r * lpad + c;
      s = gpart[idx];
      for (int z = 1; z < ksplit; ++z) s += gpart[(int64_t)z * split_stride + idx];
      g_out[idx] = s;
    }
    tile[threadIdx.y][threadIdx.x] = s;
  }
  __syncthreads();
  {
    const int t = threadIdx.y * 32 + threadIdx.x;
    const int c = c0 + (t >> 3), r = r0 + (t & 7);
    if (r < rows) {
      const float s = tile[t & 7][t >> 3];
      const float h = ptx::to_tf32(s);
      ghiT[(int64_t)c * ldt + r] = h;
      gloT[(int64_t)c * ldt + r] = ptx::to_tf32(s - h);
    }
  }
}

// ------------------------------------------------------------ H += A^T G
template <int LPAD>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_h_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tGhi,
            const __grid_constant__ CUtensorMap tGlo, int rows, int n, int rseg,
            float *__restrict__ hpart, int64_t h_split_stride, double *__restrict__ cspart,
            int accumulate, int kahan) {
  using C = TcCfgH<LPAD>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full_bar[STAGES], conv_bar[STAGES], empty_bar[STAGES], tmem_bar;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int rb = blockIdx.y * rseg;
  const int re = min(rows, rb + rseg);
  const int nk = (re - rb + 31) / 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&conv_bar[s], 128);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(&tmem_bar, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch(&tA);
    ptx::tma_prefetch(&tGhi);
    ptx::tma_prefetch(&tGlo);
  }
  if (warp == 1) ptx::tmem_alloc(&tmem_base, LPAD);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base;

  // stage layout: [raw A 16K][A_hi (K-major) 16K][A_lo 16K][G^T hi][G^T lo]
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t it = kb / STAGES;
        if (kb >= STAGES) ptx::mbar_wait(&empty_bar[s], (it - 1) & 1);
        uint8_t *st = smem + s * C::STAGE_BYTES;
        ptx::mbar_arrive_expect_tx(&full_bar[s], C::A_BYTES + 2 * C::W_BYTES);
        const int r = rb + kb * 32;
#pragma unroll
        for (int j = 0; j < 4; ++j) ptx::tma_load_2d(st + j * 4096, &tA, &full_bar[s], n0 + 32 * j, r);
        ptx::tma_load_2d(st + 3 * C::A_BYTES, &tGhi, &full_bar[s], r, 0);
        ptx::tma_load_2d(st + 3 * C::A_BYTES + C::W_BYTES, &tGlo, &full_bar[s], r, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_tf32(128, LPAD, 0, 0);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t it = kb / STAGES;
        ptx::mbar_wait(&conv_bar[s], it & 1);
        ptx::tc_fence_after();
        const uint32_t base = ptx::smem_u32(smem + s * C::STAGE_BYTES);
        const uint32_t a_hi = base + C::A_BYTES, a_lo = base + 2 * C::A_BYTES;
        const uint32_t g_hi = base + 3 * C::A_BYTES, g_lo = g_hi + C::W_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t off = kk * 32;
          const uint64_t dah = ptx::sdesc_sw128(a_hi + off, 16, 1024);
          const uint64_t dal = ptx::sdesc_sw128(a_lo + off, 16, 1024);
          const uint64_t dgh = ptx::sdesc_sw128(g_hi + off, 16, 1024);
          const uint64_t dgl = ptx::sdesc_sw128(g_lo + off, 16, 1024);
          ptx::mma_tf32(tmem, dah, dgh, idesc, (kb | kk) ? 1u : 0u);
          ptx::mma_tf32(tmem, dah, dgl, idesc, 1u);
          ptx::mma_tf32(tmem, dal, dgh, idesc, 1u);
        }
        ptx::mma_commit(&empty_bar[s]);
      }
      ptx::mma_commit(&tmem_bar);
    }
  } else if (warp >= 4) {
    // converter thread t owns column n0 + t of the tile: raw atom j = t/32, nn = t%32
    const int t = threadIdx.x - 128;
    const int j = t >> 5, nn = t & 31;
    double cs = 0.0, cc = 0.0;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t it = kb / STAGES;
      ptx::mbar_wait(&full_bar[s], it & 1);
      const float *raw = reinterpret_cast<const float *>(smem + s * C::STAGE_BYTES + j * 4096);
      float4 *hi_row = reinterpret_cast<float4 *>(smem + s * C::STAGE_BYTES + C::A_BYTES + t * 128);
      float4 *lo_row = reinterpret_cast<float4 *>(smem + s * C::STAGE_BYTES + 2 * C::A_BYTES + t * 128);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int k = 4 * c + e;  // row of A within this K block
          v[e] = raw[k * 32 + (((nn >> 2) ^ (k & 7)) << 2) + (nn & 3)];
          if (kahan) {
            const double y = (double)v[e] - cc;
            const double tt = cs + y;
            cc = (tt - cs) - y;
            cs = tt;
          } else {
            cs += (double)v[e];
          }
        }
        const float4 x = make_float4(v[0], v[1], v[2], v[3]);
        const float4 h = tf32x4(x);
        const int pos = c ^ (t & 7);  // SWIZZLE_128B position of K chunk c in row t
        hi_row[pos] = h;
        lo_row[pos] = tf32x4(make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w));
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&conv_bar[s]);
    }
    const int col = n0 + t;
    if (col < n) cspart[(int64_t)blockIdx.y * n + col] = cs;

    ptx::mbar_wait(&tmem_bar, 0);
    ptx::tc_fence_after();
    const int q = warp - 4;
    float *hp = hpart + (int64_t)blockIdx.y * h_split_stride + (int64_t)col * LPAD;
#pragma unroll 1
    for (int c = 0; c < LPAD; c += 16) {
      float v[16];
      ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
      if (col < n) {
        float4 *o4 = reinterpret_cast<float4 *>(hp + c);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float4 w = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
          if (accumulate) {
            const float4 o = o4[e];
            w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
          }
          o4[e] = w;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, LPAD);
  }
}

// Omega (fp64 n x l, rounded to fp32) -> Omega^T hi/lo (lpad x n, zero padded)
__global__ void tc_omega_prepare(const double *__restrict__ om64, int n, int l, int lpad,
                                 float *__restrict__ whi, float *__restrict__ wlo) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < (int64_t)lpad * n; idx += stride) {
    const int j = (int)(idx / n);
    const int i = (int)(idx - (int64_t)j * n);
    const float v = j < l ? (float)om64[(int64_t)i * l + j] : 0.f;
    const float h = ptx::to_tf32(v);
    whi[idx] = h;
    wlo[idx] = ptx::to_tf32(v - h);
  }
}

}  // namespace spca
