// sketch_tc.cuh — tcgen05 tensor-core sketch path (sm_100a), fp32 data.
//
// Split precision "3xTF32": every fp32 operand x is split on chip into
// x_hi = rna_tf32(x) and x_lo = rna_tf32(x - x_hi), and each contraction is
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi (+ A_lo B_lo where it is free)
// with fp32 accumulation (dropped terms ~2^-22 relative). Every operand the
// tensor core reads is an exact tf32 value.
//
// Accumulator promotion. Measured on B200: each tcgen05.mma accumulate into
// fp32 TMEM truncates toward zero, so a long accumulation drifts: relative
// bias ~ -(number of MMAs into one accumulator) x 2^-25 (e.g. -9e-5 over a
// 16k-row H accumulation, vs ~1e-9 for FFMA). The MMAs therefore run in
// periods of P K-blocks into one of two TMEM accumulators; at the end of a
// period the converter warps fold that accumulator into fp32 registers
// (round-to-nearest adds) while the MMAs continue into the other one. The
// residual bias is bounded by one period (~6e-7) regardless of the length.
//
// Shared-memory bandwidth is the scarce resource of a split-precision
// tall-skinny contraction, so the A-side operand (the data matrix) never
// goes back to shared memory: converter warps read each A tile once from
// the TMA landing buffer, split it in registers and store hi / lo straight
// into TMEM (tcgen05.st); the MMAs take A from TMEM. Only the narrow B-side
// operand (Omega^T or G^T, l_pad x 32 per K block) is read from shared
// memory. Three decoupled rings keep the HBM stream deep: the raw A landing
// ring is released as soon as the converters have read a tile, the B ring by
// MMA completion, and the TMEM operand ring sits between converters and MMA.
//
// Per canonical chunk of R rows:
//   tc_g_kernel    partial G (128-row tile x l_pad) over a K (= n) split.
//                  Converter thread (t, half) owns row t and 16 of the 32 K
//                  values of each block: reads them from the swizzled TMA
//                  tile, flags non-finite values, splits; it also owns half
//                  of row t's output columns for promotion and epilogue.
//   tc_g_finalize  fixed-order sum of the K-split partials -> G (output,
//                  fp32) and G^T hi / lo (K-major B operands of the H pass).
//   tc_h_kernel    H tile (128 n x l_pad) over a row split. Converter
//                  thread (t, half) owns column n0+t and 16 of the 32 rows
//                  of each block: reads them down the TMA tile (row-major as
//                  stored), accumulates the column sum in fp64, splits, and
//                  stores the transposed K-major A^T operand.
// Warps: 0 A producer, 1 TMEM allocator + MMA issuer, 2 B producer,
// 4..11 converters / promoters / epilogue (two warps per TMEM lane quarter).
// TMEM (512 columns): two accumulators of ACC_COLS, then NT operand stages
// of 64 columns (hi in +0..31, lo in +32..63; one K element per column).
#pragma once

#include <cuda.h>

#include "tc_ptx.cuh"

namespace spca {

constexpr int kTcThreads = 384;
constexpr int kTcConv = 256;  // converter threads (warps 4..11)
constexpr uint32_t kTmemCols = 512;
constexpr int kPromote = 4;   // K blocks per accumulator period

// optional per-CTA timeline (profiling): 16 globaltimer stamps per CTA, then
// per-chunk kernel spans {G start, G end, H start, H end} at kTraceTimeline
constexpr int kTraceTimeline = 4096 * 16;
#define TRACE_AT(slot)                                                                    \
  do {                                                                                    \
    if (trace) trace[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + (slot)] = ptx::globaltimer(); \
  } while (0)

// Measured on B200: a kind::tf32 M=128 MMA costs ~70 cycles for N <= 128
// (N = 128 runs at ~85% of the tf32 peak, N = 64 at ~45%). So for l_pad = 64
// the B operand is the contiguous [W_hi | W_lo] pair (N = 128) and each K
// step issues A_hi [W_hi|W_lo] + A_lo [W_hi|W_lo] (all four products, two
// MMAs); promotion adds the two column halves. For l_pad = 128 the three
// products run as N = 128 MMAs into one accumulator.
template <int LPAD>
struct TcCfg {
  static_assert(LPAD == 64 || LPAD == 128, "tensor-core path covers l <= 128");
  static constexpr bool FOUR = LPAD == 64;            // 4-product, N = 2 l_pad
  static constexpr int ACC_COLS = 128;                // one accumulator
  static constexpr int NA = LPAD == 64 ? 8 : 5;       // raw A ring
  static constexpr int NB = 4;                        // B operand ring
  static constexpr int NT = (kTmemCols - 2 * ACC_COLS) / 64;  // TMEM operand ring (4)
  static constexpr int HALF_COLS = LPAD / 2;          // output columns per converter thread
  static constexpr uint32_t A_BYTES = 128 * 32 * 4;   // raw A tile (16 KB)
  static constexpr uint32_t W_BYTES = LPAD * 32 * 4;  // B operand tile: l_pad x 32 K
  static constexpr uint32_t B_STAGE = 2 * W_BYTES;    // hi | lo
  static constexpr uint32_t B_OFF = NA * A_BYTES;     // B ring after the A ring
  static constexpr uint32_t SMEM = NA * A_BYTES + NB * B_STAGE + 1024;
  static constexpr uint32_t A_TMEM = 2 * ACC_COLS;    // first operand column
  static_assert(SMEM <= 227 * 1024 - 2048, "shared memory budget");
};

// round-to-nearest (ties away) to tf32 for finite values in two integer ops:
// add half an ulp of the 10-bit mantissa, clear the 13 low bits. Infinities
// stay infinite and NaNs stay NaN (their inputs are flagged anyway).
__device__ __forceinline__ float rna_tf32_fast(float v) {
  return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}

// tf32 split of v: hi = rna(v), lo = rna(v - hi); v - hi is exact in fp32
__device__ __forceinline__ void split3(float v, float &hi, float &lo) {
  hi = rna_tf32_fast(v);
  lo = rna_tf32_fast(v - hi);
}

// The MMAs of one 32-deep K block into accumulator `acc` (TMEM column).
template <int LPAD>
__device__ __forceinline__ void tc_mma_stage(uint32_t tmem, uint32_t acc, int ts, uint32_t wbase,
                                             bool first) {
  using C = TcCfg<LPAD>;
  const uint32_t a_hi = tmem + C::A_TMEM + 64 * ts;
  const uint32_t a_lo = a_hi + 32;
  const uint32_t w_hi = wbase, w_lo = wbase + C::W_BYTES;
  if constexpr (C::FOUR) {
    constexpr uint32_t idesc2 = ptx::idesc_tf32(128, 2 * LPAD, 0, 0);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t dw = ptx::sdesc_sw128(w_hi + kk * 32, 16, 1024);  // rows: W_hi then W_lo
      ptx::mma_tf32_ts(acc, a_hi + kk * 8, dw, idesc2, (first && kk == 0) ? 0u : 1u);
      ptx::mma_tf32_ts(acc, a_lo + kk * 8, dw, idesc2, 1u);
    }
  } else {
    constexpr uint32_t idesc = ptx::idesc_tf32(128, LPAD, 0, 0);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t dwh = ptx::sdesc_sw128(w_hi + kk * 32, 16, 1024);
      const uint64_t dwl = ptx::sdesc_sw128(w_lo + kk * 32, 16, 1024);
      ptx::mma_tf32_ts(acc, a_hi + kk * 8, dwh, idesc, (first && kk == 0) ? 0u : 1u);
      ptx::mma_tf32_ts(acc, a_hi + kk * 8, dwl, idesc, 1u);
      ptx::mma_tf32_ts(acc, a_lo + kk * 8, dwh, idesc, 1u);
    }
  }
}

// pipeline state shared by both kernels
template <int LPAD>
struct TcBars {
  using C = TcCfg<LPAD>;
  uint64_t a_full[C::NA], a_empty[C::NA];
  uint64_t b_full[C::NB], b_empty[C::NB];
  uint64_t t_full[C::NT], t_empty[C::NT];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
  double cs_x[128];  // H kernel: column-sum exchange between the two halves
};

template <int LPAD>
__device__ __forceinline__ void tc_prologue(TcBars<LPAD> &b, const CUtensorMap *m0,
                                            const CUtensorMap *m1, const CUtensorMap *m2) {
  using C = TcCfg<LPAD>;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NA; ++s) {
      ptx::mbar_init(&b.a_full[s], 1);
      ptx::mbar_init(&b.a_empty[s], kTcConv / 32);  // one elected arrive per converter warp
    }
    for (int s = 0; s < C::NB; ++s) {
      ptx::mbar_init(&b.b_full[s], 1);
      ptx::mbar_init(&b.b_empty[s], 1);
    }
    for (int s = 0; s < C::NT; ++s) {
      ptx::mbar_init(&b.t_full[s], kTcConv / 32);
      ptx::mbar_init(&b.t_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&b.acc_full[s], 1);
      ptx::mbar_init(&b.acc_empty[s], kTcConv / 32);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch(m0);
    ptx::tma_prefetch(m1);
    ptx::tma_prefetch(m2);
  }
  if ((threadIdx.x >> 5) == 1) ptx::tmem_alloc(&b.tmem_base, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
}

// MMA issuer loop (warp 1, one lane): TMEM operand ring x B ring -> the two
// period accumulators
template <int LPAD>
__device__ __forceinline__ void tc_mma_loop(TcBars<LPAD> &b, uint8_t *smem, uint32_t tmem, int nk,
                                            bool skip_wait, bool skip_mma) {
  using C = TcCfg<LPAD>;
  for (int kb = 0; kb < nk; ++kb) {
    const int ts = kb % C::NT, bs = kb % C::NB;
    const int q = kb / kPromote, buf = q & 1;
    const bool first = (kb % kPromote) == 0;
    if (first && q >= 2) ptx::mbar_wait(&b.acc_empty[buf], ((q >> 1) - 1) & 1);
    if (!skip_wait) {
      ptx::mbar_wait(&b.t_full[ts], (kb / C::NT) & 1);
      ptx::mbar_wait(&b.b_full[bs], (kb / C::NB) & 1);
    }
    ptx::tc_fence_after();
    if (!skip_mma)
      tc_mma_stage<LPAD>(tmem, tmem + buf * C::ACC_COLS, ts,
                         ptx::smem_u32(smem + C::B_OFF + bs * C::B_STAGE), first);
    ptx::mma_commit(&b.t_empty[ts]);
    ptx::mma_commit(&b.b_empty[bs]);
    if ((kb % kPromote) == kPromote - 1 || kb == nk - 1) ptx::mma_commit(&b.acc_full[buf]);
  }
}

// converter hand-off of one K block: wait for a free TMEM stage, store the
// split operand, publish it to the MMA issuer (one arrive per warp)
template <int LPAD>
__device__ __forceinline__ void tc_publish(TcBars<LPAD> &b, uint32_t lane_base, int kb, int half,
                                           const float *hi, const float *lo, bool skip_st = false) {
  using C = TcCfg<LPAD>;
  const int ts = kb % C::NT;
  if (kb >= C::NT) ptx::mbar_wait(&b.t_empty[ts], ((kb / C::NT) - 1) & 1);
  ptx::tc_fence_after();
  if (!skip_st) {  // profiling knob: leave TMEM untouched
    ptx::tmem_st16(lane_base + C::A_TMEM + 64 * ts + 16 * half, hi);
    ptx::tmem_st16(lane_base + C::A_TMEM + 64 * ts + 32 + 16 * half, lo);
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&b.t_full[ts]);
}

// Fold accumulator period q into this thread's fp32 registers (its row /
// column-half of the result), then hand the accumulator back to the MMAs.
template <int LPAD>
__device__ __forceinline__ void tc_promote(TcBars<LPAD> &b, uint32_t lane_base, int q, int half,
                                           float *racc) {
  using C = TcCfg<LPAD>;
  const int buf = q & 1;
  ptx::mbar_wait(&b.acc_full[buf], (q >> 1) & 1);
  ptx::tc_fence_after();
  const uint32_t base = lane_base + buf * C::ACC_COLS + half * C::HALF_COLS;
#pragma unroll
  for (int c = 0; c < C::HALF_COLS; c += 16) {
    float v[16];
    ptx::tmem_ld16(base + c, v);
    if constexpr (C::FOUR) {  // W_lo half of the accumulator
      float w[16];
      ptx::tmem_ld16(base + LPAD + c, w);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += w[i];
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) racc[c + i] += v[i];
  }
  ptx::tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&b.acc_empty[buf]);
}

// ------------------------------------------------------------- G = A Omega
template <int LPAD>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_g_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tWhi,
            const __grid_constant__ CUtensorMap tWlo, int rows, int n, int kseg, int row_base,
            float *__restrict__ gpart, int64_t split_stride, int64_t first_row,
            unsigned long long *__restrict__ bad_row, int dbg,
            unsigned long long *__restrict__ trace, int seq) {
  if (threadIdx.x == 0) TRACE_AT(0);
  if (threadIdx.x == 0 && trace) atomicMin(&trace[kTraceTimeline + 4 * (seq & 1023) + 0], ptx::globaltimer());
  using C = TcCfg<LPAD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ TcBars<LPAD> bars;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * 128;
  const int kbeg = blockIdx.y * kseg;
  const int kend = min(n, kbeg + kseg);
  const int nk = kend > kbeg ? (kend - kbeg + 31) / 32 : 0;

  tc_prologue<LPAD>(bars, &tA, &tWhi, &tWlo);
  const uint32_t tmem = bars.tmem_base;
  if (threadIdx.x == 0) TRACE_AT(1);

  if (warp == 0) {
    if (lane == 0) {  // A producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::NA;
        if (kb >= C::NA) ptx::mbar_wait(&bars.a_empty[s], ((kb / C::NA) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&bars.a_full[s], C::A_BYTES);
        ptx::tma_load_2d(smem + s * C::A_BYTES, &tA, &bars.a_full[s], kbeg + kb * 32, row_base + row0);
        if (kb == 0) TRACE_AT(2);
      }
      TRACE_AT(3);
    }
  } else if (warp == 2) {
    if (lane == 0) {  // B producer (Omega^T hi | lo)
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::NB;
        if (kb >= C::NB) ptx::mbar_wait(&bars.b_empty[s], ((kb / C::NB) - 1) & 1);
        uint8_t *st = smem + C::B_OFF + s * C::B_STAGE;
        if ((dbg & 4) && kb >= C::NB) {  // profiling knob: reuse stale Omega tiles
          ptx::mbar_arrive(&bars.b_full[s]);
          continue;
        }
        ptx::mbar_arrive_expect_tx(&bars.b_full[s], C::B_STAGE);
        ptx::tma_load_2d(st, &tWhi, &bars.b_full[s], kbeg + kb * 32, 0);
        ptx::tma_load_2d(st + C::W_BYTES, &tWlo, &bars.b_full[s], kbeg + kb * 32, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      TRACE_AT(4);
      tc_mma_loop<LPAD>(bars, smem, tmem, nk, false, (dbg & 2) != 0);
      TRACE_AT(5);
    }
  } else if (warp >= 4) {
    const int ct = threadIdx.x - 128;
    const int t = ct & 127;   // row of the tile == TMEM lane
    const int half = ct >> 7; // which 16 of the 32 K values per block / which output half
    const uint32_t lane_base = tmem + ((uint32_t)(t & ~31) << 16);
    float racc[C::HALF_COLS];
#pragma unroll
    for (int i = 0; i < C::HALF_COLS; ++i) racc[i] = 0.f;
    float chk = 0.f;  // becomes NaN iff this row holds a non-finite value
    const int nq = (nk + kPromote - 1) / kPromote;
    int promoted = 0;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::NA;
      ptx::mbar_wait(&bars.a_full[s], (kb / C::NA) & 1);
      if (kb == 0 && ct == 0) TRACE_AT(6);
      float4 v[4];
      const uint32_t row = ptx::smem_u32(smem + s * C::A_BYTES + t * 128);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) v[cc] = ptx::lds128(row + (((4 * half + cc) ^ (t & 7)) << 4));
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bars.a_empty[s]);  // landing slot free again
      float hi[16], lo[16];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        // x * 0 is 0 for finite x and NaN for +-inf / NaN: one FFMA per value
        chk = fmaf(v[cc].x, 0.f, fmaf(v[cc].y, 0.f, fmaf(v[cc].z, 0.f, fmaf(v[cc].w, 0.f, chk))));
        split3(v[cc].x, hi[4 * cc + 0], lo[4 * cc + 0]);
        split3(v[cc].y, hi[4 * cc + 1], lo[4 * cc + 1]);
        split3(v[cc].z, hi[4 * cc + 2], lo[4 * cc + 2]);
        split3(v[cc].w, hi[4 * cc + 3], lo[4 * cc + 3]);
      }
      if (dbg & 1) {
#pragma unroll
        for (int i = 0; i < 16; ++i) hi[i] = lo[i] = 0.f;
      }
      tc_publish<LPAD>(bars, lane_base, kb, half, hi, lo, (dbg & 32) != 0);
      // fold the period that ended one period ago (the MMAs run ahead meanwhile)
      if ((kb + 1) % kPromote == 0 && (kb + 1) / kPromote >= 2) {
        tc_promote<LPAD>(bars, lane_base, promoted, half, racc);
        ++promoted;
      }
    }
    for (; promoted < nq; ++promoted) tc_promote<LPAD>(bars, lane_base, promoted, half, racc);
    if (ct == 0) TRACE_AT(7);
    if (!(chk == 0.f) && row0 + t < rows) report_bad_row(bad_row, first_row + row0 + t);

    // epilogue: this thread's row, its half of the columns
    if (ct == 0) TRACE_AT(8);
    const int r = row0 + t;
    if (r < rows) {
      float4 *o4 = reinterpret_cast<float4 *>(gpart + (int64_t)blockIdx.y * split_stride +
                                              (int64_t)r * LPAD + half * C::HALF_COLS);
#pragma unroll
      for (int i = 0; i < C::HALF_COLS / 4; ++i)
        o4[i] = make_float4(racc[4 * i], racc[4 * i + 1], racc[4 * i + 2], racc[4 * i + 3]);
    }
    if (ct == 0) TRACE_AT(9);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
    if (lane == 0) TRACE_AT(10);
    if (lane == 0 && trace) atomicMax(&trace[kTraceTimeline + 4 * (seq & 1023) + 1], ptx::globaltimer());
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
      float h, lo;
      split3(s, h, lo);
      ghiT[(int64_t)c * ldt + r] = h;
      gloT[(int64_t)c * ldt + r] = lo;
    }
  }
}

// ------------------------------------------------------------ H += A^T G
template <int LPAD>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_h_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tGhi,
            const __grid_constant__ CUtensorMap tGlo, int rows, int n, int rseg, int row_base,
            float *__restrict__ hpart, int64_t h_split_stride, double *__restrict__ cspart,
            int accumulate, int kahan, int dbg,
            unsigned long long *__restrict__ trace, int seq) {
  if (threadIdx.x == 0) TRACE_AT(0);
  if (threadIdx.x == 0 && trace) atomicMin(&trace[kTraceTimeline + 4 * (seq & 1023) + 2], ptx::globaltimer());
  using C = TcCfg<LPAD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ TcBars<LPAD> bars;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int rb = blockIdx.y * rseg;
  const int re = min(rows, rb + rseg);
  const int nk = re > rb ? (re - rb + 31) / 32 : 0;  // trailing splits may be empty

  tc_prologue<LPAD>(bars, &tA, &tGhi, &tGlo);
  const uint32_t tmem = bars.tmem_base;
  if (threadIdx.x == 0) TRACE_AT(1);

  if (warp == 0) {
    if (lane == 0) {  // A producer: 4 atoms of 32 rows x 32 n
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::NA;
        if (kb >= C::NA) ptx::mbar_wait(&bars.a_empty[s], ((kb / C::NA) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&bars.a_full[s], C::A_BYTES);
        uint8_t *st = smem + s * C::A_BYTES;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          ptx::tma_load_2d(st + j * 4096, &tA, &bars.a_full[s], n0 + 32 * j, row_base + rb + kb * 32);
        if (kb == 0) TRACE_AT(2);
      }
      TRACE_AT(3);
    }
  } else if (warp == 2) {
    if (lane == 0) {  // B producer (G^T hi | lo)
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::NB;
        if (kb >= C::NB) ptx::mbar_wait(&bars.b_empty[s], ((kb / C::NB) - 1) & 1);
        uint8_t *st = smem + C::B_OFF + s * C::B_STAGE;
        ptx::mbar_arrive_expect_tx(&bars.b_full[s], C::B_STAGE);
        ptx::tma_load_2d(st, &tGhi, &bars.b_full[s], rb + kb * 32, 0);
        ptx::tma_load_2d(st + C::W_BYTES, &tGlo, &bars.b_full[s], rb + kb * 32, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      TRACE_AT(4);
      tc_mma_loop<LPAD>(bars, smem, tmem, nk, false, (dbg & 2) != 0);
      TRACE_AT(5);
    }
  } else if (warp >= 4) {
    // converter thread (t, half) owns column n0 + t, rows 16*half..16*half+15 of each block,
    // and half of that column's output (sketch) columns
    const int ct = threadIdx.x - 128;
    const int t = ct & 127, half = ct >> 7;
    const int j = t >> 5, nn = t & 31;
    const uint32_t lane_base = tmem + ((uint32_t)(t & ~31) << 16);
    float racc[C::HALF_COLS];
#pragma unroll
    for (int i = 0; i < C::HALF_COLS; ++i) racc[i] = 0.f;
    double cs = 0.0, cc = 0.0;
    const int nq = (nk + kPromote - 1) / kPromote;
    int promoted = 0;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::NA;
      ptx::mbar_wait(&bars.a_full[s], (kb / C::NA) & 1);
      if (kb == 0 && ct == 0) TRACE_AT(6);
      const uint32_t raw = ptx::smem_u32(smem + s * C::A_BYTES + j * 4096);
      float v[16];
#pragma unroll
      for (int kq = 0; kq < 16; ++kq) {
        const int k = 16 * half + kq;
        v[kq] = ptx::lds32(raw + ((k * 32 + (((nn >> 2) ^ (k & 7)) << 2) + (nn & 3)) << 2));
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bars.a_empty[s]);  // landing slot free again
      float hi[16], lo[16];
      double part[4] = {0.0, 0.0, 0.0, 0.0};  // fp64 partial sums, four chains
#pragma unroll
      for (int kq = 0; kq < 16; ++kq) {
        split3(v[kq], hi[kq], lo[kq]);
        part[kq & 3] += (double)v[kq];
      }
      const double blk = (part[0] + part[1]) + (part[2] + part[3]);
      if (kahan) {
        const double y = blk - cc;
        const double tt = cs + y;
        cc = (tt - cs) - y;
        cs = tt;
      } else {
        cs += blk;
      }
      if (dbg & 1) {
#pragma unroll
        for (int i = 0; i < 16; ++i) hi[i] = lo[i] = 0.f;
      }
      tc_publish<LPAD>(bars, lane_base, kb, half, hi, lo);
      if ((kb + 1) % kPromote == 0 && (kb + 1) / kPromote >= 2) {
        tc_promote<LPAD>(bars, lane_base, promoted, half, racc);
        ++promoted;
      }
    }
    for (; promoted < nq; ++promoted) tc_promote<LPAD>(bars, lane_base, promoted, half, racc);
    if (ct == 0) TRACE_AT(7);
    // column sums: half 1 hands its partial to half 0 (fixed order)
    if (half == 1) bars.cs_x[t] = cs;
    ptx::named_bar(1, kTcConv);
    const int col = n0 + t;
    if (half == 0 && col < n) cspart[(int64_t)blockIdx.y * n + col] = cs + bars.cs_x[t];

    if (ct == 0) TRACE_AT(8);
    if (col < n) {
      float4 *o4 = reinterpret_cast<float4 *>(hpart + (int64_t)blockIdx.y * h_split_stride +
                                              (int64_t)col * LPAD + half * C::HALF_COLS);
#pragma unroll
      for (int i = 0; i < C::HALF_COLS / 4; ++i) {
        float4 w = make_float4(racc[4 * i], racc[4 * i + 1], racc[4 * i + 2], racc[4 * i + 3]);
        if (accumulate) {
          const float4 o = o4[i];
          w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
        }
        o4[i] = w;
      }
    }
    if (ct == 0) TRACE_AT(9);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
    if (lane == 0) TRACE_AT(10);
    if (lane == 0 && trace) atomicMax(&trace[kTraceTimeline + 4 * (seq & 1023) + 3], ptx::globaltimer());
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
    split3(v, whi[idx], wlo[idx]);
  }
}

}  // namespace spca
