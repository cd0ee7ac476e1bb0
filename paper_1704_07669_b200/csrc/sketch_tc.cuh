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
// Building blocks of the pass kernel (sketch_fused.cuh): tile configuration,
// the tf32 split and the MMA stage of one 32-deep K block.
// TMEM (512 columns): two accumulators of ACC_COLS, then NT operand stages
// of 64 columns (hi in +0..31, lo in +32..63; one K element per column).
#pragma once

#include <cuda.h>

#include "tc_ptx.cuh"

namespace spca {

// Warps: 0 A producer, 1 TMEM allocator + MMA issuer (leader CTA), 2 B
// producer, 3 idle, 4..11 converters / promoters, 12..15 epilogue.
constexpr int kTcThreads = 512;
constexpr int kTcConv = 256;    // converter threads (warps 4..11)
constexpr int kTcEpi = 128;     // epilogue threads (warps 12..15)
constexpr int kTcEpiBase = 384; // first epilogue thread
constexpr uint32_t kTmemCols = 512;
constexpr int kPromote = 4;     // K blocks per accumulator period

// Measured on B200 (tools/mma_bench.cu, tools/mma2_test.cu): a kind::tf32
// K=8 MMA takes 64 cycles per SM at N = 128 (the full tf32 rate), 44 at N = 64
// and 128 at N = 256, with A from TMEM or SMEM, for one CTA (M = 128) and for
// a CTA pair (cta_group::2, M = 256). The pass runs on CTA pairs: each CTA
// keeps its own 128 rows of the A operand in TMEM and HALF of the N = 128 B
// operand in SMEM, which halves B's shared-memory and L2->SM traffic per SM
// (the SM ingress, ~94 GB/s per SM measured with tools/l2_bench.cu, is what
// bounds a single-CTA version).
//   l_pad = 64:  B = [W_hi | W_lo] (N = 128; rank 0 holds W_hi, rank 1 W_lo);
//                two MMAs per K step: A_hi B + A_lo B (all four products);
//                promotion adds the two column halves of the accumulator.
//   l_pad = 128: B = W_hi and B = W_lo (N = 128 each; rank r holds rows
//                64r..64r+63 of both); three MMAs: A_hi W_hi + A_hi W_lo + A_lo W_hi.
template <int LPAD>
struct TcCfg {
  static_assert(LPAD == 64 || LPAD == 128, "tensor-core path covers l <= 128");
  static constexpr bool FOUR = LPAD == 64;
  static constexpr int ACC_COLS = 128;                // one accumulator
  static constexpr int NA = LPAD == 64 ? 8 : 5;       // raw A ring
  static constexpr int NB = 4;                        // B operand ring
  static constexpr int NT = (kTmemCols - 2 * ACC_COLS) / 64;  // TMEM operand ring (4)
  static constexpr int HALF_COLS = LPAD / 2;          // output columns per converter thread
  static constexpr uint32_t A_BYTES = 128 * 32 * 4;   // raw A tile (16 KB)
  static constexpr uint32_t BH_BYTES = 64 * 32 * 4;   // this CTA's half of one B matrix tile (8 KB)
  static constexpr uint32_t B_STAGE = FOUR ? BH_BYTES : 2 * BH_BYTES;
  static constexpr uint32_t STG_BYTES = 128 * LPAD * 4;  // epilogue staging tile
  static constexpr uint32_t B_OFF = NA * A_BYTES;
  static constexpr uint32_t STG_OFF = B_OFF + NB * B_STAGE;
  static constexpr uint32_t SMEM = STG_OFF + STG_BYTES + 1024;
  static constexpr uint32_t A_TMEM = 2 * ACC_COLS;    // first operand column
  static_assert(SMEM <= 227 * 1024 - 4096, "shared memory budget");
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

// The pair MMAs (M = 256) of one 32-deep K block into accumulator `acc`;
// `bstage` is the B stage address (same offset in both CTAs).
template <int LPAD>
__device__ __forceinline__ void tc_mma_stage2(uint32_t tmem, uint32_t acc, int ts, uint32_t bstage,
                                              bool first) {
  using C = TcCfg<LPAD>;
  const uint32_t a_hi = tmem + C::A_TMEM + 64 * ts;
  const uint32_t a_lo = a_hi + 32;
  constexpr uint32_t idesc = ptx::idesc_tf32(256, 128, 0, 0);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint32_t acc_flag = (first && kk == 0) ? 0u : 1u;
    if constexpr (C::FOUR) {
      const uint64_t db = ptx::sdesc_sw128(bstage + kk * 32, 16, 1024);
      ptx::mma2_tf32_ts(acc, a_hi + kk * 8, db, idesc, acc_flag);
      ptx::mma2_tf32_ts(acc, a_lo + kk * 8, db, idesc, 1u);
    } else {
      const uint64_t dh = ptx::sdesc_sw128(bstage + kk * 32, 16, 1024);
      const uint64_t dl = ptx::sdesc_sw128(bstage + C::BH_BYTES + kk * 32, 16, 1024);
      ptx::mma2_tf32_ts(acc, a_hi + kk * 8, dh, idesc, acc_flag);
      ptx::mma2_tf32_ts(acc, a_hi + kk * 8, dl, idesc, 1u);
      ptx::mma2_tf32_ts(acc, a_lo + kk * 8, dh, idesc, 1u);
    }
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
