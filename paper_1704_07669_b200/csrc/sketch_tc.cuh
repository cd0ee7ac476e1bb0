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
// producer, 3 idle, 4..11 converters (two groups of four warps, one warp per
// TMEM lane quarter; group g takes the K blocks kb = g mod 2), then the
// promoter warps (fold each accumulator period into fp32 registers and stage
// the unit's result; 64 output columns per warp) and 4 epilogue warps.
// converter groups (TcCfg<LPAD>::GROUPS): group g takes the K blocks kb = g (mod
// GROUPS). Two. Three for l_pad 64 (768 threads, 80 registers, ~70 bytes of
// spills) measured no better: the skeleton (no loads, no MMAs, no epilogue)
// went 1.013 -> 0.964 ms, the full pass 1.667 -> 1.694 ms, and one of two runs
// hung (profiles/r6_groups_ab.txt) - the converter stage's group count is not
// what bounds the pipeline.
#ifndef SPCA_GROUPS_64
#define SPCA_GROUPS_64 2
#endif
// K blocks per iteration of the MMA-issuing warp (l_pad 64). That warp's loop
// is serial - wait for the operand stage, fence, issue, commit - and its waits
// and commits cost 60-100 cycles each: with one K block per iteration it took
// 620-750 cycles per block (fine trace, profiles/r6_fine_trace.txt: 396 cycles
// of "issue + commit" with NO MMAs issued) against 384 tensor cycles, while the
// converters ran five blocks ahead - the issuing warp bounded the pipeline.
// With 2, the two converter groups' blocks 2j and 2j + 1 share one "stage full"
// barrier and one commit: one wait, 24 MMAs, one commit per iteration. Every
// unit then has an even number of K blocks (FusedSched::kp; an odd tail gets
// one more block of TMA zero fill).
// Build option (SPCA_BUILD_KPAIR=1), off by default: it lifts the block rate
// (G units 14.6 -> 11.8 us per 32 K blocks; passes whose A is L2-resident or
// whose epilogue is idle run 5-9% faster), but the full config-2 pass is bound
// elsewhere (G -> G^T latency against the L2 capacity): equal
// in 20-pass bursts (1.670 vs 1.670 ms), 0.7% slower over 300 back-to-back
// passes under the power cap (1.880 vs 1.867 ms) and 7% more DRAM reads
// (6.98 vs 6.46 GB) because the faster G units put more data between a
// tile's two reads (profiles/r6_kpair.txt, r6_kpair_sustained.txt).
#ifndef SPCA_KPAIR
#define SPCA_KPAIR 0
#endif
// Experiment (off): G units' phase B (wait for the tile's other K segments,
// slice reduction, G^T) on a reduction team - the idle warp 3 (1), or warp 3 and
// one more warp (2) - instead of on the four epilogue warps, l_pad 64. The
// epilogue warps are busy ~75% of the time and pick a G unit's staged result
// up 6.8 us late at the median (r6_kpair.txt trace), which delays G^T and with
// it the H units; but the slice reduction on 32 / 64 threads instead of 128 is
// itself slower, and G^T's latency is what the H units wait for: config 2
// 1.663 (off) -> 1.894 (one warp) / 1.729 ms (two warps, which also caps the
// kernel at 80 registers: 21 warps put six on one SM sub-partition)
// (profiles/r6_gteam_ab.txt).
// Experiment (off): G slice reduction with ten partial loads in flight per half
// instead of 1 + 4 + 4 + 1 (same order of additions): config 2 1.694 vs 1.688 ms,
// config 5 61.3 vs 61.9 ms - within noise (profiles/r6_gwide_ab.txt)
#ifndef SPCA_GRED_WIDE
#define SPCA_GRED_WIDE 0
#endif
#ifndef SPCA_GRED_TEAM
#define SPCA_GRED_TEAM 0
#endif
constexpr int kTcEpi = 128;     // epilogue threads
constexpr uint32_t kTmemCols = 512;
#ifndef SPCA_PROMOTE
#define SPCA_PROMOTE 4
#endif
constexpr int kPromote = SPCA_PROMOTE;  // K blocks per accumulator period

// Measured on B200 (tools/mma_bench.cu, tools/mma2_test.cu): a kind::tf32
// K=8 MMA takes 64 cycles per SM at N = 128 (the full tf32 rate), 44 at N = 64
// and 128 at N = 256, with A from TMEM or SMEM, for one CTA (M = 128) and for
// a CTA pair (cta_group::2, M = 256). The pass runs on CTA pairs: each CTA
// keeps its own 128 rows of the A operand in TMEM and HALF of every B operand
// in shared memory, which halves B's shared-memory and L2->SM traffic per SM
// (the per-SM ingress, ~90 GB/s measured with tools/l2_bench.cu and
// tools/tma_bench.cu, is what bounds a single-CTA version).
// Three products per K step into one accumulator of N = l_pad columns:
// A_hi W_hi + A_hi W_lo + A_lo W_hi (the dropped A_lo W_lo is ~2^-22 of a
// product). B stage per CTA: rows [r * l_pad/2, (r+1) * l_pad/2) of W_hi, then
// the same rows of W_lo (rank r). l_pad = 64 keeps the accumulators at 64
// columns, leaving TMEM for six A operand stages: the MMA completion latency
// needs that depth when every K block's operand is produced on chip.
// converters relay the B ring (wait b_full before arriving, release b_empty
// after the block's MMAs): the MMA warp waits and commits once per K block
#ifndef SPCA_RELAY
#define SPCA_RELAY 1
#endif
// l_pad = 64 MMA form: 0 = three N = 64 MMAs per step (default, measured
// faster: 8 KB B stages, six TMEM operand stages), 1 = stacked N = 128 + 64
#ifndef SPCA_STACKED_64
#define SPCA_STACKED_64 0
#endif
// B operand layout: 1 = hi and lo rows of each CTA's half interleaved in one
// matrix (rows ((2g + half) * 2 + part) * l_pad/2 + r for column group g), so
// a CTA's B stage is ONE TMA box of l_pad rows per K block (TMA request rate,
// not bytes, limits the per-SM stream: tools/mc_bench.cu); 0 = separate hi /
// lo matrices, two boxes per K block
#ifndef SPCA_BCOMB
#define SPCA_BCOMB 1
#endif
// Experiment (off): A ring in pairs of 16 KB slots, one TMA request bringing
// two K blocks (a 3-D box of two 128 x 32 tiles for G units, a 64-row box for
// H units), the two converter groups sharing the pair's barriers. In
// isolation 2 x 16 KB boxes stream at 118 GB/s per SM from L2 vs 63 GB/s for
// 16 KB boxes (tools/mc_bench.cu), but in the pass it measured no faster at
// config 2 (1.699 vs 1.703 ms) and 5% slower at config 3 (shallower ring):
// the A request rate does not bound the pass.
#ifndef SPCA_PAIRA
#define SPCA_PAIRA 0
#endif
// B operand as raw fp32 (1): Omega^T and G^T reach shared memory unsplit (half
// the B bytes through L2 -> SM, the pass's scarcest resource: 24 -> 20 KB of
// ingress per CTA and K block at l_pad = 64), and the converter group of the
// block writes lo = rna_tf32(b - trunc_tf32(b)) next to it in shared memory.
// The tensor core reads the raw b as tf32 by dropping its 13 low mantissa
// bits, i.e. as trunc_tf32(b), so hi + lo = b as in the host split.
// 0 = hi / lo split once in global memory (Omega^T at create, G^T in the G
// epilogue), both loaded per K block. Measured (round 2): parity unchanged
// (which confirms the truncating read), but config 2 1.647 -> 1.676 ms and
// config 3 11.60 -> 12.35 ms: the L2 -> SM bytes of B are not what bounds
// the pass, the converters' extra wait and shared-memory traffic cost more.
#ifndef SPCA_BRAW
#define SPCA_BRAW 0
#endif
// epilogue staging buffers for l_pad = 64. Two (at the cost of two A stages)
// measured no faster and failed 1 run in 8 (a launch fault not yet understood):
// kept at one; the staging code is written for either.
#ifndef SPCA_NSTG_64
#define SPCA_NSTG_64 1
#endif
// Epilogue data movement on the TMA engine (1): the staged unit result leaves
// shared memory as ONE bulk copy (G: K-split partial -> its slot) or as one
// bulk fp32 reduce-add per H row (performed at L2: H += partial, in chunk
// order under hseq as before), instead of 128 epilogue threads loading,
// adding and storing 32-64 KB per unit. The staging tile is then unswizzled
// ([128][l_pad], the layout of the partial slots and of H's rows). Measured
// (round 2): parity unchanged, but config 2 1.647 -> 1.680 ms, config 3
// 11.60 -> 12.28 ms, 512-row chunks 1.709 -> 1.766 ms: the bulk operations
// queue on the same per-SM TMA engine as the A and B loads of the next unit.
#ifndef SPCA_BULK_EPI
#define SPCA_BULK_EPI 0
#endif
// G units' K-split partials written to global memory by the promoter warps
// straight from their registers (the epilogue then only waits for the tile's
// segments and reduces its slice, and the staging tile is free at once):
// 0 = off (staged, copied by the epilogue), 1 = l_pad 128 only, 2 = both.
// Measured (round 2, =2): parity green; config 2 1.652 -> 1.735 ms, config 3
// 11.31 -> 11.55, config 5 59.7 -> 60.3: the G epilogue's time is its wait for
// the tile's other K segments (23 us at config 3 with or without the copy),
// and the promoters' global stores delay the next unit's accumulator folds.
#ifndef SPCA_PROMO_GP
#define SPCA_PROMO_GP 0
#endif
template <int LPAD>
struct TcCfg {
  static_assert(LPAD == 64 || LPAD == 128, "tensor-core path covers l <= 128");
  // l_pad = 64: "stacked" form, two MMAs per 8-deep step: A_hi [W_hi | W_lo]
  // (N = 128) and A_lo W_hi (N = 64) into the first half; the accumulator is
  // 128 columns and promotion adds its halves. l_pad = 128: three N = 128 MMAs.
  static constexpr bool STACKED = LPAD == 64 && SPCA_STACKED_64;
  static constexpr int ACC_COLS = STACKED ? 128 : LPAD;  // one accumulator
  static constexpr int NS = (kTmemCols - 2 * ACC_COLS) / 64;  // TMEM A operand stages
  // K blocks per MMA-warp iteration (SPCA_KPAIR: 1 = l_pad 64 only, 2 = l_pad 128 as well)
  static constexpr int KP = ((LPAD == 64 || SPCA_KPAIR == 2) && SPCA_KPAIR && !SPCA_PAIRA) ? 2 : 1;
  static_assert(NS % KP == 0 && SPCA_PROMOTE % KP == 0, "operand stages / accumulator period in whole iterations");
  // B ring: deep enough to cover an L2 round trip (~1-2 us) at the MMA rate
  static constexpr int GROUPS = LPAD == 64 ? SPCA_GROUPS_64 : 2;  // converter groups
  static constexpr int CONV = 128 * GROUPS;                       // converter threads
  static constexpr int PROMO_WARPS = 4 * (LPAD / 64);  // promoters: 64 output columns per thread
  static constexpr int PROMO_BASE = 128 + CONV;        // first promoter thread
  static constexpr int EPI_BASE = PROMO_BASE + 32 * PROMO_WARPS;  // first epilogue thread
  // one more warp when the G slice reductions run on their own team (with the idle warp 3)
#ifdef SPCA_FINE_TRACE
  static constexpr bool GT = false;  // warp 3 records MMA completions
#else
  static constexpr bool GT = LPAD == 64 && SPCA_GRED_TEAM;
#endif
  // team size: warp 3 alone (SPCA_GRED_TEAM 1), or with one more warp (2: 21 warps
  // put six on one SM sub-partition, which caps the kernel at 80 registers)
  static constexpr int GT_THREADS = SPCA_GRED_TEAM == 2 ? 64 : 32;
  static constexpr int THREADS = EPI_BASE + kTcEpi + ((GT && GT_THREADS == 64) ? 32 : 0);
  static constexpr uint32_t A_BYTES = 128 * 32 * 4;   // raw A tile (16 KB)
  static constexpr uint32_t BH_BYTES = (LPAD / 2) * 32 * 4;  // l_pad/2 rows of one B matrix tile
  // B stage per CTA (rank r). Stacked: [R0 | R1 | R2] of 32 rows each:
  //   rank 0: W_hi[0:32], W_hi[32:64], W_hi[0:32];  rank 1: W_lo[0:32], W_lo[32:64], W_hi[32:64]
  // (R0..R1 = this CTA's 64 rows of [W_hi | W_lo], R2 = its 32 rows of W_hi).
  // Otherwise: W_hi rows [r*l_pad/2, (r+1)*l_pad/2) then the same rows of W_lo.
  static constexpr uint32_t B_STAGE = STACKED ? 3 * BH_BYTES : 2 * BH_BYTES;
  static constexpr int NB = STACKED ? 7 : (LPAD == 64 ? 8 : 4);  // B ring (12 | 8 | 16 KB stages)
  static constexpr int NSTG = LPAD == 64 ? SPCA_NSTG_64 : 1;  // epilogue staging buffers
  static constexpr int NA = SPCA_PAIRA ? (LPAD == 64 ? 6 : 4)
                                       : (STACKED ? 6 : (LPAD == 64 ? (NSTG == 2 ? 5 : 7) : 5));  // raw A ring (16 KB stages)
  static constexpr int NP = NA / 2;  // A slot pairs (SPCA_PAIRA)
  static_assert(!SPCA_PAIRA || (NA % 2 == 0 && !STACKED), "paired A slots");
  static_assert(!SPCA_BRAW || (!STACKED && !SPCA_PAIRA), "raw B operand: three-MMA form");
  static constexpr uint32_t STG_BYTES = 128 * LPAD * 4;  // epilogue staging tile
  static constexpr uint32_t B_OFF = NA * A_BYTES;
  static constexpr uint32_t STG_OFF = B_OFF + NB * B_STAGE;
  static constexpr uint32_t SMEM = STG_OFF + NSTG * STG_BYTES + 1024;
  static constexpr uint32_t A_TMEM = 2 * ACC_COLS;    // first operand column
  static_assert(SMEM <= 227 * 1024 - 4096, "shared memory budget");
};

// round-to-nearest (ties away) to tf32 for finite values in two integer ops:
// add half an ulp of the 10-bit mantissa, clear the 13 low bits. Infinities
// stay infinite and NaNs stay NaN (their inputs are flagged anyway).
__device__ __forceinline__ float rna_tf32_fast(float v) {
  return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}

// tf32 by truncation (the low 13 mantissa bits cleared): v - trunc(v) is exact
__device__ __forceinline__ float trunc_tf32(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// tf32 split of v: hi = rna(v), lo = rna(v - hi); v - hi is exact in fp32
__device__ __forceinline__ void split3(float v, float &hi, float &lo) {
  hi = rna_tf32_fast(v);
  lo = rna_tf32_fast(v - hi);
}

// The pair MMAs (M = 256) of one 32-deep K block into accumulator `acc`.
// `db` is the shared-memory descriptor of the B stage (hi half at +0, lo half
// at +BH_BYTES; same offset in both CTAs): the per-MMA descriptors differ
// only in the 14-bit start-address field (16-byte units), so they are formed
// by small adds instead of re-encoding (the issuing warp's per-block
// bookkeeping must stay well under the 384 tensor cycles of a block).
template <int LPAD>
__device__ __forceinline__ void tc_mma_stage2(uint32_t a_hi, uint32_t acc, uint64_t db, bool first) {
  using C = TcCfg<LPAD>;
  if constexpr (C::STACKED) {
    constexpr uint32_t idesc1 = ptx::idesc_tf32(256, 2 * LPAD, 0, 0);
    constexpr uint32_t idesc2 = ptx::idesc_tf32(256, LPAD, 0, 0);
    constexpr uint64_t R2 = (2 * C::BH_BYTES) >> 4;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // +32 bytes per 8-deep step
      ptx::mma2_tf32_ts(acc, a_hi + kk * 8, db + 2 * kk, idesc1, (first && kk == 0) ? 0u : 1u);
      ptx::mma2_tf32_ts(acc, a_hi + 32 + kk * 8, db + R2 + 2 * kk, idesc2, 1u);
    }
  } else {
    constexpr uint32_t idesc = ptx::idesc_tf32(256, LPAD, 0, 0);
    constexpr uint64_t LO = C::BH_BYTES >> 4;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t dh = db + 2 * kk, dl = db + LO + 2 * kk;
      ptx::mma2_tf32_ts(acc, a_hi + kk * 8, dh, idesc, (first && kk == 0) ? 0u : 1u);
      ptx::mma2_tf32_ts(acc, a_hi + kk * 8, dl, idesc, 1u);
      ptx::mma2_tf32_ts(acc, a_hi + 32 + kk * 8, dh, idesc, 1u);
    }
  }
}

// row of the combined B matrix holding element j (0 <= j < lpad) of part
// (0 = hi, 1 = lo), column groups of lp
__host__ __device__ __forceinline__ int bcomb_row(int j, int part, int lp) {
  const int hr = lp / 2, g = j / lp, jj = j - g * lp, half = jj / hr;
  return ((2 * g + half) * 2 + part) * hr + (jj - half * hr);
}

// Omega -> the combined B matrix (2 lpad x n): Omega^T hi / lo rows interleaved per CTA half
__global__ void tc_omega_prepare_comb(const double *__restrict__ om64, int n, int l, int lpad, int lp,
                                      float *__restrict__ w2, int ldw) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < (int64_t)lpad * n; idx += stride) {
    const int j = (int)(idx / n);
    const int i = (int)(idx - (int64_t)j * n);
    const float v = j < l ? (float)om64[(int64_t)i * l + j] : 0.f;
    float hi, lo;
    split3(v, hi, lo);
    w2[(int64_t)bcomb_row(j, 0, lp) * ldw + i] = hi;
    w2[(int64_t)bcomb_row(j, 1, lp) * ldw + i] = lo;
  }
}

// Omega (fp64 n x l, rounded to fp32) -> raw Omega^T (lpad x n, zero padded,
// row stride ldw) for the raw B operand (SPCA_BRAW)
__global__ void tc_omega_prepare_raw(const double *__restrict__ om64, int n, int l, int lpad,
                                     float *__restrict__ w, int ldw) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < (int64_t)lpad * n; idx += stride) {
    const int j = (int)(idx / n);
    const int i = (int)(idx - (int64_t)j * n);
    w[(int64_t)j * ldw + i] = j < l ? (float)om64[(int64_t)i * l + j] : 0.f;
  }
}

// lo part of a raw B value as the tensor core completes it: it reads b as
// trunc_tf32(b); the remainder (exact in fp32) is rounded to tf32
__device__ __forceinline__ float braw_lo(float b) { return rna_tf32_fast(b - trunc_tf32(b)); }

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
