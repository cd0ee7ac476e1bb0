// sketch_fused.cuh — the fused tensor-core sketch pass (sm_100a, fp32).
//
// One persistent kernel per push walks the pushed rows in canonical chunks of
// R0 rows (R0 * n * 4 B ~ 40 MB) and computes, per chunk c (reference
// sketch.py:85-113, paper Alg. 4 steps 5-7):
//
//   G_c = A_c Omega          ("G units": 128-row tile x K segment of n)
//   H  += A_c^T G_c          ("H units": 128-column tile x row segment of R0)
//   col_sums += 1^T A_c      (inside the H units)
//
// A_c is read from HBM by the G units (TMA, L2 evict_last) and re-read by the
// H units a stage later (evict_first). The re-read is meant to hit L2, but
// only about half of it does: ncu measures ~1.7x the bytes of A read from
// DRAM at config 2 (7.0 GB per 4 GB pass at lag 1; 8.2 GB at lag 2; 512-row
// chunks read 1.2x but run slower). The units form one global
// sequence of stages {G(s), H(s-1)}, s = 0..C, dealt round robin to CTA
// pairs (clusters of 2, one CTA per SM), so the H contraction of chunk c
// overlaps the G contraction of chunk c+1 inside one launch and every pair
// does the same work over a push. A pair unit covers two adjacent tiles (one
// per CTA) that share the B operand: the leader CTA issues M = 256 pair MMAs
// (cta_group::2), each CTA holding its own A tile in TMEM and half of B in
// shared memory (sketch_tc.cuh).
//
// Ordering between CTAs uses counters in global memory (acquire / release);
// every wait points at units dealt no later than the waiting one, so with all
// CTAs resident the pass cannot deadlock:
//   * G(c, t, seg) writes its K-split partial into slot c % kSlots, counts
//     itself in seg_cnt[c][t], waits until all S segments of the tile are
//     there, then reduces ITS slice of the tile's rows over the S partials
//     in fixed order -> G rows (output) and the split G^T hi / lo operands,
//     and counts the slice in ready[c]. Partial and G^T slots are reused
//     kSlots chunks later, after ready / hdone of that chunk say so.
//   * H(c, x, rs) loads its B operand (G^T of chunk c) once ready[c] counts
//     every slice; it adds its fp32 partial into the running H and its column
//     sums into the fp64 running sums in chunk order (hseq[x]), so results
//     are bitwise reproducible and independent of how rows were pushed.
//
// Warp roles per CTA (sketch_tc.cuh): A producer, MMA issuer (leader only),
// B producer, converters (tf32 split into TMEM, accumulator promotion) and
// epilogue warps, which take each finished unit from a staging tile in
// shared memory so the converters go straight on with the next unit.
#pragma once

#include "sketch_tc.cuh"

namespace spca {

constexpr int kMaxLag = 3;               // largest stage lag D of the H units
constexpr int kSlots = kMaxLag + 2;      // chunks whose G partials / G^T may be in flight

// optional timeline (SPCA_TC_TRACE): per CTA kTraceStride globaltimer stamps:
// [0] start, [1] end, then per unit i < kTraceUnits, 8 stamps at 8 + 8i:
//   0 converters start, 1 converters' main loop done, 2 promoters staged the result,
//   3 epilogue took it, 4 epilogue done, 5 MMA first issue, 6 promoters folded the
//   last period (MMA done), 7 B producer passed its dependency wait
constexpr int kTraceStride = 1024;
constexpr int kTraceUnits = 127;
constexpr int kTraceMma = 2048;  // leader of pair 0: 4 stamps for each of its first K blocks
constexpr int kTraceConv = 1024;  // converter thread 0 of CTA 0: 6 stamps for each of its first blocks
constexpr int kTraceWords = 256 * kTraceStride + 4 * kTraceMma + 6 * kTraceConv + kTraceMma;
#define SPCA_TRACE(i, k)                                                         \
  do {                                                                           \
    if (trace && (i) < kTraceUnits) trace[8 + 8 * (i) + (k)] = ptx::globaltimer(); \
  } while (0)

struct FusedSched {
  int C;          // chunks in this launch
  int R0;         // canonical chunk rows (multiple of 256)
  int rows_last;  // rows of the last chunk (<= R0)
  int T, Tl;      // 256-row tile pairs of a full / the last chunk
  int nt, ntl;    // real 128-row tiles of a full / the last chunk
  int S, kseg;    // G: K segments over n, K blocks per segment
  int nkb;        // K blocks over n
  int X, nx;      // H: 256-column tile pairs, real 128-column tiles over n
  int RS, hseg;   // H: row segments per chunk, K blocks per segment
  int D;          // stage lag of a chunk's H units behind its G units
  int kp;         // every unit's K block count is a multiple of kp (TcCfg::KP; kseg, hseg too)
  int Gr;         // column groups of 128 sketched together (l > 128: each unit
                  // covers one group; a unit's groups are dealt side by side, so
                  // they read the same A tile at the same time: one DRAM read)
  int total;      // pair units in this launch
  const int *order;  // device: unit u -> kind << 30 | chunk << 15 | index (null: closed form, lag D)
};

struct FusedArgs {
  FusedSched s;
  int n;
  int row_base;             // first launch row in the A tensor maps
  float *gpart;             // [kSlots][2T][S][128][LPAD] K-split partials
  float *gT;                // [kSlots][2][LPAD][R0] G^T hi, lo
  float *g_out;             // G rows of this launch, [rows][LPAD]
  float *hpart;             // [n][LPAD] running H (fp32, flushed to fp64 by the host)
  const float *cshift;      // column shift c (zero padded to a multiple of 128) or null:
                            //   every value a[r][j] enters as a[r][j] - c[j] (spca_sketch_set_shift)
  const float *left;        // co-sketch operand rows of this launch ([rows][gld]) or null:
                            //   the H units then take L instead of G (spca_sketch_set_left)
  double *colsum;           // [n] running column sums (fp64)
  double *carry;            // [n] Kahan carry, or null
  int *seg_cnt;             // [C][2T] partials written per tile
  int *ready;               // [C] reduced row slices
  int *hdone;               // [C] finished H units
  int *hseq;                // [2X] H units applied to column tile x (chunk-major)
  int *trdy;                // [C][2T] reduced row slices per 128-row tile (S = the tile's G is complete)
  int tile_ready;           // H units wait per 128-row tile of G^T (trdy) instead of for the whole chunk
  int64_t gpart_group;      // elements of gpart per column group (Gr > 1)
  int64_t gT_group;         // elements of gT per column group
  int gT_rows_group;        // rows of the G^T tensor map per column group
  int ctr_group;            // ordering-counter words per column group
  int accumulate;           // H of the launch's first chunk adds to hpart
  int64_t first_row;        // global index of the launch's first row
  const float *a;           // the launch's rows (row_base = 0) and their stride, for the
  int64_t lda;              //   exact non-finite re-check of a flagged row
  unsigned long long *bad_row;
  unsigned long long *trace;  // null unless profiling
  // fused row normalisation (normalize_rows, sketch.py:142-153), or all null / 0:
  int norm;
  float *rstat_part;          // [kSlots][2T][S][128][2] per-segment sums of d, d^2 (d = a - a0)
  float *row_a0;              // [kSlots][R0] a0 = each row's first value (the shift)
  float *row_inv;             // [kSlots][R0] 1 / ||a - mean|| (1 for a zero norm)
  double *row_coef;           // [launch rows] (mean - a0) / norm, for the finish-time corrections
  const float *wsum;          // [LPAD] column sums of this group's Omega (as used)
  int wy0;                    // first Omega^T row of this launch's column group
  int gld;                    // row stride (floats) of g_out and hpart (all column groups)
  int colsum_on;              // this launch also accumulates the column sums (group 0)
  int g3d;                    // tAg3 (3-D box of two K blocks) is valid: n % 32 == 0
  int dbg;                    // profiling knobs (SPCA_TC_DEBUG), 0 in production:
                              // 1 converters skip the split, 2 no MMAs, 4 no B loads, 8 no A loads,
                              // 2048 A tiles at one address (L2), 16384 no epilogue, 32768 no G^T
                              // stores, 65536 no H read-modify-write, 131072 no G partial copy

};

// The state of column group g of a unit: Omega^T rows, partial / G^T slots,
// output columns, ordering counters (identical to the launch's for g = 0)
struct GroupView {
  int wy0;            // first Omega^T row of the group
  int gt_row0;        // first row of the group's G^T slots in the tensor map
  float *gpart, *gT, *g_out, *hpart;
  const float *left, *wsum;
  int *seg_cnt, *ready, *hdone, *hseq, *trdy;
  int colsum_on;
};

struct FusedUnit {
  int kind;   // 0 = G, 1 = H
  int c;      // chunk
  int g;      // column group (0 unless Gr > 1)
  int a, b;   // G: tile pair, segment; H: column-tile pair, row segment
  int k0, nk; // first K block and count (G: over n; H: over the chunk's rows)
  int rows;   // rows of chunk c
};

// Stage s holds G(s) (if s < C) and H(s - D) (if 0 <= s - D < C): the H
// units of a chunk come D stages after its G units, which leaves the G^T
// reduction of the chunk D - 1 stages of slack (A of D + 1 chunks in L2).
__host__ __device__ inline int fused_total(const FusedSched &s) {
  const int TS = s.T * s.S * s.Gr, TlS = s.Tl * s.S * s.Gr, XR = s.X * s.RS * s.Gr;
  return (s.C - 1) * TS + TlS + s.C * XR;
}

// MULTI = false: a one-group launch (l_pad 64 always is), the group
// arithmetic folds away
template <bool MULTI = true>
__host__ __device__ __forceinline__ FusedUnit fused_decode(const FusedSched &s, int u) {
  const int Gr = MULTI ? s.Gr : 1;
  const int TS = s.T * s.S * Gr, TlS = s.Tl * s.S * Gr, XR = s.X * s.RS * Gr, F = TS + XR, D = s.D;
  int kind = 0, c = 0, r = 0;
#ifdef __CUDA_ARCH__
  if (s.order) {  // host-built order (tc_unit_order): any lag, including fractional stages
    const int e = __ldg(s.order + u);
    kind = e >> 30;
    c = (e >> 15) & 0x7fff;
    r = e & 0x7fff;
  } else
#endif
  {
  // region 1: stages 0 .. min(C, D) - 1, G units only
  const int size1 = s.C <= D ? (s.C - 1) * TS + TlS : D * TS;
  if (u < size1) {
    c = min(u / TS, s.C - 1);
    r = u - c * TS;
  } else {
    u -= size1;
    const int n2 = s.C > D ? s.C - D : 0;  // region 2: stages D .. C - 1, G(s) then H(s - D)
    bool done = false;
    if (n2 > 0) {
      if (u < (n2 - 1) * F) {
        const int st = D + u / F;
        r = u - (st - D) * F;
        if (r < TS) {
          c = st;
        } else {
          kind = 1;
          c = st - D;
          r -= TS;
        }
        done = true;
      } else {
        u -= (n2 - 1) * F;
        if (u < TlS + XR) {
          if (u < TlS) {
            c = s.C - 1;
            r = u;
          } else {
            kind = 1;
            c = s.C - 1 - D;
            r = u - TlS;
          }
          done = true;
        } else {
          u -= TlS + XR;
        }
      }
    }
    if (!done) {  // region 3: stages max(C, D) .. C + D - 1, H units only
      const int st = (s.C > D ? s.C : D) + u / XR;
      kind = 1;
      c = st - D;
      r = u % XR;
    }
  }
  }
  FusedUnit f;
  f.kind = kind;
  f.c = c;
  f.g = r % Gr;  // a unit's column groups are adjacent in the sequence
  r /= Gr;
  f.rows = c == s.C - 1 ? s.rows_last : s.R0;
  if (kind == 0) {
    f.a = r / s.S;
    f.b = r - f.a * s.S;
    f.k0 = f.b * s.kseg;
    f.nk = min(s.kseg, s.nkb - f.k0);
  } else {  // row-segment major: consecutive units of one column tile are X apart
    f.b = r / s.X;
    f.a = r - f.b * s.X;
    f.k0 = f.b * s.hseg;
    f.nk = max(0, min(s.hseg, (f.rows + 31) / 32 - f.k0));
  }
  // whole MMA-warp iterations: an odd tail takes one more K block, which reads
  // zeros (columns >= n / rows beyond the launch are TMA out-of-bounds fill)
  if (s.kp > 1) f.nk = (f.nk + s.kp - 1) / s.kp * s.kp;
  return f;
}

template <int LPAD>
__device__ __forceinline__ GroupView group_view(const FusedArgs &a, int g) {
  if (LPAD == 64) g = 0;  // l_pad 64 sketches are one group: the offsets fold away
  GroupView v;
  const int64_t w = (int64_t)g * a.ctr_group;
  v.wy0 = a.wy0 + g * LPAD;
  v.gt_row0 = g * a.gT_rows_group;
  v.gpart = a.gpart + g * a.gpart_group;
  v.gT = a.gT + g * a.gT_group;
  v.g_out = a.g_out + g * LPAD;
  v.hpart = a.hpart + g * LPAD;
  v.left = a.left ? a.left + g * LPAD : nullptr;
  v.wsum = a.wsum ? a.wsum + g * LPAD : nullptr;
  v.seg_cnt = a.seg_cnt + w;
  v.ready = a.ready + w;
  v.hdone = a.hdone + w;
  v.hseq = a.hseq + w;
  v.trdy = a.trdy + w;
  v.colsum_on = a.colsum_on && g == 0;
  return v;
}

__device__ __forceinline__ int fused_real_tiles(const FusedSched &s, int c) {
  return c == s.C - 1 ? s.ntl : s.nt;
}

template <int LPAD>
struct PairBars {
  using C = TcCfg<LPAD>;
  uint64_t a_full[C::NA], a_empty[C::NA];  // local: A producer <-> converters
  uint64_t kb_full[C::NS];                 // leader: both CTAs' converters stored the TMEM stage
  uint64_t kb_empty[C::NS];                // each CTA: MMAs done with the TMEM stage
  uint64_t b_full[C::NB];                  // leader: both CTAs' B halves landed
  uint64_t b_empty[C::NB];                 // each CTA: MMAs done with the B stage
  uint64_t acc_full[2];                    // each CTA: accumulator period complete
  uint64_t acc_empty[2];                   // leader: both CTAs folded the period
  uint64_t epi_full[2], epi_empty[2];      // local: converters/promoters <-> epilogue staging
  uint32_t tmem_base;
};

// DUAL: clusters of four CTAs = two CTA pairs sketching two column groups of
// the same rows (l_pad 256 as two groups of 128): pair 0 loads every A tile
// once and multicasts it to the matching CTA of pair 1 (each A tile leaves
// L2 once for both groups), pair p computes group p. The cluster shape is
// compiled in (2, or 4 for DUAL): with the shape given as a launch attribute
// the cooperative launch failed under ncu (LaunchFailed, round 2 session 4),
// and the driver lists the smoke test's kernels with ncu.
template <int LPAD, bool NORM, bool SHIFT = false, bool DUAL = false>
__global__ void __cluster_dims__(DUAL ? 4 : 2, 1, 1) __launch_bounds__(TcCfg<LPAD>::THREADS, 1)
tc_pass_kernel(const __grid_constant__ CUtensorMap tAg, const __grid_constant__ CUtensorMap tAh,
               const __grid_constant__ CUtensorMap tWhi, const __grid_constant__ CUtensorMap tWlo,
               const __grid_constant__ CUtensorMap tGT,
#if SPCA_PAIRA
               const __grid_constant__ CUtensorMap tAg3, const __grid_constant__ CUtensorMap tAh2,
#endif
               const FusedArgs args) {
  using C = TcCfg<LPAD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ PairBars<LPAD> bars;
  __shared__ double stg_cs[C::NSTG][C::GROUPS * 128];  // H: per converter group, column-sum partial
  __shared__ int stg_bad[128];              // G epilogue: row of the tile has a non-finite partial
  __shared__ __align__(16) float sst[C::NA][64];      // norm, H blocks: a0 and 1/norm of the block's 32 rows
  __shared__ double stg_rs[C::NSTG][2][C::GROUPS * 128];  // norm, G units: per group sums of d and d^2
  __shared__ float sl_stat[128][2];                   // norm, G slice reduction: mean_d, inv per row
  const FusedSched &sc = args.s;

  static_assert(!DUAL || (!NORM && !SPCA_PAIRA && LPAD == 128), "dual pairs: plain / shift l_pad 128");
  // G slice reductions on their own two warps (fused normalisation keeps them on the epilogue warps)
  constexpr bool GTEAM = C::GT && !NORM && !DUAL;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = ptx::cluster_rank();
  const uint32_t rank = crank & 1u;              // rank in the CTA pair
  const uint32_t pid = DUAL ? crank >> 1 : 0u;   // pair in the cluster = column group (DUAL)
  const uint32_t leader = crank & ~1u;           // the pair's leader CTA (cluster rank)
  const uint16_t pmask = (uint16_t)(3u << (2 * pid));  // the pair's cluster ranks
  constexpr int CS = DUAL ? 4 : 2;               // CTAs per cluster
  const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  unsigned long long *trace = args.trace ? args.trace + (size_t)blockIdx.x * kTraceStride : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = ptx::globaltimer();

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NA; ++s) {
      ptx::mbar_init(&bars.a_full[s], 1);
      // the four warps of one converter group; paired slots: both groups (barriers [0, NP))
      // DUAL: pair 0's slot is also released by the matching CTA of pair 1 (multicast)
      ptx::mbar_init(&bars.a_empty[s], SPCA_PAIRA ? 8 : ((DUAL && pid == 0) ? 8 : 4));
    }
    for (int s = 0; s < C::NS; ++s) {
      ptx::mbar_init(&bars.kb_full[s], 2 * 4 * C::KP);  // KP converter groups (4 warps each) in each CTA
      ptx::mbar_init(&bars.kb_empty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      ptx::mbar_init(&bars.b_full[s], 1);
      ptx::mbar_init(&bars.b_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&bars.acc_full[s], 1);
      ptx::mbar_init(&bars.acc_empty[s], 2 * C::PROMO_WARPS);
    }
    for (int s = 0; s < C::NSTG; ++s) {
      ptx::mbar_init(&bars.epi_full[s], C::CONV + 32 * C::PROMO_WARPS);  // converters (column sums) + promoters
      ptx::mbar_init(&bars.epi_empty[s], kTcEpi);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch(&tAg);
    ptx::tma_prefetch(&tAh);
    ptx::tma_prefetch(&tWhi);
    ptx::tma_prefetch(&tWlo);
    ptx::tma_prefetch(&tGT);
#if SPCA_PAIRA
    ptx::tma_prefetch(&tAg3);
    ptx::tma_prefetch(&tAh2);
#endif
  }
  if (threadIdx.x < 128) stg_bad[threadIdx.x] = 0;
  if (warp == 1) ptx::tmem_alloc2(&bars.tmem_base, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // both CTAs' barriers exist before any cross-CTA arrive
  ptx::tc_fence_after();
  const uint32_t tmem = bars.tmem_base;

  // Phase B of a G unit's epilogue, once every K segment of the tile has written
  // its partial: reduce THIS segment's slice of the tile's rows over the S
  // partials in fixed order -> G rows (output), the split G^T operand of the H
  // units, the readiness counters. Run by the epilogue warps (nth = 128) or by
  // the reduction team (GTEAM: warp 3 and the last warp, nth = 64).
  auto g_phase_b = [&](const FusedUnit &f, const GroupView &gv, const int tile, const int e, const int nth,
                       const uint32_t barid) {
    constexpr int NQ = LPAD / 4;
    const int twoT = 2 * sc.T;
    const int gslot = f.c % kSlots;
    // reduce this segment's slice of the tile's rows over the S partials (fixed order)
    const int r0 = (f.b * 128) / sc.S, r1 = ((f.b + 1) * 128) / sc.S;
    const float *p0 = gv.gpart + (((size_t)gslot * twoT + tile) * sc.S) * 128 * LPAD;
#if SPCA_BRAW
    float *ghi = gv.gT + (size_t)gslot * LPAD * sc.R0;  // raw G^T of the slot
#else
    float *ghi = gv.gT + (size_t)(2 * gslot) * LPAD * sc.R0;
    float *glo = ghi + (size_t)LPAD * sc.R0;
#endif
    if (NORM) {
      // row statistics of the slice over the S segments (fixed order, fp64):
      // mean_d = mean(a) - a0, norm = ||a - mean(a)||, from sums of d = a - a0
      if (e < r1 - r0) {
        const int r = r0 + e, rc = tile * 128 + r;
        const double *rp = reinterpret_cast<const double *>(args.rstat_part) +
                           (((size_t)gslot * twoT + tile) * sc.S * 128 + r) * 2;
        double t1 = 0.0, t2 = 0.0;
        for (int z = 0; z < sc.S; ++z) {
          t1 += __ldcg(rp + (size_t)z * 256);
          t2 += __ldcg(rp + (size_t)z * 256 + 1);
        }
        const double md = t1 / (double)args.n;
        const double nrm = sqrt(fmax(t2 - t1 * md, 0.0));
        const double inv = nrm > 0.0 ? 1.0 / nrm : 1.0;
        const bool valid = rc < f.rows;
        const int64_t grow = (int64_t)f.c * sc.R0 + rc;
        sl_stat[r][0] = (float)md;
        sl_stat[r][1] = (float)inv;
        const size_t so = (size_t)gslot * sc.R0 + rc;
        args.row_a0[so] = valid ? __ldg(args.a + grow * args.lda) : 0.f;
        args.row_inv[so] = valid ? (float)inv : 1.f;
        if (valid) args.row_coef[grow] = md * inv;
      }
      ptx::named_bar(barid, nth);
    }
    // items = (row, 8-column group), ROW fastest: consecutive threads take
    // consecutive rows, so each G^T store of a warp covers consecutive rows
    // of one G^T row (coalesced; the row-major order scattered them one
    // row of G^T per lane: 1.5 ms of config 3's pass); a thread's two
    // float4 loads per partial fill one 32-byte sector
    const int nrs = r1 - r0;
    constexpr int NO = LPAD / 8;  // 8-column groups
#pragma unroll 1
    for (int it = e; it < nrs * NO; it += nth) {
      const int r = r0 + it % nrs, o = it / nrs;
      const int rc = tile * 128 + r;  // row within the chunk
      const bool valid = rc < f.rows;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int q = 2 * o + h2;
        // partials of other CTAs: read through L2 (.cg), never a stale L1 line
        const float4 *src = reinterpret_cast<const float4 *>(p0 + (size_t)r * LPAD) + q;
        float4 acc = __ldcg(src);
        int z = 1;
#if SPCA_GRED_WIDE
        // nine more loads in flight behind the first (config 2's ten K segments: one
        // L2 round trip per half instead of four), added in order z as below: the
        // reduction's latency is in front of G^T, which the H units wait for
        for (; z + 9 <= sc.S; z += 9) {
          float4 b9[9];
#pragma unroll
          for (int j = 0; j < 9; ++j) b9[j] = __ldcg(src + (size_t)(z + j) * 128 * NQ);
#pragma unroll
          for (int j = 0; j < 9; ++j) {
            acc.x += b9[j].x; acc.y += b9[j].y; acc.z += b9[j].z; acc.w += b9[j].w;
          }
        }
#endif
        for (; z + 4 <= sc.S; z += 4) {  // four loads in flight, added in order z
          float4 b4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) b4[j] = __ldcg(src + (size_t)(z + j) * 128 * NQ);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc.x += b4[j].x; acc.y += b4[j].y; acc.z += b4[j].z; acc.w += b4[j].w;
          }
        }
        for (; z < sc.S; ++z) {
          const float4 b4 = __ldcg(src + (size_t)z * 128 * NQ);
          acc.x += b4.x; acc.y += b4.y; acc.z += b4.z; acc.w += b4.w;
        }
        float a4[4] = {acc.x, acc.y, acc.z, acc.w};
        float b4[4] = {acc.x, acc.y, acc.z, acc.w};  // B operand of the H units
        if (gv.left != nullptr && valid) {  // co-sketch: H += A^T L
          const float4 l4 = __ldg(reinterpret_cast<const float4 *>(
                                      gv.left + ((int64_t)f.c * sc.R0 + rc) * args.gld) + q);
          b4[0] = l4.x; b4[1] = l4.y; b4[2] = l4.z; b4[3] = l4.w;
        }
        if (NORM) {  // G_hat = (d Omega - mean_d * 1^T Omega) / norm; the H units take G_hat / norm
          const float md = sl_stat[r][0], inv = sl_stat[r][1];
          const float4 w4 = __ldg(reinterpret_cast<const float4 *>(gv.wsum) + q);
          const float ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            a4[j] = fmaf(-md, ws[j], a4[j]) * inv;
            b4[j] = (gv.left != nullptr ? b4[j] : a4[j]) * inv;
          }
        }
        if (valid)
          reinterpret_cast<float4 *>(gv.g_out + ((int64_t)f.c * sc.R0 + rc) * args.gld)[q] =
              make_float4(a4[0], a4[1], a4[2], a4[3]);
#if SPCA_BRAW
#pragma unroll
        for (int j = 0; j < 4; ++j) ghi[(size_t)(4 * q + j) * sc.R0 + rc] = valid ? b4[j] : 0.f;
#else
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (args.dbg & 32768) break;  // profiling knob: no G^T stores
          float h1 = 0.f, l1 = 0.f;
          if (valid) split3(b4[j], h1, l1);
#if SPCA_BCOMB
          ghi[(size_t)bcomb_row(4 * q + j, 0, LPAD) * sc.R0 + rc] = h1;
          ghi[(size_t)bcomb_row(4 * q + j, 1, LPAD) * sc.R0 + rc] = l1;
#else
          ghi[(size_t)(4 * q + j) * sc.R0 + rc] = h1;
          glo[(size_t)(4 * q + j) * sc.R0 + rc] = l1;
#endif
        }
#endif
      }
    }
    ptx::fence_proxy_async_global();
    __threadfence();
    ptx::named_bar(barid, nth);
    if (e == 0) {
      atomicAdd(&gv.trdy[f.c * twoT + tile], 1);
      atomicAdd(&gv.ready[f.c], 1);
    }
  };

  if (warp == 0) {  // ---------------------------------------------- A producer
    // L2 policy of A: the G units' loads (from HBM) must survive until the H
    // units re-read the chunk D stages later; the H units' loads are the last use
    const uint64_t keep = (args.dbg & 4096) ? ptx::policy_evict_normal() : ptx::policy_evict_last();
    const uint64_t drop = (args.dbg & 8192) ? ptx::policy_evict_normal() : ptx::policy_evict_first();
    int gkb = 0;
#pragma unroll 1
    for (int u = cid; u < sc.total; u += ncl) {
      const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
      const int rbase = args.row_base + f.c * sc.R0;
      const int tile = 2 * f.a + (int)rank;
      const bool hstats = NORM && f.kind == 1 && f.nk > 0;
      if (hstats) {  // the row shifts / scales of chunk c come from its G reductions
        if (ptx::elect_one()) {
          if (args.tile_ready) {  // every tile this unit reads
            const int t0 = f.k0 >> 2, t1 = (f.k0 + f.nk - 1) >> 2;
            for (int t = t0; t <= t1; ++t) ptx::spin_until_geq(&gv.trdy[f.c * 2 * sc.T + t], sc.S);
          } else {
            ptx::spin_until_geq(&gv.ready[f.c], fused_real_tiles(sc, f.c) * sc.S);
          }
          ptx::fence_proxy_async_global();
        }
        __syncwarp();
      }
#if SPCA_PAIRA
      // pairs of K blocks: one request (3-D box of two K blocks / 64-row box) per pair
#pragma unroll 1
      for (int kb = 0; kb < f.nk; kb += 2, ++gkb) {
        const int p = gkb % C::NP, nb = min(2, f.nk - kb);
        if (gkb >= C::NP) ptx::mbar_wait(&bars.a_empty[p], ((gkb / C::NP) - 1) & 1);
        if (ptx::elect_one()) {
          uint8_t *st = smem + 2 * p * C::A_BYTES;
          if (args.dbg & 8) {
            ptx::mbar_arrive(&bars.a_full[p]);
          } else {
            ptx::mbar_arrive_expect_tx(&bars.a_full[p], nb * (C::A_BYTES + (hstats ? 256u : 0u)));
            if (hstats) {
              for (int j = 0; j < nb; ++j) {
                const size_t o = (size_t)(f.c % kSlots) * sc.R0 + (size_t)(f.k0 + kb + j) * 32;
                ptx::bulk_load(&sst[2 * p + j][0], args.row_a0 + o, 128, &bars.a_full[p]);
                ptx::bulk_load(&sst[2 * p + j][32], args.row_inv + o, 128, &bars.a_full[p]);
              }
            }
            if (f.kind == 0) {  // 128 rows x 32 k per block, row-major (swizzled)
              if (nb == 2 && args.g3d) {
                ptx::tma_load_3d_hint(st, &tAg3, &bars.a_full[p], 0, rbase + tile * 128, f.k0 + kb, keep);
              } else {
                for (int j = 0; j < nb; ++j)
                  ptx::tma_load_2d_hint(st + j * C::A_BYTES, &tAg, &bars.a_full[p], (f.k0 + kb + j) * 32,
                                        rbase + tile * 128, keep);
              }
            } else {            // 32 rows x 128 columns per block, unswizzled: one box of 64 rows
              ptx::tma_load_2d_hint(st, nb == 2 ? &tAh2 : &tAh, &bars.a_full[p], tile * 128,
                                    rbase + (f.k0 + kb) * 32, drop);
            }
          }
        }
        __syncwarp();
      }
#else
#pragma unroll 1
      for (int kb = 0; kb < f.nk; ++kb, ++gkb) {
        const int s = gkb % C::NA;
        if (gkb >= C::NA) ptx::mbar_wait(&bars.a_empty[s], ((gkb / C::NA) - 1) & 1);
        if (ptx::elect_one()) {
          uint8_t *st = smem + s * C::A_BYTES;
          if (args.dbg & 8) {
            ptx::mbar_arrive(&bars.a_full[s]);
          } else {
            ptx::mbar_arrive_expect_tx(&bars.a_full[s], C::A_BYTES + (hstats ? 256u : 0u));
            if (hstats) {
              const size_t o = (size_t)(f.c % kSlots) * sc.R0 + (size_t)(f.k0 + kb) * 32;
              ptx::bulk_load(&sst[s][0], args.row_a0 + o, 128, &bars.a_full[s]);
              ptx::bulk_load(&sst[s][32], args.row_inv + o, 128, &bars.a_full[s]);
            }
            const int kx = (args.dbg & 2048) ? 0 : (f.k0 + kb) * 32;  // profiling knob: L2-resident A
            const int ry = (args.dbg & 2048) ? 0 : rbase;
            if (DUAL) {
              // pair 0 fetches the tile once for both pairs: same offset in this CTA and in
              // the matching CTA of pair 1 (whose producer only posts its expected bytes)
              if (pid == 0) {
                const uint16_t mc = (uint16_t)((1u << crank) | (1u << (crank + 2)));
                if (f.kind == 0)
                  ptx::tma_load_2d_mc(st, &tAg, &bars.a_full[s], kx, ry + tile * 128, mc, keep);
                else
                  ptx::tma_load_2d_mc(st, &tAh, &bars.a_full[s], tile * 128,
                                      ry + ((args.dbg & 2048) ? 0 : (f.k0 + kb) * 32), mc, drop);
              }
            } else if (f.kind == 0) {  // 128 rows x 32 k, row-major (swizzled)
              ptx::tma_load_2d_hint(st, &tAg, &bars.a_full[s], kx, ry + tile * 128, keep);
            } else {            // 32 rows x 128 columns, one unswizzled box
              ptx::tma_load_2d_hint(st, &tAh, &bars.a_full[s], tile * 128, ry + ((args.dbg & 2048) ? 0 : (f.k0 + kb) * 32), drop);
            }
          }
        }
        __syncwarp();
      }
#endif
    }
  } else if (warp == 2) {  // ---------------------------------- B producer (half)
    const uint64_t keep = ptx::policy_evict_last();
    int gkb = 0, ui = 0;
#pragma unroll 1
    for (int u = cid; u < sc.total; u += ncl, ++ui) {
      const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
      const int gslot = f.c % kSlots;
      const bool hwait = f.kind == 1 && f.nk > 0 && !(args.dbg & 16384);
      if (hwait && !args.tile_ready) {  // G^T of chunk c must be complete
        if (ptx::elect_one()) {
          ptx::spin_until_geq(&gv.ready[f.c], fused_real_tiles(sc, f.c) * sc.S);
          ptx::fence_proxy_async_global();
        }
        __syncwarp();
      }
      if (lane == 0) SPCA_TRACE(ui, 7);
      int wtile = -1;  // tile_ready: last 128-row tile of G^T known complete
#pragma unroll 1
      for (int kb = 0; kb < f.nk; ++kb, ++gkb) {
        if (hwait && args.tile_ready && ((f.k0 + kb) >> 2) != wtile) {  // the block's rows' G^T
          wtile = (f.k0 + kb) >> 2;
          if (ptx::elect_one()) {
            ptx::spin_until_geq(&gv.trdy[f.c * 2 * sc.T + wtile], sc.S);
            ptx::fence_proxy_async_global();
          }
          __syncwarp();
        }
        const int s = gkb % C::NB;
        if (gkb >= C::NB) ptx::mbar_wait(&bars.b_empty[s], ((gkb / C::NB) - 1) & 1);
        if (ptx::elect_one()) {
          uint8_t *st = smem + C::B_OFF + s * C::B_STAGE;
          const uint32_t bar = ptx::mapa(ptx::smem_u32(&bars.b_full[s]), leader);
          const int k = (f.k0 + kb) * 32;
#if SPCA_BRAW
          (void)bar;
          if (args.dbg & 4) {
            ptx::mbar_arrive(&bars.b_full[s]);
          } else {
            // this CTA's l_pad/2 raw rows of Omega^T (G units) or of G^T slot (H units),
            // completing on its own barrier (its converters split them)
            constexpr int HR = LPAD / 2;
            ptx::mbar_arrive_expect_tx(&bars.b_full[s], C::BH_BYTES);
            const int y = (f.kind == 0 ? gv.wy0 : gv.gt_row0 + gslot * LPAD) + HR * (int)rank;
            ptx::tma_load_2d_hint(st, f.kind == 0 ? &tWhi : &tGT, &bars.b_full[s], k, y, keep);
          }
#else
          if (args.dbg & 4) {
            if (rank == 0) ptx::mbar_arrive(&bars.b_full[s]);
          } else {
          if (rank == 0) ptx::mbar_arrive_expect_tx(&bars.b_full[s], 2 * C::B_STAGE);
          constexpr int HR = LPAD / 2;  // rows per B box
          // rows of W_hi / W_lo in the maps: Omega^T (G units) or G^T slot (H units)
          const CUtensorMap *mh = f.kind == 0 ? &tWhi : &tGT, *ml = f.kind == 0 ? &tWlo : &tGT;
          const int yh = f.kind == 0 ? gv.wy0 : gv.gt_row0 + 2 * gslot * LPAD,
                    yl = f.kind == 0 ? gv.wy0 : gv.gt_row0 + (2 * gslot + 1) * LPAD;
          if constexpr (C::STACKED) {
            const CUtensorMap *m01 = rank == 0 ? mh : ml;
            const int y01 = rank == 0 ? yh : yl;
            ptx::tma_load_2d_pair(st, m01, bar, k, y01, keep);
            ptx::tma_load_2d_pair(st + C::BH_BYTES, m01, bar, k, y01 + HR, keep);
            ptx::tma_load_2d_pair(st + 2 * C::BH_BYTES, mh, bar, k, yh + HR * (int)rank, keep);
          } else if (SPCA_BCOMB) {  // this CTA's hi and lo rows: one box of LPAD rows
            const int yc = f.kind == 0 ? 2 * gv.wy0 + LPAD * (int)rank : gv.gt_row0 + (2 * gslot + (int)rank) * LPAD;
            ptx::tma_load_2d_pair(st, mh, bar, k, yc, keep);
          } else {
            ptx::tma_load_2d_pair(st, mh, bar, k, yh + HR * (int)rank, keep);
            ptx::tma_load_2d_pair(st + C::BH_BYTES, ml, bar, k, yl + HR * (int)rank, keep);
          }
          }
#endif
        }
        __syncwarp();
      }
    }
#ifdef SPCA_FINE_TRACE
  } else if (warp == 3) {  // profiling: completion time of each K block's MMAs (pair 0, leader)
    if (trace && cid == 0 && rank == 0 && lane == 0) {
      unsigned long long *ct_ = args.trace + 256 * kTraceStride + 4 * kTraceMma + 6 * kTraceConv;
      int gkb = 0;
      for (int u = cid; u < sc.total && gkb < kTraceMma; u += ncl) {
        const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
        for (int kb = 0; kb < f.nk && gkb < kTraceMma; ++kb, ++gkb) {
          ptx::mbar_wait(&bars.kb_empty[(gkb % C::NS) / C::KP], (gkb / C::NS) & 1);
          ct_[gkb] = clock64();
        }
      }
    }
#endif
  } else if (warp == 1) {  // ------------------------- MMA issuer (leader CTA)
    if (rank == 0) {
      const uint64_t bdesc0 = ptx::sdesc_sw128(ptx::smem_u32(smem + C::B_OFF), 16, 1024);
      int gkb = 0, gq = 0, ui = 0;
#pragma unroll 1
      for (int u = cid; u < sc.total; u += ncl, ++ui) {
        const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
#pragma unroll 1
        for (int kb = 0; kb < f.nk; kb += C::KP, gkb += C::KP) {
          if (lane == 0 && kb == 0) SPCA_TRACE(ui, 5);
          const int ks = gkb % C::NS, bs = gkb % C::NB;
          const int q = gq + kb / kPromote, buf = q & 1;
          const bool first = (kb % kPromote) == 0;
#ifdef SPCA_FINE_TRACE
          unsigned long long *mt = (trace && cid == 0 && lane == 0 && gkb < kTraceMma)
                                       ? args.trace + 256 * kTraceStride + 4 * gkb : nullptr;
#else
          constexpr unsigned long long *mt = nullptr;
#endif
          if (mt) mt[0] = clock64();
          if (first && q >= 2) ptx::mbar_wait(&bars.acc_empty[buf], ((q >> 1) - 1) & 1);
          if (mt) mt[1] = clock64();
          ptx::mbar_wait(&bars.kb_full[ks / C::KP], (gkb / C::NS) & 1);
          if (mt) mt[2] = clock64();
#if !SPCA_RELAY
          static_assert(C::KP == 1, "the B ring handshake through the MMA warp is per K block");
          ptx::mbar_wait(&bars.b_full[bs], (gkb / C::NB) & 1);
#endif
          if (mt) mt[3] = clock64();
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            if (!(args.dbg & 2)) {
#pragma unroll
              for (int j = 0; j < C::KP; ++j)  // the iteration's K blocks: operand stages ks + j, B stages (gkb + j) % NB
                tc_mma_stage2<LPAD>(tmem + C::A_TMEM + 64 * (ks + j), tmem + buf * C::ACC_COLS,
                                    bdesc0 + (uint64_t)((((gkb + j) % C::NB) * C::B_STAGE) >> 4), first && j == 0);
            }
            ptx::mma2_commit_both(&bars.kb_empty[ks / C::KP], pmask);
#if !SPCA_RELAY
            ptx::mma2_commit_both(&bars.b_empty[bs], pmask);
#endif
            if (((kb + C::KP - 1) % kPromote) == kPromote - 1 || kb + C::KP >= f.nk)
              ptx::mma2_commit_both(&bars.acc_full[buf], pmask);
          }
          __syncwarp();
        }
        gq += (f.nk + kPromote - 1) / kPromote;
      }
    }
  } else if (warp >= 4 && warp < 4 + C::CONV / 32) {  // -------------------- converters
    const int ct = threadIdx.x - 128;
    const int t = ct & 127;    // TMEM lane: G row / H column within the tile
    const int grp = ct >> 7;   // converts the K blocks kb = grp (mod GROUPS)
    const uint32_t lane_base = tmem + ((uint32_t)(t & ~31) << 16);
    const uint32_t kbfull_l = ptx::mapa(ptx::smem_u32(&bars.kb_full[0]), leader);
    int gkb = 0, ui = 0, gpa = 0;  // gpa: A slot pairs consumed (SPCA_PAIRA)
#pragma unroll 1
    for (int u = cid; u < sc.total; u += ncl, ++ui) {
      const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
      float cs = 0.f, cc = 0.f;   // H: column sum (fp32 Kahan over the unit)
      // fused normalisation, G units: shift every value of the row by its first
      // value a0 (d = a - a0; exact for nearby values) and sum d, d^2 (Kahan)
      float a0 = 0.f, s1 = 0.f, s1c = 0.f, s2 = 0.f, s2c = 0.f;
      if (NORM && f.kind == 0) {
        const int rt = (2 * f.a + (int)rank) * 128 + t;  // row within the chunk
        if (rt < f.rows) a0 = __ldg(args.a + ((int64_t)f.c * sc.R0 + rt) * args.lda);
      }
      if (ct == 0) SPCA_TRACE(ui, 0);
#pragma unroll 1
      for (int kb = grp; kb < f.nk; kb += C::GROUPS) {
        const int gk = gkb + kb;
#if SPCA_PAIRA
        const int ga = gpa + (kb >> 1), ab = ga % C::NP;  // A slot pair of this block
        const int s = 2 * ab + (kb & 1), ts = gk % C::NS;
#else
        const int ga = gk, ab = gk % C::NA;
        const int s = ab, ts = gk % C::NS;
#endif
#ifdef SPCA_FINE_TRACE
        unsigned long long *ctr = (trace && blockIdx.x == 0 && ct == 0 && (gk >> 1) < kTraceConv)
                                      ? args.trace + 256 * kTraceStride + 4 * kTraceMma + 6 * (gk >> 1) : nullptr;
#else
        constexpr unsigned long long *ctr = nullptr;
#endif
        if (ctr) ctr[0] = clock64();
        ptx::mbar_wait(&bars.a_full[ab], (ga / (SPCA_PAIRA ? C::NP : C::NA)) & 1);
        if (ctr) ctr[1] = clock64();
        // Load and split first, then wait for the TMEM stage: the stage is held
        // only for the two stores, which keeps the stage round trip (converters
        // -> MMA -> commit -> converters) short; the TMEM ring is shallow.
        // All 32 K values of this row (G) / column (H): hi = v with its low 13
        // mantissa bits cleared, lo = v - hi (exact); the tensor core reads lo as
        // tf32 (low 13 bits dropped): the operand keeps ~21 significant bits.
        // Non-finite inputs are found from their G rows in the epilogue.
        float v[32], hi[32];
        if (!(args.dbg & 1)) {
          if (f.kind == 0) {
            const uint32_t row = ptx::smem_u32(smem + s * C::A_BYTES + t * 128);
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
              const float4 x = ptx::lds128(row + ((q4 ^ (t & 7)) << 4));
              v[4 * q4] = x.x; v[4 * q4 + 1] = x.y; v[4 * q4 + 2] = x.z; v[4 * q4 + 3] = x.w;
            }
            if (SHIFT) {  // column shift (zero beyond n: padded)
              const float4 *cp = reinterpret_cast<const float4 *>(args.cshift + (f.k0 + kb) * 32);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const float4 c4 = __ldg(cp + q4);
                v[4 * q4] -= c4.x; v[4 * q4 + 1] -= c4.y; v[4 * q4 + 2] -= c4.z; v[4 * q4 + 3] -= c4.w;
              }
            }
            if (NORM) {  // d = a - a0 on the row's real columns; d, d^2 pairwise then Kahan
              const int col0 = (f.k0 + kb) * 32;
              float p1[16], p2[16];
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = col0 + i < args.n ? v[i] - a0 : 0.f;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                p1[i] = v[2 * i] + v[2 * i + 1];
                p2[i] = fmaf(v[2 * i], v[2 * i], v[2 * i + 1] * v[2 * i + 1]);
              }
#pragma unroll
              for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
                for (int i = 0; i < w; ++i) {
                  p1[i] = p1[i] + p1[i + w];
                  p2[i] = p2[i] + p2[i + w];
                }
              float y = p1[0] - s1c, tt = s1 + y;
              s1c = (tt - s1) - y;
              s1 = tt;
              y = p2[0] - s2c;
              tt = s2 + y;
              s2c = (tt - s2) - y;
              s2 = tt;
            }
          } else {
            const uint32_t raw = ptx::smem_u32(smem + s * C::A_BYTES + t * 4);  // column t
#pragma unroll
            for (int kq = 0; kq < 32; ++kq) v[kq] = ptx::lds32(raw + kq * 512);
            if (SHIFT) {  // column shift on the chunk's real rows only
              const float cj = __ldg(args.cshift + (2 * f.a + (int)rank) * 128 + t);
              const int r0 = (f.k0 + kb) * 32;
#pragma unroll
              for (int kq = 0; kq < 32; ++kq) v[kq] = r0 + kq < f.rows ? v[kq] - cj : 0.f;
            }
            float p16[16];  // pairwise sum of the 32 values, then one Kahan step
            if (NORM) {  // d = a - a0 per row; the column sum weights rows by 1/norm
              const uint32_t st_ = ptx::smem_u32(&sst[s][0]);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const float4 s0 = ptx::lds128(st_ + 16 * q4), w4 = ptx::lds128(st_ + 128 + 16 * q4);
                v[4 * q4] -= s0.x; v[4 * q4 + 1] -= s0.y; v[4 * q4 + 2] -= s0.z; v[4 * q4 + 3] -= s0.w;
                hi[4 * q4] = v[4 * q4] * w4.x;
                hi[4 * q4 + 1] = v[4 * q4 + 1] * w4.y;
                hi[4 * q4 + 2] = v[4 * q4 + 2] * w4.z;
                hi[4 * q4 + 3] = v[4 * q4 + 3] * w4.w;
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) p16[i] = hi[2 * i] + hi[2 * i + 1];
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) p16[i] = v[2 * i] + v[2 * i + 1];
            }
#pragma unroll
            for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
              for (int i = 0; i < w; ++i) p16[i] = p16[i] + p16[i + w];
            const float y = p16[0] - cc;
            const float tt = cs + y;
            cc = (tt - cs) - y;
            cs = tt;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            hi[i] = trunc_tf32(v[i]);
            v[i] -= hi[i];
          }
        }
        // every lane's loads were consumed by the split above: the landing slot
        // can go back to TMA (one lane's arrive would not order the other lanes'
        // outstanding shared loads against the next TMA write)
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&bars.a_empty[ab]);
          // DUAL, pair 1: the slot's data came from pair 0's multicast; its producer
          // refills this CTA's slot too, so it waits for this release as well
          if (DUAL && pid == 1) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&bars.a_empty[ab]), crank - 2));
        }
        if (gk >= C::NS) {
          ptx::mbar_wait(&bars.kb_empty[ts / C::KP], ((gk / C::NS) - 1) & 1);
#if SPCA_RELAY
          // block gk - NS is done: its B stage goes back to this CTA's B producer
          // (one arrival per block: lane 0 of the group's first warp)
          if (t == 0) ptx::mbar_arrive(&bars.b_empty[(gk - C::NS) % C::NB]);
#endif
        }
        if (ctr) ctr[2] = clock64();
        ptx::tc_fence_after();
        const uint32_t tst = lane_base + C::A_TMEM + 64 * ts;
        if (!(args.dbg & 1)) {
          ptx::tmem_st32(tst, hi);
          ptx::tmem_st32(tst + 32, v);
        }
        if (ctr) ctr[3] = clock64();
        ptx::tmem_wait_st();
        if (ctr) ctr[4] = clock64();
#if SPCA_BRAW
        {  // this CTA's raw B half landed: write its lo part beside it (16-byte
           // chunks at the same offsets, so the swizzled layout carries over)
          const int bs = gk % C::NB;
          ptx::mbar_wait(&bars.b_full[bs], (gk / C::NB) & 1);
          const uint32_t b0 = ptx::smem_u32(smem + C::B_OFF + bs * C::B_STAGE);
          constexpr int PER = (int)(C::BH_BYTES / (16 * 128));  // chunks per thread of the group
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const uint32_t off = (uint32_t)(i * 128 + t) * 16;
            const float4 x = ptx::lds128(b0 + off);
            ptx::st_shared_v4(b0 + C::BH_BYTES + off,
                              make_float4(braw_lo(x.x), braw_lo(x.y), braw_lo(x.z), braw_lo(x.w)));
          }
          ptx::fence_proxy_async_smem();  // generic writes -> the tensor core's reads
        }
#elif SPCA_RELAY
        // the leader's converters also vouch for the block's B stage (both CTAs'
        // halves complete on the leader's barrier): the MMA warp waits on kb_full only
        if (rank == 0) ptx::mbar_wait(&bars.b_full[gk % C::NB], (gk / C::NB) & 1);
#endif
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(kbfull_l + 8 * (ts / C::KP));
        if (ctr) ctr[5] = clock64();
      }
#if SPCA_PAIRA
      if (grp == 1 && (f.nk & 1)) {  // the unit's last pair holds one block: release the empty half
        const int ga = gpa + (f.nk >> 1), ab = ga % C::NP;
        ptx::mbar_wait(&bars.a_full[ab], (ga / C::NP) & 1);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&bars.a_empty[ab]);
      }
      gpa += (f.nk + 1) >> 1;
#endif
      gkb += f.nk;
      if (ct == 0) SPCA_TRACE(ui, 1);
      // hand the column-sum partial to the epilogue with the unit's staging
      const int sb = ui % C::NSTG;  // staging buffer of this unit
      if (ui >= C::NSTG) ptx::mbar_wait(&bars.epi_empty[sb], ((ui / C::NSTG) - 1) & 1);
      if (f.kind == 1) stg_cs[sb][grp * 128 + t] = (double)cs - (double)cc;
      if (NORM && f.kind == 0) {
        stg_rs[sb][0][grp * 128 + t] = (double)s1 - (double)s1c;
        stg_rs[sb][1][grp * 128 + t] = (double)s2 - (double)s2c;
      }
      ptx::mbar_arrive(&bars.epi_full[sb]);
    }
  } else if (warp >= C::PROMO_BASE / 32 && warp < C::EPI_BASE / 32) {  // ----- promoters
    const int pt = threadIdx.x - C::PROMO_BASE;
    const int t = pt & 127;              // TMEM lane: G row / H column within the tile
    const int c0 = (pt >> 7) * 64;       // this thread's 64 output columns
    const uint32_t lane_base = tmem + ((uint32_t)(t & ~31) << 16);
    const uint32_t accempty_l = ptx::mapa(ptx::smem_u32(&bars.acc_empty[0]), leader);
    const uint32_t stg_row = ptx::smem_u32(smem + C::STG_OFF + t * LPAD * 4);
    int gq = 0, ui = 0;
#pragma unroll 1
    for (int u = cid; u < sc.total; u += ncl, ++ui) {
      const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
      const int nq = (f.nk + kPromote - 1) / kPromote;
      float racc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) racc[i] = 0.f;
      // fold each accumulator period into fp32 registers (round-to-nearest adds:
      // the tensor core's own accumulation truncates) and hand it back
#pragma unroll 1
      for (int qq = 0; qq < nq; ++qq, ++gq) {
        const int buf = gq & 1;
        ptx::mbar_wait(&bars.acc_full[buf], (gq >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t base = lane_base + buf * C::ACC_COLS + c0;
        if (!(args.dbg & 512))
#pragma unroll
        for (int c = 0; c < 64; c += 8) {
          float v[8];
          ptx::tmem_ld8(base + c, v);
          if constexpr (C::STACKED) {  // + the A_hi W_lo half of the accumulator
            float w[8];
            ptx::tmem_ld8(base + LPAD + c, w);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += w[i];
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) racc[c + i] += v[i];
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(accempty_l + 8 * buf);
      }
      if (pt == 0) SPCA_TRACE(ui, 6);
      constexpr bool kPGP = SPCA_PROMO_GP == 2 || (SPCA_PROMO_GP == 1 && LPAD == 128);
      const int sb = ui % C::NSTG;  // staging buffer of this unit
      if (kPGP && f.kind == 0) {
        // G partial straight to its slot (row t, columns c0..c0+63); the slot was
        // last used kSlots chunks ago: its slices must have been reduced
        const int tile = 2 * f.a + (int)rank;
        float chk = 0.f;
        if (tile < fused_real_tiles(sc, f.c) && !(args.dbg & 131072)) {
          if (f.c >= kSlots) {
            if (lane == 0) ptx::spin_until_geq(&gv.ready[f.c - kSlots], sc.nt * sc.S);
            __syncwarp();
          }
          float4 *gp = reinterpret_cast<float4 *>(
              gv.gpart + ((((size_t)(f.c % kSlots) * 2 * sc.T + tile) * sc.S + f.b) * 128 + t) * LPAD + c0);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            gp[i] = make_float4(racc[4 * i], racc[4 * i + 1], racc[4 * i + 2], racc[4 * i + 3]);
            chk = fmaf(racc[4 * i], 0.f, fmaf(racc[4 * i + 1], 0.f, fmaf(racc[4 * i + 2], 0.f, fmaf(racc[4 * i + 3], 0.f, chk))));
          }
          __threadfence();  // the partial is visible before the epilogue counts it
        }
        // the epilogue has cleared the previous unit's flags once it released that unit
        if (ui >= C::NSTG) ptx::mbar_wait(&bars.epi_empty[sb], ((ui / C::NSTG) - 1) & 1);
        if (!(chk == 0.f)) stg_bad[t] = 1;  // a non-finite value in this row's partial
        if (pt == 0) SPCA_TRACE(ui, 2);
        ptx::mbar_arrive(&bars.epi_full[sb]);
        continue;
      }
      // stage the result for the epilogue warps (16-byte chunks XOR-swizzled by row)
      if (ui >= C::NSTG) ptx::mbar_wait(&bars.epi_empty[sb], ((ui / C::NSTG) - 1) & 1);
      if (pt == 0) SPCA_TRACE(ui, 2);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int q = c0 / 4 + i;
        ptx::st_shared_v4(stg_row + sb * C::STG_BYTES + ((SPCA_BULK_EPI ? q : (q ^ (t & 7))) << 4),
                          make_float4(racc[4 * i], racc[4 * i + 1], racc[4 * i + 2], racc[4 * i + 3]));
      }
      if (SPCA_BULK_EPI) ptx::fence_proxy_async_smem();  // the staging leaves through the TMA engine
      ptx::mbar_arrive(&bars.epi_full[sb]);
    }
  } else if (GTEAM && (warp == 3 || (C::GT_THREADS == 64 && warp == C::THREADS / 32 - 1))) {  // reduction team
    // G units only: wait (on the global segment counter) until every K segment of
    // the unit's tile has published its partial, then run phase B. Decoupled from
    // the epilogue warps: no local hand-off is needed, the counter says it all.
    const int tb = (warp == 3 ? 0 : 32) + lane;
#pragma unroll 1
    for (int u = cid; u < sc.total; u += ncl) {
      const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      if (f.kind != 0 || (args.dbg & 16384)) continue;
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
      const int tile = 2 * f.a + (int)rank;
      if (tile >= fused_real_tiles(sc, f.c)) continue;
      if (tb == 0) {
        ptx::spin_until_geq(&gv.seg_cnt[f.c * 2 * sc.T + tile], sc.S);  // every segment's partial is in
        if (f.c >= kSlots) ptx::spin_until_geq(&gv.hdone[f.c - kSlots], sc.nx * sc.RS);
      }
      ptx::named_bar(3, C::GT_THREADS);
      g_phase_b(f, gv, tile, tb, C::GT_THREADS, 3u);
    }
  } else if (warp >= C::EPI_BASE / 32) {  // --------------------------------- epilogue
    const int e = threadIdx.x - C::EPI_BASE;  // row (G) / column (H) of the tile
    constexpr int NQ = LPAD / 4;             // 16-byte chunks per row
    const int twoT = 2 * sc.T;
    int ui = 0;
#pragma unroll 1
    for (int u = cid; u < sc.total; u += ncl, ++ui) {
      const FusedUnit f = fused_decode<(LPAD != 64) && !DUAL>(sc, u);
      const GroupView gv = group_view<LPAD>(args, DUAL ? (int)pid : f.g);
      const int tile = 2 * f.a + (int)rank;
      const int sb = ui % C::NSTG;  // staging buffer of this unit
      ptx::mbar_wait(&bars.epi_full[sb], (ui / C::NSTG) & 1);
      if (e == 0) SPCA_TRACE(ui, 3);
      if (args.dbg & 16384) {  // profiling knob: no epilogue work (results are garbage)
        ptx::mbar_arrive(&bars.epi_empty[sb]);
        continue;
      }
      if (f.kind == 0) {  // ---------------------------------- G epilogue
        const int gslot = f.c % kSlots;
        const bool real = tile < fused_real_tiles(sc, f.c);
        const int row = tile * 128 + e;
        bool flagged = false;
        constexpr bool kPGP = SPCA_PROMO_GP == 2 || (SPCA_PROMO_GP == 1 && LPAD == 128);
        if (kPGP && real) {  // the promoters wrote the partial and flagged non-finite rows
          ptx::named_bar(2, kTcEpi);
          if (NORM) {  // this segment's row sums of d, d^2 (the two converter groups, in order)
            double *rp = reinterpret_cast<double *>(args.rstat_part) +
                         ((((size_t)gslot * twoT + tile) * sc.S + f.b) * 128 + e) * 2;
            double r0s = stg_rs[sb][0][e], r1s = stg_rs[sb][1][e];
#pragma unroll
            for (int g2 = 1; g2 < C::GROUPS; ++g2) {
              r0s += stg_rs[sb][0][g2 * 128 + e];
              r1s += stg_rs[sb][1][g2 * 128 + e];
            }
            rp[0] = r0s;
            rp[1] = r1s;
          }
          flagged = stg_bad[e] != 0;
          ptx::named_bar(2, kTcEpi);  // every flag read before it is cleared for the next unit
          stg_bad[e] = 0;
        } else if (real) {
          // the partial slot was last used kSlots chunks ago: its slices must be reduced
          if (f.c >= kSlots && e == 0) ptx::spin_until_geq(&gv.ready[f.c - kSlots], sc.nt * sc.S);
          ptx::named_bar(2, kTcEpi);
          // copy the staged tile to its partial slot, NQ consecutive lanes per row
          // (each warp store covers whole rows: coalesced)
          float4 *gp = reinterpret_cast<float4 *>(
              gv.gpart + (((size_t)gslot * twoT + tile) * sc.S + f.b) * 128 * LPAD);
          const uint32_t stg0 = ptx::smem_u32(smem + C::STG_OFF + sb * C::STG_BYTES);
#if SPCA_BULK_EPI
          if (e == 0) {  // the whole staged tile -> its partial slot, one bulk copy
            ptx::bulk_store(gp, stg0, 128 * LPAD * 4);
            ptx::bulk_commit();
          }
#pragma unroll 4
          for (int it = e; it < 128 * NQ; it += kTcEpi) {  // non-finite check only
            const int r = it / NQ, q = it % NQ;
            const float4 x = ptx::lds128(stg0 + r * LPAD * 4 + (q << 4));
            const float chk = fmaf(x.x, 0.f, fmaf(x.y, 0.f, fmaf(x.z, 0.f, x.w * 0.f)));
            if (!(chk == 0.f)) stg_bad[r] = 1;
          }
          if (e == 0) ptx::bulk_wait_read0();
#else
#pragma unroll 4
          for (int it = e; it < 128 * NQ; it += kTcEpi) {
            const int r = it / NQ, q = it % NQ;
            const float4 x = ptx::lds128(stg0 + r * LPAD * 4 + ((q ^ (r & 7)) << 4));
            const float chk = fmaf(x.x, 0.f, fmaf(x.y, 0.f, fmaf(x.z, 0.f, x.w * 0.f)));
            if (!(chk == 0.f)) stg_bad[r] = 1;
            if (!(args.dbg & 131072)) gp[it] = x;  // profiling knob: no partial copy
          }
#endif
          if (NORM) {  // this segment's row sums of d, d^2 (the two converter groups, in order)
            double *rp = reinterpret_cast<double *>(args.rstat_part) +
                         ((((size_t)gslot * twoT + tile) * sc.S + f.b) * 128 + e) * 2;
            double r0s = stg_rs[sb][0][e], r1s = stg_rs[sb][1][e];
#pragma unroll
            for (int g2 = 1; g2 < C::GROUPS; ++g2) {
              r0s += stg_rs[sb][0][g2 * 128 + e];
              r1s += stg_rs[sb][1][g2 * 128 + e];
            }
            rp[0] = r0s;
            rp[1] = r1s;
          }
          ptx::named_bar(2, kTcEpi);
          flagged = stg_bad[e] != 0;
          stg_bad[e] = 0;
        }
        ptx::mbar_arrive(&bars.epi_empty[sb]);
        if (real) {
          // a non-finite input makes its G row non-finite: confirm on the raw row
          // segment (a huge finite row may also overflow G; the reference only
          // rejects non-finite values)
          if (flagged && row < f.rows) {
            const int64_t grow = (int64_t)f.c * sc.R0 + row;
            const float *ar = args.a + grow * args.lda;
            const int k1 = min(args.n, (f.k0 + f.nk) * 32);
            bool bad = false;
            for (int k = f.k0 * 32; k < k1 && !bad; ++k) bad = !isfinite(ar[k]);
            if (bad) report_bad_row(args.bad_row, args.first_row + grow);
          }
          // every writer fences its own stores before the count (a fence by one
          // thread does not drain the other warps' outstanding stores)
#if SPCA_BULK_EPI
          if (e == 0) {  // the partial's bulk copy is performed and ordered before the count
            ptx::bulk_wait0();
            ptx::fence_proxy_async_global();
          }
#endif
          __threadfence();
          ptx::named_bar(2, kTcEpi);
          int *cnt = &gv.seg_cnt[f.c * twoT + tile];
          if constexpr (GTEAM) {
            // the reduction team (warp 3 + the last warp) takes the unit from here: it
            // waits for the tile's other K segments and reduces this segment's slice,
            // so these warps are free for the next unit's staged result at once
            if (e == 0) atomicAdd(cnt, 1);
          } else {
            if (e == 0) {
              atomicAdd(cnt, 1);
              ptx::spin_until_geq(cnt, sc.S);  // every segment's partial is in
              if (f.c >= kSlots) ptx::spin_until_geq(&gv.hdone[f.c - kSlots], sc.nx * sc.RS);
            }
            ptx::named_bar(2, kTcEpi);
            g_phase_b(f, gv, tile, e, kTcEpi, 2u);
          }
        }
      } else {  // ------------------------------------------------ H epilogue
        const bool real = tile < sc.nx;
        const int seq = f.c * sc.RS + f.b;
        const int col = tile * 128 + e;
        double csv = 0.0;
        if (real) {
          if (e == 0) ptx::spin_until_geq(&gv.hseq[tile], seq);
          ptx::named_bar(2, kTcEpi);
#if SPCA_BULK_EPI
          {  // H row e += staged row e, one bulk reduce-add per row (at L2); the launch
             // zeroed H when it does not accumulate (the first unit of a tile adds to 0)
            const uint32_t stg0 = ptx::smem_u32(smem + C::STG_OFF + sb * C::STG_BYTES);
            if (col < args.n) {
              ptx::bulk_reduce_add_f32(gv.hpart + (int64_t)col * args.gld, stg0 + e * LPAD * 4, LPAD * 4);
              ptx::bulk_commit();
              ptx::bulk_wait_read0();
            }
          }
#else
          {  // H rows of the tile's columns, NQ consecutive lanes per column (coalesced)
            float *hp0 = gv.hpart + (int64_t)tile * 128 * args.gld;
            const bool overwrite = !args.accumulate && seq == 0;
            const uint32_t stg0 = ptx::smem_u32(smem + C::STG_OFF + sb * C::STG_BYTES);
            const int items = min(128, args.n - tile * 128) * NQ;
            // batches of 8 items: the 8 old values are loaded before any store
            // (a store between loads would serialize them on the L2 round trip:
            // the compiler cannot tell the rows apart)
            constexpr int kB = 8;
            for (int it0 = e; it0 < ((args.dbg & 65536) ? 0 : items); it0 += kB * kTcEpi) {  // knob: no H RMW
              float4 o[kB];
#pragma unroll
              for (int j = 0; j < kB; ++j) {
                const int it = it0 + j * kTcEpi;
                o[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (!overwrite && it < items)
                  o[j] = __ldcg(reinterpret_cast<const float4 *>(hp0 + (int64_t)(it / NQ) * args.gld) + it % NQ);
              }
#pragma unroll
              for (int j = 0; j < kB; ++j) {
                const int it = it0 + j * kTcEpi;
                if (it >= items) break;
                const int r = it / NQ, q = it % NQ;
                float4 w = ptx::lds128(stg0 + r * LPAD * 4 + ((q ^ (r & 7)) << 4));
                w.x += o[j].x; w.y += o[j].y; w.z += o[j].z; w.w += o[j].w;
                reinterpret_cast<float4 *>(hp0 + (int64_t)r * args.gld)[q] = w;
              }
            }
          }
#endif
          csv = stg_cs[sb][e];
#pragma unroll
          for (int g2 = 1; g2 < C::GROUPS; ++g2) csv += stg_cs[sb][g2 * 128 + e];
        }
        ptx::mbar_arrive(&bars.epi_empty[sb]);
        if (real) {
          if (col < args.n && gv.colsum_on) {
            if (args.carry) {
              const double y = csv - __ldcg(args.carry + col);
              const double s0 = __ldcg(args.colsum + col);
              const double tt = s0 + y;
              args.carry[col] = (tt - s0) - y;
              args.colsum[col] = tt;
            } else {
              args.colsum[col] = __ldcg(args.colsum + col) + csv;
            }
          }
#if SPCA_BULK_EPI
          if (col < args.n) {  // this row's reduce-add is performed before the release
            ptx::bulk_wait0();
            ptx::fence_proxy_async_global();
          }
#endif
          __threadfence();
          ptx::named_bar(2, kTcEpi);
          if (e == 0) {
            ptx::st_release(&gv.hseq[tile], seq + 1);
            atomicAdd(&gv.hdone[f.c], 1);
          }
        }
      }
      if (e == 0) SPCA_TRACE(ui, 4);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // the peer's TMEM and barriers stay live until the leader is done
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, kTmemCols);
  }
  if (trace && threadIdx.x == 0) trace[1] = ptx::globaltimer();
}

}  // namespace spca
