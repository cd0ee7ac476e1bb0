// postpass.cuh — the blocked QB post-pass on hand-written fp64 kernels.
//
// Reference: blocked_qb (/root/reference/pkg/src/streampca/qb.py:59-135),
// Algorithm 4 steps 9-17. For sketch block i (columns
// [c0, c0 + b) of G, Q = the c0 columns already accepted):
//
//   y   = G_i - Q (B Omega_i)                          qb.py:96
//   Q_i R_i = qr(y)          (CholeskyQR2)             qb.py:97
//   Q_i Rt  = qr(Q_i - Q (Q^T Q_i))   (re-orth., CholeskyQR2)  qb.py:111-114
//   R_i <- Rt R_i;  B_i from R_i^-T (H_i^T - (y^T Q) B - (Omega_i^T B^T) B)  qb.py:115-118
//
// The tall-skinny work of a block (Q is m x c0 with m up to 5e6) is six
// sweeps over the rows. Every sweep is ONE kernel computing, per row,
//
//   t = y M - Q X        (M: b x b, X: c0 x b; either term may be absent)
//
// and folding t^T [Q | t] into per-CTA partial sums; the sweeps differ only
// in M, X, the output and the sums kept:
//
//   S1  M = I,               X = B Omega_i   write y = t;  [t^T Q | t^T t]
//   S2  M = R1^-1                            t^T t
//   S3  M = R1^-1 R2^-1                      t^T Q      (-> X of S4, transposed)
//   S4  M = R1^-1 R2^-1,     X = Q^T Q2      write z = t;  t^T t
//   S5  M = R3^-1                            t^T t
//   S6  M = R3^-1 R4^-1                      write Q[:, c0:c0+b] = t
//
// (CholeskyQR2: R = chol(y^T y), Q1 = y R^-1, twice). The right-side
// triangular solves of the library form become products with the inverse
// triangular factors (formed once per block, b <= 16), so a sweep is a pure
// fp64 tensor-core contraction: M = rows, N = b, K = b + c0 — no serial
// per-row substitution holding the tile. One fixed-order reduction of the
// partials and one single-warp kernel for the b x b algebra follow each
// reducing sweep (Cholesky factors, triangular inverses, CholeskyQR2's
// acceptance test, the deficiency test |r_jj| < RANK_TOL max ||G_j|| of
// qb.py:100 and solve_rt's singularity guard of linalg.py:131-135). Any
// failed test sets a device flag; the host checks it once per factorization
// and falls back to the general (Householder / repair) path. No float
// atomics: results are bitwise reproducible.
//
// Roofline: HBM. Per block the sweeps read Q three times (S1, S3, S4) and
// the m x b blocks y / z seven times: ~ 8 m (3 c0 + 9 b) bytes; the DMMA work
// (b padded to 16 columns) stays below the fp64 tensor rate for c0 <= 512.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tc_ptx.cuh"

namespace spca {

constexpr int kQbMaxB = 16;     // block sizes up to 16 (the reference's default is 10)
constexpr int kQbMaxCat = 256;  // c0 + b columns reduced per sweep (l <= 256: config 5 has 250)
constexpr int kQbThreads = 256; // 8 warps; thread 0 also issues the TMA loads
constexpr int kQbWarps = kQbThreads / 32;
// Row strides (doubles) of the t tile and of the [M; -X] operand block: 24
// = 8 mod 16, so a DMMA fragment load (4 rows x 8 consecutive doubles) hits
// each bank once per 128-byte wavefront (a stride of 16 made it 4-way)
constexpr int kQbLdt = 24;
constexpr int kQbLdw = 24;
constexpr int kQbNtw = kQbMaxCat / 8 / kQbWarps;   // 8-column tiles of [Q | t] per warp (at most)
constexpr int kQbMaxStages = 3;
constexpr double kQbCq1Cond = 16.0;  // one-pass CholeskyQR up to this Frobenius condition number

struct QbSweepArgs {
  int64_t m;
  int c0, b, tr, stages;  // accepted Q columns, block width, rows per tile (16/32/64), ring depth (2/3)
  int nslab;              // 16-column slabs of Q loaded per tile (0: Q not read)
  const double *mt;       // b x b (row-major): t = y mt, or null (identity)
  const double *x;        // c0 x b: t -= Q x, or null
  double *out;            // m x b output rows (row stride ldo) or null
  int64_t ldo;
  double *part;           // [gridDim.x][b][c0 + b]
  const double *y1d;      // y rows as one contiguous m x b block (row stride b): each tile is
                          // one 1-D bulk copy instead of a tensor-map box of narrow rows
  const double *skip;     // nonzero *skip: the sweep is not needed (one-pass CholeskyQR), or null
};

// fp64 tensor-core step D(16x8) += A(16x4, row) B(4x8, col) (fragments: a0 =
// A[g][t], a1 = A[g+8][t], b = B[t][g]; d = D[g][2t..2t+1], D[g+8][2t..2t+1];
// g = lane / 4, t = lane % 4)
__device__ __forceinline__ void qb_dmma(double (&d)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b));
}

// Stage layout (bytes): nslab Q slabs of [tr][16] doubles with the TMA's
// 128-byte swizzle (16-byte chunk c of row r at chunk c ^ (r & 7)), then the
// y tile [tr][b] (unswizzled).
__host__ __device__ inline size_t qb_stage_bytes(int nslab, int b, int tr) {
  return (size_t)nslab * tr * 128 + (((size_t)tr * b * 8 + 1023) & ~(size_t)1023);
}
// operand block [M; -X] as one K x 16 matrix, K = b (padded to 4) + c0 (padded to 4)
__host__ __device__ inline int qb_km(int b) { return (b + 3) & ~3; }
__host__ __device__ inline int qb_kb(int c0, int b) { return qb_km(b) + ((c0 + 3) & ~3); }
__host__ __device__ inline size_t qb_sweep_smem(int c0, int b, int tr, int nslab, int stages) {
  return 1024 + stages * qb_stage_bytes(nslab, b, tr) +
         sizeof(double) * ((size_t)tr * kQbLdt + (size_t)qb_kb(c0, b) * kQbLdw + kQbThreads * 4);
}
// element (r, k) of a swizzled Q slab set
__device__ __forceinline__ double qb_qs(const uint8_t *qs, int tr, int r, int k) {
  const int j = k >> 4, kk = k & 15;
  return *reinterpret_cast<const double *>(qs + (size_t)j * tr * 128 + r * 128 + ((((kk >> 1) ^ (r & 7))) << 4) +
                                           ((kk & 1) << 3));
}

// One sweep over the rows in tiles of tr. Thread 0 streams each tile's Q
// slabs and y rows into a two- or three-stage ring (tensor-map boxes; the
// contiguous y scratch as one bulk copy); a stage is refilled as soon as
// the tile it held is done. KIND (compile time): kX t -= Q X, kP reduce
// t^T Q, kW reduce t^T t, kOut write t. Per tile:
//   A. t = y M - Q X on the fp64 tensor cores (DMMA m16n8k4): one task per
//      (16-row tile, 8-column half of b), K = b (padded to 4) then c0; the
//      task writes its fragments to the output rows and to the t tile;
//   B. accumulate t^T [Q | t] (M = b padded to 16, N = 8-column tiles,
//      K = the tile's rows): the Q part in ceil(c0 / 8) column tiles, the t
//      part in NH tiles after them, dealt to the warps; with fewer tiles than
//      warps the rows are split over the warps (kspl row groups), whose sums
//      are added in a fixed order at the end.
constexpr int kQbX = 1, kQbP = 2, kQbW = 4, kQbOut = 8;
template <int B, int KIND>
__global__ void __launch_bounds__(kQbThreads, 2) qb_sweep_kernel(const __grid_constant__ CUtensorMap tq,
                                                                 const __grid_constant__ CUtensorMap ty,
                                                                 const QbSweepArgs a) {
  extern __shared__ __align__(1024) uint8_t qsm_raw[];
  // 1024-byte aligned base by offset arithmetic on the shared pointer (an
  // integer round trip would hide the address space: generic loads)
  uint8_t *qsm = qsm_raw + ((1024u - (ptx::smem_u32(qsm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kQbMaxStages];
  constexpr int b = B;
  constexpr int NH = B > 8 ? 2 : 1;  // 8-column halves of b
  constexpr int KM = (B + 3) & ~3;   // rows of M in the operand block
  constexpr bool HX = KIND & kQbX, WP = KIND & kQbP, WW = KIND & kQbW, WO = KIND & kQbOut;
  if (a.skip && *a.skip != 0.0) return;  // uniform over the grid
  const int c0 = a.c0, tr = a.tr, nslab = a.nslab, nst = a.stages;
  const int c04 = (c0 + 3) & ~3, kb = qb_kb(c0, b);
  const size_t sbytes = qb_stage_bytes(nslab, b, tr);
  const size_t qbytes = (size_t)nslab * tr * 128;
  double *ts = reinterpret_cast<double *>(qsm + nst * sbytes);  // [tr][kQbLdt]
  double *ws = ts + (size_t)tr * kQbLdt;                        // [kb][kQbLdw]: M rows [0, KM), -X rows [KM, kb)
  double *red = ws + (size_t)kb * kQbLdw;                       // [warps][32][4] end-of-sweep sums
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fg = lane >> 2, ft = lane & 3;
  const int64_t ntiles = (a.m + tr - 1) / tr;
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_mbar_init();
  }
  for (int i = tid; i < kb * kQbLdw; i += kQbThreads) {
    const int k = i / kQbLdw, j = i - k * kQbLdw;
    double v = 0.0;
    if (k < KM) {
      if (k < b && j < b) v = a.mt ? a.mt[k * b + j] : (k == j ? 1.0 : 0.0);
    } else if (HX && k - KM < c0 && j < b) {
      v = -a.x[(k - KM) * b + j];
    }
    ws[i] = v;
  }
  for (int i = tid; i < tr * kQbLdt; i += kQbThreads) ts[i] = 0.0;
  __syncthreads();
  auto issue = [&](int it) {  // tile `it` of this CTA -> stage it % nst
    const int64_t tile = blockIdx.x + (int64_t)it * gridDim.x;
    if (tile >= ntiles) return;
    const int s = it % nst;
    uint8_t *st = qsm + s * sbytes;
    const int y0 = (int)(tile * tr);
    const int rows = (int)(a.m - y0 < (int64_t)tr ? a.m - y0 : (int64_t)tr);
    // tensor-map boxes arrive whole (rows past m as zeros); the bulk copy
    // takes the valid rows only (consumers mask the rest)
    const uint32_t ybytes = a.y1d ? (uint32_t)rows * b * 8 : (uint32_t)tr * b * 8;
    ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)qbytes + ybytes);
    for (int j = 0; j < nslab; ++j) ptx::tma_load_2d(st + (size_t)j * tr * 128, &tq, &full[s], 16 * j, y0);
    if (a.y1d)
      ptx::bulk_load(st + qbytes, a.y1d + (size_t)y0 * b, ybytes, &full[s]);
    else
      ptx::tma_load_2d(st + qbytes, &ty, &full[s], 0, y0);
  };
  if (tid == 0)
    for (int it = 0; it < nst; ++it) issue(it);

  // column tiles of the reduction: [0, ntq) Q columns 8 nt.., [ntq, ntq + NH) t columns
  const int ntq = WP ? (c0 + 7) / 8 : 0;
  const int nlive = ntq + (WW ? NH : 0);
  // row groups: the split minimising the busiest warp's share of part B,
  // ceil(nlive / (warps / kspl)) tiles of tr / kspl rows each (at most
  // kQbNtw tiles per warp; ties to fewer groups). nlive = 10 (c0 = 60) was
  // dealt 2 tiles to two warps and 1 to the rest (kspl 1); kspl 2 gives 3
  // half-height tiles to every column group.
  int kspl = 8;
  {
    int best = 1 << 30;
    for (int k = 1; k <= kQbWarps; k *= 2) {
      const int per = (nlive + kQbWarps / k - 1) / (kQbWarps / k);
      if (per > kQbNtw) continue;
      const int cost = per * (kQbWarps / k);  // per / k in units of 1 / warps
      if (cost < best) {
        best = cost;
        kspl = k;
      }
    }
  }
  const int cgs = kQbWarps / kspl;                                                  // column-tile stride
  const int rsub = warp % kspl, cg = warp / kspl;
  double acc[kQbNtw][4];
#pragma unroll
  for (int u = 0; u < kQbNtw; ++u)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[u][i] = 0.0;

  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % nst;
    ptx::mbar_wait(&full[s], (it / nst) & 1);
    const uint8_t *qs = qsm + s * sbytes;
    const double *ys = reinterpret_cast<const double *>(qs + qbytes);
    const int64_t row0 = tile * tr;
    const int rows = (int)(a.m - row0 < (int64_t)tr ? a.m - row0 : (int64_t)tr);
    // A. t = y M - Q X
    for (int task = warp; task < (tr / 16) * NH; task += kQbWarps) {
      const int rt = task / NH, nh = task - rt * NH;
      const int r0 = rt * 16 + fg, col = 8 * nh + fg;
      double d[4][4] = {};  // four independent accumulation chains, summed in a fixed order
#pragma unroll
      for (int k = 0; k < KM; k += 4) {  // y M (K = b padded to 4)
        const int kk = k + ft;
        const double a0 = kk < b && r0 < rows ? ys[r0 * b + kk] : 0.0;
        const double a1 = kk < b && r0 + 8 < rows ? ys[(r0 + 8) * b + kk] : 0.0;
        qb_dmma(d[(k >> 2) & 3], a0, a1, ws[kk * kQbLdw + col]);
      }
      if (HX) {  // - Q X
        const double *wx = ws + (size_t)(KM + ft) * kQbLdw + col;
        int k = 0;
        for (; k + 16 <= c04; k += 16) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int kc = k + 4 * c + ft;
            qb_dmma(d[c], qb_qs(qs, tr, r0, kc), qb_qs(qs, tr, r0 + 8, kc), wx[(k + 4 * c) * kQbLdw]);
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // the last K steps (fewer than 16)
          if (k + 4 * c < c04) {
            const int kc = k + 4 * c + ft;
            qb_dmma(d[c], qb_qs(qs, tr, r0, kc), qb_qs(qs, tr, r0 + 8, kc), wx[(k + 4 * c) * kQbLdw]);
          }
        }
      }
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (d[0][q] + d[1][q]) + (d[2][q] + d[3][q]);
      const int cc = 8 * nh + 2 * ft;  // this lane's two columns; rows r0 and r0 + 8
      double *t0 = ts + (size_t)r0 * kQbLdt + cc;
      t0[0] = v[0];
      t0[1] = v[1];
      t0[8 * kQbLdt] = v[2];
      t0[8 * kQbLdt + 1] = v[3];
      if (WO && cc < b) {  // b is even: both columns are real
        if (r0 < rows) *reinterpret_cast<double2 *>(a.out + (row0 + r0) * a.ldo + cc) = make_double2(v[0], v[1]);
        if (r0 + 8 < rows)
          *reinterpret_cast<double2 *>(a.out + (row0 + r0 + 8) * a.ldo + cc) = make_double2(v[2], v[3]);
      }
    }
    if (WP || WW) {
      __syncthreads();  // t complete
      // B. acc[u] += t^T [Q | t], column tile cg + u cgs of this warp, its row group
#pragma unroll 2
      for (int r = 4 * rsub; r < tr; r += 4 * kspl) {
        const double a0 = ts[(r + ft) * kQbLdt + fg], a1 = B > 8 ? ts[(r + ft) * kQbLdt + fg + 8] : 0.0;
#pragma unroll
        for (int u = 0; u < kQbNtw; ++u) {
          const int nt = cg + u * cgs;
          if (nt >= nlive) break;
          const double bv = nt < ntq ? qb_qs(qs, tr, r + ft, nt * 8 + fg)
                                     : ts[(r + ft) * kQbLdt + (nt - ntq) * 8 + fg];
          qb_dmma(acc[u], a0, a1, bv);
        }
      }
    }
    __syncthreads();  // every warp is done with stage s and ts: refill the stage
    if (tid == 0) issue(it + nst);
  }
  if (!(WP || WW)) return;
  // this CTA's partial [t^T Q | t^T t] (b x (c0 + b)): the row groups of a
  // column tile added in the fixed order rsub = 0, 1, .. (one owned tile
  // per round through shared memory)
  const int ncat = c0 + b;
  double *p = a.part + (size_t)blockIdx.x * b * ncat;
#pragma unroll
  for (int u = 0; u < kQbNtw; ++u) {
    if (u * cgs >= nlive) break;  // uniform over the CTA
#pragma unroll
    for (int q = 0; q < 4; ++q) red[(warp * 32 + lane) * 4 + q] = acc[u][q];
    __syncthreads();
    const int nt = cg + u * cgs;
    if (rsub == 0 && nt < nlive) {
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[q] = 0.0;
        for (int g = 0; g < kspl; ++g) v[q] += red[((warp + g) * 32 + lane) * 4 + q];
      }
      // columns of [Q | t]: Q tiles cover [8 nt, 8 nt + 8) (only < c0 kept),
      // t tiles cover t columns [8 (nt - ntq), ..) (only < b kept)
      const bool isq = nt < ntq;
      const int kc = (isq ? nt : nt - ntq) * 8 + 2 * ft, lim = isq ? c0 : b, off = isq ? 0 : c0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = fg + 8 * h;
        if (i >= b) continue;
        if (kc < lim) p[(size_t)i * ncat + off + kc] = v[2 * h];
        if (kc + 1 < lim) p[(size_t)i * ncat + off + kc + 1] = v[2 * h + 1];
      }
    }
    __syncthreads();
  }
}

// red[e] = sum of part[z][e] over z in a fixed order: a block takes 32
// entries, its 8 warps the parts z = w (mod 8), each lane summing its
// entry's parts in order; the 8 partial sums are combined pairwise in a
// fixed tree (deterministic). Only the entries of the sweep's reduced
// columns are meaningful. xt (optional): c0 x b transpose of the t^T Q part,
// the next sweep's X.
__global__ void __launch_bounds__(256) qb_reduce_kernel(const double *__restrict__ part, int nparts, int b,
                                                        int ncat, double *red, double *xt, int c0) {
  __shared__ double sh[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int ne = b * ncat;
  double s = 0.0;
  if (e < ne) {
    int z = w;
    for (; z + 8 * 7 < nparts; z += 8 * 8) {  // eight loads in flight, added in order
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = part[(size_t)(z + 8 * j) * ne + e];
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
    for (; z < nparts; z += 8) s += part[(size_t)z * ne + e];
  }
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < ne) {
    const double v = ((sh[0][lane] + sh[1][lane]) + (sh[2][lane] + sh[3][lane])) +
                     ((sh[4][lane] + sh[5][lane]) + (sh[6][lane] + sh[7][lane]));
    red[e] = v;
    const int i = e / ncat, k = e - i * ncat;
    if (xt && k < c0) xt[(size_t)k * b + i] = v;
  }
}

// ------------------------------------------------- b x b algebra (one warp)
// upper Cholesky W = R^T R (row-major b x b in shared memory); false when W
// is not numerically positive definite (cholesky_ex info != 0)
__device__ bool qb_chol_upper_w(const double *w, double *r, int b) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < b * b; e += 32) r[e] = 0.0;
  __syncwarp();
  bool ok = true;
  for (int j = 0; j < b; ++j) {
    if (lane == 0) {
      double d = w[j * b + j];
      for (int k = 0; k < j; ++k) d = fma(-r[k * b + j], r[k * b + j], d);
      r[j * b + j] = d > 0.0 ? sqrt(d) : nan("");
    }
    __syncwarp();
    const double rjj = r[j * b + j];
    ok = ok && rjj > 0.0;
    const int i = j + 1 + lane;
    if (i < b) {
      double s = w[j * b + i];
      for (int k = 0; k < j; ++k) s = fma(-r[k * b + j], r[k * b + i], s);
      r[j * b + i] = s / rjj;
    }
    __syncwarp();
  }
  return ok;
}
// c = x y for upper triangular b x b matrices
__device__ void qb_mul_upper_w(const double *x, const double *y, double *c, int b) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < b * b; e += 32) {
    const int i = e / b, j = e - i * b;
    double s = 0.0;
    for (int k = i; k <= j; ++k) s = fma(x[i * b + k], y[k * b + j], s);
    c[e] = j >= i ? s : 0.0;
  }
  __syncwarp();
}
// ri = r^-1 (upper triangular): lane j solves r x = e_j by back substitution
__device__ void qb_inv_upper_w(const double *r, double *ri, int b) {
  const int j = threadIdx.x & 31;
  if (j < b) {
    double x[kQbMaxB];
#pragma unroll
    for (int i = 0; i < kQbMaxB; ++i) x[i] = 0.0;
    x[j] = 1.0 / r[j * b + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s = fma(r[i * b + k], x[k], s);
      x[i] = -s / r[i * b + i];
    }
    for (int i = 0; i < b; ++i) ri[i * b + j] = x[i];
  }
  __syncwarp();
}

// Small b x b algebra between sweeps (b <= 16, one warp). `st` holds the
// block's matrices, each b x b row-major:
//   [0] R1  [1] R2  [2] r_i = R2 R1  [3] R3  [4] R4  [5] R_i = R4 R3 r_i
//   [6] R1^-1  [7] R1^-1 R2^-1  [8] R3^-1  [9] R3^-1 R4^-1
//  op 1: R1 = chol(W), [6]
//  op 2: CholeskyQR2 test on W = Q1^T Q1 (max |W - I| < 1e-5), R2 = chol(W),
//        r_i, [7], deficiency test |r_i,jj| >= tol (qb.py:100)
//  op 3: R3 = chol(W), [8]
//  op 4: test on W = Z1^T Z1, R4 = chol(W), R_i, [9], singularity guard on
//        diag(R_i) (linalg.py:131-135)
// the b x b algebra of one step on W (shared memory, row-major b x b), by
// warp 0 of the calling block
__device__ void qb_small_ops(int op, int b, const double *w, double *st, int *flag, const double *tol,
                             bool allow_one = false, double *skip_out = nullptr) {
  __shared__ double f[10][kQbMaxB * kQbMaxB], tmp[kQbMaxB * kQbMaxB];
  const int bb = b * b, lane = threadIdx.x & 31;
  for (int e = lane; e < bb; e += 32)
    for (int q = 0; q < 10; ++q) f[q][e] = st[q * bb + e];
  __syncwarp();
  bool ok = true;
  if (op == 1 || op == 3) {
    double *R = op == 1 ? f[0] : f[3];
    double *Ri = op == 1 ? f[6] : f[8];
    ok = qb_chol_upper_w(w, R, b);
    qb_inv_upper_w(R, Ri, b);
    // One-pass CholeskyQR suffices when the block is well conditioned: its
    // orthogonality defect is ~ eps cond(y)^2, so with cond_F(R) = ||R||_F
    // ||R^-1||_F <= kQbCq1Cond (cond_2 <= cond_F) the second pass would only
    // correct ~1e-13. Then R2 = I (R4 = I): the steps of op 2 (op 4) run here
    // and the second pass's sweep and reduction are skipped on the device.
    double fr = 0.0, fi = 0.0;
    for (int e = lane; e < bb; e += 32) {
      fr += R[e] * R[e];
      fi += Ri[e] * Ri[e];
    }
    for (int o = 16; o > 0; o >>= 1) {
      fr += __shfl_xor_sync(0xffffffffu, fr, o);
      fi += __shfl_xor_sync(0xffffffffu, fi, o);
    }
    const bool one = allow_one && ok && sqrt(fr) * sqrt(fi) <= kQbCq1Cond && isfinite(fr * fi);
    if (one) {
      double *Rb = op == 1 ? f[1] : f[4];
      for (int e = lane; e < bb; e += 32) {
        Rb[e] = (e / b == e % b) ? 1.0 : 0.0;
        (op == 1 ? f[7] : f[9])[e] = Ri[e];
      }
      __syncwarp();
      if (op == 1) {
        for (int e = lane; e < bb; e += 32) f[2][e] = R[e];  // r_i = R1
        __syncwarp();
        const double tl = *tol;
        for (int j = lane; j < b; j += 32) {
          const double d = f[2][j * b + j];
          ok = ok && isfinite(d) && !(fabs(d) < tl);
        }
      } else {
        qb_mul_upper_w(f[3], f[2], f[5], b);  // R_i = R3 r_i
        double mx = 0.0;
        for (int j = 0; j < b; ++j) mx = fmax(mx, fabs(f[5][j * b + j]));
        for (int j = lane; j < b; j += 32) {
          const double d = fabs(f[5][j * b + j]);
          ok = ok && isfinite(d) && !(d < 1e-300) && !(d < 1e-15 * mx);
        }
      }
    }
    if (lane == 0 && skip_out) *skip_out = one ? 1.0 : 0.0;
  } else {
    double defect = 0.0;
    for (int e = lane; e < bb; e += 32) defect = fmax(defect, fabs(w[e] - (e % (b + 1) == 0 ? 1.0 : 0.0)));
    for (int o = 16; o > 0; o >>= 1) defect = fmax(defect, __shfl_xor_sync(0xffffffffu, defect, o));
    ok = defect < 1e-5 && isfinite(defect);
    double *R = op == 2 ? f[1] : f[4];
    ok = qb_chol_upper_w(w, R, b) && ok;
    qb_inv_upper_w(R, tmp, b);
    qb_mul_upper_w(op == 2 ? f[6] : f[8], tmp, op == 2 ? f[7] : f[9], b);  // Ra^-1 Rb^-1
    if (op == 2) {
      qb_mul_upper_w(f[1], f[0], f[2], b);  // r_i = R2 R1
      const double tl = *tol;
      for (int j = lane; j < b; j += 32) {
        const double d = f[2][j * b + j];
        ok = ok && isfinite(d) && !(fabs(d) < tl);
      }
    } else {
      qb_mul_upper_w(f[4], f[3], tmp, b);  // Rt = R4 R3
      qb_mul_upper_w(tmp, f[2], f[5], b);  // R_i = Rt r_i
      double mx = 0.0;
      for (int j = 0; j < b; ++j) mx = fmax(mx, fabs(f[5][j * b + j]));
      for (int j = lane; j < b; j += 32) {
        const double d = fabs(f[5][j * b + j]);
        ok = ok && isfinite(d) && !(d < 1e-300) && !(d < 1e-15 * mx);
      }
    }
  }
  ok = __all_sync(0xffffffffu, ok);
  for (int e = lane; e < bb; e += 32)
    for (int q = 0; q < 10; ++q) st[q * bb + e] = f[q][e];
  if (lane == 0 && !ok) *flag = 1;
}

// Small b x b algebra between sweeps (b <= 16, one warp). `st` holds the
// block's matrices, each b x b row-major:
//   [0] R1  [1] R2  [2] r_i = R2 R1  [3] R3  [4] R4  [5] R_i = R4 R3 r_i
//   [6] R1^-1  [7] R1^-1 R2^-1  [8] R3^-1  [9] R3^-1 R4^-1
//  op 1: R1 = chol(W), [6]
//  op 2: CholeskyQR2 test on W = Q1^T Q1 (max |W - I| < 1e-5), R2 = chol(W),
//        r_i, [7], deficiency test |r_i,jj| >= tol (qb.py:100)
//  op 3: R3 = chol(W), [8]
//  op 4: test on W = Z1^T Z1, R4 = chol(W), R_i, [9], singularity guard on
//        diag(R_i) (linalg.py:131-135)
// W is the t^T t block of the reduced [t^T Q | t^T t] (b x ncat).
__global__ void qb_small_kernel(int op, int b, int ncat, int c0, const double *redm, double *st, int *flag,
                                const double *tol, int allow_one, double *skip_out) {
  __shared__ double w[kQbMaxB * kQbMaxB];
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < b * b; e += 32) w[e] = redm[(size_t)(e / b) * ncat + c0 + e % b];
  __syncwarp();
  qb_small_ops(op, b, w, st, flag, tol, allow_one != 0, skip_out);
}

// W-only sweeps (S2, S4, S5): the fixed-order reduction of the t^T t block
// of the partials AND the b x b step in one launch (one block): thread
// (entry e, group g) sums the parts z = g (mod 8) eight loads at a time, the
// eight group sums are added in a fixed tree, then warp 0 runs the step.
__global__ void __launch_bounds__(256) qb_wfinish_kernel(int op, int b, int ncat, int c0,
                                                         const double *__restrict__ part, int nparts, double *st,
                                                         int *flag, const double *tol, const double *skip,
                                                         int allow_one, double *skip_out) {
  __shared__ double sh[8][kQbMaxB * kQbMaxB], w[kQbMaxB * kQbMaxB];
  if (skip && *skip != 0.0) return;  // one-pass CholeskyQR: op 1 / op 3 did this step
  const int bb = b * b, ne = b * ncat;
  for (int i = threadIdx.x; i < 8 * bb; i += blockDim.x) {
    const int g = i / bb, e = i - g * bb;
    const size_t col = (size_t)(e / b) * ncat + c0 + e % b;  // t^T t entry in the b x ncat partial
    double s = 0.0;
    int z = g;
    for (; z + 8 * 7 < nparts; z += 8 * 8) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = part[(size_t)(z + 8 * j) * ne + col];
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
    for (; z < nparts; z += 8) s += part[(size_t)z * ne + col];
    sh[g][e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < bb; e += blockDim.x)
    w[e] = ((sh[0][e] + sh[1][e]) + (sh[2][e] + sh[3][e])) + ((sh[4][e] + sh[5][e]) + (sh[6][e] + sh[7][e]));
  __syncthreads();
  if (threadIdx.x < 32) qb_small_ops(op, b, w, st, flag, tol, allow_one != 0, skip_out);
}

}  // namespace spca

namespace spca {

// ------------------------------------------------ B side of a QB block
// The two n-long products of a block (qb.py:96 and :115-118) on fp64 CUDA
// cores: they read the accepted rows of B (c0 x n, up to 384 MB at config 5)
// once each, where library GEMMs of these skinny shapes ran at 1-3 TB/s.
//
// X = B[:c0] Omega_i (c0 x b), K = n split over the CTAs: a CTA stages its
// K-chunk of Omega_i (chunk x b) in shared memory; warp w takes rows
// w, w + 8, ... in groups of R, every lane a strided subset of the chunk's
// k, accumulating R x b sums that are butterfly-reduced across the warp in a
// fixed pattern; partials [chunk][c0][b] are reduced in a fixed order by
// qb_reduce_kernel (bitwise reproducible).
template <int B>
__global__ void __launch_bounds__(256, 2) qb_omega_proj_kernel(int64_t n, int c0, const double *__restrict__ bm,
                                                               int64_t ldb, const double *__restrict__ om,
                                                               int64_t ldo, int64_t kchunk,
                                                               double *__restrict__ part) {
  extern __shared__ __align__(16) double osm[];  // [B][kchunk]: lane-consecutive k, conflict-free
  constexpr int R = 2, U = 8;  // rows per warp pass, 32-wide k steps in flight (R * U loads per lane)
  const int64_t k0 = (int64_t)blockIdx.x * kchunk;
  const int kn = (int)(kchunk < n - k0 ? kchunk : n - k0);
  const int kc = (int)kchunk;
#pragma unroll 8
  for (int i = threadIdx.x; i < kn * B; i += blockDim.x) {  // eight loads in flight per thread
    const int k = i / B, j = i - k * B;
    osm[j * kc + k] = __ldg(om + (k0 + k) * ldo + j);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *p = part + (size_t)blockIdx.x * c0 * B;
  for (int r0 = warp * R; r0 < c0; r0 += 8 * R) {
    double acc[R][B];
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int j = 0; j < B; ++j) acc[q][j] = 0.0;
    for (int kb = 0; kb < kn; kb += 32 * U) {
      double bv[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kb + 32 * u + lane;
#pragma unroll
        for (int q = 0; q < R; ++q)
          bv[u][q] = (k < kn && r0 + q < c0) ? __ldg(bm + (size_t)(r0 + q) * ldb + k0 + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kb + 32 * u + lane;
        if (k < kn) {
#pragma unroll
          for (int j = 0; j < B; ++j) {
            const double ov = osm[j * kc + k];
#pragma unroll
            for (int q = 0; q < R; ++q) acc[q][j] = fma(bv[u][q], ov, acc[q][j]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int j = 0; j < B; ++j) {
        double v = acc[q][j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[q][j] = v;
      }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (r0 + q < c0)
#pragma unroll
          for (int j = 0; j < B; ++j) p[(size_t)(r0 + q) * B + j] = acc[q][j];
  }
}

// B_i (rows [c0, c0 + b) of B, all n columns) in one pass over B[:c0]:
//   B_i = R_i^-T (H_i^T - (y^T Q + X^T) B[:c0])       (qb.py:115-118)
// one thread per column k: rhs = H[k, c0:c0+b] - M B[:c0, k] with
// M = y^T Q + X^T (b x c0, in shared memory, read as broadcasts), then the
// lower-triangular solve with R_i^T by forward substitution.
template <int B>
__global__ void __launch_bounds__(256) qb_b_rows_kernel(int64_t n, int c0, const double *__restrict__ bm,
                                                        int64_t ldb, const double *__restrict__ h, int64_t ldh,
                                                        const double *__restrict__ p_out,
                                                        const double *__restrict__ x,
                                                        const double *__restrict__ ri, double *__restrict__ bout) {
  extern __shared__ __align__(16) double msm[];  // [c0][B]: M^T, then R_i (B x B)
  double *rs = msm + (size_t)c0 * B;
  const int ncat = c0 + B;
  for (int i = threadIdx.x; i < c0 * B; i += blockDim.x) {
    const int r = i / B, j = i - r * B;
    msm[i] = p_out[(size_t)j * ncat + r] + x[(size_t)r * B + j];
  }
  for (int i = threadIdx.x; i < B * B; i += blockDim.x) rs[i] = ri[i];
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double acc[B];
#pragma unroll
  for (int j = 0; j < B; ++j) acc[j] = h[k * ldh + j];
  int r = 0;
  for (; r + 8 <= c0; r += 8) {  // eight loads of B in flight
    double bv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) bv[u] = __ldg(bm + (size_t)(r + u) * ldb + k);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double *mr = msm + (r + u) * B;
#pragma unroll
      for (int j = 0; j < B; ++j) acc[j] = fma(-mr[j], bv[u], acc[j]);
    }
  }
  for (; r < c0; ++r) {
    const double bv = __ldg(bm + (size_t)r * ldb + k);
    const double *mr = msm + r * B;
#pragma unroll
    for (int j = 0; j < B; ++j) acc[j] = fma(-mr[j], bv, acc[j]);
  }
  // R_i^T z = acc: z_j = (acc_j - sum_{i<j} R[i][j] z_i) / R[j][j]
#pragma unroll
  for (int j = 0; j < B; ++j) {
    double s = acc[j];
#pragma unroll
    for (int i = 0; i < j; ++i) s = fma(-rs[i * B + j], acc[i], s);
    acc[j] = s / rs[j * B + j];
    bout[(size_t)j * ldb + k] = acc[j];
  }
}

}  // namespace spca
