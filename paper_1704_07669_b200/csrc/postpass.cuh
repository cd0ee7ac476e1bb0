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
// sweeps over the rows, each ONE kernel that streams its operands once and
// folds every product the step needs into per-CTA partial sums:
//
//   S1  t = G_i - Q X            write y = t;  reduce [t^T Q | t^T t]   (X = B Omega_i)
//   S2  t = y R1^-1                            reduce t^T t
//   S3  t = (y R1^-1) R2^-1                    reduce t^T Q
//   S4  t = (y R1^-1) R2^-1 - Q P2^T  write z = t;  reduce t^T t
//   S5  t = z R3^-1                            reduce t^T t
//   S6  t = (z R3^-1) R4^-1           write Q[:, c0:c0+b] = t
//
// (the triangular solves are applied per row by substitution, as a right-side
// trsm does), with one fixed-order reduction of the partials and one small
// single-CTA kernel for the b x b algebra after each reducing sweep
// (Cholesky factors, CholeskyQR2's acceptance test, the deficiency test
// |r_jj| < RANK_TOL max ||G_j|| of qb.py:100 and solve_rt's singularity
// guard of linalg.py:131-135). Any failed test sets a device flag; the host
// checks it once per factorization and falls back to the general
// (Householder / repair) path, which handles every such block. No float
// atomics: results are bitwise reproducible.
//
// Roofline: HBM. Per block the sweeps read Q three times (S1, S3, S4) and
// the m x b blocks y / z seven times: ~ 8 m (3 c0 + 9 b) bytes; the DFMA work
// (~4 m c0 b per block) stays below the fp64 rate for c0 <= 512.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace spca {

constexpr int kQbThreads = 256;
constexpr int kQbMaxB = 16;    // block sizes up to 16 (the reference's default is 10)
constexpr int kQbMaxCat = 512; // c0 + b columns reduced per sweep (2 per thread)

struct QbSweepArgs {
  int64_t m;
  int c0, b, tr;          // accepted Q columns, block width, rows per tile
  const double *q;        // m x c0 (row stride ldq) or null when c0 == 0
  int64_t ldq;
  const double *yin;      // m x b input rows (row stride ldy)
  int64_t ldy;
  const double *ra, *rb;  // b x b upper triangular (row-major): t = (yin ra^-1) rb^-1, either may be null
  const double *x;        // c0 x b: t -= Q x, or null
  double *out;            // m x b output rows (row stride ldo) or null
  int64_t ldo;
  int want_p, want_w;     // reduce t^T Q (b x c0) / t^T t (b x b)
  double *part;           // [gridDim.x][b][c0 + b]
};

// right-side substitution t <- t R^-1 (R upper, row-major b x b): solves
// x R = t column by column, x_j = (t_j - sum_{i<j} x_i R_ij) / R_jj
__device__ __forceinline__ void qb_rsolve(double *t, const double *r, int b) {
#pragma unroll
  for (int j = 0; j < kQbMaxB; ++j) {
    if (j < b) {
      double s = t[j];
#pragma unroll
      for (int i = 0; i < kQbMaxB; ++i)
        if (i < j) s = fma(-t[i], r[i * b + j], s);
      t[j] = s / r[j * b + j];
    }
  }
}

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// shared-memory doubles of one sweep CTA (two tile stages of [Q | y] plus t,
// x and the two triangular factors)
__host__ __device__ inline size_t qb_sweep_smem(int c0, int b, int tr) {
  const int ldqs = c0 | 1;
  return sizeof(double) * ((size_t)2 * tr * (ldqs + b) + (size_t)tr * (kQbMaxB + 1) + (size_t)c0 * b + 2 * b * b);
}

// One sweep: rows in tiles of tr, staged in shared memory by cp.async two
// tiles deep (the next tile streams in while this one is computed).
__global__ void __launch_bounds__(kQbThreads) qb_sweep_kernel(const QbSweepArgs a) {
  extern __shared__ double qsm[];
  const int c0 = a.c0, b = a.b, tr = a.tr;
  const int ldqs = c0 | 1;                  // odd row stride: conflict-free column reads
  const int ldt = kQbMaxB + 1;
  const bool need_q = c0 > 0 && (a.x != nullptr || a.want_p);
  double *qst[2], *yst[2];
  qst[0] = qsm;
  yst[0] = qst[0] + (size_t)tr * ldqs;
  qst[1] = yst[0] + (size_t)tr * b;
  yst[1] = qst[1] + (size_t)tr * ldqs;
  double *ts = yst[1] + (size_t)tr * b;     // [tr][ldt]
  double *xs = ts + (size_t)tr * ldt;       // [c0][b]
  double *ras = xs + (size_t)c0 * b;        // [b][b]
  double *rbs = ras + b * b;                // [b][b]
  const int tid = threadIdx.x;
  for (int i = tid; i < c0 * b; i += kQbThreads) xs[i] = a.x ? a.x[i] : 0.0;
  for (int i = tid; i < b * b; i += kQbThreads) {
    ras[i] = a.ra ? a.ra[i] : 0.0;
    rbs[i] = a.rb ? a.rb[i] : 0.0;
  }
  const int ncat = c0 + b;
  double acc[2][kQbMaxB];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int i = 0; i < kQbMaxB; ++i) acc[u][i] = 0.0;

  const int64_t ntiles = (a.m + tr - 1) / tr;
  auto issue = [&](int64_t tile, int st) {  // tile -> stage st (rows past m read as zeros)
    if (tile >= ntiles) return;
    const int64_t row0 = tile * tr;
    const int rows = (int)(a.m - row0 < (int64_t)tr ? a.m - row0 : (int64_t)tr);
    if (need_q) {
      for (int i = tid; i < tr * c0; i += kQbThreads) {
        const int r = i / c0, k = i - r * c0;
        if (r < rows) cp_async8(qst[st] + r * ldqs + k, a.q + (row0 + r) * a.ldq + k);
        else qst[st][r * ldqs + k] = 0.0;
      }
    }
    for (int i = tid; i < tr * b; i += kQbThreads) {
      const int r = i / b, j = i - r * b;
      if (r < rows) cp_async8(yst[st] + r * b + j, a.yin + (row0 + r) * a.ldy + j);
      else yst[st][r * b + j] = 0.0;
    }
  };
  int st = 0;
  issue(blockIdx.x, 0);
  cp_async_commit();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, st ^= 1) {
    issue(tile + gridDim.x, st ^ 1);  // the other stage was released by the last barrier
    cp_async_commit();
    cp_async_wait1();                 // this tile's group has landed (for this thread)
    __syncthreads();                  // ... and for every thread
    const int64_t row0 = tile * tr;
    const int rows = (int)(a.m - row0 < (int64_t)tr ? a.m - row0 : (int64_t)tr);
    const double *qs = qst[st], *ys = yst[st];
    for (int r = tid; r < tr; r += kQbThreads) {  // triangular solves: one thread per row
      double t[kQbMaxB];
#pragma unroll
      for (int j = 0; j < kQbMaxB; ++j) t[j] = j < b ? ys[r * b + j] : 0.0;
      if (a.ra) qb_rsolve(t, ras, b);
      if (a.rb) qb_rsolve(t, rbs, b);
#pragma unroll
      for (int j = 0; j < kQbMaxB; ++j)
        if (j < b) ts[r * ldt + j] = r < rows ? t[j] : 0.0;
    }
    if (a.x && c0 > 0) {  // t -= Q x: (row, column) pairs over all threads
      __syncthreads();
      for (int i = tid; i < tr * b; i += kQbThreads) {
        const int r = i / b, j = i - r * b;
        const double *qr = qs + r * ldqs;
        double s = 0.0;
        for (int k = 0; k < c0; ++k) s = fma(qr[k], xs[k * b + j], s);
        ts[r * ldt + j] -= s;  // only this thread touches (r, j)
      }
    }
    __syncthreads();
    if (a.out) {
      for (int i = tid; i < rows * b; i += kQbThreads) {
        const int r = i / b, j = i - r * b;
        a.out[(row0 + r) * a.ldo + j] = ts[r * ldt + j];
      }
    }
    if (a.want_p || a.want_w) {  // thread owns columns k = tid, tid + 256 of [Q | t]
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = tid + u * kQbThreads;
        if (k >= ncat) continue;
        const bool isq = k < c0;
        if ((isq && !a.want_p) || (!isq && !a.want_w)) continue;
        for (int r = 0; r < rows; ++r) {
          const double cv = isq ? qs[r * ldqs + k] : ts[r * ldt + (k - c0)];
          const double *tr_ = ts + r * ldt;
#pragma unroll
          for (int i = 0; i < kQbMaxB; ++i)
            if (i < b) acc[u][i] = fma(tr_[i], cv, acc[u][i]);
        }
      }
    }
    __syncthreads();  // stage st and ts are free for the next issue / tile
  }
  if (a.want_p || a.want_w) {
    double *p = a.part + (size_t)blockIdx.x * b * ncat;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = tid + u * kQbThreads;
      if (k >= ncat) continue;
      for (int i = 0; i < b; ++i) p[(size_t)i * ncat + k] = acc[u][i];
    }
  }
}

// red[i][k] = sum over the parts in order (fixed-order, deterministic);
// xt (optional): c0 x b transpose of the t^T Q part, the next sweep's x
__global__ void qb_reduce_kernel(const double *__restrict__ part, int nparts, int b, int ncat, double *red,
                                 double *xt, int c0) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= b * ncat) return;
  double s = 0.0;
  for (int z = 0; z < nparts; ++z) s += part[(size_t)z * b * ncat + e];
  red[e] = s;
  const int i = e / ncat, k = e - i * ncat;
  if (xt && k < c0) xt[(size_t)k * b + i] = s;
}

// upper Cholesky W = R^T R of a b x b symmetric matrix (row-major); false
// when W is not numerically positive definite (cholesky_ex info != 0)
__device__ bool qb_chol_upper(const double *w, int ldw, double *r, int b) {
  for (int i = 0; i < b * b; ++i) r[i] = 0.0;
  for (int j = 0; j < b; ++j) {
    double d = w[j * ldw + j];
    for (int k = 0; k < j; ++k) d = fma(-r[k * b + j], r[k * b + j], d);
    if (!(d > 0.0)) return false;
    const double rjj = sqrt(d);
    r[j * b + j] = rjj;
    for (int i = j + 1; i < b; ++i) {
      double s = w[j * ldw + i];
      for (int k = 0; k < j; ++k) s = fma(-r[k * b + j], r[k * b + i], s);
      r[j * b + i] = s / rjj;
    }
  }
  return true;
}

// c = a b for upper triangular b x b matrices (row-major)
__device__ void qb_mul_upper(const double *x, const double *y, double *c, int b) {
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) {
      double s = 0.0;
      for (int k = i; k <= j; ++k) s = fma(x[i * b + k], y[k * b + j], s);
      c[i * b + j] = j >= i ? s : 0.0;
    }
}

// Small b x b algebra between sweeps (one thread; b <= 16). `st` holds the
// block's factors: [R1 | R2 | r_i | R3 | R4 | R_i], each b x b.
//  op 1: R1 = chol(W)
//  op 2: CholeskyQR2 test on W = Q1^T Q1 (max |W - I| < 1e-5), R2 = chol(W),
//        r_i = R2 R1, deficiency test |r_i,jj| >= tol (qb.py:100)
//  op 3: R3 = chol(W)
//  op 4: test on W = Z1^T Z1, R4 = chol(W), R_i = (R4 R3) r_i, singularity
//        guard on diag(R_i) (linalg.py:131-135)
__global__ void qb_small_kernel(int op, int b, int ncat, int c0, const double *red, double *st, int *flag,
                                const double *tol) {
  if (threadIdx.x != 0) return;
  const double *w = red + c0;  // the t^T t block of the reduced [t^T Q | t^T t]
  const int bb = b * b;
  double *R1 = st, *R2 = st + bb, *ri = st + 2 * bb, *R3 = st + 3 * bb, *R4 = st + 4 * bb, *Ri = st + 5 * bb;
  bool ok = true;
  if (op == 1 || op == 3) {
    ok = qb_chol_upper(w, ncat, op == 1 ? R1 : R3, b);
  } else {
    double defect = 0.0;
    for (int i = 0; i < b; ++i)
      for (int j = 0; j < b; ++j) defect = fmax(defect, fabs(w[i * ncat + j] - (i == j ? 1.0 : 0.0)));
    ok = defect < 1e-5 && isfinite(defect);
    ok = qb_chol_upper(w, ncat, op == 2 ? R2 : R4, b) && ok;
    if (op == 2) {
      qb_mul_upper(R2, R1, ri, b);
      for (int j = 0; j < b; ++j) ok = ok && isfinite(ri[j * b + j]) && !(fabs(ri[j * b + j]) < *tol);
    } else {
      double rt[kQbMaxB * kQbMaxB];
      qb_mul_upper(R4, R3, rt, b);
      qb_mul_upper(rt, ri, Ri, b);
      double mx = 0.0;
      for (int j = 0; j < b; ++j) mx = fmax(mx, fabs(Ri[j * b + j]));
      for (int j = 0; j < b; ++j) {
        const double d = fabs(Ri[j * b + j]);
        ok = ok && isfinite(d) && !(d < 1e-300) && !(d < 1e-15 * mx);
      }
    }
  }
  if (!ok) *flag = 1;
}

}  // namespace spca
