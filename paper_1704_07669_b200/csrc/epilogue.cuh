// epilogue.cuh — small fixed-order reduction / conversion kernels around the
// contraction kernels. None of them uses float atomics, so every result is
// bitwise reproducible run to run.
#pragma once

#include "common.cuh"

namespace spca {

// colsum64[i] += sum_z cspart[z][i]  (plain or Kahan; sketch.py:105-111)
__global__ void colsum_accumulate(const double *__restrict__ cspart, int splits, int n,
                                  double *__restrict__ colsum, double *__restrict__ carry) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = cspart[i];
  if (carry == nullptr) {
    for (int z = 1; z < splits; ++z) s += cspart[(int64_t)z * n + i];
  } else {
    double c = 0.0;
    for (int z = 1; z < splits; ++z) {
      double y = cspart[(int64_t)z * n + i] - c;
      double t = s + y;
      c = (t - s) - y;
      s = t;
    }
  }
  if (carry == nullptr) {
    colsum[i] += s;
  } else {
    double c = carry[i], t0 = colsum[i];
    double y = s - c;
    double t = t0 + y;
    carry[i] = (t - t0) - y;
    colsum[i] = t;
  }
}

// H64[i][j] += sum_z Hpart[z][i][j] for j < l  (Hpart row stride ldh)
template <typename T>
__global__ void h_flush(const T *__restrict__ hpart, int splits, int64_t split_stride, int n,
                        int l, int ldh, double *__restrict__ h64) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t count = (int64_t)n * l;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < count; idx += stride) {
    int64_t i = idx / l;
    int j = (int)(idx - i * l);
    const T *p = hpart + i * ldh + j;
    double s = (double)p[0];
    for (int z = 1; z < splits; ++z) s += (double)p[(int64_t)z * split_stride];
    h64[idx] += s;
  }
}

// G64 (rows x l) <- G (rows x ldg) widened
template <typename T>
__global__ void g_widen(const T *__restrict__ g, int ldg, int64_t rows, int l,
                        double *__restrict__ g64) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t count = rows * l;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < count; idx += stride) {
    int64_t r = idx / l;
    int j = (int)(idx - r * l);
    g64[idx] = (double)g[r * ldg + j];
  }
}

// out[j] = sum_r X[r][j] (X rows x l, fp64), one block per column, fixed-order tree.
__global__ void column_sums64(const double *__restrict__ x, int64_t rows, int l,
                              double *__restrict__ out) {
  __shared__ double red[256];
  int j = blockIdx.x;
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) s += x[r * l + j];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = red[0];
}

// w[j] = sum_i mu[i] * omega64[i][j]  (mu^T Omega; sketch.py:137)
__global__ void mu_omega(const double *__restrict__ mu, const double *__restrict__ om, int n,
                         int l, double *__restrict__ w) {
  __shared__ double red[256];
  int j = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += mu[i] * om[(int64_t)i * l + j];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) w[j] = red[0];
}

// mu = colsum / m
__global__ void mean_from_colsum(const double *__restrict__ colsum, int n, double inv_m,
                                 double *__restrict__ mu) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) mu[i] = colsum[i] * inv_m;
}

// G -= 1 w^T  (rows x l)
__global__ void g_center(double *__restrict__ g, int64_t rows, int l, const double *__restrict__ w) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < rows * l; idx += stride) g[idx] -= w[idx % l];
}

// H -= mu gsum^T (n x l); colsum <- 0
__global__ void h_center(double *__restrict__ h, int n, int l, const double *__restrict__ mu,
                         const double *__restrict__ gsum, double *__restrict__ colsum) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < (int64_t)n * l; idx += stride) {
    int64_t i = idx / l;
    int j = (int)(idx - i * l);
    h[idx] -= mu[i] * gsum[j];
  }
  idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; idx < n; idx += stride) colsum[idx] = 0.0;
}

// Omega (n x l fp64, row-major) -> compute-precision copy with row stride ldw
// (zero padded), plus the fp64 "as used" copy (omega rounded to T, widened).
template <typename T>
__global__ void omega_prepare(const double *__restrict__ om, int n, int l, int ldw,
                              T *__restrict__ w, double *__restrict__ om_used) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; idx < (int64_t)n * ldw; idx += stride) {
    int64_t i = idx / ldw;
    int j = (int)(idx - i * ldw);
    T v = (j < l) ? (T)om[i * l + j] : T(0);
    w[idx] = v;
    if (j < l) om_used[i * l + j] = (double)v;
  }
}

// fused row normalisation, finish-time corrections (sketch_fused.cuh):
// out[j] = sum_r g[r][j] * coef[r] for j < l, out[l] = sum_r coef[r]
__global__ void norm_coef_sums(const double *__restrict__ g, int64_t rows, int l,
                               const double *__restrict__ coef, double *__restrict__ out) {
  __shared__ double red[256];
  const int j = blockIdx.x;
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) s += j < l ? g[r * l + j] * coef[r] : coef[r];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = red[0];
}

// H[i][j] -= c[j], colsum[i] -= c[l]  (hcs = [H (n x l) | colsum (n)])
__global__ void norm_correct(double *__restrict__ hcs, int n, int l, const double *__restrict__ c) {
  const int64_t total = (int64_t)n * (l + 1);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < (int64_t)n * l) hcs[idx] -= c[idx % l];
    else hcs[idx] -= c[l];
  }
}

// dst (rows x n, stride ldd) <- src (stride lds): device rows whose stride the
// pass kernel's TMA cannot address, re-strided into the staging ring
template <typename T>
__global__ void restride_rows(const T *__restrict__ src, int64_t lds, int64_t rows, int n, T *__restrict__ dst,
                              int64_t ldd) {
  const int64_t total = rows * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / n;
    const int c = (int)(idx - r * n);
    dst[r * ldd + c] = src[r * lds + c];
  }
}

// Column shift (spca_sketch_set_shift): c = the mean of the pass's first
// `rows` rows (fp64 sum, rounded to fp32; a non-finite mean becomes 0), zero
// padded to `pad` entries. Rows of stride ld.
template <typename T>
__global__ void shift_capture(const T *__restrict__ a, int rows, int64_t ld, int n, int pad,
                              float *__restrict__ c) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < pad; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (j < n)
      for (int r = 0; r < rows; ++r) s += (double)a[(int64_t)r * ld + j];
    const float v = (float)(s / (double)rows);
    c[j] = isfinite(v) ? v : 0.f;
  }
}

// dst = src - 1 c^T on `rows` rows (SIMT path: the shifted chunk in a workspace)
template <typename T>
__global__ void shift_rows(const T *__restrict__ src, int64_t rows, int n, int64_t lds, const float *__restrict__ c,
                           T *__restrict__ dst, int64_t ldd) {
  const int64_t total = rows * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / n;
    const int j = (int)(idx - r * n);
    dst[r * ldd + j] = src[r * lds + j] - (T)c[j];
  }
}

// w[j] = sum_i c[i] Omega[i][j] (fp64, Omega as used), one block per column;
// gs[j] = sum_r X[r][j] over the finished (shifted) G or the co-sketch operand
__global__ void shift_terms(const float *__restrict__ c, const double *__restrict__ om, int n, int l,
                            const double *__restrict__ x, int64_t rows, double *__restrict__ w,
                            double *__restrict__ gs) {
  __shared__ double red[2][256];
  const int j = blockIdx.x;
  double s = 0.0, t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += (double)c[i] * om[(int64_t)i * l + j];
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) t += x[r * l + j];
  red[0][threadIdx.x] = s;
  red[1][threadIdx.x] = t;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[0][threadIdx.x] += red[0][threadIdx.x + o];
      red[1][threadIdx.x] += red[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    w[j] = red[0][0];
    gs[j] = red[1][0];
  }
}

// Undo the shift at finish (A = A' + 1 c^T, G = G' + 1 w^T, w = Omega^T c):
//   plain    H = H' + colsum' w^T + c gsum'^T + m c w^T
//   co-sketch H = H' + c lsum^T
//   colsum = colsum' + m c;  G += 1 w^T (separately, g_add_row)
__global__ void shift_fix_h(double *__restrict__ hcs, int n, int l, const float *__restrict__ c,
                            const double *__restrict__ w, const double *__restrict__ gs, int64_t m,
                            int cosketch) {
  const int64_t nl = (int64_t)n * l;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < nl;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / l;
    const int j = (int)(idx - i * l);
    const double ci = (double)c[i];
    hcs[idx] += cosketch ? ci * gs[j] : hcs[nl + i] * w[j] + ci * gs[j] + (double)m * ci * w[j];
  }
}

__global__ void shift_fix_colsum(double *__restrict__ colsum, int n, const float *__restrict__ c, int64_t m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) colsum[i] += (double)m * (double)c[i];
}

__global__ void g_add_row(double *__restrict__ g, int64_t rows, int l, const double *__restrict__ w) {
  const int64_t total = rows * l;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    g[idx] += w[idx % l];
}

// fp64 column sums of Omega (as used) -> fp32, zero padded to lpad
__global__ void omega_colsums(const double *__restrict__ om, int n, int l, int lpad, float *__restrict__ out) {
  __shared__ double red[256];
  const int j = blockIdx.x;
  double s = 0.0;
  if (j < l)
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += om[(int64_t)i * l + j];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = (float)red[0];
}

}  // namespace spca
