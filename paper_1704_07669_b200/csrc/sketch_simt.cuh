// sketch_simt.cuh — CUDA-core (FFMA fp32 / DFMA fp64) sketch kernels.
//
// One canonical chunk of R rows of A (row-major, stride lda) is processed by
//   simt_g_kernel   G_c = A_c Omega            (reference sketch.py:103)
//                   + first non-finite row      (sketch.py:45-49)
//   simt_g_reduce   fixed-order sum of split-K partials of G_c
//   simt_h_kernel   Hpart[z] (+)= A_c^T G_c     (sketch.py:104)
//                   + per-chunk column sums     (sketch.py:106) in fp64
// fp32: register-tiled FFMA (4x4 outputs per thread, 256 threads); fp64: the
// same CTA tiles fed to the fp64 tensor cores with warp-level DMMA
// (mma.sync m16n8k4 .f64: each warp one 16-row tile x four 8-column tiles).
// Both use double-buffered shared-memory tiles loaded with 16-byte vector
// loads when alignment allows. This is the SIMT path (SPCA_PREC_SIMT) and the
// fp64 path; the tensor-core path for fp32 lives in sketch_tc.cuh.
#pragma once

#include "common.cuh"

namespace spca {

constexpr int kSimtThreads = 256;

// fp64 tensor-core step: D(16x8) += A(16x4, row) B(4x8, col), fp64 throughout
// (fragment: a0 = A[g][t], a1 = A[g+8][t], b = B[t][g], d = D[g][2t..2t+1],
// D[g+8][2t..2t+1] with g = lane / 4, t = lane % 4)
__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b));
}

// shared-row padding: fp64 tiles are read as 4 k-rows x 8 consecutive values
// per warp load, conflict-free when the row stride is 64 mod 128 bytes
template <typename T, int W>
struct SimtRow {
  static constexpr int value = sizeof(T) == 8 ? W + 8 : W + 16 / (int)sizeof(T);
};

// ---------------------------------------------------------------- G = A W
// grid = (row tiles, l tiles, k splits). W is n x ldw (ldw % BL == 0, zero
// padded beyond l). out: [split][rows][ldo] (split stride `out_split_stride`).
template <typename T, int BM, int BL, int BK, bool VEC>
__global__ void __launch_bounds__(kSimtThreads)
simt_g_kernel(const T *__restrict__ A, int64_t lda, int rows, int n,
              const T *__restrict__ W, int ldw, T *__restrict__ out, int ldo,
              int64_t out_split_stride, int kseg, int64_t first_row,
              unsigned long long *__restrict__ bad_row) {
  constexpr int TM = 4, TL = 4;
  constexpr int NTL = BL / TL;
  constexpr int NTM = BM / TM;
  static_assert(sizeof(T) == 8 || NTL * NTM == kSimtThreads, "thread tiling");
  constexpr int VN = Vec<T>::n;
  constexpr int A_PER = BM * BK / kSimtThreads;  // elements per thread
  constexpr int W_PER = BK * BL / kSimtThreads;
  static_assert(A_PER % VN == 0 && W_PER % VN == 0, "vector tiling");
  __shared__ __align__(16) T As[2][BK][SimtRow<T, BM>::value];
  __shared__ __align__(16) T Ws[2][BK][sizeof(T) == 8 ? BL + 8 : BL];

  const int tid = threadIdx.x;
  const int tl = tid % NTL, tm = tid / NTL;
  const int m0 = blockIdx.x * BM;
  const int j0 = blockIdx.y * BL;
  const int kb = blockIdx.z * kseg;
  const int ke = min(n, kb + kseg);
  const bool check = (blockIdx.y == 0);

  T ra[A_PER];
  T rw[W_PER];
  int bad_local = INT32_MAX;

  auto load_tiles = [&](int k0) {
    if constexpr (VEC) {
#pragma unroll
      for (int i = 0; i < A_PER / VN; ++i) {
        int v = tid + i * kSimtThreads;
        int r = v / (BK / VN), kk = (v % (BK / VN)) * VN;
        int gr = m0 + r, gk = k0 + kk;
        typename Vec<T>::type x;
        if (gr < rows && gk < ke) {
          x = *reinterpret_cast<const typename Vec<T>::type *>(A + (int64_t)gr * lda + gk);
        } else {
          x = typename Vec<T>::type{};
        }
        const T *px = reinterpret_cast<const T *>(&x);
#pragma unroll
        for (int e = 0; e < VN; ++e) {
          ra[i * VN + e] = px[e];
          if (check && !finite_val(px[e])) bad_local = min(bad_local, gr);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < A_PER; ++i) {
        int e = tid + i * kSimtThreads;
        int r = e / BK, kk = e % BK;
        int gr = m0 + r, gk = k0 + kk;
        T x = (gr < rows && gk < ke) ? A[(int64_t)gr * lda + gk] : T(0);
        ra[i] = x;
        if (check && !finite_val(x)) bad_local = min(bad_local, gr);
      }
    }
#pragma unroll
    for (int i = 0; i < W_PER / VN; ++i) {
      int v = tid + i * kSimtThreads;
      int kk = v / (BL / VN), jj = (v % (BL / VN)) * VN;
      int gk = k0 + kk;
      typename Vec<T>::type x;
      if (gk < ke) {
        x = *reinterpret_cast<const typename Vec<T>::type *>(W + (int64_t)gk * ldw + j0 + jj);
      } else {
        x = typename Vec<T>::type{};
      }
      const T *px = reinterpret_cast<const T *>(&x);
#pragma unroll
      for (int e = 0; e < VN; ++e) rw[i * VN + e] = px[e];
    }
  };
  auto store_tiles = [&](int buf) {
    if constexpr (VEC) {
#pragma unroll
      for (int i = 0; i < A_PER / VN; ++i) {
        int v = tid + i * kSimtThreads;
        int r = v / (BK / VN), kk = (v % (BK / VN)) * VN;
#pragma unroll
        for (int e = 0; e < VN; ++e) As[buf][kk + e][r] = ra[i * VN + e];
      }
    } else {
#pragma unroll
      for (int i = 0; i < A_PER; ++i) {
        int e = tid + i * kSimtThreads;
        As[buf][e % BK][e / BK] = ra[i];
      }
    }
#pragma unroll
    for (int i = 0; i < W_PER / VN; ++i) {
      int v = tid + i * kSimtThreads;
      int kk = v / (BL / VN), jj = (v % (BL / VN)) * VN;
      *reinterpret_cast<typename Vec<T>::type *>(&Ws[buf][kk][jj]) =
          *reinterpret_cast<typename Vec<T>::type *>(&rw[i * VN]);
    }
  };

  T acc[TM][TL];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TL; ++j) acc[i][j] = T(0);
  // fp64: warp (wm, wn) owns rows [16 wm, 16 wm + 16) x columns [32 wn, 32 wn + 32)
  // fp64: warps WM (rows) x WN (32-column slices); each warp MPW 16-row tiles x four 8-column tiles
  constexpr int WN = BL / 32 > 0 ? BL / 32 : 1, WM = (kSimtThreads / 32) / WN, MPW = BM / 16 / WM;
  static_assert(sizeof(T) == 4 || (MPW >= 1 && MPW * WM * 16 == BM && WN * 32 == BL), "DMMA warp tiling");
  const int lane = tid & 31, wid = tid >> 5, wm = wid % WM, wn = wid / WM;
  const int fg = lane >> 2, ft = lane & 3;
  double dacc[MPW][4][4];
#pragma unroll
  for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dacc[mi][i][j] = 0.0;

  const int ntiles = (ke > kb) ? (ke - kb + BK - 1) / BK : 0;
  if (ntiles > 0) {
    load_tiles(kb);
    store_tiles(0);
    __syncthreads();
  }
  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ntiles) load_tiles(kb + (t + 1) * BK);
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int k = 0; k < BK; ++k) {
        T a[TM], w[TL];
        float4 av = *reinterpret_cast<const float4 *>(&As[buf][k][tm * TM]);
        float4 wv = *reinterpret_cast<const float4 *>(&Ws[buf][k][tl * TL]);
        a[0] = av.x; a[1] = av.y; a[2] = av.z; a[3] = av.w;
        w[0] = wv.x; w[1] = wv.y; w[2] = wv.z; w[3] = wv.w;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TL; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
      }
    } else {  // fp64: DMMA, four k-steps of 4 per tile
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double a0[MPW], a1[MPW];
#pragma unroll
        for (int mi = 0; mi < MPW; ++mi) {
          a0[mi] = As[buf][ks + ft][(wm * MPW + mi) * 16 + fg];
          a1[mi] = As[buf][ks + ft][(wm * MPW + mi) * 16 + fg + 8];
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const double bw = Ws[buf][ks + ft][wn * 32 + nt * 8 + fg];
#pragma unroll
          for (int mi = 0; mi < MPW; ++mi) dmma_16x8x4(dacc[mi][nt], a0[mi], a1[mi], bw);
        }
      }
    }
    if (t + 1 < ntiles) {
      store_tiles(buf ^ 1);
    }
    __syncthreads();
  }

  if (check) {
    // warp-level min, one atomic per warp that saw a bad row
    for (int o = 16; o > 0; o >>= 1) bad_local = min(bad_local, __shfl_xor_sync(0xffffffffu, bad_local, o));
    if ((tid & 31) == 0 && bad_local != INT32_MAX) report_bad_row(bad_row, first_row + bad_local);
  }

  T *o = out + (int64_t)blockIdx.z * out_split_stride;
  if constexpr (sizeof(T) == 8) {
#pragma unroll
    for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m0 + (wm * MPW + mi) * 16 + fg + 8 * h;
        if (r >= rows) continue;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          *reinterpret_cast<double2 *>(o + (int64_t)r * ldo + j0 + wn * 32 + nt * 8 + 2 * ft) =
              make_double2(dacc[mi][nt][2 * h], dacc[mi][nt][2 * h + 1]);
      }
    return;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int r = m0 + tm * TM + i;
    if (r >= rows) continue;
    T *dst = o + (int64_t)r * ldo + j0 + tl * TL;
#pragma unroll
    for (int j = 0; j < TL; j += VN) {
      typename Vec<T>::type v;
      T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
      for (int e = 0; e < VN; ++e) pv[e] = acc[i][j + e];
      *reinterpret_cast<typename Vec<T>::type *>(dst + j) = v;
    }
  }
}

// Fixed-order sum of `splits` partial G slabs into G (rows x ld).
template <typename T>
__global__ void simt_g_reduce(const T *__restrict__ part, int splits, int64_t split_stride,
                              int64_t count, T *__restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < count; i += stride) {
    T s = part[i];
    for (int z = 1; z < splits; ++z) s += part[(int64_t)z * split_stride + i];
    out[i] = s;
  }
}

// ---------------------------------------------------------- Hpart += A^T G
// grid = (n tiles, l tiles, row splits). Hpart: [split][n][ldh]; cspart: [split][n].
template <typename T, int BN, int BL, int BK, bool VEC>
__global__ void __launch_bounds__(kSimtThreads)
simt_h_kernel(const T *__restrict__ A, int64_t lda, int rows, int n,
              const T *__restrict__ G, int ldg, T *__restrict__ Hpart, int ldh,
              int64_t h_split_stride, double *__restrict__ cspart, int rseg,
              int accumulate, int kahan) {
  constexpr int TN = 4, TL = 4;
  constexpr int NTL = BL / TL;
  constexpr int NTN = BN / TN;
  static_assert(sizeof(T) == 8 || NTL * NTN == kSimtThreads, "thread tiling");
  constexpr int VN = Vec<T>::n;
  constexpr int A_PER = BK * BN / kSimtThreads;
  constexpr int G_PER = BK * BL / kSimtThreads;
  static_assert(A_PER % VN == 0 && G_PER % VN == 0, "vector tiling");
  __shared__ __align__(16) T As[2][BK][sizeof(T) == 8 ? BN + 8 : BN];
  __shared__ __align__(16) T Gs[2][BK][sizeof(T) == 8 ? BL + 8 : BL];

  const int tid = threadIdx.x;
  const int tl = tid % NTL, tn = tid / NTL;
  const int n0 = blockIdx.x * BN;
  const int j0 = blockIdx.y * BL;
  const int rb = blockIdx.z * rseg;
  const int re = min(rows, rb + rseg);
  // column sums: fp32 path, the threads of l-tile 0 for their 4 columns; fp64
  // path, thread c < BN for column c (the MMA fragments do not own columns)
  const bool do_cs = (blockIdx.y == 0) && (sizeof(T) == 4 ? (tl == 0) : (tid < BN));

  T ra[A_PER];
  T rg[G_PER];

  auto load_tiles = [&](int r0) {
    if constexpr (VEC) {
#pragma unroll
      for (int i = 0; i < A_PER / VN; ++i) {
        int v = tid + i * kSimtThreads;
        int r = v / (BN / VN), c = (v % (BN / VN)) * VN;
        int gr = r0 + r, gc = n0 + c;
        typename Vec<T>::type x;
        if (gr < re && gc < n) {
          x = *reinterpret_cast<const typename Vec<T>::type *>(A + (int64_t)gr * lda + gc);
        } else {
          x = typename Vec<T>::type{};
        }
        const T *px = reinterpret_cast<const T *>(&x);
#pragma unroll
        for (int e = 0; e < VN; ++e) ra[i * VN + e] = px[e];
      }
    } else {
#pragma unroll
      for (int i = 0; i < A_PER; ++i) {
        int e = tid + i * kSimtThreads;
        int r = e / BN, c = e % BN;
        int gr = r0 + r, gc = n0 + c;
        ra[i] = (gr < re && gc < n) ? A[(int64_t)gr * lda + gc] : T(0);
      }
    }
#pragma unroll
    for (int i = 0; i < G_PER / VN; ++i) {
      int v = tid + i * kSimtThreads;
      int r = v / (BL / VN), jj = (v % (BL / VN)) * VN;
      int gr = r0 + r;
      typename Vec<T>::type x;
      if (gr < re) {
        x = *reinterpret_cast<const typename Vec<T>::type *>(G + (int64_t)gr * ldg + j0 + jj);
      } else {
        x = typename Vec<T>::type{};
      }
      const T *px = reinterpret_cast<const T *>(&x);
#pragma unroll
      for (int e = 0; e < VN; ++e) rg[i * VN + e] = px[e];
    }
  };
  auto store_tiles = [&](int buf) {
    if constexpr (VEC) {
#pragma unroll
      for (int i = 0; i < A_PER / VN; ++i) {
        int v = tid + i * kSimtThreads;
        int r = v / (BN / VN), c = (v % (BN / VN)) * VN;
        *reinterpret_cast<typename Vec<T>::type *>(&As[buf][r][c]) =
            *reinterpret_cast<typename Vec<T>::type *>(&ra[i * VN]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < A_PER; ++i) {
        int e = tid + i * kSimtThreads;
        As[buf][e / BN][e % BN] = ra[i];
      }
    }
#pragma unroll
    for (int i = 0; i < G_PER / VN; ++i) {
      int v = tid + i * kSimtThreads;
      int r = v / (BL / VN), jj = (v % (BL / VN)) * VN;
      *reinterpret_cast<typename Vec<T>::type *>(&Gs[buf][r][jj]) =
          *reinterpret_cast<typename Vec<T>::type *>(&rg[i * VN]);
    }
  };

  T acc[TN][TL];
#pragma unroll
  for (int i = 0; i < TN; ++i)
#pragma unroll
    for (int j = 0; j < TL; ++j) acc[i][j] = T(0);
  double cs[TN] = {0.0, 0.0, 0.0, 0.0};
  double cc[TN] = {0.0, 0.0, 0.0, 0.0};  // Kahan carries (compensated mode)
  // fp64: warps WM (columns) x WN (32-wide l slices); each warp MPW 16-column tiles x four 8-wide tiles
  constexpr int WN = BL / 32 > 0 ? BL / 32 : 1, WM = (kSimtThreads / 32) / WN, MPW = BN / 16 / WM;
  static_assert(sizeof(T) == 4 || (MPW >= 1 && MPW * WM * 16 == BN && WN * 32 == BL), "DMMA warp tiling");
  const int lane = tid & 31, wid = tid >> 5, wm = wid % WM, wn = wid / WM;
  const int fg = lane >> 2, ft = lane & 3;
  double dacc[MPW][4][4];
#pragma unroll
  for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dacc[mi][i][j] = 0.0;

  const int ntiles = (re > rb) ? (re - rb + BK - 1) / BK : 0;
  if (ntiles > 0) {
    load_tiles(rb);
    store_tiles(0);
    __syncthreads();
  }
  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ntiles) load_tiles(rb + (t + 1) * BK);
    if constexpr (sizeof(T) == 8) {  // fp64: DMMA (A^T: m = column, k = row) + column sums
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double a0[MPW], a1[MPW];
#pragma unroll
        for (int mi = 0; mi < MPW; ++mi) {
          a0[mi] = As[buf][ks + ft][(wm * MPW + mi) * 16 + fg];
          a1[mi] = As[buf][ks + ft][(wm * MPW + mi) * 16 + fg + 8];
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const double bg = Gs[buf][ks + ft][wn * 32 + nt * 8 + fg];
#pragma unroll
          for (int mi = 0; mi < MPW; ++mi) dmma_16x8x4(dacc[mi][nt], a0[mi], a1[mi], bg);
        }
      }
      if (do_cs) {
#pragma unroll
        for (int k = 0; k < BK; ++k) {
          const double x = As[buf][k][tid];
          if (kahan) {
            const double y = x - cc[0];
            const double t2 = cs[0] + y;
            cc[0] = (t2 - cs[0]) - y;
            cs[0] = t2;
          } else {
            cs[0] += x;
          }
        }
      }
    } else
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[TN], g[TL];
      {
        float4 av = *reinterpret_cast<const float4 *>(&As[buf][k][tn * TN]);
        float4 gv = *reinterpret_cast<const float4 *>(&Gs[buf][k][tl * TL]);
        a[0] = av.x; a[1] = av.y; a[2] = av.z; a[3] = av.w;
        g[0] = gv.x; g[1] = gv.y; g[2] = gv.z; g[3] = gv.w;
      }
#pragma unroll
      for (int i = 0; i < TN; ++i)
#pragma unroll
        for (int j = 0; j < TL; ++j) acc[i][j] = fma(a[i], g[j], acc[i][j]);
      if (do_cs) {
        if (kahan) {
#pragma unroll
          for (int i = 0; i < TN; ++i) {
            double y = (double)a[i] - cc[i];
            double t = cs[i] + y;
            cc[i] = (t - cs[i]) - y;
            cs[i] = t;
          }
        } else {
#pragma unroll
          for (int i = 0; i < TN; ++i) cs[i] += (double)a[i];
        }
      }
    }
    if (t + 1 < ntiles) store_tiles(buf ^ 1);
    __syncthreads();
  }

  T *hp = Hpart + (int64_t)blockIdx.z * h_split_stride;
  if constexpr (sizeof(T) == 8) {
#pragma unroll
    for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = n0 + (wm * MPW + mi) * 16 + fg + 8 * h;
      if (c >= n) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double2 *dst = reinterpret_cast<double2 *>(hp + (int64_t)c * ldh + j0 + wn * 32 + nt * 8 + 2 * ft);
        double2 v = make_double2(dacc[mi][nt][2 * h], dacc[mi][nt][2 * h + 1]);
        if (accumulate) {
          const double2 old = *dst;
          v.x += old.x;
          v.y += old.y;
        }
        *dst = v;
      }
    }
    if (do_cs && n0 + tid < n) cspart[(int64_t)blockIdx.z * n + n0 + tid] = cs[0];
    return;
  }
#pragma unroll
  for (int i = 0; i < TN; ++i) {
    int c = n0 + tn * TN + i;
    if (c >= n) continue;
    T *dst = hp + (int64_t)c * ldh + j0 + tl * TL;
#pragma unroll
    for (int j = 0; j < TL; j += VN) {
      typename Vec<T>::type v;
      T *pv = reinterpret_cast<T *>(&v);
      if (accumulate) {
        typename Vec<T>::type old = *reinterpret_cast<const typename Vec<T>::type *>(dst + j);
        const T *po = reinterpret_cast<const T *>(&old);
#pragma unroll
        for (int e = 0; e < VN; ++e) pv[e] = po[e] + acc[i][j + e];
      } else {
#pragma unroll
        for (int e = 0; e < VN; ++e) pv[e] = acc[i][j + e];
      }
      *reinterpret_cast<typename Vec<T>::type *>(dst + j) = v;
    }
    if (do_cs) cspart[(int64_t)blockIdx.z * n + c] = cs[i];
  }
}

}  // namespace spca
