// Row normalisation: each row to zero mean, then unit Euclidean norm; a
// constant row becomes the zero row (reference normalize_rows,
// /root/reference/pkg/src/streampca/sketch.py:142-153). HBM-bound: one read
// of the row from HBM, two re-reads that hit L2 (the row was just touched),
// one write. fp64 arithmetic for either element type.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"

namespace spca {

constexpr int kNormThreads = 256;

// block-wide fp64 sum; every thread gets the total
__device__ __forceinline__ double block_sum64(double v, double *red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // red[] free from a previous call
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) t += red[i];
  return t;
}

// grid-stride over rows, one CTA per row at a time
template <typename T>
__global__ void __launch_bounds__(kNormThreads)
normalize_rows_kernel(const T *__restrict__ src, int64_t rows, int64_t n, int64_t lds,
                      T *__restrict__ dst, int64_t ldd) {
  __shared__ double red[kNormThreads / 32];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const T *x = src + r * lds;
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += kNormThreads) s += (double)x[j];
    const double mean = block_sum64(s, red) / (double)n;
    double q = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += kNormThreads) {
      const double d = (double)x[j] - mean;
      q = fma(d, d, q);
    }
    const double norm = sqrt(block_sum64(q, red));
    // one fp64 division per row; the elements are scaled by its reciprocal
    // (within 1.5 ulp of the reference's per-element division)
    const double inv = 1.0 / (norm == 0.0 ? 1.0 : norm);
    T *y = dst + r * ldd;
    for (int64_t j = threadIdx.x; j < n; j += kNormThreads) y[j] = (T)(((double)x[j] - mean) * inv);
  }
}

// Register-resident variant: one CTA per row, the row held in registers as
// 16-byte vectors (NV per thread) -> one HBM read and one write per element.
// Needs n a multiple of the vector width, 16-byte aligned rows and
// n <= kNormThreads * NV * (16 / sizeof(T)).
template <typename T, int NV>
__global__ void __launch_bounds__(kNormThreads)
normalize_rows_vec_kernel(const T *__restrict__ src, int64_t rows, int64_t n, int64_t lds,
                          T *__restrict__ dst, int64_t ldd) {
  constexpr int E = 16 / sizeof(T);  // elements per vector
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  __shared__ double red[kNormThreads / 32];
  const int nv = (int)(n / E);
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const V *x = reinterpret_cast<const V *>(src + r * lds);
    T v[NV][E];
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int j = threadIdx.x + i * kNormThreads;
      if (j < nv) {
        const V w = __ldcs(x + j);  // streamed once: do not keep it in L2
        const T *pw = reinterpret_cast<const T *>(&w);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          v[i][e] = pw[e];
          s += (double)pw[e];
        }
      }
    }
    const double mean = block_sum64(s, red) / (double)n;
    double q = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (threadIdx.x + i * kNormThreads < nv) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double d = (double)v[i][e] - mean;
          q = fma(d, d, q);
        }
      }
    }
    const double norm = sqrt(block_sum64(q, red));
    const double inv = 1.0 / (norm == 0.0 ? 1.0 : norm);
    V *y = reinterpret_cast<V *>(dst + r * ldd);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int j = threadIdx.x + i * kNormThreads;
      if (j < nv) {
        V w;
        T *pw = reinterpret_cast<T *>(&w);
#pragma unroll
        for (int e = 0; e < E; ++e) pw[e] = (T)(((double)v[i][e] - mean) * inv);
        y[j] = w;
      }
    }
  }
}

}  // namespace spca
