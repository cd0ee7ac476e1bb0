// Row normalisation: each row to zero mean, then unit Euclidean norm; a
// constant row becomes the zero row (reference normalize_rows,
// /root/reference/pkg/src/streampca/sketch.py:142-153). HBM-bound: one read
// of the row from HBM, two re-reads that hit L2 (the row was just touched),
// one write. fp64 arithmetic for either element type.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
    const double safe = norm == 0.0 ? 1.0 : norm;
    T *y = dst + r * ldd;
    for (int64_t j = threadIdx.x; j < n; j += kNormThreads) y[j] = (T)(((double)x[j] - mean) / safe);
  }
}

}  // namespace spca
