// common.cuh — shared helpers for the libspca kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define SPCA_DEVINL __device__ __forceinline__

namespace spca {

constexpr int64_t kNoBadRow = INT64_MAX;

template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int n = 2; };

SPCA_DEVINL bool finite_val(float x) { return isfinite(x); }
SPCA_DEVINL bool finite_val(double x) { return isfinite(x); }

// Smallest offending absolute row wins (sketch.py:46 reports the first bad row).
SPCA_DEVINL void report_bad_row(unsigned long long *bad, int64_t row) {
  atomicMin(bad, (unsigned long long)row);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace spca
