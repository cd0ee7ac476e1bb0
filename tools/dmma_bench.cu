// FP64 throughput on B200: mma.sync m16n8k4 / m16n8k8 / m16n8k16 .f64 (DMMA)
// versus DFMA, one CTA of 8 warps per SM, register-resident operands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_bench tools/dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void __launch_bounds__(256) dmma(int iters, double *out) {
  double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0}, d[4] = {0, 0, 0, 0};
  for (int i = 0; i < K / 2; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < K / 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int it = 0; it < iters; ++it) {
    if constexpr (K == 4) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[1]), "d"(a[0]), "d"(b[0]));
    } else if constexpr (K == 8) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                   : "d"(a[1]), "d"(a[0]), "d"(a[3]), "d"(a[2]), "d"(b[1]), "d"(b[0]));
    } else {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                   : "d"(a[1]), "d"(a[0]), "d"(a[3]), "d"(a[2]), "d"(a[5]), "d"(a[4]), "d"(a[7]), "d"(a[6]),
                     "d"(b[1]), "d"(b[0]), "d"(b[3]), "d"(b[2]));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] + c[1] + c[2] + c[3] + d[0] + d[1] + d[2] + d[3];
}

__global__ void __launch_bounds__(256) dfma(int iters, double *out) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = 1e-3 * (threadIdx.x + i);
  const double y = 0.999, z = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y, z);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *out;
  cudaMalloc(&out, 148 * 4 * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 16;
  for (int blocks : {148, 296, 592}) {
    float ms;
    auto run = [&](auto kern, double flops_per_iter_per_warp, const char *name) {
      kern<<<blocks, 256>>>(iters / 16, out);
      cudaEventRecord(e0);
      kern<<<blocks, 256>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = flops_per_iter_per_warp * iters * blocks * 8;
      printf("%-22s blocks %3d: %7.2f TFLOP/s (%s)\n", name, blocks, flops / (ms * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    };
    run(dmma<4>, 2 * 2.0 * 16 * 8 * 4, "mma m16n8k4 f64");
    run(dmma<8>, 2 * 2.0 * 16 * 8 * 8, "mma m16n8k8 f64");
    run(dmma<16>, 2 * 2.0 * 16 * 8 * 16, "mma m16n8k16 f64");
    run(dfma, 8 * 2.0 * 32, "dfma");
  }
  return 0;
}
