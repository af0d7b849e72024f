// fp64 FMA throughput by operand source: register, kernel-param (c-bank),
// __constant__ table (ld.const -> LDCU/uniform register), inline immediate.
#include <cuda_runtime.h>
__constant__ double ctab[4] = {0.99999912345678, 1.2345678912345e-7, 0.0, 0.0};
template <int MODE>
__global__ void __launch_bounds__(256) op_probe(double* sink, const double* gab, int iters, double pa, double pb) {
  double a, b;
  if (MODE == 0) { a = gab[0]; b = gab[1]; }
  if (MODE == 1) { a = pa; b = pb; }
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (MODE == 0 || MODE == 1) x[k] = fma(x[k], a, b);
      if (MODE == 2) asm volatile("{ .reg .f64 t, u; ld.const.f64 t, [ctab]; ld.const.f64 u, [ctab+8]; fma.rn.f64 %0, %0, t, u; }" : "+d"(x[k]));
      if (MODE == 3) asm volatile("fma.rn.f64 %0, %0, 0d3FEFFFFE2D1A3F0B, 0d3E8092A6D1A2C7E1;" : "+d"(x[k]));
      if (MODE == 4) asm volatile("fma.rn.f64 %0, %0, 0d3FF0000000000000, 0d3E80000000000000;" : "+d"(x[k]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == -1.2345) sink[threadIdx.x] = s;
}
extern "C" int op_probe_launch(int mode, int blocks, int iters, double* sink, const double* gab, void* st) {
  cudaStream_t s = (cudaStream_t)st;
  switch (mode) {
    case 0: op_probe<0><<<blocks, 256, 0, s>>>(sink, gab, iters, 0.999999, 1e-7); break;
    case 1: op_probe<1><<<blocks, 256, 0, s>>>(sink, gab, iters, 0.999999, 1e-7); break;
    case 2: op_probe<2><<<blocks, 256, 0, s>>>(sink, gab, iters, 0.999999, 1e-7); break;
    case 3: op_probe<3><<<blocks, 256, 0, s>>>(sink, gab, iters, 0.999999, 1e-7); break;
    case 4: op_probe<4><<<blocks, 256, 0, s>>>(sink, gab, iters, 0.999999, 1e-7); break;
  }
  return (int)cudaGetLastError();
}
