// rbd_peak.cu -- measures the CUDA-core FMA roofline (fp64 and fp32) on the
// running GPU.  MEASURED_PEAKS.json carries HBM and bf16-tensor peaks only; the
// dynamics kernels are scalar fp64/fp32 FMA work, so bench.py measures this
// denominator in the same run (nominal B200: ~37 TF fp64, ~74 TF fp32).
//
//   int rbd_fma_peak(int dtype, int blocks, int iters, void* sink, void* stream)
// launches `blocks` x 256 threads, each running 16 independent FMA chains for
// `iters` iterations: flops = 2 * 16 * iters * 256 * blocks.
#include <cuda_runtime.h>
#include <stdint.h>

template <typename T>
__global__ void __launch_bounds__(256) rbd_fma_peak_kernel(T* sink, int iters, T a, T b) {
  T x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (T)(threadIdx.x + k);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == (T)-1.2345) sink[threadIdx.x] = s;  // keep the chains alive
}

extern "C" int rbd_fma_peak(int dtype, int blocks, int iters, void* sink, void* stream) {
  if (dtype == 1)
    rbd_fma_peak_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(
        (double*)sink, iters, 0.999999, 1e-7);
  else
    rbd_fma_peak_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(
        (float*)sink, iters, 0.999999f, 1e-7f);
  return (int)cudaGetLastError();
}
