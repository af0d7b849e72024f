// TMEM as a per-thread spill tier for straight-line fp64 programs (probe).
//
// A thread-per-knot program keeps values that do not fit its registers in a
// per-thread "row".  Today the row is shared memory ([slot][33] layout);
// this probe measures tensor memory (tcgen05.st / tcgen05.ld, 32x32b shape:
// lane = thread of the warp's lane quadrant) as that tier: latency of a
// store -> load round trip, and throughput of reload batches interleaved
// with DFMA work at 4 and 8 warps/SM, against the same loop on shared memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ void tst2(unsigned addr, double v) {
  unsigned lo, hi;
  asm volatile("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(lo), "r"(hi) : "memory");
}
__device__ __forceinline__ double tld2(unsigned addr) {
  unsigned lo, hi;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(addr) : "memory");
  double v;
  asm volatile("mov.b64 %0, {%1, %2};" : "=d"(v) : "r"(lo), "r"(hi));
  return v;
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// one CTA = W warps; warps w and w+4 share lane quadrant w%4 and split its columns
template <int W, int NSLOT, int BATCH, int FMAS, bool TMEM>
__global__ void __launch_bounds__(W * 32, 1) k_tier(double* out, int iters, long long* cycles) {
  __shared__ unsigned s_taddr;
  extern __shared__ double s_row[];  // [NSLOT * (W/4 ... )][33] per quadrant group when !TMEM
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NCOL = (W > 4 ? 2 : 1) * 2 * NSLOT;  // columns per lane quadrant
  constexpr int ALLOC = NCOL <= 32 ? 32 : NCOL <= 64 ? 64 : NCOL <= 128 ? 128 : NCOL <= 256 ? 256 : 512;
  unsigned my = 0;
  if (TMEM) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&s_taddr)), "n"(ALLOC));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    my = s_taddr + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 2 * NSLOT);
  }
  double* row = s_row + (size_t)warp * NSLOT * 33 + lane;
  double seed = 1.0 + 1e-9 * (threadIdx.x + blockIdx.x);
  for (int s = 0; s < NSLOT; ++s) {
    if (TMEM)
      tst2(my + 2 * s, seed + s);
    else
      row[s * 33] = seed + s;
  }
  if (TMEM) twait_st();
  __syncwarp();
  long long t0 = clock64();
  double sink = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < NSLOT / BATCH; ++b) {
      double v[BATCH];
#pragma unroll
      for (int j = 0; j < BATCH; ++j) v[j] = TMEM ? tld2(my + 2 * (b * BATCH + j)) : row[(b * BATCH + j) * 33];
      if (TMEM) twait_ld();
#pragma unroll
      for (int f = 0; f < FMAS; ++f)
#pragma unroll
        for (int j = 0; j < BATCH; ++j) v[j] = fma(v[j], 0.999999999, 1e-12);
#pragma unroll
      for (int j = 0; j < BATCH; ++j) {
        if (TMEM)
          tst2(my + 2 * (b * BATCH + j), v[j]);
        else
          row[(b * BATCH + j) * 33] = v[j];
      }
      sink += v[0];
    }
    if (TMEM) twait_st();
  }
  long long t1 = clock64();
  if (lane == 0 && warp == 0) cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
  if (TMEM) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "n"(ALLOC));
  }
}

// round-trip latency: st -> wait::st -> ld -> wait::ld, dependent
__global__ void k_lat(double* out, int iters, long long* cycles) {
  __shared__ unsigned s_taddr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&s_taddr)), "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  unsigned a = s_taddr;
  double v = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    tst2(a, v);
    twait_st();
    v = tld2(a);
    twait_ld();
    v = v * 1.0000001;
  }
  long long t1 = clock64();
  cycles[0] = t1 - t0;
  out[threadIdx.x] = v;
  // ld only (independent address, no preceding store in the loop)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double w = tld2(a + 2);
    twait_ld();
    v += w;
  }
  t1 = clock64();
  cycles[1] = t1 - t0;
  out[threadIdx.x] += v;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "n"(32));
}

template <int W, int NSLOT, int BATCH, int FMAS, bool TMEM>
void run(const char* name) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int ctas = sms;  // one CTA per SM (TMEM alloc is per CTA)
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, sizeof(double) * ctas * W * 32));
  CK(cudaMalloc(&cyc, sizeof(long long) * ctas));
  size_t smem = TMEM ? 0 : sizeof(double) * W * NSLOT * 33;
  auto k = k_tier<W, NSLOT, BATCH, FMAS, TMEM>;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int iters = 200;
  k<<<ctas, W * 32, smem>>>(out, 4, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<ctas, W * 32, smem>>>(out, iters, cyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c0;
  CK(cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost));
  double per_it = (double)c0 / iters;
  // per SM per iteration: W warps x NSLOT values loaded + stored (8 B x 32 lanes each)
  double bytes = (double)W * NSLOT * 32 * 8;
  double flops = (double)ctas * W * 32 * NSLOT * FMAS * 2.0 * iters;
  printf("%-6s W=%d slots=%3d batch=%2d fmas=%2d: %8.1f cyc/iter  ld %.1f B/cyc/SM  (ld+st %.1f)  %.2f TF fp64  %.3f ms\n",
         name, W, NSLOT, BATCH, FMAS, per_it, bytes / per_it, 2 * bytes / per_it, flops / (ms * 1e-3) / 1e12, ms);
  CK(cudaFree(out));
  CK(cudaFree(cyc));
}

int main() {
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, sizeof(double) * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * 2));
  k_lat<<<1, 32>>>(out, 1000, cyc);
  CK(cudaDeviceSynchronize());
  long long c[2];
  CK(cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost));
  printf("latency: st+wait::st+ld+wait::ld+dmul %.1f cyc/iter; ld+wait::ld+dadd %.1f cyc/iter\n", c[0] / 1000.0,
         c[1] / 1000.0);
  // pure streaming of the tier (few FMAs) and with DFMA work in between
  run<4, 64, 8, 1, true>("tmem");
  run<4, 64, 8, 1, false>("smem");
  run<8, 64, 8, 1, true>("tmem");
  run<8, 64, 8, 1, false>("smem");
  run<4, 64, 16, 1, true>("tmem");
  run<4, 64, 4, 1, true>("tmem");
  run<4, 64, 1, 1, true>("tmem");
  run<4, 64, 8, 8, true>("tmem");
  run<4, 64, 8, 8, false>("smem");
  run<8, 64, 8, 8, true>("tmem");
  run<8, 64, 8, 8, false>("smem");
  run<4, 128, 8, 4, true>("tmem");
  run<8, 64, 8, 4, true>("tmem");
  run<8, 64, 8, 4, false>("smem");
  run<4, 200, 8, 4, true>("tmem");
  return 0;
}
