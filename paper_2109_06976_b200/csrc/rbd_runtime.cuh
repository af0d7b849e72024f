// rbd_runtime.cuh -- batch kernel template, launchers and the host-buffer
// session shared by every generated per-robot library (see include/rbd_b200.h).
//
// A generated library defines, per (algorithm, dtype), a knot struct K with
//   typedef T;  NDOF, NIN (1 or 3 inputs), E0/E1/E2 (per-knot output extents),
//   BK (knots per CTA = threads per CTA), STAGE (stage outputs in smem),
//   SIN/SOUT (per-knot smem row lengths, odd -> bank-conflict-free rows),
//   __device__ static void run_dev(T* my_row, T* o0, T* o1, T* o2, unsigned valid)
// -- the straight-line, fully constant-folded program for ONE knot point
// (a short C++ sin/cos prologue + one inline-PTX block).
// This header turns it into a batched sm_100a kernel: one thread per knot, the
// CTA's [BK x n] input slabs staged through shared memory with coalesced loads,
// outputs staged per thread in shared memory and written back coalesced
// (knot-major global layout, reference output_map order).
#pragma once

#if defined(__CUDACC__)
#include <cuda_runtime.h>
#endif
#include <stdint.h>
#include <string.h>
#include <math.h>
#if defined(__CUDACC__)
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>
#endif

#include "rbd_b200.h"

#if defined(__CUDACC__)
#define RBD_HD __device__ __forceinline__
#define RBD_HDC __host__ __device__
#else
#define RBD_HD inline
#define RBD_HDC
#endif

RBD_HD void rbd_sincos(double x, double* s, double* c) {
#if defined(__CUDA_ARCH__)
  sincos(x, s, c);
#else
  *s = sin(x);
  *c = cos(x);
#endif
}

RBD_HD void rbd_sincos(float x, float* s, float* c) {
#if defined(__CUDA_ARCH__)
  sincosf(x, s, c);
#else
  *s = sinf(x);
  *c = cosf(x);
#endif
}

// sin and cos of N angles evaluated side by side (fp64): Cody-Waite
// reduction by pi/2 in two parts, then the classic minimax kernels on
// [-pi/4, pi/4] (the fdlibm __kernel_sin / __kernel_cos coefficients) and a
// quadrant select.  N independent chains share each coefficient (one uniform
// register pair per coefficient, not one per call) and give the scheduler
// N-way ILP; ~1-2 ulp, well inside the 1e-9 parity bound.  Angles beyond
// |x| > 2^20 (where the 2-part reduction loses bits) take sincos().
#if defined(__CUDACC__)
// out-of-line fallback, so the rarely taken path adds a call, not N inlined
// copies of libdevice's reduction, to the straight-line kernel body
static __device__ __noinline__ double2 rbd_sincos_slow(double x) {
  double2 v;
  sincos(x, &v.x, &v.y);
  return v;
}
#endif

template <int N>
RBD_HD void rbd_sincos_batch(const double* x, double* s, double* c) {
#if defined(__CUDA_ARCH__)
  // pi/2 = P1 + P2 + O(1e-33); with FMA, x - k P1 is rounded once
  const double TWO_OVER_PI = 6.366197723675814e-01;
  const double P1 = 1.5707963267948966e+00, P2 = 6.123233995736766e-17;
  const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
               S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
               S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
  const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
               C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
               C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
  bool big = false;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double k = rint(x[j] * TWO_OVER_PI);
    const double r = fma(-k, P2, fma(-k, P1, x[j]));
    const double z = r * r;
    const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, S6, S5), S4), S3), S2), S1);
    const double sn = fma(r * z, ps, r);
    const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, C6, C5), C4), C3), C2), C1);
    const double cs = fma(z * z, pc, fma(-0.5, z, 1.0));
    const int q = (int)(long long)k & 3;
    const double a = (q & 1) ? cs : sn, b = (q & 1) ? sn : cs;
    s[j] = (q & 2) ? -a : a;
    c[j] = ((q + 1) & 2) ? -b : b;
    big |= fabs(x[j]) > 1048576.0;
  }
  if (big) {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (fabs(x[j]) > 1048576.0) {
        const double2 v = rbd_sincos_slow(x[j]);
        s[j] = v.x;
        c[j] = v.y;
      }
  }
#else
  for (int j = 0; j < N; ++j) {
    s[j] = sin(x[j]);
    c[j] = cos(x[j]);
  }
#endif
}

RBD_HD void rbd_sincos_fast(double x, double* s, double* c) { rbd_sincos_batch<1>(&x, s, c); }
RBD_HD void rbd_sincos_fast(float x, float* s, float* c) { rbd_sincos(x, s, c); }

RBD_HD double rbd_fma(double a, double b, double c) { return fma(a, b, c); }
RBD_HD float rbd_fma(float a, float b, float c) { return fmaf(a, b, c); }

#if defined(__CUDACC__)

// ---------------------------------------------------------------------------
// batch kernel: CTA = BK knots, thread t = knot (blockIdx.x * BK + t)
// ---------------------------------------------------------------------------
// parked-output list length / identity flag (PARK kernels only)
template <class K, class = void>
struct rbd_park_traits {
  static constexpr int nout = 0;
  static constexpr bool ofull = true;
};
template <class K>
struct rbd_park_traits<K, decltype((void)K::NOUT, void())> {
  static constexpr int nout = K::NOUT;
  static constexpr bool ofull = K::OFULL;
};
template <class K, class = void>
struct rbd_prog_traits {
  static constexpr int nprog = 1;
};
template <class K>
struct rbd_prog_traits<K, decltype((void)K::NPROG, void())> {
  static constexpr int nprog = K::NPROG;
};
template <class K>
__host__ __device__ constexpr int rbd_nprog() { return rbd_prog_traits<K>::nprog; }

template <class K>
__host__ __device__ constexpr int rbd_nout() { return rbd_park_traits<K>::nout; }
// widest per-knot input window of a kernel's inputs (registers for staging)
template <class K>
__host__ __device__ constexpr int rbd_max_inw() {
  int w = 0;
  for (int a = 0; a < K::NIN; ++a) w = K::inw(a) > w ? K::inw(a) : w;
  return w;
}

template <class K>
__host__ __device__ constexpr bool rbd_ofull() { return rbd_park_traits<K>::ofull; }
template <class K, class = void>
struct rbd_l2pf_traits {
  static constexpr int waves = 0;
};
template <class K>
struct rbd_l2pf_traits<K, decltype((void)K::L2PF, void())> {
  static constexpr int waves = K::L2PF;
};

template <class K, class = void>
struct rbd_zmap_traits {
  static constexpr int n = 0;
};
template <class K>
struct rbd_zmap_traits<K, decltype((void)K::NZM, void())> {
  static constexpr int n = K::NZM;
};
template <class K>
__host__ __device__ constexpr int rbd_nzm() { return rbd_zmap_traits<K>::n; }

template <class K, class = void>
struct rbd_bulk_traits {
  static constexpr bool on = false;
};
template <class K>
struct rbd_bulk_traits<K, decltype((void)K::BULK, void())> {
  static constexpr bool on = K::BULK;
};

// TMA bulk store of one output array's CTA range: src = [nk][E] staged
// array-major in shared memory, dst = the knots' contiguous global rows.
// One elected thread issues it (bulk-group completion); the caller waits for
// the shared-memory reads before the staging is reused or the CTA exits.
// Falls back to a cooperative 16-byte copy when the range is not a whole
// number of 16-byte units or dst is not 16-byte aligned (bulk-copy rule).
template <class T, int E, int NT>
__device__ __forceinline__ bool rbd_bulk_store(T* dst, const T* src, int nk, int tid) {
  const unsigned bytes = (unsigned)(nk * E * (int)sizeof(T));
  const bool ok = (bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  if (ok) {
    if (tid == 0)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"((unsigned)__cvta_generic_to_shared(src)), "r"(bytes)
                   : "memory");
  } else {
    for (int i = tid; i < nk * E; i += NT) __stcs(dst + i, src[i]);
  }
  return ok;
}

// TMA bulk prefetch into L2 of the input slabs of the CTA `waves` waves
// ahead (one wave = %nsmid SMs x MINB CTAs: roughly the CTA that will take
// this SM slot): its input loads then hit L2
// instead of waiting on HBM behind the output write stream.  One thread per
// input array; the slab is [BK knots][ins(a)] contiguous (a part program's
// window is inside it); the 16-byte-aligned body only (bulk-copy rule).
template <class K>
__device__ __forceinline__ void rbd_prefetch_slabs(const void* q, const void* qd, const void* u, const void* fx,
                                                   long long N, int tid) {
  constexpr int waves = rbd_l2pf_traits<K>::waves;
  if constexpr (waves > 0) {
    typedef typename K::T T;
    if (tid < K::NIN) {
      unsigned nsm;
      asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));  // SMs on this GPU (148 on B200)
      const long long nb = (long long)blockIdx.x + (long long)waves * nsm * K::MINB;
      const long long k0 = nb * K::BK;
      if (k0 < N) {
        const long long nk = N - k0 < K::BK ? N - k0 : K::BK;
        const void* arr = tid == 0 ? q : (tid == 1 ? qd : (tid == 2 ? u : fx));
        const char* lo = reinterpret_cast<const char*>(arr) + k0 * K::ins(tid) * (long long)sizeof(T);
        const char* hi = lo + nk * K::ins(tid) * (long long)sizeof(T);
        const char* a = reinterpret_cast<const char*>((reinterpret_cast<uintptr_t>(lo) + 15) & ~(uintptr_t)15);
        const unsigned bytes = (unsigned)((hi - a) & ~15LL);
        if (hi > a && bytes)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
      }
    }
  }
}

// coalesced write-back of nk knots x E elements of one output array, 16-byte
// streaming stores when E is a multiple of the vector width and dst is
// 16-byte aligned (else 8/4-byte stores); get(k, e) yields knot k's element e
template <class T>
struct rbd_vec16;
template <>
struct rbd_vec16<double> {
  typedef double2 t;
};
template <>
struct rbd_vec16<float> {
  typedef float4 t;
};
template <class T, int E, int NT, class F>
__device__ __forceinline__ void rbd_write_back(T* dst, int nk, int tid, F get) {
  constexpr int VW = 16 / (int)sizeof(T);
  if (E % VW == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    typedef typename rbd_vec16<T>::t V;
    V* vd = reinterpret_cast<V*>(dst);
    for (int p = tid; p < nk * (E / VW); p += NT) {
      const int idx = p * VW, k = idx / E, e = idx - k * E;
      V v;
      T* pv = reinterpret_cast<T*>(&v);
#pragma unroll
      for (int j = 0; j < VW; ++j) pv[j] = get(k, e + j);
      __stcs(vd + p, v);
    }
  } else {
    for (int idx = tid; idx < nk * E; idx += NT) {
      const int k = idx / E, e = idx - k * E;
      __stcs(dst + idx, get(k, e));
    }
  }
}

// write-back through an element map (element e of a knot's output row ->
// slot map[e] of that knot's staged row, or -1 for a structural 0).  With
// 16-byte vectors, thread t's vectors start at elements (VW t + i NT VW)
// mod E, which repeat with period P = lcm(NT VW, E) / (NT VW) in i: the
// thread reads its P x VW map entries once into registers instead of one
// shared-memory map load per element (quad12 fp32: P = 9; gradFD 2^20
// 341 -> 328 us, gradID 300 -> 291).  Falls back to the
// per-element form when the period is long or vectors do not tile a row.
RBD_HDC constexpr int rbd_gcd(int a, int b) { return b == 0 ? a : rbd_gcd(b, a % b); }
template <class T, int E, int NT>
__device__ __forceinline__ void rbd_write_back_map(T* dst, int nk, int tid, const short* map, const T* rows,
                                                   int stride) {
  constexpr int VW = 16 / (int)sizeof(T);
  constexpr int STEP = NT * VW;
  constexpr int P = E / rbd_gcd(STEP, E);  // lcm(STEP, E) / STEP
  if constexpr (E % VW == 0 && P * VW <= 40) {
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      short m[P][VW];
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const int e0 = (tid * VW + r * STEP) % E;
#pragma unroll
        for (int j = 0; j < VW; ++j) m[r][j] = map[e0 + j];
      }
      typedef typename rbd_vec16<T>::t V;
      V* vd = reinterpret_cast<V*>(dst);
      const int nv = nk * (E / VW);
      for (int i0 = 0; i0 * NT < nv; i0 += P) {
#pragma unroll
        for (int r = 0; r < P; ++r) {
          const int p = tid + (i0 + r) * NT;
          if (p < nv) {
            const int k = (p * VW) / E;
            V v;
            T* pv = reinterpret_cast<T*>(&v);
#pragma unroll
            for (int j = 0; j < VW; ++j) pv[j] = m[r][j] >= 0 ? rows[k * stride + m[r][j]] : T(0);
            __stcs(vd + p, v);
          }
        }
      }
      return;
    }
  }
  rbd_write_back<T, E, NT>(dst, nk, tid, [=](int k, int e) {
    const int sl = map[e];
    return sl >= 0 ? rows[k * stride + sl] : T(0);
  });
}

template <class K>
__global__ void __launch_bounds__(K::BK, K::MINB)
rbd_batch_kernel(const typename K::T* __restrict__ q, const typename K::T* __restrict__ qd,
                 const typename K::T* __restrict__ u, const typename K::T* __restrict__ fx,
                 typename K::T* __restrict__ o0, typename K::T* __restrict__ o1,
                 typename K::T* __restrict__ o2, long long N, typename K::T* __restrict__ xs) {
  typedef typename K::T T;
  constexpr int BK = K::BK, n = K::NDOF;
  extern __shared__ __align__(16) unsigned char rbd_smem[];
  T* s_in = reinterpret_cast<T*>(rbd_smem);  // [BK][SIN], SIN odd -> conflict-free rows
  // [BK][SOUT] when staging; with the row in TMEM (TROW) the output staging
  // aliases the input staging (the program copies its inputs to TMEM and
  // passes a CTA barrier before its first output store)
  T* s_out = K::TROW ? s_in : s_in + BK * K::SIN;
  const long long base = (long long)blockIdx.x * BK;
  const long long left = N - base;
  const int nk = left < BK ? (int)left : BK;
  const int tid = threadIdx.x;
  rbd_prefetch_slabs<K>(q, qd, u, fx, N, tid);

  // all input loads of this thread are issued before the first smem store
  // (one HBM round trip per CTA, not one per element); input a contributes
  // its window of inw(a) scalars per knot (a part program's dof window; 6 per
  // dof for f_ext), at offset ing(a) of the knot's global row of ins(a)
  constexpr int NT = K::inr(K::NIN - 1) + K::inw(K::NIN - 1);
  T v[NT];
#pragma unroll
  for (int a = 0; a < K::NIN; ++a) {
    const T* src = (a == 0 ? q : (a == 1 ? qd : (a == 2 ? u : fx))) + base * K::ins(a) + K::ing(a);
#pragma unroll
    for (int r = 0; r < K::inw(a); ++r) {
      const int idx = tid + r * BK;
      const int k = idx / K::inw(a), j = idx - k * K::inw(a);
      v[K::inr(a) + r] = (idx < nk * K::inw(a)) ? __ldg(src + k * K::ins(a) + j) : T(0);
    }
  }
#pragma unroll
  for (int a = 0; a < K::NIN; ++a) {
#pragma unroll
    for (int r = 0; r < K::inw(a); ++r) {
      const int idx = tid + r * BK;
      const int k = idx / K::inw(a), j = idx - k * K::inw(a);
      s_in[k * K::SIN + K::inr(a) + j] = v[K::inr(a) + r];
    }
  }
  short* s_map = reinterpret_cast<short*>(s_in + BK * K::SIN);  // PARK: output list -> row slot
  unsigned short* s_elem = reinterpret_cast<unsigned short*>(s_map + rbd_nout<K>());
  if constexpr (K::PARK) {
    for (int j = tid; j < rbd_nout<K>(); j += BK) {
      s_map[j] = K::omap()[j];
      if constexpr (!rbd_ofull<K>()) s_elem[j] = K::oelem()[j];
    }
  }
  // TMEM row with structural zeros unstaged: element -> dense staging slot (or -1)
  short* s_zm = reinterpret_cast<short*>(s_in + BK * (K::SIN > K::SOUT ? K::SIN : K::SOUT));
  if constexpr (rbd_nzm<K>() > 0) {
    for (int j = tid; j < rbd_nzm<K>(); j += BK) s_zm[j] = K::zmap()[j];
  }
  __syncthreads();
  // tensor memory for the imports a split column kernel homes there: one
  // allocation per CTA (4k warps, warp w -> TMEM lanes [32 (w % 4), +32)),
  // released at the end so the SM's other CTAs can allocate
  unsigned tm = 0;
  if constexpr (K::TCOLS > 0) {
    __shared__ unsigned s_tmem;
    if ((tid >> 5) == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&s_tmem)), "n"(K::TCOLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // lane quadrant of the warp; warps w and w + 4 (, w + 8 ...) split the columns
    tm = s_tmem + ((unsigned)(32 * ((tid >> 5) & 3)) << 16) + (unsigned)((tid >> 7) * (K::TCOLS / (BK / 128)));
  }
  T* my = s_in + tid * K::SIN;  // this knot's inputs + its sin/cos scratch
  // split prefix kernel: this knot's export slots in the scratch ([32-knot chunk][slot][lane])
  T* xb = K::NX ? xs + ((size_t)((base + tid) >> 5) * K::NX * 32 + ((base + tid) & 31)) : nullptr;

  if constexpr (K::PARK) {
    // the program parks every output value in its row; write the CTA's
    // contiguous output ranges back coalesced (structural zeros from the map)
    K::run_dev(my, nullptr, nullptr, nullptr, 1u, xb, tm);
    __syncthreads();
    if constexpr (rbd_nout<K>() == 0) {
      // nothing parked (a split prefix whose outputs all come from the columns)
    } else if constexpr (!rbd_ofull<K>()) {
      // a part program (subset of the root trees): only its own elements
      constexpr int M = rbd_nout<K>();
      for (int idx = tid; idx < nk * M; idx += BK) {
        const int k = idx / M, j = idx - k * M;
        const int e = s_elem[j], sl = s_map[j];
        const T v = sl >= 0 ? s_in[k * K::SIN + sl] : T(0);
        if (e < K::E0)
          __stcs(o0 + (base + k) * K::E0 + e, v);
        else if (e < K::E0 + K::E1)
          __stcs(o1 + (base + k) * K::E1 + (e - K::E0), v);
        else
          __stcs(o2 + (base + k) * K::E2 + (e - K::E0 - K::E1), v);
      }
    } else {
      rbd_write_back_map<T, K::E0, BK>(o0 + base * K::E0, nk, tid, s_map, s_in, K::SIN);
      if constexpr (K::E1 > 0) rbd_write_back_map<T, K::E1, BK>(o1 + base * K::E1, nk, tid, s_map + K::E0, s_in, K::SIN);
      if constexpr (K::E2 > 0)
        rbd_write_back_map<T, K::E2, BK>(o2 + base * K::E2, nk, tid, s_map + K::E0 + K::E1, s_in, K::SIN);
    }
  } else if constexpr (rbd_bulk_traits<K>::on) {
    // array-major staging [BK][E0] | [BK][E1] | [BK][E2]: each array's CTA
    // range is one contiguous block in shared and in global memory
    T* so1 = s_out + BK * K::E0;
    T* so2 = so1 + BK * K::E1;
    K::run_dev(my, s_out + tid * K::E0, so1 + tid * K::E1, so2 + tid * K::E2, 1u, xb, tm);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> TMA reads
    __syncthreads();
    rbd_bulk_store<T, K::E0, BK>(o0 + base * K::E0, s_out, nk, tid);
    if constexpr (K::E1 > 0) rbd_bulk_store<T, K::E1, BK>(o1 + base * K::E1, so1, nk, tid);
    if constexpr (K::E2 > 0) rbd_bulk_store<T, K::E2, BK>(o2 + base * K::E2, so2, nk, tid);
    if (tid == 0) {
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging read before the CTA exits
    }
  } else if constexpr (K::STAGE) {
    T* o = s_out + tid * K::SOUT;
    K::run_dev(my, o, o + K::E0, o + K::E0 + K::E1, 1u, xb, tm);
    __syncthreads();
    if constexpr (K::TPART) {
      // a part program's elements, staged densely: element map write-back
      constexpr int M = K::NOUT;
      const unsigned short* oe = K::oelem();
      for (int idx = tid; idx < nk * M; idx += BK) {
        const int k = idx / M, j = idx - k * M;
        const int e = oe[j];
        const T v = s_out[k * K::SOUT + j];
        if (e < K::E0)
          __stcs(o0 + (base + k) * K::E0 + e, v);
        else if (e < K::E0 + K::E1)
          __stcs(o1 + (base + k) * K::E1 + (e - K::E0), v);
        else
          __stcs(o2 + (base + k) * K::E2 + (e - K::E0 - K::E1), v);
      }
    } else if constexpr (rbd_nzm<K>() > 0) {
      // per-element map loads here: the register-cached map of
      // rbd_write_back_map raises quad12 fp64's kernel from 164 to 178
      // registers, which drops the third (TMEM-waiting) CTA per SM: 440 -> 546 us
      auto zm = [&](int off) {
        return [=](int k, int e) {
          const int j = s_zm[off + e];
          return j >= 0 ? s_out[k * K::SOUT + j] : T(0);
        };
      };
      rbd_write_back<T, K::E0, BK>(o0 + base * K::E0, nk, tid, zm(0));
      if constexpr (K::E1 > 0) rbd_write_back<T, K::E1, BK>(o1 + base * K::E1, nk, tid, zm(K::E0));
      if constexpr (K::E2 > 0) rbd_write_back<T, K::E2, BK>(o2 + base * K::E2, nk, tid, zm(K::E0 + K::E1));
    } else {
      // coalesced write-back, one output array at a time
      auto staged = [&](int off) { return [=](int k, int e) { return s_out[k * K::SOUT + off + e]; }; };
      rbd_write_back<T, K::E0, BK>(o0 + base * K::E0, nk, tid, staged(0));
      if constexpr (K::E1 > 0) rbd_write_back<T, K::E1, BK>(o1 + base * K::E1, nk, tid, staged(K::E0));
      if constexpr (K::E2 > 0) rbd_write_back<T, K::E2, BK>(o2 + base * K::E2, nk, tid, staged(K::E0 + K::E1));
    }
  } else {
    // every thread runs the program (CTA barriers inside); stores of the
    // padding threads of the last CTA are predicated off
    const long long k = base + (tid < nk ? tid : 0);
    K::run_dev(my, o0 + k * K::E0, K::E1 ? o1 + k * K::E1 : nullptr,
               K::E2 ? o2 + k * K::E2 : nullptr, tid < nk ? 1u : 0u, xb, tm);
  }
  if constexpr (K::TCOLS > 0) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if ((tid >> 5) == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(K::TCOLS));  // warp 0: tm is the allocation base
  }
}

// ---------------------------------------------------------------------------
// warp-specialised kernel: CTA = W warps on a group of 32 knots (lane = knot);
// the generated run_group() runs the program's tasks phase by phase.
// Persistent: CTAs loop over 32-knot groups so a global (L2-resident) arena
// is sized by the grid, not by N.
// ---------------------------------------------------------------------------
#define RBD_WS_LANES 33
template <class K>
__global__ void __launch_bounds__(K::W * 32, K::MINB)
rbd_ws_kernel(const typename K::T* __restrict__ q, const typename K::T* __restrict__ qd,
              const typename K::T* __restrict__ u, const typename K::T* __restrict__ fx,
              typename K::T* __restrict__ o0, typename K::T* __restrict__ o1,
              typename K::T* __restrict__ o2, long long N, typename K::T* __restrict__ garena) {
  typedef typename K::T T;
  constexpr int n = K::NDOF, NT = K::W * 32, L = RBD_WS_LANES;
  extern __shared__ __align__(16) unsigned char rbd_smem[];
  T* s_in = reinterpret_cast<T*>(rbd_smem);         // [SIN][33]
  T* s_ar = s_in + K::SIN * L;                        // [NA][33] when ARENA_SMEM
  T* s_out = s_ar + (K::ARENA_SMEM ? K::NA * L : 0);  // [SOUT][33] when STAGE
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long groups = (N + 31) / 32;
  for (long long g = blockIdx.x; g < groups; g += gridDim.x) {
    const long long base = g * 32;
    const int nk = (N - base) < 32 ? (int)(N - base) : 32;
    // input a: 32 knots x inw(a) scalars, PER(a) loads per thread, all in flight
    constexpr int WMAX = rbd_max_inw<K>();  // widest input row (f_ext 6 per dof, a split scratch nx)
    constexpr int PMAX = (32 * WMAX + NT - 1) / NT;
    T v[K::NIN][PMAX];
#pragma unroll
    for (int a = 0; a < K::NIN; ++a) {
      const T* src = (a == 0 ? q : (a == 1 ? qd : (a == 2 ? u : fx))) + base * K::ins(a) + K::ing(a);
#pragma unroll
      for (int r = 0; r < (32 * K::inw(a) + NT - 1) / NT; ++r) {
        const int idx = tid + r * NT;
        const int k = idx / K::inw(a), j = idx - k * K::inw(a);
        v[a][r] = (idx < nk * K::inw(a)) ? __ldg(src + k * K::ins(a) + j) : T(0);
      }
    }
#pragma unroll
    for (int a = 0; a < K::NIN; ++a) {
#pragma unroll
      for (int r = 0; r < (32 * K::inw(a) + NT - 1) / NT; ++r) {
        const int idx = tid + r * NT;
        if (idx < 32 * K::inw(a)) {
          const int k = idx / K::inw(a), j = idx - k * K::inw(a);
          s_in[(K::inr(a) + j) * L + k] = v[a][r];
        }
      }
    }
    __syncthreads();
    K::prologue(s_in, warp, lane);
    __syncthreads();
    const unsigned a_in = (unsigned)__cvta_generic_to_shared(s_in + lane);
    typename K::arena_t a_ar;
    if constexpr (K::ARENA_SMEM)
      a_ar = (unsigned)__cvta_generic_to_shared(s_ar + lane);
    else if constexpr (K::ARENA_GROUP)  // split columns: the prefix kernel's exports of this group
      a_ar = (unsigned long long)(garena + (size_t)g * K::NA * 32 + lane);
    else  // one arena per resident CTA (grid row y of NVAR variant rows)
      a_ar = (unsigned long long)(garena + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * K::NA * 32 + lane);
    typename K::out_t a0, a1, a2;
    const int kk = lane < nk ? lane : 0;
    if constexpr (K::STAGE) {
      a0 = (unsigned)__cvta_generic_to_shared(s_out + lane);
      a1 = (unsigned)__cvta_generic_to_shared(s_out + K::E0 * L + lane);
      a2 = (unsigned)__cvta_generic_to_shared(s_out + (K::E0 + K::E1) * L + lane);
    } else {
      a0 = (unsigned long long)(o0 + (base + kk) * K::E0);
      a1 = (unsigned long long)(K::E1 ? o1 + (base + kk) * K::E1 : o0);
      a2 = (unsigned long long)(K::E2 ? o2 + (base + kk) * K::E2 : o0);
    }
    K::run_group(blockIdx.y, warp, a_in, a_ar, a0, a1, a2, lane < nk ? 1u : 0u);  // ends with a barrier
    if constexpr (K::STAGE) {
      {
        T* dst = o0 + base * K::E0;
        for (int idx = tid; idx < nk * K::E0; idx += NT) {
          const int k = idx / K::E0, e = idx - k * K::E0;
          __stcs(dst + idx, s_out[e * L + k]);
        }
      }
      if constexpr (K::E1 > 0) {
        T* dst = o1 + base * K::E1;
        for (int idx = tid; idx < nk * K::E1; idx += NT) {
          const int k = idx / K::E1, e = idx - k * K::E1;
          __stcs(dst + idx, s_out[(K::E0 + e) * L + k]);
        }
      }
      if constexpr (K::E2 > 0) {
        T* dst = o2 + base * K::E2;
        for (int idx = tid; idx < nk * K::E2; idx += NT) {
          const int k = idx / K::E2, e = idx - k * K::E2;
          __stcs(dst + idx, s_out[(K::E0 + K::E1 + e) * L + k]);
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// fine-grained warp-specialised kernel (fsched.py): CTA = W warps on a group
// of 32 knots (lane = knot); warp w runs ONE straight-line block holding its
// share of the op-level list schedule, phases separated by `bar.sync 1`, its
// values in registers across phases; values another warp reads go through a
// [slot][33] shared-memory arena.  blockIdx.y = column variant (a gradient
// program's prefix + one share of its columns).  Persistent over groups.
// ---------------------------------------------------------------------------
template <class K>
__global__ void __launch_bounds__(K::W * 32, K::MINB)
rbd_fs_kernel(const typename K::T* __restrict__ q, const typename K::T* __restrict__ qd,
              const typename K::T* __restrict__ u, const typename K::T* __restrict__ fx,
              typename K::T* __restrict__ o0, typename K::T* __restrict__ o1,
              typename K::T* __restrict__ o2, long long N) {
  typedef typename K::T T;
  constexpr int NT = K::W * 32, L = RBD_WS_LANES;
  extern __shared__ __align__(16) unsigned char rbd_smem[];
  T* s_in = reinterpret_cast<T*>(rbd_smem);  // [SIN][33]
  T* s_ar = s_in + K::SIN * L;                // [NA][33]
  T* s_out = s_ar + K::NA * L;                // [SOUT][33] when STAGE
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int var = blockIdx.y;
  const long long groups = (N + 31) / 32;
  for (long long g = blockIdx.x; g < groups; g += gridDim.x) {
    const long long base = g * 32;
    const int nk = (N - base) < 32 ? (int)(N - base) : 32;
    constexpr int WMAX = rbd_max_inw<K>();  // widest input row (f_ext 6 per dof, a split scratch nx)
    constexpr int PMAX = (32 * WMAX + NT - 1) / NT;
    T v[K::NIN][PMAX];
#pragma unroll
    for (int a = 0; a < K::NIN; ++a) {
      const T* src = (a == 0 ? q : (a == 1 ? qd : (a == 2 ? u : fx))) + base * K::ins(a) + K::ing(a);
#pragma unroll
      for (int r = 0; r < (32 * K::inw(a) + NT - 1) / NT; ++r) {
        const int idx = tid + r * NT;
        const int k = idx / K::inw(a), j = idx - k * K::inw(a);
        v[a][r] = (idx < nk * K::inw(a)) ? __ldg(src + k * K::ins(a) + j) : T(0);
      }
    }
#pragma unroll
    for (int a = 0; a < K::NIN; ++a) {
#pragma unroll
      for (int r = 0; r < (32 * K::inw(a) + NT - 1) / NT; ++r) {
        const int idx = tid + r * NT;
        if (idx < 32 * K::inw(a)) {
          const int k = idx / K::inw(a), j = idx - k * K::inw(a);
          s_in[(K::inr(a) + j) * L + k] = v[a][r];
        }
      }
    }
    __syncthreads();
    K::prologue(s_in, warp, lane);
    __syncthreads();
    const unsigned a_in = (unsigned)__cvta_generic_to_shared(s_in + lane);
    const unsigned a_ar = (unsigned)__cvta_generic_to_shared(s_ar + lane);
    typename K::out_t a0, a1, a2;
    const int kk = lane < nk ? lane : 0;
    if constexpr (K::STAGE) {
      a0 = (unsigned)__cvta_generic_to_shared(s_out + lane);
      a1 = (unsigned)__cvta_generic_to_shared(s_out + K::E0 * L + lane);
      a2 = (unsigned)__cvta_generic_to_shared(s_out + (K::E0 + K::E1) * L + lane);
    } else {
      a0 = (unsigned long long)(o0 + (base + kk) * K::E0);
      a1 = (unsigned long long)(K::E1 ? o1 + (base + kk) * K::E1 : o0);
      a2 = (unsigned long long)(K::E2 ? o2 + (base + kk) * K::E2 : o0);
    }
    K::run(var, warp, a_in, a_ar, a0, a1, a2, lane < nk ? 1u : 0u);
    __syncthreads();
    if constexpr (K::STAGE) {
      {
        T* dst = o0 + base * K::E0;
        for (int idx = tid; idx < nk * K::E0; idx += NT) {
          const int k = idx / K::E0, e = idx - k * K::E0;
          __stcs(dst + idx, s_out[e * L + k]);
        }
      }
      if constexpr (K::E1 > 0) {
        T* dst = o1 + base * K::E1;
        for (int idx = tid; idx < nk * K::E1; idx += NT) {
          const int k = idx / K::E1, e = idx - k * K::E1;
          __stcs(dst + idx, s_out[(K::E0 + e) * L + k]);
        }
      }
      if constexpr (K::E2 > 0) {
        T* dst = o2 + base * K::E2;
        for (int idx = tid; idx < nk * K::E2; idx += NT) {
          const int k = idx / K::E2, e = idx - k * K::E2;
          __stcs(dst + idx, s_out[(K::E0 + K::E1 + e) * L + k]);
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// fused rollout (warp-specialised program, FD or gradFD): B trajectories x H
// semi-implicit Euler steps in ONE launch.  A CTA owns a 32-trajectory group
// for the whole horizon: per step it stages (q_k, qd_k, tau_k), runs the
// program (outputs of step k to global), then advances the group's states
// in place -- qd_{k+1} = qd_k + dt qdd_k, q_{k+1} = q_k + dt qd_{k+1} --
// before the next step.  Time-major arrays: q, qd [H+1][B][n] (step 0 set by
// the caller), tau / qdd [H][B][n], gradients [H][B][n*n].  States written in
// the launch are re-read with plain (coherent) loads, not __ldg.
// ---------------------------------------------------------------------------
template <class K>
__global__ void __launch_bounds__(K::W * 32, K::MINB)
rbd_ws_rollout_kernel(typename K::T* __restrict__ q, typename K::T* __restrict__ qd,
                      const typename K::T* __restrict__ tau, typename K::T* __restrict__ o0,
                      typename K::T* __restrict__ o1, typename K::T* __restrict__ o2, long long B, int H,
                      typename K::T dt, typename K::T* __restrict__ garena) {
  typedef typename K::T T;
  constexpr int n = K::NDOF, NT = K::W * 32, L = RBD_WS_LANES;
  static_assert(K::LO == 0 && K::NP == K::NDOF && K::NIN == 3 && K::NVAR == 1, "rollout: whole-robot program");
  // qdd is the last output: FD -> out0 [n], gradFD -> out2 [n]
  constexpr int EQ = K::E2 ? K::E2 : K::E0;
  static_assert(EQ == n, "rollout: FD / gradFD programs only");
  extern __shared__ __align__(16) unsigned char rbd_smem[];
  T* s_in = reinterpret_cast<T*>(rbd_smem);
  T* s_ar = s_in + K::SIN * L;
  T* s_out = s_ar + (K::ARENA_SMEM ? K::NA * L : 0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long groups = (B + 31) / 32;
  for (long long g = blockIdx.x; g < groups; g += gridDim.x) {
    const long long base = g * 32;
    const int nk = (B - base) < 32 ? (int)(B - base) : 32;
    {  // step 0: q_0, qd_0, tau_0; later steps keep q, qd in shared memory
      const T* src3[3] = {q, qd, tau};
      for (int a = 0; a < 3; ++a)
        for (int idx = tid; idx < 32 * n; idx += NT) {
          const int kn = idx / n, j = idx - kn * n;
          s_in[(K::inr(a) + j) * L + kn] = kn < nk ? src3[a][(base + kn) * n + j] : T(0);
        }
      __syncthreads();
    }
    for (int k = 0; k < H; ++k) {
      const size_t st = (size_t)k * B * n;
      K::prologue(s_in, warp, lane);
      __syncthreads();
      const unsigned a_in = (unsigned)__cvta_generic_to_shared(s_in + lane);
      typename K::arena_t a_ar;
      if constexpr (K::ARENA_SMEM)
        a_ar = (unsigned)__cvta_generic_to_shared(s_ar + lane);
      else
        a_ar = (unsigned long long)(garena + (size_t)blockIdx.x * K::NA * 32 + lane);
      T* p0 = o0 + (size_t)k * B * K::E0;
      T* p1 = K::E1 ? o1 + (size_t)k * B * K::E1 : o0;
      T* p2 = K::E2 ? o2 + (size_t)k * B * K::E2 : o0;
      typename K::out_t a0, a1, a2;
      const int kk = lane < nk ? lane : 0;
      if constexpr (K::STAGE) {
        a0 = (unsigned)__cvta_generic_to_shared(s_out + lane);
        a1 = (unsigned)__cvta_generic_to_shared(s_out + K::E0 * L + lane);
        a2 = (unsigned)__cvta_generic_to_shared(s_out + (K::E0 + K::E1) * L + lane);
      } else {
        a0 = (unsigned long long)(p0 + (base + kk) * K::E0);
        a1 = (unsigned long long)(p1 + (base + kk) * K::E1);
        a2 = (unsigned long long)(p2 + (base + kk) * K::E2);
      }
      K::run_group(0, warp, a_in, a_ar, a0, a1, a2, lane < nk ? 1u : 0u);  // ends with a barrier
      // the program is done with tau_k: fetch tau_{k+1} into its rows with
      // asynchronous copies that land under the write-back and the Euler update
      if (k + 1 < H) {
        const T* tn = tau + (size_t)(k + 1) * B * n;
        for (int idx = tid; idx < nk * n; idx += NT) {
          const int kn = idx / n, j = idx - kn * n;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(s_in + (K::inr(2) + j) * L + kn);
          asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sa), "l"(tn + (base + kn) * n + j),
                       "n"((int)sizeof(T)) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      if constexpr (K::STAGE) {
        for (int b = 0; b < 3; ++b) {
          const int E = b == 0 ? K::E0 : (b == 1 ? K::E1 : K::E2);
          const int off = b == 0 ? 0 : (b == 1 ? K::E0 : K::E0 + K::E1);
          T* dst = (b == 0 ? p0 : (b == 1 ? p1 : p2)) + base * E;
          for (int idx = tid; idx < nk * E; idx += NT) {
            const int kn = idx / E, e = idx - kn * E;
            __stcs(dst + idx, s_out[(off + e) * L + kn]);
          }
        }
      }
      __syncthreads();  // this step's qdd (global or staged) is visible to the whole CTA
      // semi-implicit Euler from the staged states; the new states go to the
      // trajectory (global) and stay in shared memory for the next step
      const T* qddk = (K::E2 ? p2 : p0) + base * n;
      const size_t nx = (size_t)(k + 1) * B * n;
      for (int idx = tid; idx < nk * n; idx += NT) {
        const int kn = idx / n, j = idx - kn * n;
        const T a = K::STAGE ? s_out[((K::E2 ? K::E0 + K::E1 : 0) + j) * L + kn] : qddk[idx];
        T& sq = s_in[(K::inr(0) + j) * L + kn];
        T& sqd = s_in[(K::inr(1) + j) * L + kn];
        const T v = sqd + dt * a;
        const T qn = sq + dt * v;
        sqd = v;
        sq = qn;
        qd[nx + (base + kn) * n + j] = v;
        q[nx + (base + kn) * n + j] = qn;
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();  // states and tau_{k+1} staged for the next step
    }
  }
}

template <class K>
constexpr size_t rbd_smem_bytes();
static inline bool rbd_capturing(cudaStream_t s);

template <class K>
static int rbd_launch_rollout(void* q, void* qd, const void* tau, void* o0, void* o1, void* o2, int64_t B, int32_t H,
                              double dt, void* stream) {
  typedef typename K::T T;
  if (B < 0 || H < 0 || !q || !qd || !tau || !o0 || (K::E1 > 0 && !o1) || (K::E2 > 0 && !o2)) return RBD_EINVAL;
  if (B == 0 || H == 0) return 0;
  constexpr size_t smem = rbd_smem_bytes<K>();
  struct cache_t {
    std::mutex lock;
    bool ready = false;
    int grid = 0;
    void* arena = nullptr;
    cudaEvent_t last = nullptr;
    bool used = false;
  };
  static cache_t cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  cache_t& c = cache[dev & 63];
  std::lock_guard<std::mutex> guard(c.lock);
  cudaError_t e = cudaSuccess;
  if (!c.ready) {
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(rbd_ws_rollout_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return (int)e;
    }
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rbd_ws_rollout_kernel<K>, K::W * 32, smem);
    if (e != cudaSuccess) return (int)e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    c.grid = (per_sm > 0 ? per_sm : 1) * sms;
    if (!K::ARENA_SMEM) {
      e = cudaMalloc(&c.arena, sizeof(T) * (size_t)c.grid * K::NA * 32);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.last, cudaEventDisableTiming);
      if (e != cudaSuccess) return (int)e;
    }
    c.ready = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const long long groups = (B + 31) / 32;
  const long long grid = groups < c.grid ? groups : c.grid;
  // a global arena is indexed by CTA: order launches that share it
  const bool chain = !K::ARENA_SMEM && !rbd_capturing(st);
  if (chain && c.used && (e = cudaStreamWaitEvent(st, c.last, 0)) != cudaSuccess) return (int)e;
  rbd_ws_rollout_kernel<K><<<(unsigned)grid, K::W * 32, smem, st>>>(
      (T*)q, (T*)qd, (const T*)tau, (T*)o0, (T*)o1, (T*)o2, (long long)B, (int)H, (T)dt, (T*)c.arena);
  e = cudaGetLastError();
  if (e == cudaSuccess && chain) {
    e = cudaEventRecord(c.last, st);
    c.used = true;
  }
  return (int)e;
}

// ---------------------------------------------------------------------------
// warp-specialised kernel over a thread-block cluster (MAP 3): one cluster of
// C CTAs x W warps per 32-knot group (lane = knot); CTA rank r runs the tasks
// the schedule put on warps [r W, (r + 1) W).  Every CTA stages the group's
// inputs and sin/cos itself; a value produced on another CTA is read from
// that CTA's shared-memory arena (DSMEM, ld.shared::cluster at the address
// mapa gives), and every phase ends with a cluster barrier (release/acquire),
// so an SM streams only its own warps' code.  Persistent over groups.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rbd_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class K>
__global__ void __launch_bounds__(K::W * 32, 1)
rbd_wc_kernel(const typename K::T* __restrict__ q, const typename K::T* __restrict__ qd,
              const typename K::T* __restrict__ u, const typename K::T* __restrict__ fx,
              typename K::T* __restrict__ o0, typename K::T* __restrict__ o1,
              typename K::T* __restrict__ o2, long long N) {
  typedef typename K::T T;
  constexpr int NT = K::W * 32, L = RBD_WS_LANES;
  extern __shared__ __align__(16) unsigned char rbd_smem[];
  T* s_in = reinterpret_cast<T*>(rbd_smem);  // [SIN][33]
  T* s_ar = s_in + K::SIN * L;                // [NA][33]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const unsigned a_in = (unsigned)__cvta_generic_to_shared(s_in + lane);
  const unsigned a_ar = (unsigned)__cvta_generic_to_shared(s_ar + lane);
  unsigned a_rem[K::C];
#pragma unroll
  for (int r = 0; r < K::C; ++r) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a_rem[r]) : "r"(a_ar), "r"(r));
  rbd_cluster_sync();  // every CTA of the cluster is running before any DSMEM access
  const long long groups = (N + 31) / 32;
  const long long ncl = gridDim.x / K::C;
  for (long long g = blockIdx.x / K::C; g < groups; g += ncl) {
    const long long base = g * 32;
    const int nk = (N - base) < 32 ? (int)(N - base) : 32;
    constexpr int WMAX = rbd_max_inw<K>();  // widest input row (f_ext 6 per dof, a split scratch nx)
    constexpr int PMAX = (32 * WMAX + NT - 1) / NT;
    T v[K::NIN][PMAX];
#pragma unroll
    for (int a = 0; a < K::NIN; ++a) {
      const T* src = (a == 0 ? q : (a == 1 ? qd : (a == 2 ? u : fx))) + base * K::ins(a) + K::ing(a);
#pragma unroll
      for (int r = 0; r < (32 * K::inw(a) + NT - 1) / NT; ++r) {
        const int idx = tid + r * NT;
        const int k = idx / K::inw(a), j = idx - k * K::inw(a);
        v[a][r] = (idx < nk * K::inw(a)) ? __ldg(src + k * K::ins(a) + j) : T(0);
      }
    }
#pragma unroll
    for (int a = 0; a < K::NIN; ++a) {
#pragma unroll
      for (int r = 0; r < (32 * K::inw(a) + NT - 1) / NT; ++r) {
        const int idx = tid + r * NT;
        if (idx < 32 * K::inw(a)) {
          const int k = idx / K::inw(a), j = idx - k * K::inw(a);
          s_in[(K::inr(a) + j) * L + k] = v[a][r];
        }
      }
    }
    __syncthreads();
    K::prologue(s_in, warp, lane);
    __syncthreads();
    const int kk = lane < nk ? lane : 0;
    const unsigned long long a0 = (unsigned long long)(o0 + (base + kk) * K::E0);
    const unsigned long long a1 = (unsigned long long)(K::E1 ? o1 + (base + kk) * K::E1 : o0);
    const unsigned long long a2 = (unsigned long long)(K::E2 ? o2 + (base + kk) * K::E2 : o0);
    // phases end with a cluster barrier; the last one also retires every
    // remote read of this group's arenas before the next group overwrites them
    K::run_group(blockIdx.y, (int)rank * K::W + warp, a_in, a_ar, a_rem, a0, a1, a2, lane < nk ? 1u : 0u);
  }
}

template <class K>
constexpr size_t rbd_smem_bytes() {
  if constexpr (K::MAP == 3)
    return sizeof(typename K::T) * (size_t)RBD_WS_LANES * (K::SIN + K::NA);
  else if constexpr (K::MAP == 2)
    return sizeof(typename K::T) * (size_t)RBD_WS_LANES * (K::SIN + K::NA + (K::STAGE ? K::SOUT : 0));
  else if constexpr (K::MAP == 1)
    return sizeof(typename K::T) * (size_t)RBD_WS_LANES *
           (K::SIN + (K::ARENA_SMEM ? K::NA : 0) + (K::STAGE ? K::SOUT : 0));
  else if constexpr (K::TROW)  // input staging and output staging aliased (+ the zero map)
    return sizeof(typename K::T) * (size_t)K::BK * (K::SIN > K::SOUT ? K::SIN : K::SOUT) +
           sizeof(short) * (size_t)rbd_nzm<K>();
  else
    return sizeof(typename K::T) * (size_t)K::BK * (K::SIN + (K::STAGE ? K::SOUT : 0)) +
           sizeof(short) * (size_t)rbd_nout<K>() * (rbd_ofull<K>() ? 1 : 2);
}

// Per-(kernel, device) launch state: occupancy-derived grid and, for the
// warp-specialised kernel with a global (L2-resident) arena, the arena and
// the event of its last launch.  Initialised once under the mutex; launches
// that share the arena are ordered across streams by an event chain, so the
// entry stays reentrant (any host thread, any stream).
struct rbd_dev_cache {
  std::mutex lock;
  bool ready = false;
  int grid = 0;
  void* arena = nullptr;
  cudaEvent_t last = nullptr;  // recorded after the last launch that used the arena
  bool used = false;
};

static inline bool rbd_capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return st != cudaStreamCaptureStatusNone;
}

template <class K>
static int rbd_launch_kernel(const void* q, const void* qd, const void* u, const void* fx, void* o0,
                             void* o1, void* o2, int64_t N, void* stream, void* xs = nullptr) {
  typedef typename K::T T;
  if (N < 0) return RBD_EINVAL;
  if (N == 0) return 0;
  if (!q || (K::NIN >= 3 && (!qd || !u)) || (K::NIN == 4 && !fx) || !o0 || (K::E1 > 0 && !o1) ||
      (K::E2 > 0 && !o2))
    return RBD_EINVAL;
  constexpr size_t smem = rbd_smem_bytes<K>();
  static rbd_dev_cache cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  rbd_dev_cache& c = cache[dev & 63];
  std::unique_lock<std::mutex> guard(c.lock);
  if (!c.ready) {
    cudaError_t e = cudaSuccess;
    // the large-shared-memory opt-in is per device
    if (smem > 48 * 1024) {
      if constexpr (K::MAP == 3)
        e = cudaFuncSetAttribute(rbd_wc_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      else if constexpr (K::MAP == 2)
        e = cudaFuncSetAttribute(rbd_fs_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      else if constexpr (K::MAP == 1)
        e = cudaFuncSetAttribute(rbd_ws_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      else
        e = cudaFuncSetAttribute(rbd_batch_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return (int)e;
    }
    if constexpr (K::MAP == 3) {
      if (K::C > 8) {
        e = cudaFuncSetAttribute(rbd_wc_kernel<K>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return (int)e;
      }
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = K::C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(K::C, K::NVAR);
      cfg.blockDim = dim3(K::W * 32);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      e = cudaOccupancyMaxActiveClusters(&ncl, rbd_wc_kernel<K>, &cfg);
      if (e != cudaSuccess) return (int)e;
      // clusters per variant row
      c.grid = (ncl > 0 ? ncl : 1) / K::NVAR;
      if (c.grid < 1) c.grid = 1;
    }
    if constexpr (K::MAP == 2) {
      int per_sm = 0, sms = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rbd_fs_kernel<K>, K::W * 32, smem);
      if (e != cudaSuccess) return (int)e;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      // CTAs per variant row: the grid has NVAR rows of them
      c.grid = ((per_sm > 0 ? per_sm : 1) * sms + K::NVAR - 1) / K::NVAR;
    }
    if constexpr (K::MAP == 1) {
      int per_sm = 0, sms = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rbd_ws_kernel<K>, K::W * 32, smem);
      if (e != cudaSuccess) return (int)e;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      // CTAs per variant row: the grid has NVAR rows of them
      int grid = ((per_sm > 0 ? per_sm : 1) * sms) / K::NVAR;
      if (grid < 1) grid = 1;
      if (!K::ARENA_SMEM && !K::ARENA_GROUP) {
        e = cudaMalloc(&c.arena, sizeof(T) * (size_t)grid * K::NVAR * K::NA * 32);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.last, cudaEventDisableTiming);
        if (e != cudaSuccess) return (int)e;
      }
      c.grid = grid;
    }
    c.ready = true;
  }
  if constexpr (K::MAP == 3) {
    guard.unlock();
    const long long groups = (N + 31) / 32;
    const long long ncl = groups < c.grid ? groups : c.grid;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K::C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(ncl * K::C), K::NVAR);
    cfg.blockDim = dim3(K::W * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, rbd_wc_kernel<K>, (const T*)q, (const T*)qd, (const T*)u, (const T*)fx,
                                   (T*)o0, (T*)o1, (T*)o2, (long long)N);
  } else if constexpr (K::MAP == 2) {
    guard.unlock();
    const long long groups = (N + 31) / 32;
    const long long grid = groups < c.grid ? groups : c.grid;
    rbd_fs_kernel<K><<<dim3((unsigned)grid, K::NVAR), K::W * 32, smem, (cudaStream_t)stream>>>(
        (const T*)q, (const T*)qd, (const T*)u, (const T*)fx, (T*)o0, (T*)o1, (T*)o2, (long long)N);
    return (int)cudaGetLastError();
  } else if constexpr (K::MAP == 1) {
    const long long groups = (N + 31) / 32;
    const long long grid = groups < c.grid ? groups : c.grid;
    if (K::ARENA_GROUP && !xs) return RBD_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const bool shared_arena = !K::ARENA_SMEM && !K::ARENA_GROUP;
    // the global arena is indexed by CTA: a launch waits for the previous
    // launch of this kernel (any stream) before reusing it.  Inside a stream
    // capture the graph's own order applies (no foreign events in a graph).
    const bool chain = shared_arena && !rbd_capturing(st);
    if (!shared_arena) guard.unlock();
    if (chain && c.used) {
      cudaError_t e = cudaStreamWaitEvent(st, c.last, 0);
      if (e != cudaSuccess) return (int)e;
    }
    rbd_ws_kernel<K><<<dim3((unsigned)grid, K::NVAR), K::W * 32, smem, st>>>(
        (const T*)q, (const T*)qd, (const T*)u, (const T*)fx, (T*)o0, (T*)o1, (T*)o2, (long long)N,
        K::ARENA_GROUP ? (T*)xs : (T*)c.arena);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && chain) {
      e = cudaEventRecord(c.last, st);
      c.used = true;
    }
    return (int)e;
  } else {
    guard.unlock();
    const long long grid = (N + K::BK - 1) / K::BK;
    if (K::NX && !xs) return RBD_EINVAL;
    // several programs (split gradient columns): grid row y runs program y
    rbd_batch_kernel<K><<<dim3((unsigned)grid, rbd_nprog<K>()), K::BK, smem, (cudaStream_t)stream>>>(
        (const T*)q, (const T*)qd, (const T*)u, (const T*)fx, (T*)o0, (T*)o1, (T*)o2, (long long)N,
        (T*)xs);
    return (int)cudaGetLastError();
  }
}

// ---------------------------------------------------------------------------
// small-batch split (wsched.split_programs): KA = the big tree's prefix as a
// warp-specialised kernel (exports -> a per-device [N][NX] scratch, the
// tree's qdd -> out2), then KB = CTA-row variants of its gradient columns
// (the scratch staged as their 4th input) and of the other root trees, on the
// caller's stream.  The scratch is shared by every stream of the device:
// launches are ordered by an event chain (as the warp-specialised global
// arena); inside a stream capture the graph's order applies.
// ---------------------------------------------------------------------------
template <class KA, class KB, long long MAXN>
static int rbd_launch_ws_split(const void* q, const void* qd, const void* u, void* o0, void* o1, void* o2,
                               int64_t N, void* stream) {
  typedef typename KA::T T;
  static_assert(KB::NIN == 4, "column variants read the scratch as their 4th input");
  if (N < 0 || N > MAXN) return RBD_EINVAL;
  if (N == 0) return 0;
  struct cache_t {
    std::mutex lock;
    T* scratch = nullptr;
    cudaEvent_t last = nullptr;
    bool used = false;
  };
  static cache_t cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  cache_t& c = cache[dev & 63];
  std::lock_guard<std::mutex> guard(c.lock);
  cudaError_t e = cudaSuccess;
  if (!c.scratch) {
    e = cudaMalloc(&c.scratch, sizeof(T) * (size_t)MAXN * KA::E0);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.last, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      if (c.scratch) cudaFree(c.scratch);
      c.scratch = nullptr;
      return (int)e;
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  const bool chain = !rbd_capturing(st);
  if (chain && c.used && (e = cudaStreamWaitEvent(st, c.last, 0)) != cudaSuccess) return (int)e;
  int rc = rbd_launch_kernel<KA>(q, qd, u, nullptr, c.scratch, KA::E1 ? o2 : nullptr, nullptr, N, stream);
  if (rc == 0) rc = rbd_launch_kernel<KB>(q, qd, u, c.scratch, o0, o1, o2, N, stream);
  if (rc == 0 && chain) {
    e = cudaEventRecord(c.last, st);
    if (e != cudaSuccess) return (int)e;
    c.used = true;
  }
  return rc;
}

// ---------------------------------------------------------------------------
// split gradient program (large root trees): the prefix kernel KA (thread per
// knot: RNEA, articulated inertias, Minv, FD, RNEA at qdd) exports the values
// the gradient columns need to a scratch; the column kernel KB (thread per
// knot) reloads them through its register plan.  Chunks of KA::CHUNK knots
// keep the scratch L2-resident.
// ---------------------------------------------------------------------------
// Side streams, events and the double-buffered scratch of the split
// pipeline, one set per (device, caller stream): calls from different
// streams (or host threads) never share a scratch buffer, and calls on one
// caller stream are ordered by that stream (each call forks from it and
// joins back into it), so the pipeline is reentrant.
struct rbd_split_state {
  bool init = false;
  int dev = -1;
  cudaStream_t caller = nullptr;
  void* scratch[2] = {nullptr, nullptr};
  size_t bytes = 0;
  cudaStream_t sa = nullptr, sb = nullptr;
  cudaEvent_t start = nullptr, join_a = nullptr, join_b = nullptr;
  cudaEvent_t done_a[2] = {nullptr, nullptr}, done_b[2] = {nullptr, nullptr};
  bool recorded[2] = {false, false};  // done_b[b] marks the last read of scratch[b]
  std::mutex lock;
};
#define RBD_SPLIT_STATES 64

template <class KA, class KB>
static rbd_split_state* rbd_split_state_of(int dev, cudaStream_t caller, bool create) {
  static rbd_split_state state[RBD_SPLIT_STATES];
  static std::mutex table;
  std::lock_guard<std::mutex> g(table);
  for (auto& st : state)
    if (st.init && st.dev == dev && st.caller == caller) return &st;
  if (!create) return nullptr;
  for (auto& st : state) {
    if (st.init) continue;
    constexpr size_t bytes = sizeof(typename KA::T) * (size_t)KA::CHUNK * KA::NX;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&st.scratch[i], bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st.sa, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st.sb, cudaStreamNonBlocking);
    cudaEvent_t* evs[] = {&st.start, &st.join_a, &st.join_b, &st.done_a[0], &st.done_a[1], &st.done_b[0],
                          &st.done_b[1]};
    for (cudaEvent_t* ev : evs)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return nullptr;
    st.bytes = bytes;
    st.dev = dev;
    st.caller = caller;
    st.init = true;
    return &st;
  }
  return nullptr;  // more than RBD_SPLIT_STATES distinct caller streams
}

// Join: the caller's stream continues after both side streams of its split
// pipeline on the current device.
template <class KA, class KB>
static int rbd_split_join(void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  rbd_split_state* st = rbd_split_state_of<KA, KB>(dev, (cudaStream_t)stream, false);
  if (!st) return 0;
  std::lock_guard<std::mutex> guard(st->lock);
  cudaStream_t s0 = (cudaStream_t)stream;
  cudaError_t e;
  if ((e = cudaEventRecord(st->join_a, st->sa)) != cudaSuccess) return (int)e;
  if ((e = cudaStreamWaitEvent(s0, st->join_a, 0)) != cudaSuccess) return (int)e;
  if ((e = cudaEventRecord(st->join_b, st->sb)) != cudaSuccess) return (int)e;
  if ((e = cudaStreamWaitEvent(s0, st->join_b, 0)) != cudaSuccess) return (int)e;
  return 0;
}

// Fork: enqueue the whole split pipeline on the side streams (after the work
// already on the caller's stream) and return without joining, so the caller
// can enqueue independent work (other root trees) meanwhile.  join = true:
// also join before returning.
template <class KA, class KB>
static int rbd_launch_split(const void* q, const void* qd, const void* u, const void* fx, void* o0,
                            void* o1, void* o2, int64_t N, void* stream, bool join = true) {
  typedef typename KA::T T;
  static_assert(KA::NX == KB::NX && KA::MAP == 0 && KB::MAP == 0, "prefix exports and column imports disagree");
  static_assert(KA::CHUNK % KA::BK == 0 && KA::BK % 32 == 0, "chunk / CTA / warp alignment");
  if (N < 0) return RBD_EINVAL;
  if (N == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t s0 = (cudaStream_t)stream;
  rbd_split_state* stp = rbd_split_state_of<KA, KB>(dev, s0, true);
  if (!stp) return (int)cudaErrorMemoryAllocation;
  rbd_split_state& st = *stp;
  {
    std::lock_guard<std::mutex> guard(st.lock);
    // pipeline over two scratch buffers: prefix(i+1) on stream A overlaps
    // columns(i) on stream B; A reuses buffer b only after B has read it
    cudaError_t e = cudaEventRecord(st.start, s0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st.sa, st.start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st.sb, st.start, 0);
    if (e != cudaSuccess) return (int)e;
    constexpr int n = KA::NDOF;
    // two host threads on one caller stream: the previous call's column
    // kernels may still read the scratch (outside a capture only; a graph
    // orders its own nodes)
    const bool ext = !rbd_capturing(s0);
    int chunk = 0;
    for (int64_t c0 = 0; c0 < N; c0 += KA::CHUNK, ++chunk) {
      const int buf = chunk & 1;
      const int64_t nk = (N - c0) < KA::CHUNK ? (N - c0) : KA::CHUNK;
      const T* cq = (const T*)q + c0 * n;
      const T* cqd = qd ? (const T*)qd + c0 * n : nullptr;
      const T* cu = u ? (const T*)u + c0 * n : nullptr;
      const T* cfx = fx ? (const T*)fx + c0 * 6 * n : nullptr;
      T* c_o0 = (T*)o0 + c0 * KA::E0;
      T* c_o1 = KA::E1 ? (T*)o1 + c0 * KA::E1 : nullptr;
      T* c_o2 = KA::E2 ? (T*)o2 + c0 * KA::E2 : nullptr;
      if ((chunk >= 2 || (ext && st.recorded[buf])) && (e = cudaStreamWaitEvent(st.sa, st.done_b[buf], 0)) != cudaSuccess)
        return (int)e;
      int rc = rbd_launch_kernel<KA>(cq, cqd, cu, cfx, c_o0, c_o1, c_o2, nk, (void*)st.sa, st.scratch[buf]);
      if (rc) return rc;
      if ((e = cudaEventRecord(st.done_a[buf], st.sa)) != cudaSuccess) return (int)e;
      if ((e = cudaStreamWaitEvent(st.sb, st.done_a[buf], 0)) != cudaSuccess) return (int)e;
      rc = rbd_launch_kernel<KB>(cq, cqd, cu, cfx, c_o0, c_o1, c_o2, nk, (void*)st.sb, st.scratch[buf]);
      if (rc) return rc;
      if ((e = cudaEventRecord(st.done_b[buf], st.sb)) != cudaSuccess) return (int)e;
      st.recorded[buf] = ext;
    }
  }
  return join ? rbd_split_join<KA, KB>(stream) : 0;
}

// ---------------------------------------------------------------------------
// dispatch table (filled by the generated file through rbd_entry_for)
// ---------------------------------------------------------------------------
typedef int (*rbd_launch_fn)(const void*, const void*, const void*, const void*, void*, void*, void*,
                             int64_t, void*);
struct rbd_entry {
  rbd_launch_fn fn;
  int32_t n_inputs;
  int64_t e0, e1, e2;
  int32_t elem;           // sizeof(T)
  int64_t copy_out_max_n;  // batches up to this size run a kernel whose output stores are not
                           // coalesced (CTA-row variants): the small-batch host path lands its
                           // outputs in device memory and copies them back once
  rbd_launch_fn fn_host;   // the small-batch host path's launcher (may prefer output-staging kernels)
};
#if defined(RBD_MAIN_TU)
static const rbd_entry* rbd_entry_for(int alg, int dtype, int fext);  // generated main TU
static int rbd_ndof();                                                 // generated main TU

extern "C" int rbd_launch(int alg, int dtype, const void* q, const void* qd, const void* u,
                          void* out0, void* out1, void* out2, int64_t N, void* stream) {
  const rbd_entry* e = rbd_entry_for(alg, dtype, 0);
  if (!e) return RBD_EINVAL;
  return e->fn(q, qd, u, nullptr, out0, out1, out2, N, stream);
}

extern "C" int rbd_launch_fext(int alg, int dtype, const void* q, const void* qd, const void* u,
                               const void* f_ext, void* out0, void* out1, void* out2, int64_t N,
                               void* stream) {
  const rbd_entry* e = rbd_entry_for(alg, dtype, 1);
  if (!e) return RBD_EINVAL;
  return e->fn(q, qd, u, f_ext, out0, out1, out2, N, stream);
}

extern "C" int rbd_alg_extents(int alg, int32_t* n_inputs, int64_t* e0, int64_t* e1, int64_t* e2) {
  const rbd_entry* e = rbd_entry_for(alg, RBD_F64, 0);
  if (!e) return RBD_EINVAL;
  if (n_inputs) *n_inputs = e->n_inputs;
  if (e0) *e0 = e->e0;
  if (e1) *e1 = e->e1;
  if (e2) *e2 = e->e2;
  return 0;
}

// ---------------------------------------------------------------------------
// host-buffer session: chunked H2D -> kernel -> D2H pipeline over `slots` streams
// ---------------------------------------------------------------------------
#define RBD_MAX_SLOTS 8
static inline size_t rbd_align256(size_t x) { return (x + 255) & ~(size_t)255; }
// small batches (<= RBD_ZC_BYTES of inputs + outputs) skip the copy engines:
// the kernel reads its inputs from and writes its outputs to page-locked
// host memory directly over PCIe (zero-copy) -- one launch + one sync.
// Caller buffers that are already pinned are used in place; pageable ones go
// through the session's pinned staging area with host memcpy.
#define RBD_ZC_BYTES (1u << 20)
struct rbd_session {
  int device;
  int64_t chunk;
  int32_t slots;
  size_t slot_bytes;
  cudaStream_t stream[RBD_MAX_SLOTS];
  unsigned char* dbuf[RBD_MAX_SLOTS];
  unsigned char* hstage;  // pinned, RBD_ZC_BYTES (+ 256: the non-finite input flag)
  unsigned* dflag;        // device view of that flag (mapped)
};

// any non-finite element of a[0, count) sets *flag (device input check of the
// chunked host path; the small-batch path checks on the host)
template <class T>
__global__ void rbd_finite_kernel(const T* __restrict__ a, long long count, unsigned* flag) {
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(a[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

template <class T>
static bool rbd_host_finite(const void* p, int64_t count) {
  const T* a = (const T*)p;
  for (int64_t i = 0; i < count; ++i)
    if (!isfinite(a[i])) return false;
  return true;
}

// device address of a host pointer when it is page-locked and mapped, else nullptr
static inline const void* rbd_mapped(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeHost && a.devicePointer) return a.devicePointer;
  return nullptr;
}

extern "C" int rbd_session_create(int device, int64_t chunk_knots, int32_t slots,
                                  rbd_session** out) {
  if (!out || chunk_knots <= 0 || slots <= 0 || slots > RBD_MAX_SLOTS) return RBD_EINVAL;
  *out = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return (int)e;
  // size for the largest per-knot footprint over all algorithms, fp64,
  // f_ext (6 per dof) included
  int64_t per_knot = 0;
  for (int a = 0; a < 5; ++a) {
    const rbd_entry* en = rbd_entry_for(a, RBD_F64, 0);
    int64_t f = (int64_t)en->n_inputs * rbd_ndof() + 6 * rbd_ndof() + en->e0 + en->e1 + en->e2;
    if (f > per_knot) per_knot = f;
  }
  rbd_session* s = new rbd_session();
  s->device = device;
  s->chunk = chunk_knots;
  s->slots = slots;
  s->slot_bytes = (size_t)per_knot * (size_t)chunk_knots * sizeof(double) + 10 * 256;
  e = cudaHostAlloc((void**)&s->hstage, RBD_ZC_BYTES + 256, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e == cudaSuccess) {
    s->dflag = (unsigned*)rbd_mapped(s->hstage + RBD_ZC_BYTES);
    if (!s->dflag) e = cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) {
    if (s->hstage) cudaFreeHost(s->hstage);
    delete s;
    cudaSetDevice(prev);
    return (int)e;
  }
  for (int i = 0; i < slots; ++i) {
    e = cudaStreamCreateWithFlags(&s->stream[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc((void**)&s->dbuf[i], s->slot_bytes);
    if (e != cudaSuccess) {
      for (int j = 0; j <= i; ++j) {
        if (s->dbuf[j]) cudaFree(s->dbuf[j]);
        if (s->stream[j]) cudaStreamDestroy(s->stream[j]);
      }
      cudaFreeHost(s->hstage);
      delete s;
      cudaSetDevice(prev);
      return (int)e;
    }
  }
  cudaSetDevice(prev);
  *out = s;
  return 0;
}

extern "C" int rbd_session_destroy(rbd_session* s) {
  if (!s) return RBD_ESESSION;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(s->device);
  for (int i = 0; i < s->slots; ++i) {
    cudaStreamSynchronize(s->stream[i]);
    cudaFree(s->dbuf[i]);
    cudaStreamDestroy(s->stream[i]);
  }
  cudaFreeHost(s->hstage);
  cudaSetDevice(prev);
  delete s;
  return 0;
}

static int rbd_run_host_impl(rbd_session* s, int alg, int dtype, const void* q, const void* qd,
                             const void* u, const void* fx, void* out0, void* out1, void* out2,
                             int64_t N) {
  if (!s) return RBD_ESESSION;
  const rbd_entry* e = rbd_entry_for(alg, dtype, fx ? 1 : 0);
  if (!e || N < 0) return RBD_EINVAL;
  if (N == 0) return 0;
  const int64_t n = rbd_ndof();
  const size_t es = (size_t)e->elem;
  const void* hin[4] = {q, qd, u, fx};
  const int64_t iext[4] = {n, n, n, 6 * n};  // per-knot input extents (f_ext: 6 per dof)
  void* hout[3] = {out0, out1, out2};
  const int64_t ext[3] = {e->e0, e->e1, e->e2};
  for (int a = 0; a < e->n_inputs; ++a)
    if (!hin[a]) return RBD_EINVAL;
  for (int b = 0; b < 3; ++b)
    if (ext[b] > 0 && !hout[b]) return RBD_EINVAL;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t err = cudaSetDevice(s->device);
  if (err != cudaSuccess) return (int)err;
  int rc = 0;
  size_t in_bytes = 0, out_bytes = 0;
  for (int a = 0; a < e->n_inputs; ++a) in_bytes += (size_t)(N * iext[a]) * es;
  for (int b = 0; b < 3; ++b) out_bytes += (size_t)(N * ext[b]) * es;
  if (in_bytes + out_bytes + 8 * 256 <= RBD_ZC_BYTES) {
    // non-finite inputs are rejected before any work (refdyn._check_state)
    for (int a = 0; a < e->n_inputs; ++a) {
      const bool ok = es == 8 ? rbd_host_finite<double>(hin[a], N * iext[a]) : rbd_host_finite<float>(hin[a], N * iext[a]);
      if (!ok) {
        cudaSetDevice(prev);
        return RBD_ENONFINITE;
      }
    }
    // small batch: the kernel reads its inputs straight from pinned host
    // memory (the caller's buffers when page-locked, else the pinned stage);
    // outputs go to device memory and come back with ONE copy -- a kernel
    // writing over PCIe pays per store, and the small-batch kernels' stores
    // are not all coalesced (CTA-row variants store straight from registers)
    const void* din[4] = {nullptr, nullptr, nullptr, nullptr};
    void* dout[3] = {nullptr, nullptr, nullptr};
    bool direct_in = true, direct_out = true;
    for (int a = 0; a < e->n_inputs && direct_in; ++a) direct_in = (din[a] = rbd_mapped(hin[a])) != nullptr;
    unsigned char* hp = s->hstage;
    if (!direct_in) {
      for (int a = 0; a < e->n_inputs; ++a) {
        const size_t bytes = (size_t)(N * iext[a]) * es;
        memcpy(hp, hin[a], bytes);
        din[a] = rbd_mapped(hp);
        hp += rbd_align256(bytes);
      }
    }
    // kernels that stage their outputs write them coalesced straight into
    // pinned host memory; the others (N <= copy_out_max_n) write device
    // memory, copied back in one transfer to the pinned stage (then to the
    // caller) or straight into each pinned caller buffer
    const bool via_device = N <= e->copy_out_max_n;
    unsigned char* dp = s->dbuf[0];
    for (int b = 0; b < 3; ++b) {
      if (!ext[b]) continue;
      void* mapped = (void*)rbd_mapped(hout[b]);
      direct_out = direct_out && mapped != nullptr;
      dout[b] = dp;
      dp += rbd_align256((size_t)(N * ext[b]) * es);
    }
    if (!via_device) {  // zero-copy outputs: the caller's pinned buffers, else the pinned stage
      unsigned char* hq = s->hstage + rbd_align256(in_bytes) + 4 * 256;
      for (int b = 0; b < 3; ++b) {
        if (!ext[b]) continue;
        if (direct_out) {
          dout[b] = (void*)rbd_mapped(hout[b]);
        } else {
          dout[b] = (void*)rbd_mapped(hq);
          hq += rbd_align256((size_t)(N * ext[b]) * es);
        }
      }
    }
    cudaStream_t st = s->stream[0];
    rc = e->fn_host(din[0], din[1], din[2], din[3], dout[0], dout[1], dout[2], N, (void*)st);
    unsigned char* ho = s->hstage + rbd_align256(in_bytes) + 4 * 256;  // after the staged inputs
    if (rc == 0 && via_device) {
      if (direct_out) {
        for (int b = 0; b < 3 && rc == 0; ++b)
          if (ext[b])
            rc = (int)cudaMemcpyAsync(hout[b], dout[b], (size_t)(N * ext[b]) * es, cudaMemcpyDeviceToHost, st);
      } else {
        rc = (int)cudaMemcpyAsync(ho, s->dbuf[0], (size_t)(dp - s->dbuf[0]), cudaMemcpyDeviceToHost, st);
      }
    }
    if (rc == 0) rc = (int)cudaStreamSynchronize(st);
    if (rc == 0 && !direct_out) {
      unsigned char* src = ho;
      for (int b = 0; b < 3; ++b) {
        if (!ext[b]) continue;
        const size_t bytes = (size_t)(N * ext[b]) * es;
        memcpy(hout[b], src, bytes);
        src += rbd_align256(bytes);
      }
    }
    cudaSetDevice(prev);
    return rc;
  }
  // non-finite inputs: each chunk's staged inputs are checked on the device
  // (one pass over bytes already in HBM), the verdict read after the final sync
  volatile unsigned* hflag = (volatile unsigned*)(s->hstage + RBD_ZC_BYTES);
  *hflag = 0u;
  for (int64_t c = 0, k0 = 0; k0 < N && rc == 0; ++c, k0 += s->chunk) {
    const int slot = (int)(c % s->slots);
    const int64_t nk = (N - k0) < s->chunk ? (N - k0) : s->chunk;
    cudaStream_t st = s->stream[slot];
    unsigned char* p = s->dbuf[slot];
    const void* din[4] = {nullptr, nullptr, nullptr, nullptr};
    void* dout[3] = {nullptr, nullptr, nullptr};
    for (int a = 0; a < e->n_inputs; ++a) {
      const size_t bytes = (size_t)(nk * iext[a]) * es;
      err = cudaMemcpyAsync(p, (const unsigned char*)hin[a] + (size_t)(k0 * iext[a]) * es, bytes,
                            cudaMemcpyHostToDevice, st);
      if (err != cudaSuccess) { rc = (int)err; break; }
      const long long cnt = (long long)(nk * iext[a]);
      const unsigned g = (unsigned)((cnt + 255) / 256 < 1184 ? (cnt + 255) / 256 : 1184);
      if (es == 8)
        rbd_finite_kernel<double><<<g, 256, 0, st>>>((const double*)p, cnt, s->dflag);
      else
        rbd_finite_kernel<float><<<g, 256, 0, st>>>((const float*)p, cnt, s->dflag);
      din[a] = p;
      p += rbd_align256(bytes);
    }
    if (rc) break;
    for (int b = 0; b < 3; ++b) {
      if (ext[b] == 0) continue;
      dout[b] = p;
      p += rbd_align256((size_t)(nk * ext[b]) * es);
    }
    rc = e->fn(din[0], din[1], din[2], din[3], dout[0], dout[1], dout[2], nk, (void*)st);
    if (rc) break;
    for (int b = 0; b < 3; ++b) {
      if (ext[b] == 0) continue;
      err = cudaMemcpyAsync((unsigned char*)hout[b] + (size_t)(k0 * ext[b]) * es, dout[b],
                            (size_t)(nk * ext[b]) * es, cudaMemcpyDeviceToHost, st);
      if (err != cudaSuccess) { rc = (int)err; break; }
    }
  }
  for (int i = 0; i < s->slots; ++i) {
    err = cudaStreamSynchronize(s->stream[i]);
    if (err != cudaSuccess && rc == 0) rc = (int)err;
  }
  if (rc == 0 && *hflag) rc = RBD_ENONFINITE;
  cudaSetDevice(prev);
  return rc;
}

extern "C" int rbd_run_host(rbd_session* s, int alg, int dtype, const void* q, const void* qd,
                            const void* u, void* out0, void* out1, void* out2, int64_t N) {
  return rbd_run_host_impl(s, alg, dtype, q, qd, u, nullptr, out0, out1, out2, N);
}

extern "C" int rbd_run_host_fext(rbd_session* s, int alg, int dtype, const void* q, const void* qd,
                                 const void* u, const void* f_ext, void* out0, void* out1,
                                 void* out2, int64_t N) {
  if (!f_ext) return RBD_EINVAL;
  return rbd_run_host_impl(s, alg, dtype, q, qd, u, f_ext, out0, out1, out2, N);
}

// ---------------------------------------------------------------------------
// several devices: one session per device, contiguous batch slices
// ---------------------------------------------------------------------------
// Knots are independent (no exchange step): slice k of ceil(N / count) knots
// runs on session k's device from its own host thread, through that
// session's own pipeline; results land in place in the caller's arrays.
static void rbd_shard(int64_t N, int32_t count, int32_t k, int64_t* begin, int64_t* len) {
  const int64_t per = (N + count - 1) / count;
  int64_t b = per * k;
  if (b > N) b = N;
  int64_t e = b + per;
  if (e > N) e = N;
  *begin = b;
  *len = e - b;
}

static int rbd_run_host_multi_impl(rbd_session* const* s, int32_t count, int alg, int dtype, const void* q,
                                   const void* qd, const void* u, const void* fx, void* out0, void* out1,
                                   void* out2, int64_t N) {
  if (!s || count <= 0) return RBD_EINVAL;
  for (int32_t k = 0; k < count; ++k)
    if (!s[k]) return RBD_ESESSION;
  const rbd_entry* e = rbd_entry_for(alg, dtype, fx ? 1 : 0);
  if (!e || N < 0) return RBD_EINVAL;
  const int64_t n = rbd_ndof();
  const size_t es = (size_t)e->elem;
  const int64_t iext[4] = {n, n, n, 6 * n};
  const int64_t ext[3] = {e->e0, e->e1, e->e2};
  std::vector<int> rc(count, 0);
  std::vector<std::thread> th;
  for (int32_t k = 0; k < count; ++k) {
    int64_t b, len;
    rbd_shard(N, count, k, &b, &len);
    if (len == 0) continue;
    auto in = [&](const void* p, int a) -> const void* {
      return p ? (const unsigned char*)p + (size_t)(b * iext[a]) * es : nullptr;
    };
    auto out = [&](void* p, int j) -> void* {
      return (p && ext[j]) ? (unsigned char*)p + (size_t)(b * ext[j]) * es : nullptr;
    };
    const void *kq = in(q, 0), *kqd = in(qd, 1), *ku = in(u, 2), *kfx = in(fx, 3);
    void *k0 = out(out0, 0), *k1 = out(out1, 1), *k2 = out(out2, 2);
    th.emplace_back([=, &rc]() {
      rc[k] = rbd_run_host_impl(s[k], alg, dtype, kq, kqd, ku, kfx, k0, k1, k2, len);
    });
  }
  for (auto& t : th) t.join();
  for (int32_t k = 0; k < count; ++k)
    if (rc[k]) return rc[k];
  return 0;
}

extern "C" int rbd_run_host_multi(rbd_session* const* sessions, int32_t count, int alg, int dtype,
                                  const void* q, const void* qd, const void* u, void* out0, void* out1,
                                  void* out2, int64_t N) {
  return rbd_run_host_multi_impl(sessions, count, alg, dtype, q, qd, u, nullptr, out0, out1, out2, N);
}

extern "C" int rbd_run_host_multi_fext(rbd_session* const* sessions, int32_t count, int alg, int dtype,
                                       const void* q, const void* qd, const void* u, const void* f_ext,
                                       void* out0, void* out1, void* out2, int64_t N) {
  if (!f_ext) return RBD_EINVAL;
  return rbd_run_host_multi_impl(sessions, count, alg, dtype, q, qd, u, f_ext, out0, out1, out2, N);
}

extern "C" int rbd_session_device(const rbd_session* s, int32_t* device) {
  if (!s || !device) return RBD_ESESSION;
  *device = s->device;
  return 0;
}

// ---------------------------------------------------------------------------
// semi-implicit Euler step of a batch of trajectories (device-resident rollouts)
//   qd' = qd + dt * qdd ;  q' = q + dt * qd'
// ---------------------------------------------------------------------------
template <typename T>
__global__ void rbd_euler_kernel(const T* __restrict__ q, const T* __restrict__ qd,
                                 const T* __restrict__ qdd, T* __restrict__ q1, T* __restrict__ qd1,
                                 long long count, T dt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const T v = fma(dt, qdd[i], qd[i]);
    qd1[i] = v;
    q1[i] = fma(dt, v, q[i]);
  }
}

extern "C" int rbd_euler_step(int dtype, const void* q, const void* qd, const void* qdd, void* q_next,
                              void* qd_next, int64_t N, double dt, void* stream) {
  if (N < 0 || !q || !qd || !qdd || !q_next || !qd_next) return RBD_EINVAL;
  if (N == 0) return 0;
  const long long count = (long long)N * rbd_ndof();
  const unsigned grid = (unsigned)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
  if (dtype == RBD_F64)
    rbd_euler_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const double*)q, (const double*)qd, (const double*)qdd, (double*)q_next, (double*)qd_next, count, dt);
  else if (dtype == RBD_F32)
    rbd_euler_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const float*)q, (const float*)qd, (const float*)qdd, (float*)q_next, (float*)qd_next, count, (float)dt);
  else
    return RBD_EINVAL;
  return (int)cudaGetLastError();
}

extern "C" int rbd_bench_host(rbd_session* s, int alg, int dtype, const void* q, const void* qd,
                              const void* u, void* out0, void* out1, void* out2, int64_t N,
                              int32_t reps, double* seconds) {
  if (!seconds || reps <= 0) return RBD_EINVAL;
  const auto t0 = std::chrono::steady_clock::now();
  for (int32_t r = 0; r < reps; ++r) {
    const int rc = rbd_run_host(s, alg, dtype, q, qd, u, out0, out1, out2, N);
    if (rc) return rc;
  }
  const auto t1 = std::chrono::steady_clock::now();
  *seconds = std::chrono::duration<double>(t1 - t0).count() / reps;
  return 0;
}
#endif  // RBD_MAIN_TU

#endif  // __CUDACC__
