// TEST-ONLY host build of a generated per-robot source (never shipped, never
// loaded by the product API): compiles the per-knot programs with g++ so the
// generator can be checked against the oracle on a machine without a GPU.
// The product path is the sm_100a build of the same source (kernels.py).
#include <stdint.h>
#include GEN_SRC

template <class K>
static void host_loop(const void* q, const void* qd, const void* u, const void* fx, void* o0,
                      void* o1, void* o2, int64_t N) {
  typedef typename K::T T;
  const T* Q = (const T*)q;
  const T* QD = (const T*)(qd ? qd : q);
  const T* U = (const T*)(u ? u : q);
  const T* FX = (const T*)(fx ? fx : q);
  T* O0 = (T*)o0;
  T* O1 = (T*)(o1 ? o1 : o0);
  T* O2 = (T*)(o2 ? o2 : o0);
  const int64_t sfx = fx ? 6 * K::NDOF : 0;
  for (int64_t k = 0; k < N; ++k)
    K::run(Q + k * K::NDOF, QD + k * K::NDOF, U + k * K::NDOF, FX + k * sfx, O0 + k * K::E0,
           O1 + k * K::E1, O2 + k * K::E2);
}

#define CASE(A, D) \
  case A##_##D: host_loop<Knot_##A##_##D>(q, qd, u, nullptr, o0, o1, o2, N); return 0;
#define CASEX(A, D) \
  case A##_##D: host_loop<Knot_##A##_##D##_X>(q, qd, u, fx, o0, o1, o2, N); return 0;

enum { ID_f32, ID_f64, Minv_f32, Minv_f64, FD_f32, FD_f64, gradID_f32, gradID_f64, gradFD_f32,
       gradFD_f64 };

extern "C" int host_eval(int alg, int dtype, const void* q, const void* qd, const void* u,
                         void* o0, void* o1, void* o2, int64_t N) {
  switch (alg * 2 + dtype) {
    CASE(ID, f32) CASE(ID, f64) CASE(Minv, f32) CASE(Minv, f64) CASE(FD, f32) CASE(FD, f64)
    CASE(gradID, f32) CASE(gradID, f64) CASE(gradFD, f32) CASE(gradFD, f64)
  }
  return -1;
}

extern "C" int host_eval_fext(int alg, int dtype, const void* q, const void* qd, const void* u,
                              const void* fx, void* o0, void* o1, void* o2, int64_t N) {
  switch (alg * 2 + dtype) {
    CASEX(ID, f32) CASEX(ID, f64) CASEX(FD, f32) CASEX(FD, f64)
    CASEX(gradID, f32) CASEX(gradID, f64) CASEX(gradFD, f32) CASEX(gradFD, f64)
  }
  return -1;
}
