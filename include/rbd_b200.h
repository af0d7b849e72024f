/*
 * rbd_b200.h -- C ABI of one generated per-robot dynamics library.
 *
 * `paper_2109_06976_b200.codegen` emits one CUDA source per robot (tree,
 * joint types, constant transforms and inertias baked in as immediates);
 * nvcc compiles it for sm_100a into lib<robot>-<hash>.so.  Every such library
 * exports exactly the symbols below.  No torch types cross this boundary:
 * plain pointers, sizes and a cudaStream_t passed as void*.
 *
 * What each entry replaces in the reference (rbdgen, pure Python):
 *   rbd_<alg>_<f32|f64>   one batched launch of the generated program;
 *                         replaces interp.interpret(program, inputs)
 *                         (rbdgen/interp.py:54-86) called once per knot, and the
 *                         per-knot refdyn functions (rbdgen/refdyn.py:91-249):
 *                           ID     = rnea                (refdyn.py:91)
 *                           Minv   = minv_direct         (refdyn.py:128)
 *                           FD     = forward_dynamics    (refdyn.py:172)
 *                           gradID = rnea_grad           (refdyn.py:178)
 *                           gradFD = fd_grad (+ qdd)     (refdyn.py:242)
 *   rbd_run_host          the spec's batch executor run_batch:
 *                         N knots from HOST buffers, chunked and pipelined
 *                         H2D / kernel / D2H on the session's streams.
 *   rbd_get_info          KernelProgram.meta (rbdgen/codegen.py:788-795).
 *
 * Data layout (all algorithms, both precisions): knot-major, row-major,
 * contiguous per knot -- q[k*n + j]; matrices out[k*n*n + i*n + j] with
 * [i, j] = d out_i / d x_j, exactly the reference output_map order
 * (rbdgen/schedule.py:208-226).  Unused pointer arguments are NULL.
 *
 * Argument meaning per algorithm (u = qdd for ID/gradID, tau for FD/gradFD):
 *   ID      (q, qd, qdd) -> out0 = tau_out[n]
 *   Minv    (q)          -> out0 = minv_out[n*n]   (full symmetric)
 *   FD      (q, qd, tau) -> out0 = qdd_out[n]
 *   gradID  (q, qd, qdd) -> out0 = dq_out[n*n], out1 = dqd_out[n*n]
 *   gradFD  (q, qd, tau) -> out0 = dq_out[n*n], out1 = dqd_out[n*n], out2 = qdd_out[n]
 *
 * Errors: every entry returns 0 on success, a cudaError_t value (> 0) from the
 * CUDA runtime, or a negative RBD_E* code for argument errors.  Device
 * entries launch asynchronously on `stream` and never synchronise or allocate.
 * All entries are reentrant: any host thread may call any entry on any stream
 * concurrently (per-stream scratch for the split pipeline, an event chain
 * for the warp-specialised kernels' shared global arena).  A session is
 * owned by one host thread at a time.
 */
#ifndef RBD_B200_H
#define RBD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBD_ABI_VERSION 1

enum rbd_alg { RBD_ID = 0, RBD_MINV = 1, RBD_FD = 2, RBD_GRADID = 3, RBD_GRADFD = 4 };
enum rbd_dtype { RBD_F32 = 0, RBD_F64 = 1 };

#define RBD_EINVAL (-1)   /* bad algorithm / dtype / NULL pointer / N < 0 */
#define RBD_ESESSION (-2) /* bad or exhausted session */
#define RBD_ENONFINITE (-3) /* host-buffer entries: an input holds NaN or Inf (the reference's
                               refdyn._check_state raises ValueError); outputs are undefined */

typedef struct rbd_info {
  int32_t abi_version;     /* RBD_ABI_VERSION */
  int32_t n_dof;           /* == n_frames after fixed-joint fusion */
  int32_t n_frames;
  int32_t n_trees;         /* independent root trees (block-diagonal Minv) */
  int32_t knots_per_block; /* CTA size of the batch kernels (one knot per thread) */
  int32_t reserved;
  const char* robot;       /* model name */
  const char* fingerprint; /* sha256 of the model numbers baked in */
} rbd_info;

int rbd_get_info(rbd_info* out);

/* Per-knot extents of algorithm `alg`: number of inputs used (1 or 3) and the
 * element counts of out0..out2 (0 when unused). */
int rbd_alg_extents(int alg, int32_t* n_inputs, int64_t* e0, int64_t* e1, int64_t* e2);

/* ---- device-pointer entries (kernel-only path) ---------------------------- */
int rbd_ID_f64(const double* q, const double* qd, const double* qdd, double* tau_out,
               double* unused1, double* unused2, int64_t N, void* stream);
int rbd_Minv_f64(const double* q, const double* unused_qd, const double* unused_u,
                 double* minv_out, double* unused1, double* unused2, int64_t N, void* stream);
int rbd_FD_f64(const double* q, const double* qd, const double* tau, double* qdd_out,
               double* unused1, double* unused2, int64_t N, void* stream);
int rbd_gradID_f64(const double* q, const double* qd, const double* qdd, double* dq_out,
                   double* dqd_out, double* unused2, int64_t N, void* stream);
int rbd_gradFD_f64(const double* q, const double* qd, const double* tau, double* dq_out,
                   double* dqd_out, double* qdd_out, int64_t N, void* stream);

int rbd_ID_f32(const float* q, const float* qd, const float* qdd, float* tau_out,
               float* unused1, float* unused2, int64_t N, void* stream);
int rbd_Minv_f32(const float* q, const float* unused_qd, const float* unused_u,
                 float* minv_out, float* unused1, float* unused2, int64_t N, void* stream);
int rbd_FD_f32(const float* q, const float* qd, const float* tau, float* qdd_out,
               float* unused1, float* unused2, int64_t N, void* stream);
int rbd_gradID_f32(const float* q, const float* qd, const float* qdd, float* dq_out,
                   float* dqd_out, float* unused2, int64_t N, void* stream);
int rbd_gradFD_f32(const float* q, const float* qd, const float* tau, float* dq_out,
                   float* dqd_out, float* qdd_out, int64_t N, void* stream);

/* Generic form of the ten entries above. */
int rbd_launch(int alg, int dtype, const void* q, const void* qd, const void* u,
               void* out0, void* out1, void* out2, int64_t N, void* stream);

/* ---- external forces (refdyn's f_ext argument, refdyn.py:79-80, :91-249) ---
 * f_ext[k*n*6 + i*6 + c]: spatial force [moment; force] on link i of knot k in
 * link-i coordinates, subtracted from the link's Newton-Euler force (ID, FD,
 * and both gradients, which hold f_ext fixed in the link frame).  Minv takes
 * no f_ext. */
int rbd_ID_f64_fext(const double* q, const double* qd, const double* qdd, const double* f_ext,
                    double* tau_out, double* unused1, double* unused2, int64_t N, void* stream);
int rbd_FD_f64_fext(const double* q, const double* qd, const double* tau, const double* f_ext,
                    double* qdd_out, double* unused1, double* unused2, int64_t N, void* stream);
int rbd_gradID_f64_fext(const double* q, const double* qd, const double* qdd, const double* f_ext,
                        double* dq_out, double* dqd_out, double* unused2, int64_t N, void* stream);
int rbd_gradFD_f64_fext(const double* q, const double* qd, const double* tau, const double* f_ext,
                        double* dq_out, double* dqd_out, double* qdd_out, int64_t N, void* stream);
int rbd_ID_f32_fext(const float* q, const float* qd, const float* qdd, const float* f_ext,
                    float* tau_out, float* unused1, float* unused2, int64_t N, void* stream);
int rbd_FD_f32_fext(const float* q, const float* qd, const float* tau, const float* f_ext,
                    float* qdd_out, float* unused1, float* unused2, int64_t N, void* stream);
int rbd_gradID_f32_fext(const float* q, const float* qd, const float* qdd, const float* f_ext,
                        float* dq_out, float* dqd_out, float* unused2, int64_t N, void* stream);
int rbd_gradFD_f32_fext(const float* q, const float* qd, const float* tau, const float* f_ext,
                        float* dq_out, float* dqd_out, float* qdd_out, int64_t N, void* stream);

/* Generic form of the eight f_ext entries (alg != RBD_MINV). */
int rbd_launch_fext(int alg, int dtype, const void* q, const void* qd, const void* u,
                    const void* f_ext, void* out0, void* out1, void* out2, int64_t N,
                    void* stream);

/* ---- host-buffer entries (end-to-end path) -------------------------------- */
typedef struct rbd_session rbd_session;

/* Device buffers for `slots` pipeline stages of up to `chunk_knots` knots each
 * (sized for the largest algorithm in fp64), one stream per stage, on `device`. */
int rbd_session_create(int device, int64_t chunk_knots, int32_t slots, rbd_session** out);
int rbd_session_destroy(rbd_session* s);

/* Run N knots whose inputs/outputs live in HOST memory (pinned for full
 * overlap; pageable works, at lower PCIe throughput).  Splits the batch in
 * chunks, issues H2D(chunk) -> kernel -> D2H(chunk) round-robin over the
 * session's streams so copies in both directions overlap the kernels, and
 * returns after the last D2H has landed. */
int rbd_run_host(rbd_session* s, int alg, int dtype, const void* q, const void* qd,
                 const void* u, void* out0, void* out1, void* out2, int64_t N);

/* rbd_run_host with per-link external forces (host buffer, layout as above). */
int rbd_run_host_fext(rbd_session* s, int alg, int dtype, const void* q, const void* qd,
                      const void* u, const void* f_ext, void* out0, void* out1, void* out2,
                      int64_t N);

/* Several GPUs (knots are independent): slice k of
 * ceil(N / count) knots runs through sessions[k] (its own device, pipeline and
 * host thread), all slices concurrently; results land in place.  Returns the
 * first failing slice's code. */
int rbd_run_host_multi(rbd_session* const* sessions, int32_t count, int alg, int dtype,
                       const void* q, const void* qd, const void* u, void* out0, void* out1,
                       void* out2, int64_t N);
int rbd_run_host_multi_fext(rbd_session* const* sessions, int32_t count, int alg, int dtype,
                            const void* q, const void* qd, const void* u, const void* f_ext,
                            void* out0, void* out1, void* out2, int64_t N);

/* Device ordinal a session was created on. */
int rbd_session_device(const rbd_session* s, int32_t* device);

/* Device-resident rollouts (the paper's trajectory-optimisation use case):
 * one semi-implicit Euler step for N knots of this robot, device pointers,
 * [N][n] arrays: qd_next = qd + dt * qdd, q_next = q + dt * qd_next. */
int rbd_euler_step(int dtype, const void* q, const void* qd, const void* qdd, void* q_next,
                   void* qd_next, int64_t N, double dt, void* stream);

/* Fused rollout: B trajectories x H semi-implicit Euler steps of FD or gradFD
 * in ONE launch (a CTA carries a 32-trajectory group through the whole
 * horizon).  Time-major device arrays: q, qd [H+1][B][n] with step 0 set by
 * the caller (steps 1..H are written), tau and qdd [H][B][n], and for gradFD
 * dq, dqd [H][B][n*n] (NULL for FD).  Per step k: qdd_k = FD(q_k, qd_k, tau_k)
 * (refdyn.py:172; gradFD also writes fd_grad, refdyn.py:242), then
 * qd_{k+1} = qd_k + dt qdd_k, q_{k+1} = q_k + dt qd_{k+1}. */
int rbd_rollout(int alg, int dtype, void* q, void* qd, const void* tau, void* qdd, void* dq, void* dqd,
                int64_t B, int32_t H, double dt, void* stream);

/* Benchmark helper (not in the reference interface): calls rbd_run_host
 * `reps` times back to back and stores the mean host wall time per call in
 * *seconds (steady clock) -- the end-to-end latency a C/C++ caller sees,
 * without any binding-language overhead. */
int rbd_bench_host(rbd_session* s, int alg, int dtype, const void* q, const void* qd,
                   const void* u, void* out0, void* out1, void* out2, int64_t N, int32_t reps,
                   double* seconds);

#ifdef __cplusplus
}
#endif
#endif /* RBD_B200_H */
