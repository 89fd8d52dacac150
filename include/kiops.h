/*
 * kiops.h -- C ABI of the B200-native KIOPS hot path (fp64, one GPU, sm_100a).
 *
 * Computes, for every requested output time T_l (KIOPS, Gaudreault, Rainwater &
 * Tokman, JCP 2018 = arXiv 1804.05126; P:n = line n of the paper text):
 *
 *     w_l = sum_{k=0..p} T_l^k phi_k(T_l A) u_k             Eq. 12, Alg. 1
 *
 * through the exponential of the augmented matrix A~ = [[A, B],[0, K]],
 * B = [u_p, ..., u_1] (Theorem 1), with adaptive substepping (Eqs. 23-28),
 * the incomplete orthogonalisation procedure of window q (Alg. 2), the
 * projected exponential exp(tau H~) (Eqs. 33, 37-38), the error estimate
 * and acceptance test (Eqs. 36, 39), the adaptivity of Alg. 4 and the
 * output update of Alg. 3.  Readings of silent or garbled passages:
 * DESIGN.md section 3 (R1-R27).
 *
 * Every step runs on the device: after kiops_apply's single host->device copy of
 * its call block, one CUDA-graph launch (device-side WHILE/IF conditional nodes)
 * runs the whole adaptive loop; one device->host copy returns the statistics.
 *
 * Conventions for every entry point:
 *  - No C++ exceptions cross the ABI; every call returns a kiops_status.
 *  - "DEVICE" pointers are CUDA global-memory pointers on the ctx's device;
 *    "HOST" pointers are ordinary (or pinned) host memory.
 *  - Borrowed pointers are never freed by the library and must outlive their use.
 *  - A ctx serves one kiops_apply at a time (single owner, not thread-safe).
 *    Distinct ctxs may run concurrently on distinct streams.
 */
#ifndef KIOPS_H
#define KIOPS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KIOPS_MAX_P 8        /* maximum number of phi terms beyond phi_0 (p)            */
#define KIOPS_MAX_OUT 64     /* maximum number of output times per call                 */
#define KIOPS_MAX_M 128      /* maximum Krylov dimension m_max (exp of <= 129^2 on one CTA) */
#define KIOPS_MAX_FORCED 256 /* maximum length of a forced (test) schedule               */
#define KIOPS_TRACE_CAP 16384

typedef struct kiops_ctx_s *kiops_ctx; /* opaque; created by kiops_create */

typedef enum {
  KIOPS_OK = 0,
  KIOPS_ERR_INVALID_ARG = 1,    /* argument outside the domain of R21; nothing launched     */
  KIOPS_ERR_UNSUPPORTED = 2,    /* valid for the method, not implemented here (m_max > 128, */
                                /* 3D planes >= 2^31 points, non-periodic stencils)          */
  KIOPS_ERR_CUDA = 3,           /* a CUDA call failed; text in kiops_last_error             */
  KIOPS_ERR_NO_CONVERGENCE = 4, /* > max_attempts attempts (R22); stats filled, w undefined */
  KIOPS_ERR_NONFINITE = 5,      /* NaN/Inf in a reduced dot, beta, H, eps or omega (R22)    */
  KIOPS_ERR_WORKSPACE = 6       /* workspace pointer NULL, misaligned or too small          */
} kiops_status;

typedef enum {
  KIOPS_OP_STENCIL1D3 = 1,          /* periodic 1D 3-point: (Ax)_i = W x_{i-1} + C x_i + E x_{i+1} + d_i x_i */
  KIOPS_OP_STENCIL2D5 = 2,          /* periodic 2D 5-point: W x_{i-1,j} + E x_{i+1,j} + S x_{i,j-1} + N x_{i,j+1} + (C + d_ij) x_ij */
  KIOPS_OP_STENCIL3D7_VARKAPPA = 3, /* periodic 3D 7-point: sum_faces (kappa_i + kappa_nb)/2 (x_nb - x_i) inv_h2 */
  KIOPS_OP_CSR = 4                  /* general CSR: int64 row_ptr[N+1], int32 col_idx[nnz], fp64 vals[nnz] */
} kiops_op_kind;

/* Operator A ("the action of the matrix A ... provided by an external
 * subroutine"; here built-in kinds).  Vectors are lexicographic, x fastest:
 * i = x + nx*(y + ny*z).  All array pointers are DEVICE, borrowed, and must
 * outlive the ctx. */
typedef struct {
  int32_t kind;           /* kiops_op_kind                                             */
  int32_t periodic;       /* stencils: must be 1 (periodic wrap)                       */
  int64_t nx, ny, nz;     /* grid; N = nx*ny*nz.  1D: ny = nz = 1; 2D: nz = 1; CSR: nx = N */
  double w[5];            /* 1D: {W, C, E}; 2D: {W, E, S, N, C}; unused for 3D and CSR  */
  const double *diag;     /* optional additive diagonal d (length N) for 1D/2D, or NULL */
  const double *kappa;    /* 3D: cell conductivity (length N)                          */
  double inv_h2;          /* 3D: 1/h^2                                                 */
  const int64_t *row_ptr; /* CSR                                                       */
  const int32_t *col_idx; /* CSR                                                       */
  const double *vals;     /* CSR                                                       */
  int64_t nnz;            /* CSR                                                       */
} kiops_operator_desc;

/* Alg. 1 inputs plus the IOP window.  Defaults (kiops_options_default):
 * tol 1e-7, m_init 10, m_min 10, m_max 128, iop_q 2, task1 0, max_attempts 10000,
 * host_staging 0, max_outputs 4, corrected 0. */
typedef struct {
  double tol;             /* Eq. 39 tolerance (absolute, 2-norm of the scaled augmented vector, R18) */
  int32_t m_init, m_min, m_max; /* 1 <= m_min <= m_max <= KIOPS_MAX_M                   */
  int32_t iop_q;          /* IOP window, 1 <= q <= m_max (q = m_max: full Arnoldi); q = 2 (Alg. 2
                           * as printed) runs the fused kernels, other q a generic 4-launch pass */
  int32_t task1;          /* 1 => output l scaled by 1/T_l^p (Alg. 1 l.31-35) */
  int64_t max_attempts;   /* accepted + rejected attempts before KIOPS_ERR_NO_CONVERGENCE */
  int32_t host_staging;   /* 1 => workspace also holds device staging for kiops_apply_host */
  int32_t max_outputs;    /* largest n_out kiops_apply_host will be called with (staging)  */
  int32_t corrected;      /* 1 => Saad's corrected scheme [46]: each output update adds
                           * beta h_{j+1,j} F(j, j+1) v_{j+1} (v_{j+1}: the last basis vector of
                           * Alg. 2); decisions (eps, omega, Alg. 4) unchanged.  Default 0 */
} kiops_options;

/* Statistics of one kiops_apply. */
typedef struct {
  int64_t substeps;       /* accepted substeps                                         */
  int64_t rejections;     /* rejected attempts                                         */
  int64_t krylov_vectors; /* Alg. 2 iterations (augmented matvecs of the method)       */
  int64_t expm_calls;     /* dense exponentials (F of Alg. 1 l.18 and F2 of Alg. 3 l.14) */
  int64_t passes;         /* fused device passes launched (krylov_vectors + one look-ahead per basis) */
  int32_t final_m;        /* m after the last Alg. 4 update (R25): warm start for the next call */
  int32_t happy_breakdowns;
  double t_reached;       /* T_end on success                                          */
  double nu, mu;          /* Eqs. 48-49 normalisation constants used                    */
  double pass_ms, ctrl_ms, gemv_ms; /* device-side kernel time (%globaltimer) of the fused
                                       passes, the controller and the GEMV in this call */
  double expm_ms;                   /* part of ctrl_ms spent in the F = exp(tau H~) of Alg. 1 l.18 */
  int64_t pass_launches;            /* launches of the pass kernel(s): one per pass, or one per Alg. 2
                                       run with the persistent inner loop (KIOPS_PERSIST=0 disables it) */
} kiops_stats;

/* One row per attempt (accepted or rejected), for oracle <-> GPU trace parity. */
typedef struct {
  int64_t attempt;
  int32_t j, happy, accept, m_new;
  double t_now, tau, beta, h_next, eps, omega, tau_new;
} kiops_trace_row;

/* Fills *o with the defaults above.  o: HOST, non-NULL. */
void kiops_options_default(kiops_options *o);

/* Bytes of DEVICE workspace kiops_create needs for this operator, p and options.
 * Returns KIOPS_ERR_INVALID_ARG / KIOPS_ERR_UNSUPPORTED like kiops_create would.
 * CSR: the workspace also holds a SELL-32 copy of the matrix (slices of 32 rows
 * padded to their longest row), so this call reads op->row_ptr from the device
 * once (KIOPS_ERR_CUDA if it cannot); row_ptr must not change before create. */
kiops_status kiops_workspace_bytes(const kiops_operator_desc *op, int p, const kiops_options *o,
                                   size_t *bytes);

/* Creates a context: validates op, p and o (R21), carves the caller-owned DEVICE
 * workspace (>= kiops_workspace_bytes, 256-byte aligned; the library never calls
 * cudaMalloc for it), builds the SELL-32 copy for CSR operators (the CSR arrays
 * are not read again by kiops_apply), and instantiates the CUDA graph on
 * `cuda_stream` (a cudaStream_t; NULL = legacy default stream).  The ctx keeps
 * op's arrays borrowed.  Synchronises the stream.  On error *out is NULL. */
kiops_status kiops_create(const kiops_operator_desc *op, int p, const kiops_options *o,
                          void *cuda_stream, void *workspace, size_t workspace_bytes,
                          kiops_ctx *out);

/* Runs Alg. 1 on the ctx stream and returns after one stream synchronisation.
 *  u:      HOST array of p+1 DEVICE pointers u_0..u_p (N doubles each; u_0 may be
 *          all zeros).  u[k] multiplies T^k phi_k (Eq. 12).
 *  tau_out: HOST array of n_out output times, 0 < T_1 < ... < T_n (R21).
 *  w:      HOST array of n_out DEVICE pointers (N doubles each), written with
 *          w(T_l); must not alias any u[k] or each other.
 *  stats:  HOST, nullable.
 * Alignment: u[k] (and, at create, op->diag / op->kappa) must be 16-byte aligned for
 * the periodic stencils with an even nx (1D/2D, and 3D with KIOPS_3D=lazy), whose
 * passes read them as 16-byte pairs; a misaligned pointer is rejected with
 * INVALID_ARG before any launch.  w and the CSR / padded-3D inputs have no alignment
 * requirement beyond 8 bytes.
 * Errors: INVALID_ARG (bad times, n_out outside 1..KIOPS_MAX_OUT, NULL or misaligned
 * pointers), NO_CONVERGENCE / NONFINITE (stats filled, w undefined), CUDA. */
kiops_status kiops_apply(kiops_ctx c, const double *const *u, const double *tau_out, int n_out,
                         double *const *w, kiops_stats *stats);

/* Same computation from HOST vectors: u is a HOST array of p+1 HOST pointers, w a
 * HOST array of n_out HOST pointers.  Needs options.host_staging = 1 and
 * n_out <= options.max_outputs at create.  The host<->device copies are part of
 * the call (cudaMemcpyAsync on the ctx stream; pinned host memory is fastest).  An
 * output buffer in pinned, device-mapped host memory (cudaHostAlloc / cudaMallocHost /
 * torch pin_memory on a UVA system) is written by the GEMV directly over the host link
 * (no staging, no separate D2H copy); any other host buffer goes through staging. */
kiops_status kiops_apply_host(kiops_ctx c, const double *const *u, const double *tau_out, int n_out,
                              double *const *w, kiops_stats *stats);

/* TEST / PROFILING HOOK (not the product path): the same computation with the
 * graph's WHILE/IF control flow run on the host -- the identical kernels are
 * launched one by one with a device->host read of the loop conditions after each.
 * Exists because Nsight Compute cannot profile kernel nodes of graphs that contain
 * conditional nodes.  Same arguments and results as kiops_apply (bitwise). */
kiops_status kiops_apply_hostloop(kiops_ctx c, const double *const *u, const double *tau_out, int n_out,
                                  double *const *w, kiops_stats *stats);

/* Copies the decision trace of the last apply (one kiops_trace_row per attempt,
 * at most KIOPS_TRACE_CAP) into host_buf (HOST, `bytes` long); *rows = rows
 * available (may exceed what fit). */
kiops_status kiops_get_trace(kiops_ctx c, void *host_buf, size_t bytes, int64_t *rows);

/* Initial Krylov size of the NEXT kiops_apply calls (Alg. 1 l.3 m_init; the Sec. 3.6
 * warm start "use the final value of m_i from the previous time step": pass the
 * previous call's stats.final_m).  0 restores options.m_init.  Clipped to
 * [m_min, m_max] like m_init.  Errors: KIOPS_ERR_INVALID_ARG for a NULL ctx or m < 0. */
kiops_status kiops_set_m_init(kiops_ctx ctx, int m_init);

/* TEST HOOK (not for users): force the next applies to run attempt i with
 * substep tau[i] and Krylov size m[i], bypassing Alg. 4, and accept it if
 * accept == NULL or accept[i] != 0 (n = 0 clears).  tau, m, accept: HOST,
 * n <= KIOPS_MAX_FORCED.  With the oracle's trace (tau, j, accept) this REPLAYS
 * the oracle's decisions (R26: the result is unique given the decision trace);
 * with accept == NULL it gives step-level parity and the semigroup pin. */
kiops_status kiops_set_forced_schedule(kiops_ctx c, const double *tau, const int32_t *m,
                                       const int32_t *accept, int n);

/* TEST HOOK: copies the projected matrix H (column-major, leading dimension
 * m_max+2, H(i,j) 1-based at h[(i-1) + (j-1)*(m_max+2)]) and the norms
 * sigma_k = ||x_k|| of the unnormalised basis vectors of the current substep.
 * h: HOST (m_max+2)^2 doubles; sig: HOST m_max+2 doubles (sig[k-1] = sigma_k);
 * *npass: number of basis vectors formed in the current substep. */
kiops_status kiops_debug_basis(kiops_ctx c, double *h, double *sig, int32_t *npass);

/* TEST HOOK: f = exp(scale * m) by the controller's own projected exponential (Pade-13
 * scaling and squaring, reading R17; the single-CTA shared-memory path for
 * n <= 48, the cluster path above), so that it can be compared with the oracle's directly.
 * m, f: HOST, n x n doubles, column-major, leading dimension n; 1 <= n <= m_max_cap + 1
 * (129).  *products (may be NULL): the number of dense products.  Uses the ctx's scratch:
 * not concurrently with kiops_apply.  NONFINITE for a zero pivot / non-finite norm. */
kiops_status kiops_debug_expm(kiops_ctx c, int n, const double *m, double scale, double *f, int32_t *products);

/* The operator's value arrays (diag, kappa, CSR vals; DEVICE, borrowed) may be rewritten
 * by the caller between applies (e.g. a new Jacobian per time step, Sec. 3.6).  Stencil
 * operators read them at every apply; a CSR operator is applied from the SELL-32 copy
 * made at kiops_create, which this call rebuilds from the current vals (same sparsity
 * pattern; asynchronous on the ctx stream).  No-op for the other kinds. */
kiops_status kiops_refresh_operator(kiops_ctx c);

/* Destroys the ctx (graph, host state).  The workspace stays owned by the caller. */
kiops_status kiops_destroy(kiops_ctx c);

/* Static strings; never NULL. */
const char *kiops_status_string(kiops_status s);
const char *kiops_last_error(kiops_ctx c);


/* ===========================================================================
 * EPIRK exponential integrators on top of kiops_apply.
 * EPIRK4s3 (Eq. 50) and EPIRK4s3A (Eq. 51) with the
 * "mixed implementation" of Sec. 2 (Eqs. 9-11); EPIRK5P1 (Eq. 52, Table 1)
 * and EXPRB5s3 (Eq. 53) with three calls per step (Sec. 4; grouping in
 * DESIGN.md readings E8-E9).  Fourth order, per constant step h,
 *   call 1 (Task I):  phi_1(c h J_n) h f(u_n) at both stage nodes c (one kiops_apply,
 *                     p = 1, T = the two nodes ascending, 1/T scaling);
 *   stages:           U_i = u_n + c_i * (call-1 output), r(U_i), b_3, b_4 (Eq. 11);
 *   call 2 (Task II): phi_1(hJ_n) h f + phi_3(hJ_n) b_3 + phi_4(hJ_n) b_4 (p = 4, T = 1);
 *   u_{n+1} = u_n + (call-2 output).
 * Each call's m starts from the same call's final m of the previous step (Sec. 3.6).
 * Problem class: u' = L u + R(u), R a cubic polynomial applied pointwise, L constant:
 * a 5-point stencil on a periodic nx x ny grid (Allen-Cahn: alpha lap(u) + u - u^3,
 * P:593-597) or a general CSR matrix (ADR with Neumann boundaries).  J(u) = L + diag(R'(u)); for this class the remainder
 * r(U) = f(U) - f(u_n) - J_n (U - u_n) equals R(U) - R(u_n) - R'(u_n)(U - u_n)
 * exactly (the linear terms cancel), which is what the stage kernel evaluates.
 * =========================================================================== */
typedef enum { KIOPS_EPIRK4S3 = 1, KIOPS_EPIRK4S3A = 2, KIOPS_EPIRK5P1 = 3, KIOPS_EXPRB5S3 = 4 } kiops_epirk_scheme;

typedef struct {
  int64_t nx, ny;          /* periodic grid, N = nx*ny, x fastest                          */
  double w[5];             /* L: {W, E, S, N, C} weights (alpha lap: alpha/dx^2 {1,1,1,1,-4}) */
  double c[4];             /* R(u) = c[0] + c[1] u + c[2] u^2 + c[3] u^3                   */
  /* Optional general linear part (non-periodic boundaries, advection, ...; e.g. the ADR
   * problem with homogeneous Neumann boundaries): when L_row_ptr != NULL, L
   * is this CSR matrix with N = nx*ny rows (DEVICE arrays, borrowed for the ctx's life,
   * constant; int64 row_ptr[N+1], int32 col_idx[nnz], fp64 vals[nnz]) and w is ignored.
   * Every row must hold its diagonal entry (kiops_epirk_create checks: INVALID_ARG).
   * The KIOPS operator h J_n = h (L + diag R'(u_n)) is then a KIOPS_OP_CSR operator whose
   * values the driver rewrites every step (kiops_refresh_operator).                    */
  const int64_t *L_row_ptr;
  const int32_t *L_col_idx;
  const double *L_vals;
  int64_t L_nnz;
} kiops_rd_problem;

typedef struct {
  int64_t steps, krylov_vectors, passes, substeps, rejections, expm_calls;
  int32_t final_m[3];      /* warm-start m of calls 1-3 after the last step (4th order: 2 calls) */
  double kiops_ms;         /* device time in the two kiops_apply calls (%globaltimer sums)  */
} kiops_epirk_stats;

typedef struct kiops_epirk_s *kiops_epirk_ctx;

/* Bytes of the caller-owned workspace for kiops_epirk_create with this scheme (one kiops
 * workspace of m_max+3 vectors per distinct call shape -- two for the fourth-order
 * schemes and EPIRK5P1, three for EXPRB5s3 -- plus 11 stage vectors; 1024^2: ~2.3 GB
 * at m_max = 128 for two shapes). */
kiops_status kiops_epirk_workspace_bytes(const kiops_rd_problem *pb, int scheme, const kiops_options *o,
                                         size_t *bytes);

/* pb, o: HOST, copied.  h > 0: the constant step.  scheme: KIOPS_EPIRK4S3,
 * KIOPS_EPIRK4S3A (two grouped calls per step), KIOPS_EPIRK5P1, KIOPS_EXPRB5S3 (three).
 * o: the KIOPS options of both calls (tol, m_*, max_attempts; task1 and staging are
 * set internally).  workspace: DEVICE, 256-byte aligned, >= the queried bytes,
 * borrowed for the ctx's life.  Errors as kiops_create. */
kiops_status kiops_epirk_create(const kiops_rd_problem *pb, int scheme, double h, const kiops_options *o,
                                void *cuda_stream, void *workspace, size_t workspace_bytes,
                                kiops_epirk_ctx *out);

/* nsteps constant steps from u (DEVICE, N doubles, updated in place).  Any KIOPS
 * failure aborts with its status (the step index is in kiops_epirk_last_error). */
kiops_status kiops_epirk_step(kiops_epirk_ctx ctx, double *u, int nsteps, kiops_epirk_stats *stats);

/* Per-call decision history of the last kiops_epirk_step (TEST / diagnostics hook; off by
 * default).  With kiops_epirk_record_history(ctx, 1), every KIOPS call of a step appends
 * one record: its step index (0-based within the last kiops_epirk_step), call index
 * (0..2), the call's counts and final m (the next call's warm start, reading E1), and the
 * Krylov size j, acceptance, omega and m_new of its first KIOPS_EPIRK_HIST_ATTEMPTS attempts (from
 * kiops_get_trace of the call's context right after it; the call has synchronised the
 * stream already).  kiops_epirk_history copies up to `cap` records into buf (HOST) and
 * sets *rows to the number available. */
#define KIOPS_EPIRK_HIST_ATTEMPTS 64
typedef struct {
  int32_t step, call, final_m, n_attempts;
  int64_t krylov_vectors, substeps, rejections;
  int16_t j[KIOPS_EPIRK_HIST_ATTEMPTS];
  int16_t m_new[KIOPS_EPIRK_HIST_ATTEMPTS];
  int8_t accept[KIOPS_EPIRK_HIST_ATTEMPTS];
  double omega[KIOPS_EPIRK_HIST_ATTEMPTS];  /* Eq. 39 of each attempt */
} kiops_epirk_call_record;
kiops_status kiops_epirk_record_history(kiops_epirk_ctx ctx, int on);
/* TEST HOOK (trace replay, R26): the forced schedule (tau_i, m_i, accept_i), i < n, of
 * call `call` (0..2) of step `step` (0-based within the next kiops_epirk_step), applied
 * with kiops_set_forced_schedule to that call only.  n = 0 with step = -1 clears every
 * schedule.  HOST arrays, copied. */
kiops_status kiops_epirk_set_forced_schedule(kiops_epirk_ctx ctx, int step, int call, const double *tau,
                                            const int32_t *m, const int32_t *accept, int n);
kiops_status kiops_epirk_history(kiops_epirk_ctx ctx, kiops_epirk_call_record *buf, int64_t cap, int64_t *rows);

kiops_status kiops_epirk_destroy(kiops_epirk_ctx ctx);
const char *kiops_epirk_last_error(kiops_epirk_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif
