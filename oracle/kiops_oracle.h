/*
 * kiops_oracle.h -- the CPU ORACLE for the KIOPS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product (paper_1804_05126_b200/, include/kiops.h) never links it and
 * shares no code, header, table or constant with it.
 *
 * Plain, slow, obviously-correct C99 following PAPER.md step by step:
 *   Alg. 1 driver, Alg. 2 IOP, Alg. 3
 *   output update, Alg. 4 adaptivity, Eqs. 36-39,
 *   Theorem 1, Eqs. 47-49, Pade-13 scaling and
 *   squaring (Higham 2005 = paper ref [47]).
 * Every silent or garbled passage is resolved by a reading R1..R27 listed in
 * DESIGN.md section 3; the code cites the reading where it applies.
 */
#ifndef KIOPS_ORACLE_H
#define KIOPS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OR_OP_STENCIL1D3 = 1,          /* periodic 1D 3-point, weights {W,C,E}              */
  OR_OP_STENCIL2D5 = 2,          /* periodic 2D 5-point, weights {W,E,S,N,C}          */
  OR_OP_STENCIL3D7_VARKAPPA = 3, /* periodic 3D 7-point, face kappa = mean of cells   */
  OR_OP_CSR = 4,                 /* general CSR (int64 row_ptr, int32 col_idx)         */
  OR_OP_DENSE = 5                /* column-major dense N x N (tiny pins only)         */
};

typedef struct {
  int kind;
  int64_t nx, ny, nz;       /* N = nx*ny*nz ; CSR/DENSE: nx = N, ny = nz = 1      */
  double w[5];              /* stencil weights                                    */
  const double *diag;       /* optional additive diagonal (length N), nullable    */
  const double *kappa;      /* 3D: cell conductivity (length N)                   */
  double inv_h2;            /* 3D: 1/h^2                                          */
  const int64_t *row_ptr;   /* CSR                                                */
  const int32_t *col_idx;
  const double *vals;
  const double *dense;      /* DENSE: column-major N x N                          */
} or_operator;

typedef struct {
  double tol;               /* Eq. 39 tolerance (default 1e-7)             */
  int m_init, m_min, m_max; /* P:252 defaults 10, 10, 128                          */
  int iop_q;                /* IOP window (2 = the paper's Alg. 2)                 */
  int task1;                /* 1 => scale output l by 1/T_l^p (Alg. 1 l.31-35)     */
  int64_t max_attempts;     /* R22 divergence guard (default 10000)                */
  int n_forced;             /* test hook: forced (tau_i, m_i[, accept_i]) schedule   */
  const double *forced_tau;
  const int *forced_m;
  const int *forced_accept; /* NULL => every forced attempt accepted; else replay     */
  int corrected;            /* 1 => Saad's corrected scheme [46]: the output  */
                            /* update adds beta h_{j+1,j} F(j,j+1) v_{j+1}             */
} or_options;

typedef struct {
  int64_t substeps, rejections, krylov_vectors, expm_calls;
  int final_m, happy_breakdowns;
  double t_reached;
  double nu, mu;            /* Eqs. 48-49 normalisation constants actually used   */
} or_stats;

typedef struct {            /* one row per attempt (accepted or rejected)         */
  int64_t attempt;
  int j, happy, accept, m_new;
  double t_now, tau, beta, h_next, eps, omega, tau_new;
} or_trace_row;

enum {
  OR_OK = 0, OR_ERR_INVALID_ARG = 1, OR_ERR_NO_CONVERGENCE = 4,
  OR_ERR_NONFINITE = 5, OR_ERR_ALLOC = 6
};

/* y = A x (N entries).  P:335 "provided by an external subroutine". */
void or_apply(const or_operator *op, const double *x, double *y);
int64_t or_n(const or_operator *op);

/* F = exp(scale*M), n x n column-major, by diagonal Pade + scaling and squaring
 * (Higham 2005 Alg. 2.3).  *n_mult counts dense products incl. squarings. */
int or_expm(int n, const double *M, double scale, double *F, int *n_mult);

/* Eqs. 48-49 with reading R12: ||B||_1 = max column abs sum of
 * B = [u_p..u_1]; nu = 2^-e, mu = 2^e, e = ceil(log2 ||B||_1); zero => 1, 1. */
void or_normalisation(int64_t N, int p, const double *const *u, double *nu, double *mu);

/* Alg. 2 lines 4-6: y = A~ v with A~ = [[A, nu*B],[0, K]].
 * u = [u_0..u_p] (B = [u_p..u_1], Thm 1).  v, y have N+p entries. */
void or_augmented_matvec(const or_operator *op, int64_t N, int p, const double *const *u,
                         double nu, const double *v, double *y);

/* Alg. 2 from scratch: V(:,1) = v0/||v0||, then IOP with window q until j == m
 * or happy breakdown.  V is (N+p) x (m+1) column-major, H is (m+1) x m
 * column-major.  Returns j (completed columns); *happy set on breakdown. */
int or_iop(const or_operator *op, int64_t N, int p, const double *const *u, double nu,
           const double *v0, int m, int q, double *V, double *H, int *happy);

/* Alg. 4 with readings R4-R10: one controller decision.
 * hist_valid/omega_old/tau_old/j_old describe the immediately preceding
 * rejected attempt of the same substep (R5).  Returns m_new, writes tau_new. */
int or_adapt(int happy, int accept, int j, int m, int m_min, int m_max, double tau,
             double omega, double t_now, double t_end, int hist_valid, double omega_old,
             double tau_old, int j_old, double *tau_new);

/* Alg. 1 + 3 + 4: w_l = sum_k T_l^k phi_k(T_l A) u_k for every output time.
 * u: p+1 input vectors u_0..u_p (N each).  T: n_out strictly increasing > 0.
 * w: n_out output vectors (N each).  trace may be NULL.                     */
/* w(0:N) = beta V(0:N, 0:j) f(0:j), V column-major with leading dimension ld (Eq. 33) */
void or_project(int64_t N, int64_t ld, int j, const double *V, const double *f, double beta, double *w);
int or_kiops(const or_operator *op, int p, const double *const *u, int n_out,
             const double *T, double *const *w, const or_options *o, or_stats *st,
             or_trace_row *trace, int64_t trace_cap, int64_t *trace_len);

/* Theorem 1 dense route for tiny pins: builds A~ (N+p)^2 explicitly and
 * returns e^{tau A~} v, v = [u_0; e_p] (N+p entries).  A must be OR_OP_DENSE
 * or any kind (applied column by column).                                   */
int or_dense_phi_combination(const or_operator *op, int p, const double *const *u,
                             double tau, double *out);

#ifdef __cplusplus
}
#endif
#endif
