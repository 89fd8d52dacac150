/*
 * kiops_oracle.c -- plain, slow, obviously-correct CPU oracle of KIOPS.
 *
 * TEST INFRASTRUCTURE ONLY (see kiops_oracle.h).  Nothing under
 * paper_1804_05126_b200/ includes, links or calls this file.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (not needed at run time).
 * Readings R1..R27 = DESIGN.md section 3.  Floating point: IEEE fp64, no
 * fast-math, no FMA contraction (built with -ffp-contract=off), every sum is a
 * plain left-to-right loop.
 */
#include "kiops_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define CM(i, j, ld) ((size_t)(j) * (size_t)(ld) + (size_t)(i)) /* column-major */

/* ------------------------------------------------------------------------- */
/* Operators: y = A x.  P:335 "the action of the matrix A ... provided by an  */
/* external subroutine"; shapes from BASELINE.json configs. */
/* ------------------------------------------------------------------------- */
int64_t or_n(const or_operator *op) { return op->nx * op->ny * op->nz; }

static int64_t wrap(int64_t i, int64_t n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

void or_apply(const or_operator *op, const double *x, double *y) {
  const int64_t N = or_n(op);
  if (op->kind == OR_OP_STENCIL1D3) {
    /* (Ax)_i = W x_{i-1} + C x_i + E x_{i+1}, periodic */
    const int64_t n = op->nx;
    for (int64_t i = 0; i < n; i++) {
      double s = op->w[0] * x[wrap(i - 1, n)] + op->w[1] * x[i] + op->w[2] * x[wrap(i + 1, n)];
      if (op->diag) s += op->diag[i] * x[i];
      y[i] = s;
    }
  } else if (op->kind == OR_OP_STENCIL2D5) {
    /* (Ax)_{x,y} = W u_{x-1,y} + E u_{x+1,y} + S u_{x,y-1} + N u_{x,y+1} + C u + d u */
    const int64_t nx = op->nx, ny = op->ny;
    for (int64_t b = 0; b < ny; b++)
      for (int64_t a = 0; a < nx; a++) {
        const int64_t i = a + nx * b;
        double s = op->w[0] * x[wrap(a - 1, nx) + nx * b] + op->w[1] * x[wrap(a + 1, nx) + nx * b] +
                   op->w[2] * x[a + nx * wrap(b - 1, ny)] + op->w[3] * x[a + nx * wrap(b + 1, ny)] +
                   op->w[4] * x[i];
        if (op->diag) s += op->diag[i] * x[i];
        y[i] = s;
      }
  } else if (op->kind == OR_OP_STENCIL3D7_VARKAPPA) {
    /* (Ax)_i = sum_{6 faces} kappa_f (x_nb - x_i) / h^2, kappa_f = (kappa_i + kappa_nb)/2 (D6) */
    const int64_t nx = op->nx, ny = op->ny, nz = op->nz;
    const double *k = op->kappa;
    for (int64_t c = 0; c < nz; c++)
      for (int64_t b = 0; b < ny; b++)
        for (int64_t a = 0; a < nx; a++) {
          const int64_t i = a + nx * (b + ny * c);
          const int64_t nb[6] = {wrap(a - 1, nx) + nx * (b + ny * c), wrap(a + 1, nx) + nx * (b + ny * c),
                                 a + nx * (wrap(b - 1, ny) + ny * c), a + nx * (wrap(b + 1, ny) + ny * c),
                                 a + nx * (b + ny * wrap(c - 1, nz)), a + nx * (b + ny * wrap(c + 1, nz))};
          double s = 0.0;
          for (int f = 0; f < 6; f++) s += 0.5 * (k[i] + k[nb[f]]) * (x[nb[f]] - x[i]);
          s *= op->inv_h2;
          if (op->diag) s += op->diag[i] * x[i];
          y[i] = s;
        }
  } else if (op->kind == OR_OP_CSR) {
    for (int64_t r = 0; r < N; r++) {
      double s = 0.0;
      for (int64_t q = op->row_ptr[r]; q < op->row_ptr[r + 1]; q++) s += op->vals[q] * x[op->col_idx[q]];
      y[r] = s;
    }
  } else { /* OR_OP_DENSE */
    for (int64_t i = 0; i < N; i++) {
      double s = 0.0;
      for (int64_t c = 0; c < N; c++) s += op->dense[CM(i, c, N)] * x[c];
      y[i] = s;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* Small dense linear algebra                                                 */
/* ------------------------------------------------------------------------- */
static void mat_mul(int n, const double *A, const double *B, double *C) { /* C = A B */
  for (int j = 0; j < n; j++)
    for (int i = 0; i < n; i++) {
      double s = 0.0;
      for (int k = 0; k < n; k++) s += A[CM(i, k, n)] * B[CM(k, j, n)];
      C[CM(i, j, n)] = s;
    }
}

static double norm1(int n, const double *A) { /* max column abs sum */
  double best = 0.0;
  for (int j = 0; j < n; j++) {
    double s = 0.0;
    for (int i = 0; i < n; i++) s += fabs(A[CM(i, j, n)]);
    if (s > best || isnan(s)) best = s;
  }
  return best;
}

/* Solve Q X = B in place (B <- X), Q n x n overwritten by its LU factors.
 * Doolittle elimination with partial pivoting (first max |.| in the column). */
static int lu_solve(int n, double *Q, double *B) {
  for (int k = 0; k < n; k++) {
    int piv = k;
    double best = fabs(Q[CM(k, k, n)]);
    for (int i = k + 1; i < n; i++)
      if (fabs(Q[CM(i, k, n)]) > best) { best = fabs(Q[CM(i, k, n)]); piv = i; }
    if (!(best > 0.0)) return -1;
    if (piv != k)
      for (int j = 0; j < n; j++) {
        double t = Q[CM(k, j, n)]; Q[CM(k, j, n)] = Q[CM(piv, j, n)]; Q[CM(piv, j, n)] = t;
        t = B[CM(k, j, n)]; B[CM(k, j, n)] = B[CM(piv, j, n)]; B[CM(piv, j, n)] = t;
      }
    for (int i = k + 1; i < n; i++) Q[CM(i, k, n)] /= Q[CM(k, k, n)];
    for (int j = k + 1; j < n; j++)
      for (int i = k + 1; i < n; i++) Q[CM(i, j, n)] -= Q[CM(i, k, n)] * Q[CM(k, j, n)];
  }
  for (int c = 0; c < n; c++) {
    for (int i = 0; i < n; i++) { /* L y = b, unit lower */
      double s = B[CM(i, c, n)];
      for (int k = 0; k < i; k++) s -= Q[CM(i, k, n)] * B[CM(k, c, n)];
      B[CM(i, c, n)] = s;
    }
    for (int i = n - 1; i >= 0; i--) { /* U x = y */
      double s = B[CM(i, c, n)];
      for (int k = i + 1; k < n; k++) s -= Q[CM(i, k, n)] * B[CM(k, c, n)];
      B[CM(i, c, n)] = s / Q[CM(i, i, n)];
    }
  }
  return 0;
}

/* ceil(log2(x)) for x > 0, exact: x = f 2^e with f in [0.5, 1). (R12, R17) */
static int ceil_log2(double x) {
  int e;
  double f = frexp(x, &e);
  return (f == 0.5) ? e - 1 : e;
}

/* Diagonal Pade + scaling and squaring, "we use a diagonal Pade
 * approximation combined with a scaling and squaring algorithm [47]".
 * [47] = Higham, SIAM J. Matrix Anal. Appl. 26 (2005), Algorithm 2.3: the
 * theta_m table (Table 2.3) and the coefficients b_j of the [m/m] Pade
 * numerator, b_j = (2m-j)! m! / ((2m)! j! (m-j)!) scaled to integers (R17). */
int or_expm(int n, const double *M, double scale, double *F, int *n_mult) {
  static const double theta3 = 1.495585217958292e-2, theta5 = 2.539398330063230e-1,
                      theta7 = 9.504178996162932e-1, theta9 = 2.097847961257068e0,
                      theta13 = 5.371920351148152e0;
  static const double b3[] = {120., 60., 12., 1.};
  static const double b5[] = {30240., 15120., 3360., 420., 30., 1.};
  static const double b7[] = {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.};
  static const double b9[] = {17643225600., 8821612800., 2075673600., 302702400., 30270240.,
                              2162160., 110880., 3960., 90., 1.};
  static const double b13[] = {64764752532480000., 32382376266240000., 7771770303897600.,
                               1187353796428800.,  129060195264000.,   10559470521600.,
                               670442572800.,      33522128640.,       1323241920.,
                               40840800.,          960960.,            16380.,
                               182.,               1.};
  const size_t nn = (size_t)n * n;
  int mult = 0, s = 0, deg;
  if (n <= 0) return -1;
  double *X = malloc(nn * sizeof(double)), *X2 = malloc(nn * sizeof(double)),
         *X4 = malloc(nn * sizeof(double)), *X6 = malloc(nn * sizeof(double)),
         *X8 = malloc(nn * sizeof(double)), *U = malloc(nn * sizeof(double)),
         *V = malloc(nn * sizeof(double)), *T = malloc(nn * sizeof(double));
  int rc = 0;
  if (!X || !X2 || !X4 || !X6 || !X8 || !U || !V || !T) { rc = -2; goto done; }
  for (size_t i = 0; i < nn; i++) X[i] = scale * M[i];
  const double nrm = norm1(n, X);
  if (!isfinite(nrm)) { rc = -3; goto done; }

  if (nrm <= theta3) deg = 3;
  else if (nrm <= theta5) deg = 5;
  else if (nrm <= theta7) deg = 7;
  else if (nrm <= theta9) deg = 9;
  else {
    deg = 13;
    s = ceil_log2(nrm / theta13);
    if (s < 0) s = 0;
    const double f = ldexp(1.0, -s);
    for (size_t i = 0; i < nn; i++) X[i] *= f;
  }

  mat_mul(n, X, X, X2); mult++;
  if (deg >= 5) { mat_mul(n, X2, X2, X4); mult++; }
  if (deg >= 7) { mat_mul(n, X2, X4, X6); mult++; }
  if (deg == 9) { mat_mul(n, X4, X4, X8); mult++; }

  if (deg < 13) {
    const double *b = deg == 3 ? b3 : deg == 5 ? b5 : deg == 7 ? b7 : b9;
    /* U = X * sum_k b_{2k+1} X^{2k},  V = sum_k b_{2k} X^{2k}   (Higham 2005 eq. 2.11) */
    for (int j = 0; j < n; j++)
      for (int i = 0; i < n; i++) {
        const size_t q = CM(i, j, n);
        const double id = (i == j) ? 1.0 : 0.0;
        double u = b[1] * id + b[3] * X2[q], v = b[0] * id + b[2] * X2[q];
        if (deg >= 5) { u += b[5] * X4[q]; v += b[4] * X4[q]; }
        if (deg >= 7) { u += b[7] * X6[q]; v += b[6] * X6[q]; }
        if (deg >= 9) { u += b[9] * X8[q]; v += b[8] * X8[q]; }
        T[q] = u; V[q] = v;
      }
    mat_mul(n, X, T, U); mult++;
  } else {
    const double *b = b13;
    /* Higham 2005 eq. 2.12:
       U = X [X6 (b13 X6 + b11 X4 + b9 X2) + b7 X6 + b5 X4 + b3 X2 + b1 I]
       V =    X6 (b12 X6 + b10 X4 + b8 X2) + b6 X6 + b4 X4 + b2 X2 + b0 I   */
    for (size_t q = 0; q < nn; q++) T[q] = b[13] * X6[q] + b[11] * X4[q] + b[9] * X2[q];
    mat_mul(n, X6, T, U); mult++;
    for (int j = 0; j < n; j++)
      for (int i = 0; i < n; i++) {
        const size_t q = CM(i, j, n);
        U[q] += b[7] * X6[q] + b[5] * X4[q] + b[3] * X2[q] + ((i == j) ? b[1] : 0.0);
      }
    mat_mul(n, X, U, T); mult++;          /* T = U (odd part) */
    for (size_t q = 0; q < nn; q++) X8[q] = b[12] * X6[q] + b[10] * X4[q] + b[8] * X2[q];
    mat_mul(n, X6, X8, V); mult++;
    for (int j = 0; j < n; j++)
      for (int i = 0; i < n; i++) {
        const size_t q = CM(i, j, n);
        V[q] += b[6] * X6[q] + b[4] * X4[q] + b[2] * X2[q] + ((i == j) ? b[0] : 0.0);
      }
    memcpy(U, T, nn * sizeof(double));
  }
  /* (V - U) R = (V + U) */
  for (size_t q = 0; q < nn; q++) { T[q] = V[q] - U[q]; F[q] = V[q] + U[q]; }
  if (lu_solve(n, T, F) != 0) { rc = -4; goto done; }
  for (int k = 0; k < s; k++) { /* R <- R^2, s times */
    mat_mul(n, F, F, T); mult++;
    memcpy(F, T, nn * sizeof(double));
  }
done:
  if (n_mult) *n_mult = mult;
  free(X); free(X2); free(X4); free(X6); free(X8); free(U); free(V); free(T);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* Theorem 1 augmentation and Sec. 3.7 normalisation                          */
/* ------------------------------------------------------------------------- */
void or_normalisation(int64_t N, int p, const double *const *u, double *nu, double *mu) {
  /* Eqs. 48-49, R12: ||B||_1 = max_k sum_i |u_k,i| over k = 1..p */
  double nb = 0.0;
  for (int k = 1; k <= p; k++) {
    double s = 0.0;
    for (int64_t i = 0; i < N; i++) s += fabs(u[k][i]);
    if (s > nb) nb = s;
  }
  if (p == 0 || nb == 0.0) { *nu = 1.0; *mu = 1.0; return; }
  const int e = ceil_log2(nb);
  *nu = ldexp(1.0, -e);
  *mu = ldexp(1.0, e);
}

/* Alg. 2 lines 4-6.  B = [u_p, ..., u_1] (Thm 1) so column
 * c (0-based) of B is u_{p-c} and pairs with tail entry N+c (R14). */
void or_augmented_matvec(const or_operator *op, int64_t N, int p, const double *const *u,
                         double nu, const double *v, double *y) {
  or_apply(op, v, y);
  for (int c = 0; c < p; c++) {
    const double t = nu * v[N + c];
    const double *b = u[p - c];
    for (int64_t i = 0; i < N; i++) y[i] += b[i] * t;
  }
  for (int c = 0; c + 1 < p; c++) y[N + c] = v[N + c + 1];
  if (p > 0) y[N + p - 1] = 0.0;
}

static double dot(int64_t n, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
  return s;
}

/* Alg. 2 with window q (R23: ascending i, one MGS pass) and the
 * breakdown threshold R3.  V: ldv = N+p rows; H: ldh rows.  *j = completed
 * columns on entry and exit.  Returns 0, or OR_ERR_NONFINITE. */
static int iop_extend(const or_operator *op, int64_t N, int p, const double *const *u, double nu,
                      double *V, double *H, int ldh, int *j, int m, int q, int *happy,
                      double *y, int64_t *kv) {
  const int64_t ld = N + p;
  while (*j < m) {
    const int jj = ++(*j); /* line 3, 1-based */
    const double *vj = V + (size_t)(jj - 1) * ld;
    or_augmented_matvec(op, N, p, u, nu, vj, y); /* lines 4-6 */
    (*kv)++;
    const double c = sqrt(dot(ld, y, y));
    const int i0 = (jj - q + 1 > 1) ? jj - q + 1 : 1; /* line 7: max(1, j-1) for q = 2 */
    for (int i = i0; i <= jj; i++) {                    /* lines 7-10 */
      const double *vi = V + (size_t)(i - 1) * ld;
      const double h = dot(ld, vi, y);
      H[CM(i - 1, jj - 1, ldh)] = h;
      for (int64_t r = 0; r < ld; r++) y[r] -= h * vi[r];
    }
    const double s = sqrt(dot(ld, y, y)); /* line 11 */
    if (!isfinite(s) || !isfinite(c)) return OR_ERR_NONFINITE;
    const double thr = (1e-12 * c > 1e-14) ? 1e-12 * c : 1e-14;
    if (s <= thr) { *happy = 1; break; } /* lines 12-15, R3 */
    H[CM(jj, jj - 1, ldh)] = s;          /* line 16, R2: H(j+1, j) = s */
    double *vn = V + (size_t)jj * ld;
    for (int64_t r = 0; r < ld; r++) vn[r] = y[r] / s; /* line 17 */
  }
  return OR_OK;
}

int or_iop(const or_operator *op, int64_t N, int p, const double *const *u, double nu,
           const double *v0, int m, int q, double *V, double *H, int *happy) {
  const int64_t ld = N + p;
  double *y = malloc((size_t)ld * sizeof(double));
  if (!y) return -1;
  const double b = sqrt(dot(ld, v0, v0));
  for (int64_t r = 0; r < ld; r++) V[r] = v0[r] / b;
  memset(H, 0, sizeof(double) * (size_t)(m + 1) * m);
  int j = 0;
  int64_t kv = 0;
  *happy = 0;
  iop_extend(op, N, p, u, nu, V, H, m + 1, &j, m, q, happy, y, &kv);
  free(y);
  return j;
}

/* ------------------------------------------------------------------------- */
/* Alg. 4, Eqs. 43-46 with readings R4-R10.           */
/* ------------------------------------------------------------------------- */
int or_adapt(int happy, int accept, int j, int m, int m_min, int m_max, double tau,
             double omega, double t_now, double t_end, int hist_valid, double omega_old,
             double tau_old, int j_old, double *tau_new) {
  const double gamma = 0.9, gamma_max = 0.6, delta = 1.4; /* Alg. 4 l.2-3 */
  const double rem = accept ? t_end - (t_now + tau) : t_end - t_now; /* R8 */
  const double om = omega > 1e-300 ? omega : 1e-300;
  double ord = j / 4.0; /* R4/R5: q = m/4 - 1 => model exponent q+1 = j/4 */
  double kappa = 2.0;   /* P:502 "a default value kappa = 2" */
  if (hist_valid) {
    const double omo = omega_old > 1e-300 ? omega_old : 1e-300;
    if (j == j_old && tau != tau_old) { /* Eq. 43 read as omega ~ C tau^ord (R4) */
      const double o = log(om / omo) / log(tau / tau_old);
      if (isfinite(o) && o > 0.0) ord = o > 1.0 ? o : 1.0;
    } else if (j != j_old && tau == tau_old) { /* Eq. 45, R6 */
      double k = pow(om / omo, 1.0 / (double)(j_old - j));
      if (!(k >= 1.1)) k = 1.1;
      if (!(k <= 10.0)) k = 10.0;
      kappa = k;
    }
  }
  if (happy) { /* Alg. 4 l.4-8 */
    *tau_new = tau < rem ? tau : rem;
    return m;
  }
  if (j == m_max) {
    double t;
    if (omega > delta) { /* l.10-13, gamma_max */
      t = tau * pow(gamma_max / om, 1.0 / ord);
      if (t < tau / 5.0) t = tau / 5.0;
      *tau_new = rem < t ? rem : t;
      return j;
    }
    /* l.15, Sec. 3.6.1: Eq. 44 with gamma = 0.9, clipped to [tau/5, 5 tau] */
    t = tau * pow(gamma / om, 1.0 / ord);
    if (t > 5.0 * tau) t = 5.0 * tau;
    if (t < tau / 5.0) t = tau / 5.0;
    *tau_new = rem < t ? rem : t;
    return m;
  }
  /* l.18, Sec. 3.6.2: Eq. 46, clip -25% / +33% and [m_min, m_max] (R7) */
  const double x = (double)j + log(om / gamma) / log(kappa);
  int lo = (3 * j) / 4, hi = (4 * j + 2) / 3;
  if (lo < m_min) lo = m_min;
  if (hi > m_max) hi = m_max;
  if (lo > hi) lo = hi;
  int mn;
  if (x >= (double)hi) mn = hi;
  else if (x <= (double)lo) mn = lo;
  else mn = (int)ceil(x);
  if (mn < lo) mn = lo;
  if (mn > hi) mn = hi;
  *tau_new = tau < rem ? tau : rem;
  return mn;
}

/* ------------------------------------------------------------------------- */
/* Alg. 1 + Alg. 3                                    */
/* ------------------------------------------------------------------------- */
/* w = beta * V(1:N, 1:j) * f(1:j), Eq. 33 as used in Alg. 3 l.15, l.20 */
static void project(int64_t N, int64_t ld, int j, const double *V, const double *f, double beta,
                    double *w) {
  for (int64_t i = 0; i < N; i++) {
    double s = 0.0;
    for (int c = 0; c < j; c++) s += V[(size_t)c * ld + i] * f[c];
    w[i] = beta * s;
  }
}

/* the same projection, exported for the CPU-baseline timing sample (bench.py) */
void or_project(int64_t N, int64_t ld, int j, const double *V, const double *f, double beta, double *w) {
  project(N, ld, j, V, f, beta, w);
}

int or_kiops(const or_operator *op, int p, const double *const *u, int n_out, const double *T,
             double *const *w, const or_options *o, or_stats *st, or_trace_row *trace,
             int64_t trace_cap, int64_t *trace_len) {
  const int64_t N = or_n(op);
  /* validation, R21 */
  if (N < 1 || p < 0 || n_out < 1 || !o || !(o->tol > 0.0) || o->m_min < 1 || o->m_min > o->m_max ||
      o->m_max > 1024 || o->iop_q < 1 || o->max_attempts < 1)
    return OR_ERR_INVALID_ARG;
  for (int l = 0; l < n_out; l++)
    if (!isfinite(T[l]) || !(T[l] > 0.0) || (l > 0 && !(T[l] > T[l - 1]))) return OR_ERR_INVALID_ARG;

  const int m_max = o->m_max, ldh = m_max + 2;
  const int64_t ld = N + p;
  const double T_end = T[n_out - 1];
  or_stats S;
  memset(&S, 0, sizeof S);
  int64_t tl = 0;
  int rc = OR_OK;

  double *V = malloc((size_t)ld * (size_t)(m_max + 1) * sizeof(double));
  double *H = calloc((size_t)ldh * (size_t)(m_max + 1), sizeof(double));
  double *Ht = malloc((size_t)(m_max + 1) * (m_max + 1) * sizeof(double));
  double *F = malloc((size_t)(m_max + 1) * (m_max + 1) * sizeof(double));
  double *F2 = malloc((size_t)(m_max + 1) * (m_max + 1) * sizeof(double));
  double *y = malloc((size_t)ld * sizeof(double));
  double *wcur = malloc((size_t)N * sizeof(double));
  double *f1 = malloc((size_t)(m_max + 1) * sizeof(double));
  if (!V || !H || !Ht || !F || !F2 || !y || !wcur || !f1) { rc = OR_ERR_ALLOC; goto out; }

  /* Sec. 3.7: nu, mu (Eqs. 48-49) */
  double nu, mu;
  or_normalisation(N, p, u, &nu, &mu);
  S.nu = nu; S.mu = mu;

  double tau = T_end;                                                    /* Alg. 1 l.2 */
  int m = o->m_init < o->m_max ? o->m_init : o->m_max;                   /* l.3 */
  if (m < o->m_min) m = o->m_min;
  double T_now = 0.0;                                                    /* l.4 */
  int j = 0, l = 0, happy = 0;                                           /* l.5-6 (R20) */
  memcpy(wcur, u[0], (size_t)N * sizeof(double));                        /* l.8 */
  double beta = 0.0;
  int hist_valid = 0, j_old = 0;
  double omega_old = 0.0, tau_old = 0.0;
  int64_t attempt = 0;

  while (T_now < T_end) { /* l.9 */
    const int forced = attempt < o->n_forced;
    if (forced) {
      tau = o->forced_tau[attempt];
      m = o->forced_m[attempt];
      if (m < 1) m = 1;
      if (m > m_max) m = m_max;
    }
    /* O3.0 / R11: never step past T_end; the attempt that reaches it is final */
    const double rem0 = T_end - T_now;
    int final = 0;
    if (tau >= rem0) { tau = rem0; final = 1; }

    if (j == 0) { /* l.10-15: exact, mu-scaled tail (Eq. 47, R13, R14), v_1 = w/||w|| */
      for (int64_t i = 0; i < N; i++) V[i] = wcur[i];
      for (int c = 0; c < p; c++) {
        const int e = p - 1 - c; /* entry N+c holds T_now^e / e! */
        double t = 1.0;
        for (int r = 1; r <= e; r++) t = t * T_now / (double)r;
        V[N + c] = mu * t;
      }
      beta = sqrt(dot(ld, V, V));
      if (!isfinite(beta)) { rc = OR_ERR_NONFINITE; goto out; }
      if (beta == 0.0) { /* R27: zero start vector (p = 0, w = 0) => w stays 0 */
        for (; l < n_out; l++) memset(w[l], 0, (size_t)N * sizeof(double));
        T_now = T_end;
        l = n_out - 1;
        memset(wcur, 0, (size_t)N * sizeof(double));
        break;
      }
      for (int64_t i = 0; i < ld; i++) V[i] = V[i] / beta;
      memset(H, 0, sizeof(double) * (size_t)ldh * (m_max + 1)); /* l.12 */
      happy = 0;
      hist_valid = 0;
    }
    if (!happy) { /* l.16: Alg. 2 */
      rc = iop_extend(op, N, p, u, nu, V, H, ldh, &j, m, o->iop_q, &happy, y, &S.krylov_vectors);
      if (rc) goto out;
    }
    /* l.17-18 with R1: H~ = [[H(1:j,1:j), e_1],[0, 0]] (Eq. 37), F = exp(tau H~) */
    const int n1 = j + 1;
    memset(Ht, 0, sizeof(double) * (size_t)n1 * n1);
    for (int c = 0; c < j; c++)
      for (int r = 0; r < j; r++) Ht[CM(r, c, n1)] = H[CM(r, c, ldh)];
    Ht[CM(0, j, n1)] = 1.0;
    if (or_expm(n1, Ht, tau, F, NULL) != 0) { rc = OR_ERR_NONFINITE; goto out; }
    S.expm_calls++;
    /* l.19, Eqs. 36-38: eps = beta h_{j+1,j} |F(j, j+1)|; Eq. 39 omega */
    const double h_next = happy ? 0.0 : H[CM(j, j - 1, ldh)];
    double eps = 0.0, omega = 0.0;
    if (!happy) {
      eps = beta * h_next * fabs(F[CM(j - 1, j, n1)]);
      omega = T_end * eps / (tau * o->tol);
    }
    if (!isfinite(omega)) { rc = OR_ERR_NONFINITE; goto out; }
    const int accept = forced ? (o->forced_accept ? o->forced_accept[attempt] != 0 : 1)
                              : (omega <= 1.4); /* P:425, delta = 1.4, R10 */
    /* l.20-21: Alg. 4 */
    double tau_new = tau;
    int m_new = m;
    if (!forced)
      m_new = or_adapt(happy, accept, j, m, o->m_min, m_max, tau, omega, T_now, T_end, hist_valid,
                       omega_old, tau_old, j_old, &tau_new);
    if (trace && tl < trace_cap) {
      or_trace_row *r = &trace[tl];
      r->attempt = attempt; r->j = j; r->happy = happy; r->accept = accept; r->m_new = m_new;
      r->t_now = T_now; r->tau = tau; r->beta = beta; r->h_next = h_next; r->eps = eps;
      r->omega = omega; r->tau_new = tau_new;
    }
    tl++;
    if (accept) { /* l.22-25: Alg. 3 */
      const double T_next = T_now + tau;
      int n_tau = 0;
      for (int k = l; k < n_out; k++)
        if (fabs(T[k]) < fabs(T_next)) n_tau++; /* Alg. 3 l.6, strict (R16), all tasks (R15) */
      /* Saad's corrected scheme [46] (option): w = beta V_{j+1} exp(tau Hbar) e_1,
       * Hbar = [[H_j, 0], [h_{j+1,j} e_j^T, 0]], whose entry (j+1, 1) is h_{j+1,j} tau
       * e_j^T phi_1(tau H_j) e_1 = h_{j+1,j} F(j, j+1) of exp(tau H~) (Eq. 38): one more
       * basis vector, v_{j+1}, in the projection.  (No v_{j+1} after a happy breakdown.) */
      const int corr = o->corrected && !happy;
      const int jc = corr ? j + 1 : j;
      for (int k = 0; k < n_tau; k++) {
        const double tt = T[l + k] - T_now;              /* l.13 */
        if (corr) {                                       /* exp(tt H~), H~ as in l.17-18 (R1) */
          if (or_expm(n1, Ht, tt, F2, NULL) != 0) { rc = OR_ERR_NONFINITE; goto out; }
          for (int c = 0; c < j; c++) f1[c] = F2[CM(c, 0, n1)];
          f1[j] = h_next * F2[CM(j - 1, j, n1)];
        } else {
          for (int c = 0; c < j; c++)                     /* H(1:j,1:j) */
            for (int r = 0; r < j; r++) Ht[CM(r, c, j)] = H[CM(r, c, ldh)];
          if (or_expm(j, Ht, tt, F2, NULL) != 0) { rc = OR_ERR_NONFINITE; goto out; } /* l.14 */
          for (int c = 0; c < j; c++) f1[c] = F2[CM(c, 0, j)];
        }
        S.expm_calls++;
        project(N, ld, jc, V, f1, beta, w[l + k]);        /* l.15 */
      }
      l += n_tau;                                         /* l.17 */
      for (int c = 0; c < j; c++) f1[c] = F[CM(c, 0, n1)];
      if (corr) f1[j] = h_next * F[CM(j - 1, j, n1)];
      project(N, ld, jc, V, f1, beta, wcur);              /* l.20 */
      T_now = final ? T_end : T_next;                     /* l.24, R11 */
      j = 0;                                              /* l.25 */
      S.substeps++;
      if (happy) S.happy_breakdowns++;
      happy = 0;
      hist_valid = 0;
    } else { /* l.26-28: keep V, H (H~ was a copy, so "restore" is implicit, R1) */
      S.rejections++;
      hist_valid = 1;
      omega_old = omega; tau_old = tau; j_old = j;
    }
    tau = tau_new;
    m = m_new;
    attempt++;
    if (T_now < T_end && attempt >= o->max_attempts) { rc = OR_ERR_NO_CONVERGENCE; break; }
  }
  if (rc == OR_OK) {
    memcpy(w[l], wcur, (size_t)N * sizeof(double)); /* l.36 */
    if (o->task1)                                   /* l.31-35 */
      for (int k = 0; k < n_out; k++) {
        const double sc = pow(1.0 / T[k], (double)p);
        for (int64_t i = 0; i < N; i++) w[k][i] = w[k][i] * sc;
      }
  }
  S.final_m = m; /* R25 */
  S.t_reached = T_now;
out:
  if (st) *st = S;
  if (trace_len) *trace_len = tl;
  free(V); free(H); free(Ht); free(F); free(F2); free(y); free(wcur); free(f1);
  return rc;
}

/* Theorem 1 evaluated densely: e^{tau A~} [u_0; e_p]. */
int or_dense_phi_combination(const or_operator *op, int p, const double *const *u, double tau,
                             double *out) {
  const int64_t N = or_n(op);
  const int n = (int)(N + p);
  double *At = calloc((size_t)n * n, sizeof(double)), *F = malloc((size_t)n * n * sizeof(double));
  double *e = calloc((size_t)N, sizeof(double)), *col = malloc((size_t)N * sizeof(double));
  if (!At || !F || !e || !col) { free(At); free(F); free(e); free(col); return -1; }
  for (int64_t c = 0; c < N; c++) { /* A block, column by column */
    e[c] = 1.0;
    or_apply(op, e, col);
    e[c] = 0.0;
    for (int64_t r = 0; r < N; r++) At[CM(r, c, n)] = col[r];
  }
  for (int c = 0; c < p; c++) /* B = [u_p, ..., u_1] */
    for (int64_t r = 0; r < N; r++) At[CM(r, N + c, n)] = u[p - c][r];
  for (int c = 0; c + 1 < p; c++) At[CM(N + c, N + c + 1, n)] = 1.0; /* K: superdiagonal */
  int rc = or_expm(n, At, tau, F, NULL);
  if (rc == 0)
    for (int r = 0; r < n; r++) {
      double s = 0.0;
      for (int64_t c = 0; c < N; c++) s += F[CM(r, c, n)] * u[0][c];
      if (p > 0) s += F[CM(r, n - 1, n)]; /* e_p */
      out[r] = s;
    }
  free(At); free(F); free(e); free(col);
  return rc;
}
