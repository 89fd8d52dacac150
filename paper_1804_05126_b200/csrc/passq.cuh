// passq.cuh -- SURVEY 8(f) row f3: IOP windows q != 2 (1 <= q <= m_max, q = m_max is
// full Arnoldi) for every operator kind.  The tuned fused kernels of passes.cuh keep
// q = 2 (Alg. 2 as printed); this generic path follows the same lazy formulation with
// the window generalised, in four launches per Krylov vector:
//   k_q_form      x_k = r_{k-1}/s_{k-1} - sum_{i in W(k-1)} H(i,k-1) x_i/s_i   (pointwise)
//   k_q_apply     r_k = (A~ x_k)_top = A x_k + nu B t_k; partials of S = x_k.x_k, R = r_k.r_k
//   k_q_dots      grid (QG, q): partials of d_i = x_i.r_k and g_i = x_i.x_k, i in W(k)
//   k_q_finalize  one CTA: fixed-order reduction; sigma_k = sqrt(S) (the Alg. 2 l.11 norm
//                 of iteration k-1, tested by R3); the window's MGS coefficients in
//                 ascending i (Alg. 2 l.7-10, R23) from the dots and the Gram entries
//                 G(i,l) = x_i.x_l of earlier passes:
//                   H(i,k) = d_i/(s_i s_k) - sum_{l in W(k), l < i} H(l,k) G(i,l)/(s_i s_l)
//                 (= v_i . (y - sum_{l<i} H(l,k) v_l) with v = x/s, y = A~ v_k); the tail of
//                 x_{k+1} and the next formation coefficients.
// W(k) = {max(1, k-q+1), ..., k} (Alg. 2 l.7).  For q = 2 the formulas reduce to the
// fused kernels' (H(k-1,k) = E1/(s_{k-1}s_k), H(k,k) = E2/s_k^2 - H(k-1,k) G/(s_{k-1}s_k)).
#pragma once

#define QG 256  // x-blocks of k_q_apply / k_q_dots (partials per dot)

__device__ __forceinline__ long long qwrap(long long g, long long n) { return g < 0 ? g + n : (g >= n ? g - n : g); }

// (A x)_i for every operator kind (plain per-point evaluation)
__device__ __forceinline__ double q_apply_point(const KParams &P, const double *__restrict__ x, long long i) {
  if (P.kind == KIOPS_OP_CSR) {
    double a = 0.0;
    for (long long q = P.row_ptr[i]; q < P.row_ptr[i + 1]; q++) a = fma(P.vals[q], x[P.col_idx[q]], a);
    return a;
  }
  if (P.kind == KIOPS_OP_STENCIL3D7_VARKAPPA) {
    const long long nx = P.nx, ny = P.ny, nz = P.nz, nxy = nx * ny;
    const long long xi = i % nx, yi = (i / nx) % ny, zi = i / nxy, b = i - xi;
    const double *kp = P.kappa;
    const long long nb[6] = {b + qwrap(xi - 1, nx), b + qwrap(xi + 1, nx), i + (qwrap(yi - 1, ny) - yi) * nx,
                             i + (qwrap(yi + 1, ny) - yi) * nx, i + (qwrap(zi - 1, nz) - zi) * nxy,
                             i + (qwrap(zi + 1, nz) - zi) * nxy};
    const double xc = x[i], kc = kp[i];
    double ra = 0.0;
#pragma unroll
    for (int d = 0; d < 6; d++) ra = fma(kc + kp[nb[d]], x[nb[d]] - xc, ra);
    return 0.5 * P.inv_h2 * ra;
  }
  // 1D3 / 2D5: w5 = {W, E, S, N, C}
  const long long nx = P.nx, ny = P.ny, xi = i % nx, yi = i / nx, b = i - xi;
  const double d = P.diag ? P.diag[i] : 0.0;
  return P.w5[0] * x[b + qwrap(xi - 1, nx)] + P.w5[1] * x[b + qwrap(xi + 1, nx)] +
         P.w5[2] * x[xi + nx * qwrap(yi - 1, ny)] + P.w5[3] * x[xi + nx * qwrap(yi + 1, ny)] + (P.w5[4] + d) * x[i];
}

__device__ __forceinline__ const double *q_slot(const KParams &P, int k) {
  return (k == 1) ? P.st->x1 : P.V + (size_t)(k - 1) * (size_t)P.ldN;
}

__global__ void __launch_bounds__(256) k_q_form(KParams P) {
  pass_guard(P);
  const DevState *st = P.st;
  const int k = st->npass + 1;
  if (k < 2 || k > P.m_max + 1) return;
  const int w0 = max(1, k - P.q);  // W(k-1) = {max(1, k-q), ..., k-1}
  double *xk = P.V + (size_t)(k - 1) * (size_t)P.ldN;
  const double a0 = P.qa[0];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.N; i += (long long)gridDim.x * blockDim.x) {
    double x = a0 * P.r[i];
    for (int l = w0; l <= k - 1; l++) x -= P.qa[l] * q_slot(P, l)[i];
    xk[i] = x;
  }
}

__global__ void __launch_bounds__(256) k_q_apply(KParams P) {
  __shared__ double red[2 * 32];
  const DevState *st = P.st;
  const int k = st->npass + 1;
  if (k > P.m_max + 1) return;
  const double nu = st->nu;
  const double *xk = q_slot(P, k);
  double btc[KMAXP];
  const double *Bc[KMAXP];
  for (int c = 0; c < KMAXP; c++) {
    btc[c] = c < P.p ? nu * P.tails[k * KMAXP + c] : 0.0;
    Bc[c] = c < P.p ? P.call->u[P.p - c] : nullptr;
  }
  double v[2] = {0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.N; i += (long long)gridDim.x * blockDim.x) {
    double r = q_apply_point(P, xk, i);
    for (int c = 0; c < P.p; c++) r = fma(Bc[c][i], btc[c], r);
    P.r[i] = r;
    const double x = xk[i];
    v[0] = fma(x, x, v[0]);
    v[1] = fma(r, r, v[1]);
  }
  block_sum<2>(v, red);
  if (threadIdx.x == 0) {
    P.qpart[0 * QG + blockIdx.x] = v[0];
    P.qpart[1 * QG + blockIdx.x] = v[1];
  }
}

__global__ void __launch_bounds__(256) k_q_dots(KParams P) {
  __shared__ double red[2 * 32];
  const DevState *st = P.st;
  const int k = st->npass + 1;
  const int i = max(1, k - P.q + 1) + (int)blockIdx.y;  // window member
  if (k > P.m_max + 1 || i > k) return;
  const double *xi = q_slot(P, i), *xk = q_slot(P, k);
  double v[2] = {0.0, 0.0};
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < P.N; n += (long long)gridDim.x * blockDim.x) {
    const double a = xi[n];
    v[0] = fma(a, P.r[n], v[0]);
    v[1] = fma(a, xk[n], v[1]);
  }
  block_sum<2>(v, red);
  if (threadIdx.x == 0) {
    P.qpart[(2 + 2 * blockIdx.y) * QG + blockIdx.x] = v[0];
    P.qpart[(3 + 2 * blockIdx.y) * QG + blockIdx.x] = v[1];
  }
}

__global__ void __launch_bounds__(256) k_q_finalize(KParams P) {
  __shared__ double sums[2 * LDH + 2];
  DevState *st = P.st;
  const int k = st->npass + 1;
  if (k > P.m_max + 1) return;
  const int w0 = max(1, k - P.q + 1), nw = k - w0 + 1;  // W(k)
  // fixed-order reductions: one warp per value
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int d = warp; d < 2 + 2 * nw; d += nwarp) {
    double s = 0.0;
    for (int b = lane; b < QG; b += 32) s += P.qpart[d * QG + b];
    s = warp_sum(s);
    if (lane == 0) sums[d] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int p = P.p;
  const double *tk = P.tails + k * KMAXP;
  double Kt[KMAXP];
  for (int c = 0; c < KMAXP; c++) Kt[c] = (c + 1 < p) ? tk[c + 1] : 0.0;  // tail of A~ x_k: K t_k
  double S = sums[0], R = sums[1];
  for (int c = 0; c < p; c++) { S += tk[c] * tk[c]; R += Kt[c] * Kt[c]; }
  st->passes++;
  st->npass = k;
  st->ns_pass += gtimer() - st->t_pass0;
  if (st->status != 0) { set_cond(P, COND_INNER, 0u); return; }
  if (!isfinite(S) || !isfinite(R)) { st->status = KIOPS_ERR_NONFINITE; set_cond(P, COND_INNER, 0u); return; }
  const double sk = sqrt(S);
  double *H = P.H;
#define HH(i, j) H[((i)-1) + (size_t)((j)-1) * LDH]
#define GG(i, j) P.gram[((i)-1) + (size_t)((j)-1) * LDH]
  if (k == 1) {  // beta = ||x_1|| (Alg. 1 l.14)
    st->beta = sk;
    P.sig[1] = sk;
    P.R2[1] = R;
    if (sk == 0.0) { st->zero_start = 1; set_cond(P, COND_INNER, 0u); return; }
  } else {
    st->kv++;
    const double skm1 = P.sig[k - 1];
    const double cn = sqrt(P.R2[k - 1]) / skm1;   // ||A~ v_{k-1}|| before projection
    const double thr = fmax(1e-12 * cn, 1e-14);   // R3
    if (sk <= thr) { st->happy = 1; set_cond(P, COND_INNER, 0u); return; }
    HH(k, k - 1) = sk;  // Alg. 2 l.16 (R2)
    P.sig[k] = sk;
    P.R2[k] = R;
  }
  // window dots with the tails; Gram row k
  double d[LDH], g[LDH];
  for (int a = 0; a < nw; a++) {
    const int i = w0 + a;
    const double *ti = P.tails + i * KMAXP;
    double di = sums[2 + 2 * a], gi = sums[3 + 2 * a];
    for (int c = 0; c < p; c++) { di += ti[c] * Kt[c]; gi += ti[c] * tk[c]; }
    d[a] = di;
    g[a] = gi;
    if (i < k) GG(k, i) = gi;
  }
  // MGS in ascending i (R23): H(i,k) = d_i/(s_i s_k) - sum_{l<i} H(l,k) G(i,l)/(s_i s_l)
  double *tn = P.tails + (k + 1) * KMAXP;
  double tnv[KMAXP];
  for (int c = 0; c < KMAXP; c++) tnv[c] = (c < p) ? Kt[c] / sk : 0.0;
  double hcol[LDH];
  for (int a = 0; a < nw; a++) {
    const int i = w0 + a;
    const double si = P.sig[i];
    double h = d[a] / (si * sk);
    for (int b = 0; b < a; b++) {
      const int l = w0 + b;
      const double gil = (i == k) ? g[b] : GG(i, l);
      h -= hcol[b] * gil / (si * P.sig[l]);
    }
    hcol[a] = h;
    HH(i, k) = h;
    const double *ti = P.tails + i * KMAXP;
    for (int c = 0; c < p; c++) tnv[c] -= h * ti[c] / si;
  }
  for (int c = 0; c < p; c++) tn[c] = tnv[c];
  // formation coefficients of x_{k+1}
  P.qa[0] = 1.0 / sk;
  for (int a = 0; a < nw; a++) P.qa[w0 + a] = hcol[a] / P.sig[w0 + a];
  set_cond(P, COND_INNER, (k < st->m + 1) ? 1u : 0u);
#undef HH
#undef GG
}
