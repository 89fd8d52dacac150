// passes.cuh -- SURVEY 8(a) rows a1 (setup), a2-a4 (fused IOP passes) for the
// built-in operators.  sm_100a CUDA C++, fp64, memory-bound (no tensor cores).
//
// Every pass k (k = npass+1, 1-based) completes Alg. 2 iteration k-1 and
// starts iteration k:
//   1. form x_k = (A~ x_{k-1})_top/s_{k-1} - H(k-2,k-1) x_{k-2}/s_{k-2}
//                 - H(k-1,k-1) x_{k-1}/s_{k-1}                     (l.7-10; l.17 folded)
//   2. r_k = A x_k + nu B t_k  (Thm 1 block matvec, l.4-6)
//   3. block partials of S = x_k.x_k, G = x_{k-1}.x_k, E1 = x_{k-1}.r_k, E2 = x_k.r_k,
//      R = r_k.r_k, then a deterministic last-CTA grid reduction (pass_finalize)
//      writing s_k = sqrt(S) = H(k,k-1) (l.11, l.16), H(k-1,k) = E1/(s_{k-1}s_k),
//      H(k,k) = E2/s_k^2 - H(k-1,k) G/(s_{k-1}s_k) -- the MGS values of l.7-10 in
//      exact arithmetic -- the breakdown test of iteration k-1 (R3), and the tail
//      of x_{k+1} (p scalars).
// The kernels in use are LAZY: (A~ x_{k-1})_top = r_{k-1} is read from the previous
// pass's output (ping-pong buffers), so step 1 is pointwise and one stencil level
// is applied per pass; HBM per pass = (q+3+p+c) 8N (SURVEY 8(d) "design" bytes).
// k_pass_stencil (generic tile kernel for odd nx) instead recomputes A~ x_{k-1} on
// chip from a halo-2 tile ("look-ahead" form, (q+1+p+c) 8N).
#pragma once
#include <type_traits>

#include "kiops_internal.cuh"

// ---------------------------------------------------------------------------
// a1: Eqs. 48-49, R12: ||B||_1 = max_c sum_i |u_c,i|; nu = 2^-e,
// mu = 2^e, e = ceil(log2 ||B||_1); and the Alg. 1 l.2-8 initial state.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ceil_log2_exact(double x) {
  int e;
  double f = frexp(x, &e);
  return (f == 0.5) ? e - 1 : e;
}

__device__ void write_exact_tail(const KParams &P, double t_now, double mu, double *t1) {
  // Eq. 47 / Alg. 1 l.13 (R13, R14): entry N+c of x_1 = mu * T_now^e / e!, e = p-1-c
  for (int c = 0; c < P.p; c++) {
    const int e = P.p - 1 - c;
    double t = 1.0;
    for (int r = 1; r <= e; r++) t = t * t_now / (double)r;
    t1[c] = mu * t;
  }
}

// Row a1 / Alg. 1 l.8 in padded mode: copy u_0 into basis slot 1 (x_1 of the first
// substep), B's columns u_p .. u_1 and kappa into their slots, ghosts included (the
// periodic images).  Called from k_setup on every call (the operator's kappa may be
// rewritten by the caller between calls; a copy costs ~2 vectors of traffic).
__device__ __forceinline__ void pad_copies(const KParams &P) {
  const CallBlock *call = P.call;
  const int Xp = P.Xp, Yp = P.Yp, nx = (int)P.nx, ny = (int)P.ny;
  const long long Np = P.Np, ldN = P.ldN;
  const int p = P.p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < Np; i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / Xp;
    const int xp = (int)(i - row * Xp);
    const long long z = row / Yp;
    const int yp = (int)(row - z * Yp);
    int x = xp - 2, y = yp - 2;
    x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
    y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
    const long long src = x + (long long)nx * (y + (long long)ny * z);
#ifdef KIOPS_BOUNDS_CHECK
    assert(x >= 0 && x < nx && y >= 0 && y < ny && src < P.N);
#endif
    P.V[i] = __ldg(call->u[0] + src);
    for (int c = 0; c < p; c++) P.V[(size_t)(P.slot_B + c) * ldN + i] = __ldg(call->u[p - c] + src);
    P.V[(size_t)P.slot_kappa * ldN + i] = __ldg(P.kappa + src);
  }
}

__global__ void __launch_bounds__(256) k_setup(KParams P) {
  const CallBlock *call = P.call;
  const int p = P.p;
  if (P.padded) pad_copies(P);
  __shared__ double red[KMAXP * 32];
  double v[KMAXP];
#pragma unroll
  for (int c = 0; c < KMAXP; c++) v[c] = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.N;
       i += (long long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < KMAXP; c++)
      if (c < p) v[c] += fabs(call->u[c + 1][i]);
  }
  block_sum<KMAXP>(v, red);
  if (threadIdx.x == 0)
    for (int c = 0; c < p; c++) P.npart[c * P.grid_max + blockIdx.x] = v[c];
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(&P.st->ticket2, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // column sums in fixed block order
  double cs[KMAXP];
#pragma unroll
  for (int c = 0; c < KMAXP; c++) {
    double s = 0.0;
    if (c < p)
      for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s += __ldcg(&P.npart[c * P.grid_max + b]);
    cs[c] = s;
  }
  block_sum<KMAXP>(cs, red);
  if (threadIdx.x != 0) return;
  DevState *st = P.st;
  st->ticket2 = 0;
  double nb = 0.0;
  for (int c = 0; c < p; c++) nb = cs[c] > nb ? cs[c] : nb;
  double nu = 1.0, mu = 1.0;
  if (p > 0 && nb > 0.0) {
    const int e = ceil_log2_exact(nb);
    nu = ldexp(1.0, -e);
    mu = ldexp(1.0, e);
  }
  st->nu = nu;
  st->mu = mu;
  const int n_out = call->n_out;
  st->t_end = call->T[n_out - 1];
  st->tau = st->t_end;                                     // Alg. 1 l.2
  const int m0 = call->m_init > 0 ? call->m_init : P.m_init;  // (warm start: kiops_set_m_init)
  int m = m0 < P.m_max ? m0 : P.m_max;                     // l.3
  st->m = m < P.m_min ? P.m_min : m;
  if (call->n_forced > 0) {
    st->tau = call->forced_tau[0];
    int fm = call->forced_m[0];
    st->m = fm < 1 ? 1 : (fm > P.m_max ? P.m_max : fm);
  }
  st->t_now = 0.0;                                         // l.4
  st->npass = 0;                                           // l.5 (j = npass - 1)
  st->l = 0;                                               // l.6
  st->happy = 0;
  st->hist_valid = 0;
  st->status = 0;
  st->zero_start = 0;
  st->accept = 0;
  st->x1 = P.padded ? P.V : call->u[0];                   // l.8 (padded: u_0 copied to slot 1)
  st->attempt = st->substeps = st->rejections = st->kv = st->expm_calls = st->passes = 0;
  st->happy_count = 0;
  st->final_m = st->m;
  st->ticket = 0;
  st->launches = 0;
  st->ns_pass = st->ns_ctrl = st->ns_gemv = st->ns_expm = 0;
  st->gemv_ticket = 0;
  write_exact_tail(P, 0.0, mu, P.tails + 1 * KMAXP);       // t_1 at T_now = 0
  set_cond(P, COND_OUTER, 1u);
  set_cond(P, COND_INNER, 1u);
  set_cond(P, COND_ACCEPT, 0u);
}

// ---------------------------------------------------------------------------
// Pass prologue: per-pass scalars (identical in every CTA).
// ---------------------------------------------------------------------------
struct PassScalars {
  int k;
  const double *xprev, *xpp;  // x_{k-1}, x_{k-2} (xpp may be NULL)
  double *xout;               // x_k destination (NULL for k = 1)
  double a0, a1, a2;          // x_k = a0 z - a2 x_{k-2} - a1 x_{k-1},  z = (A~ x_{k-1})_top
  double btp[KMAXP];          // nu * t_{k-1}
  double btc[KMAXP];          // nu * t_k
  const double *B[KMAXP];     // column c of B = u_{p-c} (Thm 1, R14)
};

// Alg. 2 l.7-10 quotients of the lazy pass's finalisation as products with the
// reciprocals is = 1/s_k, ism1 = 1/s_{k-1} (the same values in exact arithmetic as
// E1/(s_{k-1} s_k), E2/s_k^2 - h1 G/(s_{k-1} s_k), ...).  Explicit _rn operations (no
// FMA contraction): pass_finalize and the persistent loop's finalize_warp must round
// identically.
__device__ __forceinline__ double fin_h11(double E2, double is) { return __dmul_rn(__dmul_rn(E2, is), is); }
__device__ __forceinline__ double fin_h1(double E1, double ism1, double is) { return __dmul_rn(__dmul_rn(E1, ism1), is); }
__device__ __forceinline__ double fin_h2(double E2, double G, double h1, double ism1, double is) {
  return __dsub_rn(__dmul_rn(__dmul_rn(E2, is), is), __dmul_rn(__dmul_rn(__dmul_rn(h1, G), ism1), is));
}
// The p-entry tails' share of the five dots of pass k (x_k = [top; t_k], A~ x_k tail =
// K t_k): S_t = t_k.t_k, G_t = t_{k-1}.t_k, E1_t = t_{k-1}.K t_k, E2_t = t_k.K t_k,
// R_t = |K t_k|^2 (G_t, E1_t for k >= 2 only), summed apart from the grid-reduced top
// parts and added once (S = S_top + S_t, ...).  They depend only on tails known when
// pass k starts, so the persistent loop computes them during the pass body, off the
// finalisation chain; pass_finalize uses the same order.
__device__ __forceinline__ void tail_dots(int k, int p, const double *tk, const double *tkm1, double (&t)[NDOT]) {
#pragma unroll
  for (int q = 0; q < NDOT; q++) t[q] = 0.0;
#pragma unroll
  for (int c = 0; c < KMAXP; c++)
    if (c < p) {
      const double tkc = tk[c], ktc = (c + 1 < p) ? tk[c + 1 < KMAXP ? c + 1 : 0] : 0.0;
      t[0] = __fma_rn(tkc, tkc, t[0]);
      t[4] = __fma_rn(ktc, ktc, t[4]);
      t[3] = __fma_rn(tkc, ktc, t[3]);
      if (k >= 2) {
        t[1] = __fma_rn(tkm1[c], tkc, t[1]);
        t[2] = __fma_rn(tkm1[c], ktc, t[2]);
      }
    }
}

// tail of x_{k+1} (unnormalised tails, Thm 1): (K t_k / s_k - h1 t_{k-1} / s_{k-1}) - h2 t_k / s_k
__device__ __forceinline__ double fin_tail(double ktc, double tkm1c, double tkc, double h1, double h2, double ism1,
                                           double is) {
  return __dsub_rn(__dsub_rn(__dmul_rn(ktc, is), __dmul_rn(__dmul_rn(h1, tkm1c), ism1)), __dmul_rn(__dmul_rn(h2, tkc), is));
}
__device__ __forceinline__ double fin_tail1(double ktc, double tkc, double h11, double is) {
  return __dsub_rn(__dmul_rn(ktc, is), __dmul_rn(__dmul_rn(h11, tkc), is));
}

// RECIP = false (CSR path): the division form of the same quotients, kept for the
// per-pass CSR kernels, whose last-CTA finalisation is off the critical path: the
// reciprocal form changed the compiler's schedule of the inlined SELL SpMV loop
// (62 -> 48 registers, fewer gathers in flight) and cost 40% per launch at config 5.
template <bool RECIP = true>
__device__ __forceinline__ void load_pass_scalars(const KParams &P, PassScalars &s) {
  const DevState *st = P.st;
  const int k = st->npass + 1;
  s.k = (k > P.m_max + 1) ? 0 : k;  // 0 => out-of-range pass: every thread returns
  if (s.k == 0) return;
  const double nu = st->nu;
  const double *H = P.H;
  for (int c = 0; c < KMAXP; c++) s.B[c] = c < P.p ? P.call->u[P.p - c] : nullptr;
  if (k == 1) {  // x_1 is the substep's start vector: no formation
    s.xprev = st->x1;
    s.xpp = nullptr;
    s.xout = nullptr;
    s.a0 = 0.0; s.a1 = -1.0; s.a2 = 0.0;
    for (int c = 0; c < KMAXP; c++) { s.btp[c] = 0.0; s.btc[c] = c < P.p ? nu * P.tails[1 * KMAXP + c] : 0.0; }
    return;
  }
  s.xprev = slot_ptr(P, k - 1);
  s.xpp = (k >= 3) ? slot_ptr(P, k - 2) : nullptr;
  s.xout = P.V + (size_t)(k - 1) * (size_t)P.ldN;
  const double skm1 = P.sig[k - 1];
  s.a0 = 1.0 / skm1;
  if (RECIP) {
    s.a1 = __dmul_rn(H[(k - 2) + (size_t)(k - 2) * LDH], s.a0);                              // H(k-1,k-1)/s_{k-1}
    s.a2 = (k >= 3) ? __dmul_rn(H[(k - 3) + (size_t)(k - 2) * LDH], 1.0 / P.sig[k - 2]) : 0.0;  // H(k-2,k-1)/s_{k-2}
  } else {
    s.a1 = H[(k - 2) + (size_t)(k - 2) * LDH] / skm1;
    s.a2 = (k >= 3) ? H[(k - 3) + (size_t)(k - 2) * LDH] / P.sig[k - 2] : 0.0;
  }
  for (int c = 0; c < KMAXP; c++) {
    s.btp[c] = c < P.p ? nu * P.tails[(k - 1) * KMAXP + c] : 0.0;
    s.btc[c] = c < P.p ? nu * P.tails[k * KMAXP + c] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Deterministic last-CTA finalisation of pass k (all threads of the last CTA).
// ---------------------------------------------------------------------------
template <bool RECIP = true>
__device__ void pass_finalize(const KParams &P, int k, int nblocks) {
  __shared__ double red[NDOT * 32];
  double v[NDOT];
#pragma unroll
  for (int q = 0; q < NDOT; q++) v[q] = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
#pragma unroll
    for (int q = 0; q < NDOT; q++) v[q] += __ldcg(&P.partials[q * P.grid_max + b]);
  block_sum<NDOT>(v, red);
  if (threadIdx.x != 0) return;
  DevState *st = P.st;
  st->ticket = 0;
  const int p = P.p;
  const double *tk = P.tails + k * KMAXP;
  const double *tkm1 = P.tails + (k - 1) * KMAXP;
  double Kt[KMAXP];
  for (int c = 0; c < p; c++) Kt[c] = (c + 1 < p) ? tk[c + 1] : 0.0;  // tail of A~ x_k: K t_k (Alg. 2 l.5-6)
  double S = v[0], G = v[1], E1 = v[2], E2 = v[3], R = v[4];
  if (RECIP) {  // same order as the persistent loop's finalize_warp
    double t[NDOT];
    tail_dots(k, p, tk, tkm1, t);
    S = __dadd_rn(S, t[0]);
    G = __dadd_rn(G, t[1]);
    E1 = __dadd_rn(E1, t[2]);
    E2 = __dadd_rn(E2, t[3]);
    R = __dadd_rn(R, t[4]);
  } else {
    for (int c = 0; c < p; c++) {
      S += tk[c] * tk[c];
      R += Kt[c] * Kt[c];
      E2 += tk[c] * Kt[c];
      if (k >= 2) { G += tkm1[c] * tk[c]; E1 += tkm1[c] * Kt[c]; }
    }
  }
  st->passes++;
  st->npass = k;
  st->ns_pass += gtimer() - st->t_pass0;
  if (st->status != 0) {
    set_cond(P, COND_INNER, 0u);
    return;
  }
  if (!isfinite(S) || !isfinite(G) || !isfinite(E1) || !isfinite(E2) || !isfinite(R)) {
    st->status = KIOPS_ERR_NONFINITE;  // R22
    set_cond(P, COND_INNER, 0u);
    return;
  }
  const double sk = sqrt(S);
  double *H = P.H;
#define HH(i, j) H[((i)-1) + (size_t)((j)-1) * LDH]
  double *tn = P.tails + (k + 1) * KMAXP;  // tail of x_{k+1}
  if (k == 1) {  // beta = ||x_1|| (Alg. 1 l.14)
    st->beta = sk;
    P.sig[1] = sk;
    P.R2[1] = R;
    if (sk == 0.0) {  // R27
      st->zero_start = 1;
      set_cond(P, COND_INNER, 0u);
      return;
    }
    if (RECIP) {
      const double is = 1.0 / sk;
      const double h11 = fin_h11(E2, is);
      HH(1, 1) = h11;
      for (int c = 0; c < p; c++) tn[c] = fin_tail1(Kt[c], tk[c], h11, is);
    } else {
      const double h11 = E2 / (sk * sk);
      HH(1, 1) = h11;
      for (int c = 0; c < p; c++) tn[c] = Kt[c] / sk - h11 * tk[c] / sk;
    }
    set_cond(P, COND_INNER, (1 < st->m + 1) ? 1u : 0u);
    return;
  }
  // k >= 2 closes Alg. 2 iteration k-1
  st->kv++;
  const double skm1 = P.sig[k - 1];
  const double cn = sqrt(P.R2[k - 1]) / skm1;  // ||A~ v_{k-1}|| before projection
  const double thr = fmax(1e-12 * cn, 1e-14);  // R3
  if (sk <= thr) {                             // Alg. 2 l.12-15
    st->happy = 1;
    set_cond(P, COND_INNER, 0u);
    return;
  }
  HH(k, k - 1) = sk;  // l.16 (R2)
  P.sig[k] = sk;
  P.R2[k] = R;
  if (RECIP) {
    const double is = 1.0 / sk, ism1 = 1.0 / skm1;
    const double h1 = fin_h1(E1, ism1, is);
    const double h2 = fin_h2(E2, G, h1, ism1, is);
    HH(k - 1, k) = h1;
    HH(k, k) = h2;
    for (int c = 0; c < p; c++) tn[c] = fin_tail(Kt[c], tkm1[c], tk[c], h1, h2, ism1, is);
  } else {
    const double h1 = E1 / (skm1 * sk);
    const double h2 = E2 / (sk * sk) - h1 * G / (skm1 * sk);
    HH(k - 1, k) = h1;
    HH(k, k) = h2;
    for (int c = 0; c < p; c++) tn[c] = Kt[c] / sk - h1 * tkm1[c] / skm1 - h2 * tk[c] / sk;
  }
  set_cond(P, COND_INNER, (k < st->m + 1) ? 1u : 0u);
#undef HH
}

// write this CTA's partials, detect the last CTA, finalize.
template <bool RECIP = true>
__device__ __forceinline__ void pass_epilogue(const KParams &P, int k, double (&v)[NDOT]) {
  __shared__ double red[NDOT * 32];
  __shared__ bool last;
  block_sum<NDOT>(v, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NDOT; q++) P.partials[q * P.grid_max + blockIdx.x] = v[q];
    __threadfence();
    last = (atomicAdd(&P.st->ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    pass_finalize<RECIP>(P, k, gridDim.x);
  }
}

// ---------------------------------------------------------------------------
// Stencil passes: tile + halo staged in shared memory (v1 generic tile kernel).
// DIM = 1, 2, 3.  Tile TX x TY x TZ interior points; x_{k-1} (and kappa) staged on
// the halo-2 region, x_k formed on the halo-1 region, r on the interior.
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long wrapc(long long g, long long n) {
  g %= n;
  return g < 0 ? g + n : g;
}

template <int DIM, int TX, int TY, int TZ>
struct TileGeo {
  static constexpr int HX = TX + 4, HY = DIM >= 2 ? TY + 4 : 1, HZ = DIM >= 3 ? TZ + 4 : 1;
  static constexpr int GX = TX + 2, GY = DIM >= 2 ? TY + 2 : 1, GZ = DIM >= 3 ? TZ + 2 : 1;
  static constexpr int H2 = HX * HY * HZ, H1 = GX * GY * GZ, IN = TX * TY * TZ;
  static constexpr int OY = DIM >= 2 ? 1 : 0, OZ = DIM >= 3 ? 1 : 0;  // halo offsets per ring
};

template <int DIM>
__device__ __forceinline__ double stencil_at(const KParams &P, const double *s, const double *kap, int e,
                                             int sy, int sz, double d) {
  if (DIM == 1) {
    return P.w[0] * s[e - 1] + P.w[1] * s[e] + P.w[2] * s[e + 1] + d * s[e];
  } else if (DIM == 2) {
    return P.w[0] * s[e - 1] + P.w[1] * s[e + 1] + P.w[2] * s[e - sy] + P.w[3] * s[e + sy] +
           P.w[4] * s[e] + d * s[e];
  } else {
    const double xc = s[e], kc = kap[e];
    double acc = 0.5 * (kc + kap[e - 1]) * (s[e - 1] - xc);
    acc += 0.5 * (kc + kap[e + 1]) * (s[e + 1] - xc);
    acc += 0.5 * (kc + kap[e - sy]) * (s[e - sy] - xc);
    acc += 0.5 * (kc + kap[e + sy]) * (s[e + sy] - xc);
    acc += 0.5 * (kc + kap[e - sz]) * (s[e - sz] - xc);
    acc += 0.5 * (kc + kap[e + sz]) * (s[e + sz] - xc);
    return acc * P.inv_h2;
  }
}

template <int DIM, int TX, int TY, int TZ>
__global__ void __launch_bounds__(256) k_pass_stencil(KParams P) {
  using G = TileGeo<DIM, TX, TY, TZ>;
  extern __shared__ double smem[];
  double *sX1 = smem;                                  // x_{k-1} on halo-2 region
  double *sK = sX1 + G::H2;                            // kappa on halo-2 (3D) / diag on halo-1 (1D, 2D)
  double *sXK = sK + (DIM == 3 ? G::H2 : G::H1);       // x_k on halo-1 region
  double *sBT = sXK + G::H1;                           // nu B t_k on the interior

  __shared__ PassScalars S;
  pass_guard(P);
  if (threadIdx.x == 0) load_pass_scalars(P, S);
  __syncthreads();
  if (S.k == 0) return;
  const int p = P.p;
  const long long nx = P.nx, ny = P.ny, nz = P.nz;
  const long long ntx = (nx + TX - 1) / TX, nty = DIM >= 2 ? (ny + TY - 1) / TY : 1;
  const long long b = blockIdx.x;
  const long long ox = (b % ntx) * TX, oy = DIM >= 2 ? ((b / ntx) % nty) * TY : 0,
                  oz = DIM >= 3 ? (b / (ntx * nty)) * TZ : 0;
  const double *xprev = S.xprev;

  // stage 1: x_{k-1} (and kappa) on the halo-2 region
  for (int e = threadIdx.x; e < G::H2; e += blockDim.x) {
    const int a = e % G::HX, bb = (e / G::HX) % G::HY, c = e / (G::HX * G::HY);
    const long long gx = wrapc(ox + a - 2, nx);
    const long long gy = DIM >= 2 ? wrapc(oy + bb - 2, ny) : 0;
    const long long gz = DIM >= 3 ? wrapc(oz + c - 2, nz) : 0;
    const long long g = gx + nx * (gy + ny * gz);
    sX1[e] = xprev[g];
    if (DIM == 3) sK[e] = P.kappa[g];
  }
  __syncthreads();

  // stage 2: x_k on the halo-1 region (Alg. 2 l.4-10 of iteration k-1)
  for (int e = threadIdx.x; e < G::H1; e += blockDim.x) {
    const int a = e % G::GX, bb = (e / G::GX) % G::GY, c = e / (G::GX * G::GY);
    const long long gx = wrapc(ox + a - 1, nx);
    const long long gy = DIM >= 2 ? wrapc(oy + bb - 1, ny) : 0;
    const long long gz = DIM >= 3 ? wrapc(oz + c - 1, nz) : 0;
    const long long g = gx + nx * (gy + ny * gz);
    const int e2 = (a + 1) + G::HX * ((bb + G::OY) + G::HY * (c + G::OZ));
    double d = 0.0;
    if (DIM != 3) {
      d = P.diag ? P.diag[g] : 0.0;
      sK[e] = d;
    }
    double z = stencil_at<DIM>(P, sX1, sK, e2, G::HX, G::HX * G::HY, d);
    double bc = 0.0;
#pragma unroll
    for (int q = 0; q < KMAXP; q++)
      if (q < p) {
        const double bv = S.B[q][g];
        z += bv * S.btp[q];
        bc += bv * S.btc[q];
      }
    double xk = S.a0 * z - S.a1 * sX1[e2];
    if (S.xpp) xk -= S.a2 * S.xpp[g];
    sXK[e] = xk;
    const bool inner = (a >= 1 && a <= TX) && (DIM < 2 || (bb >= 1 && bb <= TY)) && (DIM < 3 || (c >= 1 && c <= TZ));
    if (inner) sBT[(a - 1) + TX * ((bb - G::OY) + TY * (c - G::OZ))] = bc;
  }
  __syncthreads();

  // stage 3: r = A~ x_k on the interior, 5 partial dots, store x_k
  double v[NDOT] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int e = threadIdx.x; e < G::IN; e += blockDim.x) {
    const int a = e % TX, bb = (e / TX) % TY, c = e / (TX * TY);
    const long long gx = ox + a, gy = oy + bb, gz = oz + c;
    if (gx >= nx || (DIM >= 2 && gy >= ny) || (DIM >= 3 && gz >= nz)) continue;
    const int e1 = (a + 1) + G::GX * ((bb + G::OY) + G::GY * (c + G::OZ));
    const int e2 = (a + 2) + G::HX * ((bb + 2 * G::OY) + G::HY * (c + 2 * G::OZ));
    const double xk = sXK[e1];
    double d = 0.0;
    if (DIM != 3) d = sK[e1];
    double r;
    if (DIM == 3) {
      // kappa of the interior point and neighbours from the halo-2 kappa tile
      const double *kap = sK;
      const int sy2 = G::HX, sz2 = G::HX * G::HY, sy1 = G::GX, sz1 = G::GX * G::GY;
      const double kc = kap[e2];
      r = 0.5 * (kc + kap[e2 - 1]) * (sXK[e1 - 1] - xk) + 0.5 * (kc + kap[e2 + 1]) * (sXK[e1 + 1] - xk) +
          0.5 * (kc + kap[e2 - sy2]) * (sXK[e1 - sy1] - xk) + 0.5 * (kc + kap[e2 + sy2]) * (sXK[e1 + sy1] - xk) +
          0.5 * (kc + kap[e2 - sz2]) * (sXK[e1 - sz1] - xk) + 0.5 * (kc + kap[e2 + sz2]) * (sXK[e1 + sz1] - xk);
      r *= P.inv_h2;
    } else {
      r = stencil_at<DIM>(P, sXK, nullptr, e1, G::GX, G::GX * G::GY, d);
    }
    r += sBT[e];
    const double xm = sX1[e2];
    v[0] += xk * xk;
    v[1] += xm * xk;
    v[2] += xm * r;
    v[3] += xk * r;
    v[4] += r * r;
    if (S.xout) S.xout[gx + nx * (gy + ny * gz)] = xk;
  }
  pass_epilogue(P, S.k, v);
}

template <int DIM, int TX, int TY, int TZ>
constexpr size_t stencil_smem_bytes() {
  using G = TileGeo<DIM, TX, TY, TZ>;
  return sizeof(double) * (size_t)(G::H2 + (DIM == 3 ? G::H2 : G::H1) + G::H1 + G::IN);
}

// ---------------------------------------------------------------------------
// CSR split form: (a) pointwise formation of x_k from r = A~ x_{k-1}, (b) SpMV with
// 8 lanes per row + the 5 dots.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_csr_form(KParams P) {
  __shared__ PassScalars S;
  if (threadIdx.x == 0 && blockIdx.x == 0) P.st->t_pass0 = gtimer();
  if (threadIdx.x == 0) load_pass_scalars<false>(P, S);
  __syncthreads();
  if (S.k <= 1) return;
  const double *r = P.r;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.N;
       i += (long long)gridDim.x * blockDim.x) {
    double xk = S.a0 * r[i] - S.a1 * S.xprev[i];
    if (S.xpp) xk -= S.a2 * S.xpp[i];
    S.xout[i] = xk;
  }
}


__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------------------
// 3D variable-kappa pass, LAZY form (SURVEY 8(a) a3 "lazy normalisation"):
// pass k forms x_k POINTWISE from the stored r_{k-1} = A~ x_{k-1} (ping-pong r
// buffers), x_{k-1} and x_{k-2}, then applies A~ once to x_k:
//     x_k = r_{k-1}/s_{k-1} - H(k-2,k-1) x_{k-2}/s_{k-2} - H(k-1,k-1) x_{k-1}/s_{k-1}
//     r_k = A x_k + nu B t_k                                  (stored for pass k+1)
// HBM per pass: read r_{k-1}, x_{k-1}, x_{k-2}, kappa, B; write x_k, r_k
// ((q+3+p+c) 8N, two vectors above the minimum) with ONE stencil level and a small
// per-thread state.  One thread per halo-1 point of a TX x TY column tile marches a
// chunk of ZC planes; x_k and kappa planes go through 2-plane shared rings,
// z-neighbours stay in registers, operands are prefetched one plane ahead.
// ---------------------------------------------------------------------------
template <int TX, int TY, int PM>
struct Lazy3 {
  static constexpr int GX = TX + 2, GY = TY + 2, S1 = GX * GY;
  static constexpr int NT = (S1 + 31) / 32 * 32;
  static constexpr int D = 2, RD = D + 1;          // operand planes in flight, private ring depth
  static constexpr int NOP = 4 + PM;               // r, x_{k-1}, x_{k-2}, kappa, B_0..B_{PM-1}
  static constexpr size_t smem_doubles = 4 * (size_t)NT + (size_t)RD * NOP * NT;
};

template <int TX, int TY, int ZC, int PM, int MINB>
__global__ void __launch_bounds__(Lazy3<TX, TY, PM>::NT, MINB) k_pass_3d_lazy(KParams P) {
  using M = Lazy3<TX, TY, PM>;
  constexpr int NT = M::NT, GX = M::GX, S1 = M::S1, D = M::D, RD = M::RD, NOP = M::NOP;
  extern __shared__ double smem[];
  double *sXK = smem;            // 2 x NT  x_k planes (shared)
  double *sKP = smem + 2 * NT;   // 2 x NT  kappa planes (shared)
  double *sOp = smem + 4 * NT;   // RD x NOP x NT  thread-private operand ring (cp.async)

  __shared__ PassScalars S;
  pass_guard(P);
  if (threadIdx.x == 0) load_pass_scalars(P, S);
  __syncthreads();
  if (S.k == 0) return;
  const int p = P.p, k = S.k;
  const long long nx = P.nx, ny = P.ny, nz = P.nz, nxy = nx * ny;
  const long long ntx = (nx + TX - 1) / TX, nty = (ny + TY - 1) / TY;
  const long long bidx = blockIdx.x;
  const long long ox = (bidx % ntx) * TX, oy = ((bidx / ntx) % nty) * TY;
  const long long z0 = (bidx / (ntx * nty)) * ZC;
  const long long z1 = (z0 + ZC < nz) ? z0 + ZC : nz;
  const int nzc = (int)(z1 - z0);
  const int t = threadIdx.x;
  const bool act = t < S1;
  const int fa = t % GX, fb = t / GX;
  const int o1 = act ? (int)(wrapc(ox + fa - 1, nx) + nx * wrapc(oy + fb - 1, ny)) : 0;
  const bool inner = act && fa >= 1 && fa <= TX && fb >= 1 && fb <= TY && (ox + fa - 1) < nx && (oy + fb - 1) < ny;
  const bool use_r = k >= 2, use_pp = S.xpp != nullptr;
  const int oo = (int)((ox + fa - 1) + nx * (oy + fb - 1));

  auto znext = [&](long long zo) { const long long n = zo + nxy; return n == nz * nxy ? 0 : n; };
  long long zoL = wrapc(z0 - 1, nz) * nxy;  // next operand plane to copy
  auto issue = [&](int slot) {
    if (act) {
      double *d = sOp + slot * NOP * NT + t;
      const long long g = zoL + o1;
      if (use_r) cp_async8(d, P.r + (size_t)((k - 1) & 1) * (size_t)P.ldN + g);
      cp_async8(d + NT, S.xprev + g);
      if (use_pp) cp_async8(d + 2 * NT, S.xpp + g);
      cp_async8(d + 3 * NT, P.kappa + g);
      if (inner)
#pragma unroll
        for (int c = 0; c < PM; c++)
          if (c < p) cp_async8(d + (4 + c) * NT, S.B[c] + g);
    }
    zoL = znext(zoL);
  };
  // plane zf = z0 - 1 + i ; x_k formed for planes z0-1 .. z1 (own column), output z0 .. z1-1
  for (int q = 0; q < D; q++) {
    issue(q);
    cp_async_commit();
  }
  double xk_m = 0.0, xk_0 = 0.0, k_m = 0.0, k_0 = 0.0, xm_0 = 0.0, bt_0 = 0.0;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, v4 = 0.0;
  long long zo_out = z0 * nxy;
  int rs = 0, ri = D;  // private ring: slot read this plane, slot issued this plane
  for (int i = 0; i <= nzc + 1; i++) {
    if (i + D <= nzc + 1) issue(ri);
    cp_async_commit();
    cp_async_wait<D>();  // this thread's copies of plane i have landed
    const double *o = sOp + rs * NOP * NT + t;
    const double xm = o[NT], kc_p = o[3 * NT];
    double xk_p = xm;
    if (use_r) xk_p = S.a0 * o[0] - S.a1 * xm - (use_pp ? S.a2 * o[2 * NT] : 0.0);
    double bt = 0.0;
    if (inner)
#pragma unroll
      for (int c = 0; c < PM; c++)
        if (c < p) bt = fma(o[(4 + c) * NT], S.btc[c], bt);
    __syncthreads();  // every thread finished the output that read slot (i & 1)
    sXK[(i & 1) * NT + t] = xk_p;
    sKP[(i & 1) * NT + t] = kc_p;
    // output plane z = zf - 1 (its in-plane x_k / kappa were published last iteration)
    if (i >= 2 && inner) {
      const double *X0 = sXK + ((i + 1) & 1) * NT, *K0 = sKP + ((i + 1) & 1) * NT;
      const double kc = k_0, xc = xk_0;
      double rx = (kc + K0[t - 1]) * (X0[t - 1] - xc);
      double ry = (kc + K0[t + 1]) * (X0[t + 1] - xc);
      rx = fma(kc + K0[t - GX], X0[t - GX] - xc, rx);
      ry = fma(kc + K0[t + GX], X0[t + GX] - xc, ry);
      rx = fma(kc + k_m, xk_m - xc, rx);
      ry = fma(kc + kc_p, xk_p - xc, ry);
      const double r = fma(rx + ry, 0.5 * P.inv_h2, bt_0);
      v0 = fma(xc, xc, v0);
      v1 = fma(xm_0, xc, v1);
      v2 = fma(xm_0, r, v2);
      v3 = fma(xc, r, v3);
      v4 = fma(r, r, v4);
      if (S.xout) S.xout[zo_out + oo] = xc;
      P.r[(size_t)(k & 1) * (size_t)P.ldN + zo_out + oo] = r;
    }
    if (i >= 2) zo_out += nxy;
    xk_m = xk_0; xk_0 = xk_p;
    k_m = k_0; k_0 = kc_p;
    xm_0 = xm;
    bt_0 = bt;
    rs = rs + 1 == RD ? 0 : rs + 1;
    ri = ri + 1 == RD ? 0 : ri + 1;
  }
  cp_async_wait<0>();
  double v[NDOT] = {v0, v1, v2, v3, v4};
  pass_epilogue(P, k, v);
}

// ---------------------------------------------------------------------------
// 16-byte cp.async (global -> shared, L2 only)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src) : "memory");
}

// Base of the dynamic shared memory of the 16-byte cp.async ring kernels, moved to a
// FIXED residue mod 128 bytes.  The extern array starts right after the kernel's
// static shared variables, so its address moved with every change to them, and the
// ring passes measured up to 20% slower at residues that are multiples of 32 than at
// 16 or 112 (sweep in profiles/r01_kernel_evolution.md, session 3): with the global
// rows at 16 mod 32, those put every 32-byte sector of a copy across two shared
// sectors.  The layouts reserve RING_SLACK extra bytes for the shift.
#ifndef KIOPS_RING_RES2D
#define KIOPS_RING_RES2D 112
#endif
#ifndef KIOPS_RING_RES3D
#define KIOPS_RING_RES3D 112
#endif
#define RING_SLACK 128
template <unsigned RES>
__device__ __forceinline__ double2 *ring_smem_base() {
  extern __shared__ __align__(128) double2 smem_ring[];  // base 128-byte aligned
  return smem_ring + RES / 16;
}

// ---------------------------------------------------------------------------
// 3D variable-kappa LAZY pass, pair version (in use for even nx, 1 <= p <= 4).
// Every thread owns TWO x-adjacent points (a 16-byte aligned pair) of the halo-1
// plane of a 64 x hb column tile, so every cp.async, shared load/store and global
// store moves 16 bytes and the x-neighbour inside the pair comes from registers;
// pairs span x in [ox-2, ox+66) (one unused point each side keeps alignment).
// Per plane: x_k = a0 r_{k-1} - a1 x_{k-1} - a2 x_{k-2} pointwise on the halo-1
// plane (operands in a thread-private cp.async ring, one plane ahead), x_k and
// kappa published in a 2-plane shared ring, one __syncthreads, then r_k = A x_k +
// nu B t_k on the interior with z-neighbours from registers; same arithmetic and
// dots as k_pass_3d_lazy.  Decomposition (lock-step persistent):
//  * the xy plane is cut into ~148 tiles of 64 x hb points (hb <= 8, balanced
//    bands, rc_tiles) and the z extent of each tile into zsplit parts, so that the
//    grid is exactly 2 CTAs per SM (config 4: 4 x 37 tiles x 2 halves = 296) and
//    every CTA has the same work (no partial last wave);
//  * all CTAs march in z in lock-step, odd parts downward, so the x/y halo rows a
//    tile shares with its neighbours, and the planes at part boundaries, are read
//    by both CTAs at about the same time (L2 hits instead of DRAM re-reads).
// Measured (config 4, ncu): 210 us, DRAM read = the 6 design read vectors exactly;
// 64 x 4 tiles at 4 CTAs/SM: slower (204 vs 166 ms of passes per call).
// ---------------------------------------------------------------------------
#define RC_SMS 148  // SMs of a B200 (host grid uses the same rule)

// tile rule shared by host and device: ntx columns of 64 points, nb bands of <= tym
// rows, about `target` tiles in all
__host__ __device__ inline void rc_tiles(long long nx, long long ny, int target, int tym, int *ntx, int *nb) {
  const int tx = (int)((nx + 63) / 64);
  int b = target / tx;
  if (b < 1) b = 1;
  if (b > ny) b = (int)ny;
  const int bmin = (int)((ny + tym - 1) / tym);
  if (b < bmin) b = bmin;
  *ntx = tx;
  *nb = b;
}
// z parts per tile: fill `ctas` CTAs, at least 2 planes per part
__host__ __device__ inline int rc_zsplit(long long nx, long long ny, long long nz, int target, int tym, int ctas) {
  int ntx, nb;
  rc_tiles(nx, ny, target, tym, &ntx, &nb);
  int zs = ctas / (ntx * nb);
  if (zs < 1) zs = 1;
  if (zs > nz / 2) zs = (int)(nz / 2 > 0 ? nz / 2 : 1);
  return zs;
}

// 7-point variable-kappa stencil on one 16-byte pair (points a = x, b = x + 1), the
// lazy pass's r expression operand for operand:
//   r = 0.5/h^2 sum_n (k_c + k_n)(x_n - x_c) + nu B t
__device__ __forceinline__ double2 stencil_pair(double2 xc, double2 kc, double xl, double xr, double kl, double kr,
                                                double2 xs, double2 xn, double2 ks, double2 kn, double2 xm,
                                                double2 km, double2 xp, double2 kp, double hh, double2 bt) {
  double ra = (kc.x + kl) * (xl - xc.x);
  double rb = (kc.y + kr) * (xr - xc.y);
  ra = fma(kc.x + kc.y, xc.y - xc.x, ra);
  rb = fma(kc.y + kc.x, xc.x - xc.y, rb);
  ra = fma(kc.x + ks.x, xs.x - xc.x, ra);
  rb = fma(kc.y + ks.y, xs.y - xc.y, rb);
  ra = fma(kc.x + kn.x, xn.x - xc.x, ra);
  rb = fma(kc.y + kn.y, xn.y - xc.y, rb);
  ra = fma(kc.x + km.x, xm.x - xc.x, ra);
  rb = fma(kc.y + km.y, xm.y - xc.y, rb);
  ra = fma(kc.x + kp.x, xp.x - xc.x, ra);
  rb = fma(kc.y + kp.y, xp.y - xc.y, rb);
  return make_double2(fma(ra, hh, bt.x), fma(rb, hh, bt.y));
}

// TYM: max tile rows; CPS: CTAs per SM (grid = CPS x 148, tiles target CPS/2 x 148)
// DD planes in flight; the private ring slot holds r, x_{k-1}, x_{k-2}, kappa for the
// NPAIR halo-1 pairs and B only for the NIN interior pairs.
template <int PM, int TYM, int CPS, int DD = 1, int NH = 1>
struct LazyQ {
  static constexpr int PX = 34, NPAIR = PX * (TYM + 2), NIN = 32 * TYM;
  static constexpr int NT = (NPAIR + 31) / 32 * 32;  // threads of one z-part (a "half")
  static constexpr int D = DD, RD = D + 1, SLOT = 4 * NPAIR + PM * NIN;
  static constexpr int TILES = RC_SMS * CPS / 2, CTAS = RC_SMS * CPS;
  static constexpr size_t half_bytes = 16 * (4 * (size_t)NPAIR + (size_t)RD * SLOT);
  static constexpr size_t smem_bytes = NH * half_bytes;
  static constexpr int BLOCK = NH * NT;
};

// NH = 2: one CTA runs the two z-parts of a tile as two thread halves that share the
// per-plane __syncthreads.  Two independent CTAs per SM (NH = 1) measured ~8% apart in
// speed (the second CTA placed on an SM is systematically slower), and the pass waits
// for the slowest; the shared barrier keeps both parts in lock-step.  Every z-march
// alternates direction with the pass parity, so a pass starts on the planes the
// previous one touched last (measured: -37 MB of DRAM reads per pass at 256^3).
template <int PM, int TYM, int CPS, int DD, int NH = 1>
__device__ __forceinline__ void body_3d_lazyq(const KParams &P, const PassScalars &S, double (&v)[NDOT]) {
  using M = LazyQ<PM, TYM, CPS, DD, NH>;
  constexpr int PX = M::PX, NPAIR = M::NPAIR, NIN = M::NIN, D = M::D, RD = M::RD, SLOT = M::SLOT, NT = M::NT;
  double2 *const smem2 = ring_smem_base<KIOPS_RING_RES3D>();
  const int h = threadIdx.x / NT, t = threadIdx.x % NT;  // half, thread within the half
  double2 *sXK = smem2 + (size_t)h * (M::half_bytes / 16);  // 2 x NPAIR   x_k pairs (plane ring)
  double2 *sKP = sXK + 2 * NPAIR;                               // 2 x NPAIR   kappa pairs
  double2 *sOp = sXK + 4 * NPAIR;                               // RD x SLOT   thread-private operand ring
  const int k = S.k;
  const long long nx = P.nx, ny = P.ny, nz = P.nz, nxy = nx * ny;
  int ntx, nb;
  rc_tiles(nx, ny, M::TILES, TYM, &ntx, &nb);
  const int ntiles = ntx * nb, zsplit = rc_zsplit(nx, ny, nz, M::TILES, TYM, M::CTAS);
  const double *rin = P.r + (size_t)((k - 1) & 1) * (size_t)P.ldN;
  double *rout = P.r + (size_t)(k & 1) * (size_t)P.ldN;
  const double *xprev = S.xprev, *xpp = S.xpp, *kap = P.kappa;
  double *xout = S.xout;
  const double a0 = S.a0, a1 = S.a1, a2 = S.a2, hh = 0.5 * P.inv_h2;
  const bool use_r = k >= 2, use_pp = xpp != nullptr;
  const double *Bc[PM];
  double btc[PM];
#pragma unroll
  for (int c = 0; c < PM; c++) {
    Bc[c] = S.B[c];
    btc[c] = S.btc[c];
  }
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, v4 = 0.0;

  for (int w = blockIdx.x; w < ntiles * (zsplit / NH); w += gridDim.x) {
    const int tile = w % ntiles, part = (w / ntiles) * NH + h;
    const long long ox = (long long)(tile % ntx) * 64, band = tile / ntx;
    const long long oy = band * ny / nb, hb = (band + 1) * ny / nb - oy;
    const long long zlo = part * nz / zsplit, zhi = (part + 1) * nz / zsplit;
    const int nzc = (int)(zhi - zlo);
    int nzmax = 0;  // longest part of this CTA (the halves share the barriers)
#pragma unroll
    for (int q = 0; q < NH; q++) {
      const int pq = (w / ntiles) * NH + q;
      const int n = (int)((pq + 1) * nz / zsplit - pq * nz / zsplit);
      nzmax = n > nzmax ? n : nzmax;
    }
    // odd parts march downward on odd passes' opposite: direction = part ^ pass parity
    const bool down = ((part ^ k) & 1) != 0;
    const int px = t % PX, py = t / PX;
    const bool act = py < hb + 2;
    const int o1 = act ? (int)(wrapc(ox - 2 + 2 * px, nx) + nx * wrapc(oy - 1 + py, ny)) : 0;
    const bool pin = act && py >= 1 && py <= hb && px >= 1 && px <= 32 && (ox - 2 + 2 * px) < nx;
    const long long oo = (ox - 2 + 2 * px) + nx * (oy - 1 + py);
    const int ib = (py - 1) * 32 + (px - 1);  // interior index (B slots)
    // logical plane j (-1 .. nzc) -> physical plane offset; the march is in j
    const long long zstep = down ? -nxy : nxy, zwrap = nz * nxy;
    long long zoL = wrapc(down ? zhi : zlo - 1, nz) * nxy;  // plane j = -1
    auto issue = [&](int slot) {
      if (act) {
        double2 *d = sOp + slot * SLOT + t;
        const long long g = zoL + o1;
        if (use_r) cp_async16(d, rin + g);
        cp_async16(d + NPAIR, xprev + g);
        if (use_pp) cp_async16(d + 2 * NPAIR, xpp + g);
        cp_async16(d + 3 * NPAIR, kap + g);
        if (pin)
#pragma unroll
          for (int c = 0; c < PM; c++) cp_async16(sOp + slot * SLOT + 4 * NPAIR + c * NIN + ib, Bc[c] + g);
      }
      zoL += zstep;
      if (zoL < 0) zoL += zwrap;
      if (zoL >= zwrap) zoL -= zwrap;
    };
    __syncthreads();  // previous part's readers are done with the rings
    for (int q = 0; q < D; q++) {
      if (q <= nzc + 1) issue(q);
      cp_async_commit();
    }
    // late issue: plane i + D is issued at the END of iteration i, into the slot of plane
    // i - 1, so during iteration i that slot (x_{k-1}, B at the output plane) and the x_k /
    // kappa shared rings (output plane's centre) still hold what the output needs: only
    // the plane below the output (x_k, kappa) is carried in registers.
    double2 xk_m = {0.0, 0.0}, k_m = {0.0, 0.0};
    long long zo_out = (down ? zhi - 1 : zlo) * nxy;
    int rs = 0, ri = D, rp = RD - 1;  // slots of planes i, i + D, i - 1
#pragma unroll 2
    for (int i = 0; i <= nzmax + 1; i++) {
      const bool live = i <= nzc + 1;
      cp_async_wait<D - 1>();
      const double2 *o = sOp + rs * SLOT + t;
      const double2 xm = o[NPAIR], kc_p = o[3 * NPAIR];
      double2 xk_p = xm;
      if (use_r) {
        const double2 rr = o[0];
        xk_p.x = a0 * rr.x - a1 * xm.x;
        xk_p.y = a0 * rr.y - a1 * xm.y;
        if (use_pp) {
          const double2 pp = o[2 * NPAIR];
          xk_p.x -= a2 * pp.x;
          xk_p.y -= a2 * pp.y;
        }
      }
      __syncthreads();  // the output that read slot (i & 1) has finished everywhere
      if (act) {
        sXK[(i & 1) * NPAIR + t] = xk_p;
        sKP[(i & 1) * NPAIR + t] = kc_p;
      }
      const double2 *X0 = sXK + ((i + 1) & 1) * NPAIR, *K0 = sKP + ((i + 1) & 1) * NPAIR;
      const double2 xk_0 = X0[t], k_0 = K0[t];
      if (i >= 2 && pin && live) {  // output logical plane i - 2 for both points of the pair
        const double2 *op = sOp + rp * SLOT;
        double2 bt = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < PM; c++) {
          const double2 b = op[4 * NPAIR + c * NIN + ib];
          bt.x = fma(b.x, btc[c], bt.x);
          bt.y = fma(b.y, btc[c], bt.y);
        }
        const double2 xm_0 = op[NPAIR + t];
        const double2 r = stencil_pair(xk_0, k_0, X0[t - 1].y, X0[t + 1].x, K0[t - 1].y, K0[t + 1].x, X0[t - PX],
                                       X0[t + PX], K0[t - PX], K0[t + PX], xk_m, k_m, xk_p, kc_p, hh, bt);
        const double2 xc = xk_0;
        v0 = fma(xc.x, xc.x, fma(xc.y, xc.y, v0));
        v1 = fma(xm_0.x, xc.x, fma(xm_0.y, xc.y, v1));
        v2 = fma(xm_0.x, r.x, fma(xm_0.y, r.y, v2));
        v3 = fma(xc.x, r.x, fma(xc.y, r.y, v3));
        v4 = fma(r.x, r.x, fma(r.y, r.y, v4));
        if (xout) *reinterpret_cast<double2 *>(xout + zo_out + oo) = xc;
        *reinterpret_cast<double2 *>(rout + zo_out + oo) = r;
      }
      if (i >= 2) zo_out += zstep;
      xk_m = xk_0;
      k_m = k_0;
      if (i + D <= nzc + 1) issue(ri);  // into the slot of plane i - 1 (= ri)
      cp_async_commit();
      rp = rs;
      rs = rs + 1 == RD ? 0 : rs + 1;
      ri = ri + 1 == RD ? 0 : ri + 1;
    }
    cp_async_wait<0>();
  }
  v[0] += v0; v[1] += v1; v[2] += v2; v[3] += v3; v[4] += v4;
}

template <int PM, int TYM, int CPS, int DD, int NH = 1>
__global__ void __launch_bounds__(LazyQ<PM, TYM, CPS, DD, NH>::BLOCK, CPS / NH) k_pass_3d_lazyq(KParams P) {
  __shared__ PassScalars S;
  pass_guard(P);
  if (threadIdx.x == 0) load_pass_scalars(P, S);
  __syncthreads();
  if (S.k == 0) return;
  double v[NDOT] = {0.0, 0.0, 0.0, 0.0, 0.0};
  body_3d_lazyq<PM, TYM, CPS, DD, NH>(P, S, v);
  pass_epilogue(P, S.k, v);
}

// ---------------------------------------------------------------------------
// 2D / 1D 5-point (+ diagonal) LAZY pass (in use for even nx): one WARP owns a
// strip of 30 interior x-pairs (+1 halo pair each side) and marches YC rows in y.
// Lane l holds the 16-byte aligned pair x = x0 - 2 + 2l, x0 + 1 - 2 + 2l.
//   x_k  = a0 r_{k-1} - a1 x_{k-1} - a2 x_{k-2}   (pointwise, every lane)
//   r_k  = W x_k(x-1) + E x_k(x+1) + S x_k(y-1) + N x_k(y+1) + (C + d) x_k + nu B t_k
// x-neighbours come from warp shuffles, y-neighbours from registers: no shared
// memory, no barriers.  Operands are prefetched one row ahead in registers.
// 1D uses the same kernel with ny = 1 and S = N = 0.
// ---------------------------------------------------------------------------
template <int PM>
struct Row2 {
  double2 r, xm, pp, d, b[PM > 0 ? PM : 1];
};

// One pass over this CTA's strips (vectors written by earlier passes of a persistent
// launch are read through L2: __ldcg, never the non-coherent path).
template <int YC, int PM>
__device__ __forceinline__ void body_2d_lazy(const KParams &P, const PassScalars &S, double (&v)[NDOT]) {
  constexpr int IP = 30;  // interior pairs per warp strip
  const int k = S.k;
  const long long nx = P.nx, ny = P.ny;
  const long long nsx = (nx + 2 * IP - 1) / (2 * IP), ncy = (ny + YC - 1) / YC;
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32;
  const bool wact = w < nsx * ncy;
  const long long sx = wact ? w % nsx : 0, cy = wact ? w / nsx : 0;
  const long long x0 = sx * 2 * IP, y0 = cy * YC;
  const long long y1 = (y0 + YC < ny) ? y0 + YC : ny;
  const long long px = x0 - 2 + 2 * lane;                 // first point of the own pair
  const long long pxw = wrapc(px, nx);
  const bool pin = wact && lane >= 1 && lane <= IP && px < nx;
  const bool use_r = k >= 2, use_pp = S.xpp != nullptr, use_d = P.diag != nullptr;
  const double *rin = P.r + (size_t)((k - 1) & 1) * (size_t)P.ldN;
  double *rout = P.r + (size_t)(k & 1) * (size_t)P.ldN;
  const double a0 = S.a0, a1 = S.a1, a2 = S.a2;
  const double Ww = P.w[0], Ew = P.w[1], Sw = P.w[2], Nw = P.w[3], Cw = P.w[4];
  double btc[PM > 0 ? PM : 1];
  const double *Bc[PM > 0 ? PM : 1];
#pragma unroll
  for (int c = 0; c < PM; c++) { btc[c] = S.btc[c]; Bc[c] = S.B[c]; }

  auto load = [&](long long y, Row2<PM> &o) {
    const long long g = pxw + nx * wrapc(y, ny);
    const double2 z2 = make_double2(0.0, 0.0);
    o.r = z2; o.pp = z2; o.d = z2;
    if (use_r) o.r = __ldcg(reinterpret_cast<const double2 *>(rin + g));
    o.xm = __ldcg(reinterpret_cast<const double2 *>(S.xprev + g));
    if (use_pp) o.pp = __ldcg(reinterpret_cast<const double2 *>(S.xpp + g));
    if (use_d) o.d = __ldg(reinterpret_cast<const double2 *>(P.diag + g));
#pragma unroll
    for (int c = 0; c < PM; c++) o.b[c] = pin ? __ldg(reinterpret_cast<const double2 *>(Bc[c] + g)) : z2;
  };
  auto form = [&](const Row2<PM> &o) {
    if (!use_r) return o.xm;
    double2 x;
    x.x = a0 * o.r.x - a1 * o.xm.x - a2 * o.pp.x;
    x.y = a0 * o.r.y - a1 * o.xm.y - a2 * o.pp.y;
    return x;
  };
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, v4 = 0.0;
  if (wact) {
    Row2<PM> cur, nxt;
    load(y0 - 1, cur);
    load(y0, nxt);
    double2 xk_m = form(cur);                 // x_k(y - 1)
    load(y0 + 1, cur);                        // row y0 + 1 (N neighbour of row y0)
    Row2<PM> row0 = nxt;                      // operands of row y (output row)
    double2 xk_0 = form(row0);                // x_k(y)
    for (long long y = y0; y < y1; y++) {
      Row2<PM> ahead;
      if (y + 2 <= y1) load(y + 2, ahead);     // prefetch row y + 2
      const double2 xk_p = form(cur);          // x_k(y + 1)
      // x-neighbours of row y: left of point a is lane-1's point b, right of b is lane+1's a
      const double xl = __shfl_up_sync(0xffffffffu, xk_0.y, 1);
      const double xr = __shfl_down_sync(0xffffffffu, xk_0.x, 1);
      double ra = Ww * xl + Ew * xk_0.y + Sw * xk_m.x + Nw * xk_p.x + (Cw + row0.d.x) * xk_0.x;
      double rb = Ww * xk_0.x + Ew * xr + Sw * xk_m.y + Nw * xk_p.y + (Cw + row0.d.y) * xk_0.y;
#pragma unroll
      for (int c = 0; c < PM; c++) {
        ra = fma(row0.b[c].x, btc[c], ra);
        rb = fma(row0.b[c].y, btc[c], rb);
      }
      if (pin) {
        const double2 xm = row0.xm;
        v0 = fma(xk_0.x, xk_0.x, fma(xk_0.y, xk_0.y, v0));
        v1 = fma(xm.x, xk_0.x, fma(xm.y, xk_0.y, v1));
        v2 = fma(xm.x, ra, fma(xm.y, rb, v2));
        v3 = fma(xk_0.x, ra, fma(xk_0.y, rb, v3));
        v4 = fma(ra, ra, fma(rb, rb, v4));
        const long long g = px + nx * y;
        if (S.xout) *reinterpret_cast<double2 *>(S.xout + g) = xk_0;
        *reinterpret_cast<double2 *>(rout + g) = make_double2(ra, rb);
      }
      xk_m = xk_0;
      xk_0 = xk_p;
      row0 = cur;
      cur = ahead;
    }
  }
  v[0] += v0; v[1] += v1; v[2] += v2; v[3] += v3; v[4] += v4;
}

// Same pass and arithmetic (identical operation order), with the operand rows
// prefetched D rows ahead by 16-byte cp.async into a warp-private shared ring
// (lane-private slots: no barriers), instead of one row ahead in registers: each
// warp's row chain then waits ~1/D of an L2/HBM latency per row.
template <int PM, int D>
struct Ring2 {
  static constexpr int NOP = 4 + PM, RD = D + 1;
  static constexpr size_t smem_bytes = 16 * (size_t)8 * RD * NOP * 32;  // 8 warps per CTA
};

// Per-warp strip geometry of the async 2D pass and the row issue (one 16-byte cp.async
// per operand and lane into ring slot si; diag and B only on output rows).
template <int YC, int PM, int D>
struct Strip2 {
  static constexpr int IP = 30;  // interior pairs per warp strip
  static constexpr int NOP = Ring2<PM, D>::NOP, RD = Ring2<PM, D>::RD;
  bool act, pin;
  int lane, nrows;
  long long px, pxw, y0, y1;
  double2 *ring;
  __device__ __forceinline__ Strip2(const KParams &P) {
    double2 *const smem2 = ring_smem_base<KIOPS_RING_RES2D>();
    const long long nx = P.nx, ny = P.ny;
    // 32-bit strip indices (strips < 2^31: N < 2^31 * 60 * YC)
    const int nsx = (int)((nx + 2 * IP - 1) / (2 * IP)), ncy = (int)((ny + YC - 1) / YC);
    lane = threadIdx.x & 31;
    const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    act = (long long)w < (long long)nsx * ncy;  // warp-uniform
    ring = smem2 + (size_t)(threadIdx.x >> 5) * RD * NOP * 32 + lane;
    const int cy = act ? w / nsx : 0, sx = act ? w - cy * nsx : 0;
    const long long x0 = (long long)sx * 2 * IP;
    y0 = (long long)cy * YC;
    y1 = (y0 + YC < ny) ? y0 + YC : ny;
    px = x0 - 2 + 2 * lane;
    pxw = wrapc(px, nx);
    pin = act && lane >= 1 && lane <= IP && px < nx;
    nrows = (int)(y1 - y0) + 2;  // logical row i = grid row y0 - 1 + i
  }
  // issue logical row ii (grid row yi) into slot si
  __device__ __forceinline__ void issue(const KParams &P, const double *rin, const double *xprev, const double *xpp,
                                        const double *const *Bc, long long yi, int si, int ii) const {
    const long long g = pxw + P.nx * yi;
    double2 *d = ring + si * NOP * 32;
    if (rin) cp_async16(d, rin + g);
    cp_async16(d + 32, xprev + g);
    if (xpp) cp_async16(d + 64, xpp + g);
    if (ii >= 1 && ii <= nrows - 2) {  // diag and B only on output rows (not the y-halo rows)
      if (P.diag) cp_async16(d + 96, P.diag + g);
      if (pin)
#pragma unroll
        for (int c = 0; c < PM; c++) cp_async16(d + (4 + c) * 32, Bc[c] + g);
    }
  }
  // the first D rows of pass k (one commit group each); rin = NULL for k = 1
  __device__ __forceinline__ void prologue(const KParams &P, const double *rin, const double *xprev, const double *xpp,
                                           const double *const *Bc) const {
    if (!act) return;
    long long yi = wrapc(y0 - 1, P.ny);
#pragma unroll
    for (int q = 0; q < D; q++) {
      if (q < nrows) issue(P, rin, xprev, xpp, Bc, yi, q, q);
      cp_async_commit();
      yi = (yi + 1 == P.ny) ? 0 : yi + 1;
    }
  }
};

template <int YC, int PM, int D>
__device__ __forceinline__ void body_2d_async(const KParams &P, const PassScalars &S, double (&v)[NDOT]) {
  const Strip2<YC, PM, D> G(P);
  constexpr int RD = Strip2<YC, PM, D>::RD, NOP = Strip2<YC, PM, D>::NOP;
  if (!G.act) return;  // warp-uniform
  const int k = S.k;
  const long long nx = P.nx, ny = P.ny;
  const bool pin = G.pin;
  const long long px = G.px, y0 = G.y0;
  const int nrows = G.nrows;
  const bool use_r = k >= 2, use_pp = S.xpp != nullptr, use_d = P.diag != nullptr;
  const double *rin = use_r ? P.r + (size_t)((k - 1) & 1) * (size_t)P.ldN : nullptr;
  double *rout = P.r + (size_t)(k & 1) * (size_t)P.ldN;
  const double *xprev = S.xprev, *xpp = S.xpp;
  double *xout = S.xout;
  const double a0 = S.a0, a1 = S.a1, a2 = S.a2;
  const double Ww = P.w[0], Ew = P.w[1], Sw = P.w[2], Nw = P.w[3], Cw = P.w[4];
  double btc[PM > 0 ? PM : 1];
  const double *Bc[PM > 0 ? PM : 1];
#pragma unroll
  for (int c = 0; c < PM; c++) { btc[c] = S.btc[c]; Bc[c] = S.B[c]; }
  G.prologue(P, rin, xprev, xpp, Bc);
  long long yi = wrapc(y0 - 1 + D, ny);  // next row to issue
  int si = D % RD, ii = D;               // its ring slot and logical index
  auto issue = [&]() {
    G.issue(P, rin, xprev, xpp, Bc, yi, si, ii);
    yi = (yi + 1 == ny) ? 0 : yi + 1;
    si = (si + 1 == RD) ? 0 : si + 1;
    ii++;
  };
  double2 *ring = G.ring;
  const double2 z2 = make_double2(0.0, 0.0);
  double2 xk_m = z2, xk_0 = z2, xm_0 = z2, d_0 = z2;
  double2 b_0[PM > 0 ? PM : 1];
#pragma unroll
  for (int c = 0; c < PM; c++) b_0[c] = z2;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0, v4 = 0.0;
  int sr = 0;  // slot of row i
  long long y = y0 - 1;
  for (int i = 0; i < nrows; i++, y++) {
    if (i + D < nrows) issue();
    cp_async_commit();
    cp_async_wait<D>();
    const double2 *o = ring + sr * NOP * 32;
    sr = (sr + 1 == RD) ? 0 : sr + 1;
    const double2 xm = o[32];
    double2 xk_p = xm;
    if (use_r) {
      const double2 rr = o[0], pp = use_pp ? o[64] : z2;
      xk_p.x = a0 * rr.x - a1 * xm.x - a2 * pp.x;
      xk_p.y = a0 * rr.y - a1 * xm.y - a2 * pp.y;
    }
    if (i >= 2) {  // output row y - 1 (x_k of rows y-2, y-1, y are xk_m, xk_0, xk_p)
      const double xl = __shfl_up_sync(0xffffffffu, xk_0.y, 1);
      const double xr = __shfl_down_sync(0xffffffffu, xk_0.x, 1);
      double ra = Ww * xl + Ew * xk_0.y + Sw * xk_m.x + Nw * xk_p.x + (Cw + d_0.x) * xk_0.x;
      double rb = Ww * xk_0.x + Ew * xr + Sw * xk_m.y + Nw * xk_p.y + (Cw + d_0.y) * xk_0.y;
#pragma unroll
      for (int c = 0; c < PM; c++) {
        ra = fma(b_0[c].x, btc[c], ra);
        rb = fma(b_0[c].y, btc[c], rb);
      }
      if (pin) {
        v0 = fma(xk_0.x, xk_0.x, fma(xk_0.y, xk_0.y, v0));
        v1 = fma(xm_0.x, xk_0.x, fma(xm_0.y, xk_0.y, v1));
        v2 = fma(xm_0.x, ra, fma(xm_0.y, rb, v2));
        v3 = fma(xk_0.x, ra, fma(xk_0.y, rb, v3));
        v4 = fma(ra, ra, fma(rb, rb, v4));
        const long long g = px + nx * (y - 1);
        if (xout) *reinterpret_cast<double2 *>(xout + g) = xk_0;
        *reinterpret_cast<double2 *>(rout + g) = make_double2(ra, rb);
      }
    }
    xk_m = xk_0;
    xk_0 = xk_p;
    xm_0 = xm;
    d_0 = use_d ? o[96] : z2;
    if (pin)
#pragma unroll
      for (int c = 0; c < PM; c++) b_0[c] = o[(4 + c) * 32];
  }
  cp_async_wait<0>();
  v[0] += v0; v[1] += v1; v[2] += v2; v[3] += v3; v[4] += v4;
}

template <int YC, int PM, int MINB = 2, int DA = 0, int NTH = 256>
__global__ void __launch_bounds__(NTH, MINB) k_pass_2d_lazy(KParams P) {
  __shared__ PassScalars S;
  pass_guard(P);
  if (threadIdx.x == 0) load_pass_scalars(P, S);
  __syncthreads();
  if (S.k == 0) return;
  double v[NDOT] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (DA > 0)
    body_2d_async<YC, PM, (DA > 0 ? DA : 1)>(P, S, v);
  else
    body_2d_lazy<YC, PM>(P, S, v);
  pass_epilogue(P, S.k, v);
}

// ---------------------------------------------------------------------------
// CSR operators run on a SELL-32 copy built at kiops_create:
// slice s = rows 32s..32s+31, padded to the slice's longest row, entry (k, lane)
// at off[s] + 32k + lane (pad: value 0, column = the row itself).  A warp = a slice:
// every value/column load is 256/128 contiguous bytes and the k-loop carries no
// dependency, so the gathers of x_k stream with full memory-level parallelism.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sell_build(long long N, const long long *__restrict__ rp,
                                                   const int *__restrict__ cols, const double *__restrict__ vals,
                                                   const long long *__restrict__ soff, int *__restrict__ scol,
                                                   double *__restrict__ sval) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < (N + 31) / 32 * 32;
       r += (long long)gridDim.x * blockDim.x) {
    const long long sl = r / 32, lane = r % 32, o0 = soff[sl], len = (soff[sl + 1] - o0) / 32;
    const long long b0 = r < N ? rp[r] : 0, n = r < N ? rp[r + 1] - b0 : 0;
    const int self = (int)(r < N ? r : 0);
    for (long long k = 0; k < len; k++) {
      const long long d = o0 + 32 * k + lane;
      scol[d] = k < n ? cols[b0 + k] : self;
      sval[d] = k < n ? vals[b0 + k] : 0.0;
    }
  }
}

__global__ void __launch_bounds__(256) k_sell_spmv(KParams P) {
  __shared__ PassScalars S;
  pass_guard(P, false);
  if (threadIdx.x == 0) load_pass_scalars<false>(P, S);
  __syncthreads();
  if (S.k == 0) return;
  const int k = S.k, p = P.p;
  const double *__restrict__ xk = (k == 1) ? S.xprev : S.xout;
  const double *__restrict__ xm = S.xprev;
  const double *__restrict__ sval = P.sell_val;
  const int *__restrict__ scol = P.sell_col;
  const long long *__restrict__ soff = P.sell_off;
  double v[NDOT] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < P.N; r += (long long)gridDim.x * blockDim.x) {
    const long long sl = r >> 5, o0 = soff[sl] + (r & 31), len = (soff[sl + 1] - soff[sl]) >> 5;
    double a0 = 0.0, a1 = 0.0;
    long long q = o0;
    int kk = 0;
#pragma unroll 4
    for (; kk + 1 < len; kk += 2, q += 64) {
      const double va = __ldg(sval + q), vb = __ldg(sval + q + 32);
      const int ca = __ldg(scol + q), cb = __ldg(scol + q + 32);
      a0 = fma(va, __ldg(xk + ca), a0);
      a1 = fma(vb, __ldg(xk + cb), a1);
    }
    if (kk < len) a0 = fma(__ldg(sval + q), __ldg(xk + __ldg(scol + q)), a0);
    double rr = a0 + a1;
#pragma unroll
    for (int c = 0; c < KMAXP; c++)
      if (c < p) rr += S.B[c][r] * S.btc[c];
    const double x = xk[r], y = xm[r];
    v[0] += x * x;
    v[1] += y * x;
    v[2] += y * rr;
    v[3] += x * rr;
    v[4] += rr * rr;
    P.r[r] = rr;
  }
  pass_epilogue<false>(P, k, v);
}
