// inner.cuh -- persistent inner loop: every pass of one Alg. 2 run (the
// inner WHILE of the graph) inside ONE launch.
//
// The per-pass kernels (passes.cuh) pay, per Krylov vector, a launch inside the
// conditional graph, a dependent prologue (state -> H, sig, tails -> the formation
// scalars) and a last-CTA epilogue (ticket atomic, partial reduction, finalisation,
// state writes).  Measured in round 1 that fixed cost is ~7-10 us per pass, which is
// the whole pass at N = 400 / 65 536 and ~half of it at 1024^2.  Here the grid stays
// resident (cooperative launch: grid <= co-resident CTAs) and between passes runs:
//   1. block sums of the five dots -> this CTA's partials (buffer k & 1);
//   2. one grid barrier (arrival counter + generation word, acquire/release);
//   3. EVERY CTA reduces all partials in the fixed block order of pass_finalize and
//      runs the same finalisation on its own copy of the carried scalars (sig, R2,
//      tails), so every CTA derives bit-identical formation scalars for pass k+1 with
//      no further global round trip; CTA 0 alone writes H, sig, R2, tails, the
//      counters and the graph conditionals for the controller.
// Arithmetic and reduction order are those of pass_finalize / load_pass_scalars, so
// results are bitwise identical to the per-pass kernels (tested).
#pragma once
#include "kiops_internal.cuh"
#include "passes.cuh"

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier over nb co-resident CTAs.  gen (thread 0's register) is the
// generation this CTA waits to leave.
__device__ __forceinline__ void grid_sync(DevState *st, unsigned nb, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (nb > 1) {
      __threadfence();
      if (atomicAdd(&st->bar_count, 1u) == nb - 1) {
        st->bar_count = 0;
        __threadfence();
        atomicAdd(&st->bar_gen, 1u);
      } else {
        while (ld_acquire_u32(&st->bar_gen) == gen) {
        }
      }
      __threadfence();
    }
    gen++;
  }
  __syncthreads();
}

// Scalars carried from the finalisation of pass k to that of pass k+1 (per CTA).
struct InnerCarry {
  double tk[KMAXP], tkm1[KMAXP];  // tails of x_k, x_{k-1}
  double skm1, R2km1;             // sig[k-1], R2[k-1]
  double nu;
  const double *x1;
  int m, status_in, go, trip;
  unsigned gen;
  unsigned long long launches;
};

// pass_finalize (passes.cuh) on the carried scalars; wr: this CTA writes the state.
// Sets C.go and, when going on, the PassScalars of pass k+1.
__device__ __noinline__ void inner_finalize(const KParams &P, int k, const double (&v)[NDOT], InnerCarry &C, PassScalars &Sn,
                               bool wr, unsigned long long &t0) {
  DevState *st = P.st;
  const int p = P.p;
  double Kt[KMAXP];
  for (int c = 0; c < p; c++) Kt[c] = (c + 1 < p) ? C.tk[c + 1] : 0.0;  // tail of A~ x_k (Alg. 2 l.5-6)
  double S = v[0], G = v[1], E1 = v[2], E2 = v[3], R = v[4];
  for (int c = 0; c < p; c++) {
    S += C.tk[c] * C.tk[c];
    R += Kt[c] * Kt[c];
    E2 += C.tk[c] * Kt[c];
    if (k >= 2) { G += C.tkm1[c] * C.tk[c]; E1 += C.tkm1[c] * Kt[c]; }
  }
  C.go = 0;
  if (wr) {
    st->passes++;
    st->npass = k;
    const unsigned long long t = gtimer();
    st->ns_pass += t - t0;
    t0 = t;
  }
  if (C.status_in != 0) {
    if (wr) set_cond(P, COND_INNER, 0u);
    return;
  }
  if (!isfinite(S) || !isfinite(G) || !isfinite(E1) || !isfinite(E2) || !isfinite(R)) {
    if (wr) {
      st->status = KIOPS_ERR_NONFINITE;  // R22
      set_cond(P, COND_INNER, 0u);
    }
    return;
  }
  const double sk = sqrt(S);
  double *H = P.H;
#define HH(i, j) H[((i)-1) + (size_t)((j)-1) * LDH]
  double tn[KMAXP];
  double a1, a2;
  if (k == 1) {  // beta = ||x_1|| (Alg. 1 l.14)
    if (wr) {
      st->beta = sk;
      P.sig[1] = sk;
      P.R2[1] = R;
    }
    if (sk == 0.0) {  // R27
      if (wr) {
        st->zero_start = 1;
        set_cond(P, COND_INNER, 0u);
      }
      return;
    }
    const double h11 = E2 / (sk * sk);
    if (wr) HH(1, 1) = h11;
    for (int c = 0; c < p; c++) tn[c] = Kt[c] / sk - h11 * C.tk[c] / sk;
    C.go = (1 < C.m + 1) ? 1 : 0;
    a1 = h11 / sk;
    a2 = 0.0;
  } else {  // k >= 2 closes Alg. 2 iteration k-1
    if (wr) st->kv++;
    const double skm1 = C.skm1;
    const double cn = sqrt(C.R2km1) / skm1;
    const double thr = fmax(1e-12 * cn, 1e-14);  // R3
    if (sk <= thr) {                             // Alg. 2 l.12-15
      if (wr) {
        st->happy = 1;
        set_cond(P, COND_INNER, 0u);
      }
      return;
    }
    if (wr) {
      HH(k, k - 1) = sk;  // l.16 (R2)
      P.sig[k] = sk;
      P.R2[k] = R;
    }
    const double h1 = E1 / (skm1 * sk);
    const double h2 = E2 / (sk * sk) - h1 * G / (skm1 * sk);
    if (wr) {
      HH(k - 1, k) = h1;
      HH(k, k) = h2;
    }
    for (int c = 0; c < p; c++) tn[c] = Kt[c] / sk - h1 * C.tkm1[c] / skm1 - h2 * C.tk[c] / sk;
    C.go = (k < C.m + 1) ? 1 : 0;
    a1 = h2 / sk;   // = H(k,k)/sig[k]          (load_pass_scalars of pass k+1)
    a2 = h1 / skm1; // = H(k-1,k)/sig[k-1]
  }
#undef HH
  if (wr) {
    double *tw = P.tails + (k + 1) * KMAXP;
    for (int c = 0; c < p; c++) tw[c] = tn[c];
    if (!C.go) set_cond(P, COND_INNER, 0u);
  }
  if (!C.go) return;
  const int kn = k + 1;  // <= m + 1 <= m_max + 1
  Sn.k = kn;
  Sn.xprev = (k == 1) ? C.x1 : P.V + (size_t)(k - 1) * (size_t)P.ldN;
  Sn.xpp = (kn >= 3) ? ((k - 1 == 1) ? C.x1 : P.V + (size_t)(k - 2) * (size_t)P.ldN) : nullptr;
  Sn.xout = P.V + (size_t)(kn - 1) * (size_t)P.ldN;
  Sn.a0 = 1.0 / sk;
  Sn.a1 = a1;
  Sn.a2 = a2;
  for (int c = 0; c < KMAXP; c++) {
    Sn.btp[c] = c < p ? C.nu * C.tk[c] : 0.0;
    Sn.btc[c] = c < p ? C.nu * tn[c] : 0.0;
    C.tkm1[c] = c < p ? C.tk[c] : 0.0;
    C.tk[c] = c < p ? tn[c] : 0.0;
  }
  C.skm1 = sk;
  C.R2km1 = R;
}

// The loop.  body(S, v) streams pass S.k over this CTA's share and accumulates the
// five dot partials into v.  All CTAs take identical control decisions.
template <class Body>
__device__ __forceinline__ void inner_loop(const KParams &P, Body &&body) {
  __shared__ PassScalars S;
  __shared__ InnerCarry C;
  __shared__ double red[NDOT * 32];
  DevState *st = P.st;
  const unsigned nb = gridDim.x;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t0 = 0;
  unsigned gen = 0;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) t0 = gtimer();
    gen = ld_acquire_u32(&st->bar_gen);
    // loop guard (pass_guard), evaluated identically by every CTA
    C.launches = st->launches + 1;
    const unsigned long long cap = (unsigned long long)(P.max_attempts + 2) * (unsigned long long)(P.m_max + 2);
    C.trip = (C.launches > cap || st->npass > P.m_max) ? 1 : 0;
    C.status_in = st->status;
    C.m = st->m;
    C.nu = st->nu;
    C.x1 = st->x1;
    load_pass_scalars(P, S);
    const int k = S.k;
    if (k >= 1) {
      for (int c = 0; c < KMAXP; c++) {
        C.tk[c] = c < P.p ? P.tails[k * KMAXP + c] : 0.0;
        C.tkm1[c] = c < P.p ? P.tails[(k - 1) * KMAXP + c] : 0.0;
      }
      C.skm1 = k >= 2 ? P.sig[k - 1] : 0.0;
      C.R2km1 = k >= 2 ? P.R2[k - 1] : 0.0;
    }
  }
  __syncthreads();
  if (C.trip || S.k == 0) {
    grid_sync(st, nb, gen);  // every CTA has read the launch counter
    if (lead) {
      st->launches = C.launches;
      if (C.trip) {
        st->status = KIOPS_ERR_CUDA;
        set_cond(P, COND_INNER, 0u);
        set_cond(P, COND_OUTER, 0u);
      }
    }
    return;
  }
  bool first = true;
  for (;;) {
    const int k = S.k;
    double v[NDOT] = {0.0, 0.0, 0.0, 0.0, 0.0};
    body(S, v);
    block_sum<NDOT>(v, red);
    double *part = P.partials + (size_t)(k & 1) * NDOT * (size_t)P.grid_max;
    if (threadIdx.x == 0)
#pragma unroll
      for (int q = 0; q < NDOT; q++) part[q * P.grid_max + blockIdx.x] = v[q];
    grid_sync(st, nb, gen);
    if (first && lead) st->launches = C.launches;
    first = false;
    double w[NDOT];
#pragma unroll
    for (int q = 0; q < NDOT; q++) w[q] = 0.0;
    for (int b = threadIdx.x; b < (int)nb; b += blockDim.x)
#pragma unroll
      for (int q = 0; q < NDOT; q++) w[q] += __ldcg(&part[q * P.grid_max + b]);
    block_sum<NDOT>(w, red);
    if (threadIdx.x == 0) inner_finalize(P, k, w, C, S, blockIdx.x == 0, t0);
    __syncthreads();
    if (!C.go) break;
  }
}

template <int YC, int PM, int MINB>
__global__ void __launch_bounds__(256, MINB) k_inner_2d_lazy(KParams P) {
  inner_loop(P, [&](const PassScalars &S, double (&v)[NDOT]) { body_2d_lazy<YC, PM>(P, S, v); });
}

template <int PM, int TYM, int CPS, int DD>
__global__ void __launch_bounds__(LazyQ<PM, TYM, CPS, DD>::NT, CPS) k_inner_3d_lazyq(KParams P) {
  inner_loop(P, [&](const PassScalars &S, double (&v)[NDOT]) { body_3d_lazyq<PM, TYM, CPS, DD>(P, S, v); });
}
