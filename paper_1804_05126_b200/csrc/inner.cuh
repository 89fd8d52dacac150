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
  double skm1, iskm1, R2km1;      // sig[k-1], 1 / sig[k-1], R2[k-1]
  double nu;
  const double *x1;
  int m, status_in, go, trip;
  unsigned long long launches;
};
// State counters CTA 0 keeps in registers and stores (never read back) every pass.
struct InnerCounters {
  long long passes, kv;
  unsigned long long ns_pass, t0;
};

// Per-CTA dot records: recs[k & 1][cta][0..4] (64-byte slots).  A CTA writes its
// block partials, then (release) adds 1 to the monotonic pass_count; one thread per
// CTA waits (acquire) until pass_count reaches base + nb * (passes so far), then the
// whole CTA reads the records in the fixed block order.  Two buffers suffice: a CTA
// writes pass k+2's record only after every CTA has counted pass k+1, i.e. finished
// reading pass k's records.
__device__ __forceinline__ double *rec_ptr(const KParams &P, int buf, int cta) {
  return P.recs + ((size_t)buf * (size_t)P.grid_max + (size_t)cta) * 8;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// pass_finalize (passes.cuh) run by the 32 lanes of warp 0 with the same expressions
// (bitwise identical results).  One reciprocal per pass: with is = 1/s_k (and
// is' = 1/s_{k-1}, carried from the previous pass), every Gram-Schmidt quotient of
// Alg. 2 l.7-10 is a product (fin_* in passes.cuh, shared with pass_finalize), so the
// chain is sqrt -> one division -> a few dependent multiplications, computed
// redundantly by every lane: no shuffles after the broadcast of the dot sums.  (The
// earlier form divided at each of three levels with shuffles between them: 4.5 k
// cycles per pass measured at config 3, now 2.4 k.)
// Lanes 4..4+KMAXP-1 own tail entry c = lane - 4.  wr: this CTA (0) writes the state.
__device__ __forceinline__ void finalize_warp(const KParams &P, int k, const double (&v0)[NDOT],
                                              const double *ts, InnerCarry &C, PassScalars &Sn, bool wr,
                                              InnerCounters &K) {
  DevState *st = P.st;
  const int lane = threadIdx.x, p = P.p;
  const unsigned FULL = 0xffffffffu;
  double v[NDOT];
#pragma unroll
  for (int q = 0; q < NDOT; q++) v[q] = __shfl_sync(FULL, v0[q], 0);
  // + the tails' share (tail_dots, computed during the pass body)
  const double S = __dadd_rn(v[0], ts[0]), G = __dadd_rn(v[1], ts[1]), E1 = __dadd_rn(v[2], ts[2]),
               E2 = __dadd_rn(v[3], ts[3]), R = __dadd_rn(v[4], ts[4]);
  const bool l0 = lane == 0;
  if (wr && l0) {
    K.passes++;
    st->passes = K.passes;
    st->npass = k;
    const unsigned long long t = gtimer();
    K.ns_pass += t - K.t0;
    K.t0 = t;
    st->ns_pass = K.ns_pass;
  }
  if (C.status_in != 0) {
    if (wr && l0) set_cond(P, COND_INNER, 0u);
    if (l0) C.go = 0;
    return;
  }
  if (!isfinite(S) || !isfinite(G) || !isfinite(E1) || !isfinite(E2) || !isfinite(R)) {
    if (wr && l0) {
      st->status = KIOPS_ERR_NONFINITE;  // R22
      set_cond(P, COND_INNER, 0u);
    }
    if (l0) C.go = 0;
    return;
  }
  const double cn = k >= 2 ? sqrt(C.R2km1) / C.skm1 : 0.0;  // carried values only: off the chain
  const double sk = sqrt(S);
  const double is = 1.0 / sk;
  const int c = lane - 4;  // tail entry owned by this lane
  const bool own = c >= 0 && c < p;
  const int cc = (c >= 0 && c < KMAXP) ? c : 0;
  const double tkc = C.tk[cc], tkm1c = C.tkm1[cc];
  const double ktc = (own && c + 1 < p) ? C.tk[cc + 1 < KMAXP ? cc + 1 : 0] : 0.0;
  double *H = P.H;
#define HH(i, j) H[((i)-1) + (size_t)((j)-1) * LDH]
  double tn = 0.0, a1, a2 = 0.0;
  int go;
  if (k == 1) {  // beta = ||x_1|| (Alg. 1 l.14)
    if (wr && l0) {
      st->beta = sk;
      P.sig[1] = sk;
      P.R2[1] = R;
    }
    if (sk == 0.0) {  // R27
      if (wr && l0) {
        st->zero_start = 1;
        set_cond(P, COND_INNER, 0u);
      }
      if (l0) C.go = 0;
      return;
    }
    const double h11 = fin_h11(E2, is);
    if (wr && l0) HH(1, 1) = h11;
    a1 = __dmul_rn(h11, is);
    if (own) tn = fin_tail1(ktc, tkc, h11, is);
    go = (1 < C.m + 1) ? 1 : 0;
  } else {  // k >= 2 closes Alg. 2 iteration k-1
    const double ism1 = C.iskm1;
    if (wr && l0) {
      K.kv++;
      st->kv = K.kv;
    }
    const double thr = fmax(1e-12 * cn, 1e-14);  // R3
    if (sk <= thr) {                             // Alg. 2 l.12-15
      if (wr && l0) {
        st->happy = 1;
        set_cond(P, COND_INNER, 0u);
      }
      if (l0) C.go = 0;
      return;
    }
    if (wr && l0) {
      HH(k, k - 1) = sk;  // l.16 (R2)
      P.sig[k] = sk;
      P.R2[k] = R;
    }
    const double h1 = fin_h1(E1, ism1, is), h2 = fin_h2(E2, G, h1, ism1, is);
    if (wr && l0) {
      HH(k - 1, k) = h1;
      HH(k, k) = h2;
    }
    a1 = __dmul_rn(h2, is);
    a2 = __dmul_rn(h1, ism1);
    if (own) tn = fin_tail(ktc, tkm1c, tkc, h1, h2, ism1, is);
    go = (k < C.m + 1) ? 1 : 0;
  }
#undef HH
  if (wr && own) P.tails[(k + 1) * KMAXP + c] = tn;
  if (wr && l0 && !go) set_cond(P, COND_INNER, 0u);
  if (l0) C.go = go;
  if (!go) return;
  if (c >= 0 && c < KMAXP) {
    Sn.btp[c] = own ? C.nu * tkc : 0.0;
    Sn.btc[c] = own ? C.nu * tn : 0.0;
    C.tkm1[c] = own ? tkc : 0.0;
    C.tk[c] = own ? tn : 0.0;
  }
  if (l0) {
    const int kn = k + 1;  // <= m + 1 <= m_max + 1
    Sn.k = kn;
    Sn.xprev = (k == 1) ? C.x1 : P.V + (size_t)(k - 1) * (size_t)P.ldN;
    Sn.xpp = (kn >= 3) ? ((k - 1 == 1) ? C.x1 : P.V + (size_t)(k - 2) * (size_t)P.ldN) : nullptr;
    Sn.xout = P.V + (size_t)(kn - 1) * (size_t)P.ldN;
    Sn.a0 = is;
    Sn.a1 = a1;
    Sn.a2 = a2;
    C.skm1 = sk;
    C.iskm1 = is;
    C.R2km1 = R;
  }
}

// Optional pass-boundary hooks: prefetch(S, C, 1) right after pass S.k's body,
// prefetch(S, C, 2) once every CTA has finished pass S.k (its records are readable),
// settle(go) after the finalisation (go: pass S.k + 1 takes place).
struct NoHooks {
  __device__ __forceinline__ void prefetch(const PassScalars &, const InnerCarry &, int) {}
  __device__ __forceinline__ void settle(bool) {}
};

// The loop.  body(S, v) streams pass S.k over this CTA's share and accumulates the
// five dot partials into v.  All CTAs take identical control decisions.
template <class Body, class Hooks = NoHooks>
__device__ __forceinline__ void inner_loop(const KParams &P, Body &&body, Hooks &&hooks = Hooks{}) {
  __shared__ PassScalars S;
  __shared__ InnerCarry C;
  __shared__ double red[NDOT * 32];
  __shared__ double ts[NDOT];
  DevState *st = P.st;
  const unsigned nb = gridDim.x;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  InnerCounters K{};
  unsigned gen = 0;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      K.t0 = gtimer();
      K.passes = st->passes;
      K.kv = st->kv;
      K.ns_pass = st->ns_pass;
    }
    gen = ld_acquire_u32(&st->bar_gen);
    // loop guard (pass_guard), evaluated identically by every CTA
    C.launches = st->launches + 1;
    const unsigned long long cap = (unsigned long long)(P.max_attempts + 2) * (unsigned long long)(P.m_max + 2);
    // No pass to run in this attempt (a rejection that only shrank tau: the basis stands,
    // also the full basis npass = m_max + 1) or an error status -- what an inner WHILE
    // node's condition would express: the launch ends through the S.k = 0 exit below, so
    // that the kernel can be a plain node of the outer loop body (flat_inner, kiops.cu).
    const bool idle = st->npass >= st->m + 1 || st->status != 0;
    C.trip = (C.launches > cap || (st->npass > P.m_max && !idle)) ? 1 : 0;
    C.status_in = st->status;
    C.m = st->m;
    C.nu = st->nu;
    C.x1 = st->x1;
    load_pass_scalars(P, S);
    if (idle) {
      S.k = 0;
      if (blockIdx.x == 0) set_cond(P, COND_INNER, 0u);
    }
    const int k = S.k;
    if (k >= 1) {
      for (int c = 0; c < KMAXP; c++) {
        C.tk[c] = c < P.p ? P.tails[k * KMAXP + c] : 0.0;
        C.tkm1[c] = c < P.p ? P.tails[(k - 1) * KMAXP + c] : 0.0;
      }
      C.skm1 = k >= 2 ? P.sig[k - 1] : 0.0;
      C.iskm1 = k >= 2 ? 1.0 / C.skm1 : 0.0;
      C.R2km1 = k >= 2 ? P.R2[k - 1] : 0.0;
    }
  }
  unsigned long long target = 0;
  if (threadIdx.x == 0) target = st->pass_count;  // stable until every CTA passed the barrier below
  // one grid barrier per launch: every CTA has read the launch and pass counters
  grid_sync(st, nb, gen);
  if (lead) st->launches = C.launches;
  if (C.trip || S.k == 0) {
    if (lead && C.trip) {
      st->status = KIOPS_ERR_CUDA;
      set_cond(P, COND_INNER, 0u);
      set_cond(P, COND_OUTER, 0u);
    }
    return;
  }
#ifdef KIOPS_PHASE_TIMERS  // debug build: CTA 0 prints body / barrier / finalise time per launch
  const int k_first = S.k;
  unsigned long long tb = 0, tw = 0, tf = 0, tp = 0, ta = gtimer(), tt;
  long long cf1 = 0;
#define PHASE(acc) do { tt = gtimer(); acc += tt - ta; ta = tt; } while (0)
#else
#define PHASE(acc) do { } while (0)
#endif
  for (;;) {
    const int k = S.k;
    double v[NDOT] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (threadIdx.x == 0) {  // the tails' share of this pass's dots, kept in shared memory (not
      double t[NDOT];        // in registers across the body, whose allocation it would change)
      tail_dots(k, P.p, C.tk, C.tkm1, t);
#pragma unroll
      for (int q = 0; q < NDOT; q++) ts[q] = t[q];
    }
    body(S, v);
    hooks.prefetch(S, C, 1);
    block_sum<NDOT>(v, red);  // (its __syncthreads order every thread's vector writes before the fence)
    PHASE(tb);
    double w[NDOT];
    if (nb == 1) {  // one CTA: its block sum is the total (= the record path's sum, + 0.0 terms)
#pragma unroll
      for (int q = 0; q < NDOT; q++) w[q] = v[q];
    } else {
    if (threadIdx.x == 0) {
      double *mine = rec_ptr(P, k & 1, blockIdx.x);
#pragma unroll
      for (int q = 0; q < NDOT; q++) __stcg(mine + q, v[q]);
      // release (cumulative: covers the CTA's x_k, r_k writes ordered before block_sum's
      // bar.sync) ... acquire on the counter, propagated to the CTA by the bar.sync below
      red_release_add_u64(&st->pass_count, 1ull);
      target += nb;
      while (ld_acquire_u64(&st->pass_count) < target) {
      }
    }
    __syncthreads();
    PHASE(tp);
    hooks.prefetch(S, C, 2);
    // every CTA's record, in the fixed block order of pass_finalize.  (Issuing pass
    // k+1's first loads here, before its scalars exist, measured slower: the extra
    // traffic delays the record loads and the finalisation more than it hides.)
#pragma unroll
    for (int q = 0; q < NDOT; q++) w[q] = 0.0;
    for (int b = threadIdx.x; b < (int)nb; b += blockDim.x) {
      const double *rr = rec_ptr(P, k & 1, b);
#pragma unroll
      for (int q = 0; q < NDOT; q++) w[q] += __ldcg(rr + q);
    }
    PHASE(tw);
    block_sum<NDOT>(w, red);
    }
    if (nb == 1) hooks.prefetch(S, C, 2);
#ifdef KIOPS_PHASE_TIMERS
    const long long c0 = clock64();
#endif
    if (threadIdx.x < 32) finalize_warp(P, k, w, ts, C, S, blockIdx.x == 0, K);
#ifdef KIOPS_PHASE_TIMERS
    const long long c1 = clock64();
    cf1 += c1 - c0;
#endif
    __syncthreads();
    PHASE(tf);
    hooks.settle(C.go != 0);
    if (!C.go) break;
  }
#ifdef KIOPS_PHASE_TIMERS
  if (threadIdx.x == 0 && k_first == 1) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("CTABODY %d %u %.2f %.2f\n", blockIdx.x, smid, tb * 1e-3, tw * 1e-3);
  }
  if (lead) printf("PHASES k_end %d body %.2f us poll %.2f us records %.2f us finalise %.2f us (warp-0 finalise %lld clk) (sums over the launch)\n", S.k,
                   tb * 1e-3, tp * 1e-3, tw * 1e-3, tf * 1e-3, cf1);
#endif
#undef PHASE
}

template <int YC, int PM, int MINB, int DA = 0, int NTH = 256>
__global__ void __launch_bounds__(NTH, MINB) k_inner_2d_lazy(KParams P) {
  inner_loop(P, [&](const PassScalars &S, double (&v)[NDOT]) {
    if (DA > 0)
      body_2d_async<YC, PM, (DA > 0 ? DA : 1)>(P, S, v);
    else
      body_2d_lazy<YC, PM>(P, S, v);
  });
}

template <int PM, int TYM, int CPS, int DD, int NH = 1>
__global__ void __launch_bounds__(LazyQ<PM, TYM, CPS, DD, NH>::BLOCK, CPS / NH) k_inner_3d_lazyq(KParams P) {
  inner_loop(P, [&](const PassScalars &S, double (&v)[NDOT]) { body_3d_lazyq<PM, TYM, CPS, DD, NH>(P, S, v); });
}

// ---------------------------------------------------------------------------
// Persistent inner loop of the CSR path for SMALL matrices (where a pass takes a few
// microseconds and the two launches + WHILE iteration per pass dominate: the EPIRK driver's
// CSR Jacobians, reduced grids).  Per pass: the pointwise formation of x_k (k_csr_form's),
// ONE grid barrier (x_k complete and visible), the SELL-32 SpMV with the five dots
// (k_sell_spmv's), then the loop's record reduction and finalisation.  x_k is gathered with
// L2 loads (.cg): it was written in this launch by other CTAs, so the non-coherent path the
// per-pass SpMV uses for its gathers is not allowed -- which is why the large matrices
// (config 5) keep the per-pass kernels.  Every thread forms and later reads r, x_{k-1},
// x_k at its own rows (the same grid-stride map in both loops).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_sync2(DevState *st, unsigned nb, unsigned &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (nb > 1) {
      __threadfence();
      if (atomicAdd(&st->bar2_count, 1u) == nb - 1) {
        st->bar2_count = 0;
        __threadfence();
        atomicAdd(&st->bar2_gen, 1u);
      } else {
        while (ld_acquire_u32(&st->bar2_gen) == gen) {
        }
      }
      __threadfence();
    }
    gen++;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_inner_csr(KParams P) {
  unsigned gen2 = 0;
  if (threadIdx.x == 0) gen2 = ld_acquire_u32(&P.st->bar2_gen);  // (before this CTA's first arrival)
  inner_loop(P, [&](const PassScalars &S, double (&v)[NDOT]) {
    const int k = S.k, p = P.p;
    const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x, di = (long long)gridDim.x * blockDim.x;
    if (k >= 2) {  // x_k = a0 r_{k-1} - a1 x_{k-1} - a2 x_{k-2}  (Alg. 2 l.7-10, l.17 folded)
      const double *r = P.r;
      for (long long i = i0; i < P.N; i += di) {
        double xk = S.a0 * r[i] - S.a1 * S.xprev[i];
        if (S.xpp) xk -= S.a2 * S.xpp[i];
        S.xout[i] = xk;
      }
    }
    grid_sync2(P.st, gridDim.x, gen2);
    const double *xk = (k == 1) ? S.xprev : S.xout;
    const double *xm = S.xprev;
    const double *__restrict__ sval = P.sell_val;
    const int *__restrict__ scol = P.sell_col;
    const long long *__restrict__ soff = P.sell_off;
    for (long long r = i0; r < P.N; r += di) {
      const long long sl = r >> 5, o0 = soff[sl] + (r & 31), len = (soff[sl + 1] - soff[sl]) >> 5;
      double a0 = 0.0, a1 = 0.0;
      long long q = o0;
      int kk = 0;
#pragma unroll 4
      for (; kk + 1 < len; kk += 2, q += 64) {
        const double va = __ldg(sval + q), vb = __ldg(sval + q + 32);
        const int ca = __ldg(scol + q), cb = __ldg(scol + q + 32);
        a0 = fma(va, __ldcg(xk + ca), a0);
        a1 = fma(vb, __ldcg(xk + cb), a1);
      }
      if (kk < len) a0 = fma(__ldg(sval + q), __ldcg(xk + __ldg(scol + q)), a0);
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
  });
}
