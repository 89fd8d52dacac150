// passrc.cuh -- the recompute pass kernels of the padded-mode 3D variable-kappa path
// (body in rc3d.cuh, Alg. 2).  The padded copies
// made at call start are pad_copies (passes.cuh, k_setup), the padded output update
// gemv_padded (controller.cuh, k_gemv).  DESIGN.md sec. 4.1 / 6.
#pragma once
#include "kiops_internal.cuh"
#include "passes.cuh"
#include "inner.cuh"
#include "rc3d.cuh"

#ifndef RC_HM
#define RC_HM 7  // tile rows (config 4 bands: 6-7 rows of 64 points)
#endif
#ifndef RC_D
#define RC_D 3  // planes in flight ahead of the two in use
#endif
template <int PM>
using RcCfg = rc3::Cfg<PM, RC_HM, RC_D>;

__device__ __forceinline__ rc3::Geom rc_geom(const KParams &P) {
  rc3::Geom G;
  G.nx = (int)P.nx; G.ny = (int)P.ny; G.nz = (int)P.nz;
  G.Xp = P.Xp; G.Yp = P.Yp;
  G.ldN = P.ldN;
  G.ntx = P.rc_ntx; G.nb = P.rc_nb; G.zsplit = P.rc_zs;
  G.slot_kappa = P.slot_kappa; G.slot_B = P.slot_B;
  G.mapA = P.tmapA; G.mapB = P.tmapB;
  G.V = P.V;
  G.hh = 0.5 * P.inv_h2;
  return G;
}

// PassScalars (load_pass_scalars / the persistent loop's finalisation) -> pass args.
// x_{k-1}, x_{k-2} are basis slots (x_1 is slot 0 in padded mode).
template <int PM>
__device__ __forceinline__ rc3::PassArgs<PM> rc_args(const KParams &P, const PassScalars &S) {
  rc3::PassArgs<PM> Q;
  Q.k = S.k;
  Q.slot_prev = (int)((S.xprev - P.V) / P.ldN);
  Q.slot_pp = S.xpp ? (int)((S.xpp - P.V) / P.ldN) : -1;
  Q.xout = S.k >= 2 ? S.xout : nullptr;
  Q.a0 = S.a0; Q.a1 = S.a1; Q.a2 = S.a2;
#pragma unroll
  for (int c = 0; c < (PM > 0 ? PM : 1); c++) {
    Q.btp[c] = c < PM ? S.btp[c] : 0.0;
    Q.btc[c] = c < PM ? S.btc[c] : 0.0;
  }
  Q.use_r = S.k >= 2;
  return Q;
}

#ifndef RC_PREFETCH
#define RC_PREFETCH 0  // measured neutral at config 4 (same-box A/B, profiles/r02_kernel_evolution.md)
#endif
// Pass-boundary prefetch: during pass k's grid reduction the first ring planes of pass
// k+1 are issued (kappa, B, x_{k-1} boxes at once; the x_k boxes once every CTA has
// finished pass k), so pass k+1 starts on landed data.  If the Alg. 2 run ends instead
// (breakdown, non-finite, status), the planes are drained.
template <int PM>
struct RcHooks {
  const KParams &P;
  const rc3::Geom &G;
  unsigned &nl;
  int &pre;
  int npend;
  __device__ __forceinline__ void prefetch(const PassScalars &S, const InnerCarry &C, int which) {
    if (!RC_PREFETCH) return;
    const int k = S.k;
    if (which == 1) npend = 0;
    if (C.status_in != 0 || k >= C.m + 1 || k + 1 > P.m_max + 1 || (which == 2 && npend == 0)) return;
    // pass k+1 reads x_k (slot k-1; x_1 is slot 0) and x_{k-1} (slot k-2, from k+1 = 3)
    npend = rc3::preissue<PM, RC_HM, RC_D>(G, k + 1, k - 1, k >= 2 ? k - 2 : -1, nl, which, pre);
  }
  __device__ __forceinline__ void settle(bool go) {
    if (!go && npend > 0) {
      rc3::drain<PM, RC_HM, RC_D>(nl, npend);
      pre = 0;
    }
    npend = 0;
  }
};

// Persistent inner loop (inner.cuh) over recompute passes: one CTA per SM.
template <int PM>
__global__ void __launch_bounds__(RcCfg<PM>::NT, 1) k_inner_3d_rc(KParams P) {
  const rc3::Geom G = rc_geom(P);
  rc3::init<PM, RC_HM, RC_D>(G);
  unsigned nl = 0;  // the ring's running fill count, carried across the passes
  int pre = 0;      // ring planes of the next pass already issued (producer thread)
  inner_loop(
      P,
      [&](const PassScalars &S, double (&v)[NDOT]) {
        const rc3::PassArgs<PM> Q = rc_args<PM>(P, S);
        rc3::body<PM, RC_HM, RC_D>(G, Q, v, nl, pre);
      },
      RcHooks<PM>{P, G, nl, pre, 0});
}

// One launch per pass (KIOPS_PERSIST=0, or a grid that is not co-resident).
template <int PM>
__global__ void __launch_bounds__(RcCfg<PM>::NT, 1) k_pass_3d_rc(KParams P) {
  __shared__ PassScalars S;
  pass_guard(P);
  if (threadIdx.x == 0) load_pass_scalars(P, S);
  const rc3::Geom G = rc_geom(P);
  rc3::init<PM, RC_HM, RC_D>(G);  // (its __syncthreads publishes S)
  if (S.k == 0) return;
  unsigned nl = 0;
  int pre = 0;
  double v[NDOT] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const rc3::PassArgs<PM> Q = rc_args<PM>(P, S);
  rc3::body<PM, RC_HM, RC_D>(G, Q, v, nl, pre);
  pass_epilogue(P, S.k, v);
}
