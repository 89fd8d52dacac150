// kiops_internal.cuh -- device-side data layout shared by the kernels of the
// B200 KIOPS path (sm_100a).  See DESIGN.md section 6 for the HBM layout.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kiops.h"

#ifdef KIOPS_BOUNDS_CHECK  // debug builds: device-side index asserts (rc3d.cuh, pad_copies, gemv_padded)
#include <cassert>
#endif

#define KMAXP KIOPS_MAX_P
#define KMAXO KIOPS_MAX_OUT
#define KMAXM KIOPS_MAX_M
#define LDH (KMAXM + 2)          // leading dimension of H and of every controller matrix
#define NSCR 12                  // controller scratch matrices (LDH x LDH each)
#define NDOT 5                   // dots reduced per pass: S, G, E1, E2, R
#define GEMV_OCHUNK 4            // outputs accumulated per GEMV chunk

// Per-call block: written by the host with ONE cudaMemcpyAsync per kiops_apply.
struct CallBlock {
  const double *u[KMAXP + 1];    // u_0..u_p (DEVICE)
  double *w[KMAXO];              // outputs (DEVICE)
  double T[KMAXO];               // output times
  int n_out;
  int m_init;                    // > 0: this call's initial m (warm start, kiops_set_m_init)
  int n_forced;                  // test hook: forced schedule
  double forced_tau[KIOPS_MAX_FORCED];
  int forced_m[KIOPS_MAX_FORCED];
  int forced_acc[KIOPS_MAX_FORCED];
};

// Controller / pass state, resident in device memory for the whole call.
struct DevState {
  double tau, t_now, t_end, beta, nu, mu;
  double omega_old, tau_old;
  int m, npass, happy, l, hist_valid, j_old, status, zero_start;
  int accept, final_m;
  // pending GEMV (Alg. 3), set by the controller, consumed by k_gemv
  int gemv_j, gemv_nout;
  const double *gemv_x1;         // x_1 of the substep being projected
  double *gemv_out[KMAXO + 1];   // targets (user outputs, running slot last)
  const double *x1;              // x_1 source for the current substep (u_0, then V slot 1)
  long long attempt, substeps, rejections, kv, expm_calls, passes, happy_count;
  unsigned int ticket;           // last-CTA counter of the grid reductions
  unsigned int ticket2;
  unsigned long long launches;   // pass launches this call (device-side loop guard)
  // device-side kernel timing (%globaltimer, ns): graph-internal kernels cannot be
  // bracketed by host events, so each kernel type accumulates its own duration
  unsigned long long t_pass0, t_gemv0, ns_pass, ns_ctrl, ns_gemv, ns_expm;
  unsigned int gemv_ticket;
  unsigned int cond[3];          // mirror of the graph conditionals (outer, inner, accept)
  int bc_accept, bc_ntau;        // controller-cluster broadcast (CTA 0 -> all CTAs)
  unsigned int bar_count, bar_gen;  // launch-start grid barrier of the persistent inner loop (inner.cuh)
  unsigned long long pass_count;    // per-pass arrivals of the persistent inner loop (monotonic)
  unsigned int bar2_count, bar2_gen;  // in-pass grid barrier of the persistent CSR loop (form -> SpMV)
};

// Frozen per-ctx parameters, passed BY VALUE to every kernel (graph node params).
struct KParams {
  int kind;
  long long nx, ny, nz, N, ldN;
  double w[5];
  double w5[5];       // 1D/2D weights as {W, E, S, N, C} for every nx (generic-q path)
  const double *diag, *kappa;
  double inv_h2;
  const long long *row_ptr;
  const int *col_idx;
  const double *vals;
  const long long *sell_off;   // CSR as SELL-32 (built at create): slice offsets (in entries)
  const int *sell_col;
  const double *sell_val;
  int p;
  double tol;
  int m_init, m_min, m_max, task1;
  long long max_attempts;
  double *V;          // basis slots: x_k at V + (k-1)*ldN, k = 1..m_max+1 (slot 1 = running solution)
  double *r;          // CSR split form: A~ x_k (top)
  DevState *st;
  CallBlock *call;
  double *H;          // LDH x LDH column-major, H(i,j) 1-based at H[(i-1) + (j-1)*LDH]
  double *sig;        // sig[k] = ||x_k||, k = 1..
  double *R2;         // R2[k] = ||A~ x_k||^2 (breakdown scale, R3)
  double *tails;      // tails[k*KMAXP + c] = tail entry N+c of x_k (unnormalised)
  double *partials;   // NDOT x grid_max
  double *recs;       // 2 x grid_max x 8: per-CTA dot records of the persistent inner loop (inner.cuh)
  double *npart;      // KMAXP x grid_max   (setup: column abs sums)
  double *scratch;    // NSCR x LDH x LDH   (controller)
  double *coef;       // (KMAXO+1) x LDH    (GEMV coefficients)
  kiops_trace_row *trace;
  int grid_pass, grid_max;
  int q;              // IOP window (2: fused kernels; else passq.cuh)
  double *qa;         // generic q: formation coefficients of the next x (LDH)
  double *gram;       // generic q: G(i,l) = x_i . x_l, LDH x LDH column-major
  double *qpart;      // generic q: (2 LDH + 2) x QG dot partials
  int no_cond;        // 1: launched outside the graph (host-loop profiling hook)
  int flat_inner;     // 1: the persistent inner kernel is a plain node of the outer WHILE body (no inner
                      //    WHILE node): COND_INNER only lives in st->cond, the kernel checks for work itself
  int corrected;      // Saad's corrected scheme (options.corrected): the GEMV also uses x_{j+1}
  // padded mode (3D variable-kappa recompute pass, rc3d.cuh / passrc.cuh): every basis
  // slot is a ghost-padded (nx+4) x (ny+4) x nz grid, and slots m_max+1 .. m_max+p hold
  // copies of B's columns (u_p .. u_1), slot m_max+p+1 a copy of kappa, made by k_setup;
  // x_1 of the first substep is V slot 1 (u_0 copied there).  N stays nx ny nz.
  int padded;
  int Xp, Yp;         // nx + 4, ny + 4
  long long Np;       // Xp Yp nz (padded vector length)
  int rc_ntx, rc_nb, rc_zs;   // recompute-pass tiles (rc3::tiles)
  int slot_B, slot_kappa;     // 0-based slots of B column 0 and of kappa
  const void *tmapA, *tmapB;  // TMA tensor maps of the 4-D tensor [Xp][Yp][nz][slots] (workspace)
  cudaGraphConditionalHandle h_outer, h_inner, h_accept;
};
enum { COND_OUTER = 0, COND_INNER = 1, COND_ACCEPT = 2 };

__device__ __forceinline__ const double *slot_ptr(const KParams &P, int k) {
  // x_k for k >= 1 ; x_1 comes from the state's source pointer
  return (k == 1) ? P.st->x1 : P.V + (size_t)(k - 1) * (size_t)P.ldN;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum of NV values per thread; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *red /* smem NV*32 */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; q++) v[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; q++) red[q * 32 + wid] = v[q];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; q++) {
      double x = lane < nw ? red[q * 32 + lane] : 0.0;
      v[q] = warp_sum(x);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void set_cond(const KParams &P, int which, unsigned v) {
  if (!P.no_cond && !(P.flat_inner && which == COND_INNER))
    cudaGraphSetConditional(which == COND_OUTER ? P.h_outer : which == COND_INNER ? P.h_inner : P.h_accept, v);
  P.st->cond[which] = v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Loop guard (block 0, thread 0 of every pass launch): the device-side WHILE loops
// can never spin forever, even if a reduction were lost.  Returns true if tripped.
__device__ __forceinline__ bool pass_guard(const KParams &P, bool start_timer = true) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return false;
  DevState *st = P.st;
  if (start_timer) st->t_pass0 = gtimer();
  const unsigned long long n = ++st->launches;
  const unsigned long long cap = (unsigned long long)(P.max_attempts + 2) * (unsigned long long)(P.m_max + 2);
  if (n > cap || st->npass > P.m_max) {
    st->status = KIOPS_ERR_CUDA;
    set_cond(P, COND_INNER, 0u);
    set_cond(P, COND_OUTER, 0u);
    return true;
  }
  return false;
}
