// controller.cuh -- SURVEY 8(a) rows a5-a8: the single-CTA controller kernel
// (projected exponential, error estimate, acceptance, Alg. 4 adaptivity, Alg. 3
// output bookkeeping) and the multi-RHS GEMV over the basis.  sm_100a, fp64.
#pragma once
#include "kiops_internal.cuh"
#include "passes.cuh"

#define CTRL_THREADS 512
#define CTRL_CL 8    // CTAs per controller cluster (portable maximum)

// ---------------------------------------------------------------------------
// Dense n x n (n <= KMAXM+1) linear algebra for ONE thread-block CLUSTER of
// CTRL_CL CTAs.  Matrices are column-major, leading dimension LDH, in global
// scratch (L2-resident).  Work is split across the cluster and ordered with
// cluster barriers (barrier.cluster arrive.release / wait.acquire), which also
// make each CTA's global writes visible to the others.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ int cl_gtid() { return (int)(cl_rank() * blockDim.x + threadIdx.x); }
__device__ __forceinline__ int cl_gsize() { return (int)(CTRL_CL * blockDim.x); }

// Named barriers of one 512-thread CTA (ids 1, 2): bar.arrive by the warp that publishes,
// bar.sync by the warps that consume (split hand-off instead of a __syncthreads).
__device__ __forceinline__ void nb_sync512(int id) { asm volatile("bar.sync %0, 512;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nb_arrive512(int id) { asm volatile("bar.arrive %0, 512;" ::"r"(id) : "memory"); }

// D += A B for one 8x8x4 FP64 tensor-core tile (mma.sync m8n8k4 .f64): fragments per
// lane g = lane/4, t = lane%4: A(g, t), B(t, g), C(g, 2t), C(g, 2t+1).
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// C = A B (ld LDH, no aliasing), n <= KMAXM+1, on the FP64 tensor cores.  CTA r owns
// the 8-column output tiles r, r+8, ...: it stages ALL of A (n x np, ld MM_LD) and its
// B column panels in shared memory (coalesced .cg loads -- other CTAs wrote them -- all
// independent, so one L2 round trip instead of one per k-step), then its warps run
// m8n8k4 DMMA from shared memory over the tile rows (zero-padded to multiples of 8).
#define MM_LD 148  // >= KMAXM+1 rounded to 8, = 4 mod 16: the fragment loads are bank-conflict free
__device__ void cl_matmul(int n, const double *__restrict__ A, const double *__restrict__ B, double *__restrict__ C,
                          double *sm) {
  const int np = (n + 7) & ~7, nt = np >> 3;
  const int rank = (int)cl_rank(), lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int ncol = (nt - rank + CTRL_CL - 1) / CTRL_CL;  // tile columns tj = rank + CTRL_CL i
  double *sA = sm;                          // np x np, ld MM_LD (A[i + ld k])
  double *sB = sm + (size_t)MM_LD * np;     // np x (8 ncol), ld MM_LD (B[k + ld j_local])
  if (ncol > 0) {
    for (int c = warp; c < np; c += nw)
      for (int r = lane; r < np; r += 32)
        sA[r + MM_LD * c] = (r < n && c < n) ? __ldcg(A + r + (size_t)LDH * c) : 0.0;
    for (int jl = warp; jl < 8 * ncol; jl += nw) {
      const int j = (rank + CTRL_CL * (jl >> 3)) * 8 + (jl & 7);
      for (int r = lane; r < np; r += 32)
        sB[r + MM_LD * jl] = (r < n && j < n) ? __ldcg(B + r + (size_t)LDH * j) : 0.0;
    }
  }
  __syncthreads();
  const int ntile = nt * ncol;  // (tile row, local tile column)
  for (int t0 = warp; t0 < ntile; t0 += 2 * nw) {
    double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    int ti[2], tl[2];
    bool on[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int tt = t0 + u * nw;
      on[u] = tt < ntile;
      ti[u] = on[u] ? (tt % nt) * 8 : 0;
      tl[u] = on[u] ? (tt / nt) * 8 : 0;
    }
    for (int k0 = 0; k0 < np; k0 += 4) {
#pragma unroll
      for (int u = 0; u < 2; u++)
        if (on[u]) dmma_8x8x4(c[u], sA[(ti[u] + g) + MM_LD * (k0 + tq)], sB[(k0 + tq) + MM_LD * (tl[u] + g)]);
    }
#pragma unroll
    for (int u = 0; u < 2; u++)
      if (on[u]) {
        const int r = ti[u] + g, jl = tl[u] + 2 * tq;
        const int cc = (rank + CTRL_CL * (jl >> 3)) * 8 + (jl & 7);
        if (r < n && cc < n) C[r + (size_t)LDH * cc] = c[u][0];
        if (r < n && cc + 1 < n) C[r + (size_t)LDH * (cc + 1)] = c[u][1];
      }
  }
  cl_sync();
}

__device__ double cta_norm1(int n, const double *A, double *red) {
  // max column abs sum, broadcast to all threads (every CTA computes the same value)
  double best = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < n; i++) s += fabs(A[i + (size_t)LDH * j]);
    best = (s > best || s != s) ? s : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, best, o);
    best = (x > best || x != x) ? x : best;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)((blockDim.x + 31) >> 5); w++) b = (red[w] > b || red[w] != red[w]) ? red[w] : b;
    red[32] = b;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

// Solve Q X = R in place (R <- X).  CTA 0 factors P Q = L U in its shared memory
// (Gaussian elimination with partial pivoting, first maximal |pivot|) and
// publishes L\U and the row permutation to global scratch; then every CTA
// solves its own block of right-hand-side columns (one thread per column:
// permutation, forward and back substitution from its shared-memory copy of L\U).
// Returns 0, or -1 for a zero pivot (every CTA).
// Q X = R (n <= KMAXM+1, ld LDH, global): CTA 0 factors Q = P L U in shared memory with
// partial pivoting (first maximal |pivot|), static column ownership (warp c mod nw owns
// column c: swaps and updates need only __syncwarp), ONE __syncthreads per step, the
// owner of column k+1 searching step k+1's pivot right after its update (look-ahead).
// L is kept in elimination order (no later row swaps of its columns), so the forward
// solve applies swap k right before eliminating with column k (LAPACK getrs order).
// Then every CTA solves its block of right-hand-side columns, one warp per column, the
// column in registers (rows lane + 32 j), pivots broadcast by shuffles.  Returns 0 or
// -1 (zero pivot) in every thread of the cluster.
#define CL_RS 5  // row slots per lane: n <= 160
__device__ int cl_solve(int n, const double *Qg, double *R, double *LUg, int *piv, int *flag, double *sm) {
  double *sQ = sm;  // n x n, ld = n
  const int rank = (int)cl_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ int s_piv[LDH];
  __shared__ int s_bad;
  if (rank == 0) {
    for (int c = warp; c < n; c += nw)
      for (int r = lane; r < n; r += 32) sQ[r + n * c] = __ldcg(Qg + r + (size_t)LDH * c);
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    // pivot of step k on column k (up to date), by its owner warp
    auto pivot = [&](int k) {
      double *C = sQ + n * k;
      double vb = -1.0;
      int rb = n;
#pragma unroll
      for (int j = 0; j < CL_RS; j++) {
        const int r = k + lane + 32 * j;
        const double a = r < n ? fabs(C[r]) : -1.0;
        if (a > vb) { vb = a; rb = r; }  // (rows ascend with j: ties keep the first)
      }
      const unsigned long long bits = vb >= 0.0 ? (unsigned long long)__double_as_longlong(vb) : 0ull;
      const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
      const unsigned mhi = __reduce_max_sync(0xffffffffu, vb >= 0.0 ? hi : 0u);
      const bool onhi = vb >= 0.0 && hi == mhi;
      const unsigned mlo = __reduce_max_sync(0xffffffffu, onhi ? lo : 0u);
      const bool top = onhi && lo == mlo;
      const int bi = (int)__reduce_min_sync(0xffffffffu, top ? (unsigned)rb : 0x7fffffffu);
      const double best = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
      if (!(best > 0.0) || bi >= n) {
        if (lane == 0) s_bad = 1;
        return;
      }
      const double pv = C[bi], ck = C[k];
      __syncwarp();
      if (lane == 0) { C[bi] = ck; C[k] = pv; }
      __syncwarp();
      const double rp = __drcp_rn(pv);
#pragma unroll
      for (int j = 0; j < CL_RS; j++) {
        const int r = k + 1 + lane + 32 * j;
        if (r < n) C[r] *= rp;  // multipliers l_r
      }
      if (lane == 0) s_piv[k] = bi;
      __syncwarp();
    };
#ifdef KIOPS_PHASE_DEBUG
    const long long f0 = clock64();
#endif
// swap rows k <-> pv of column X and subtract l_r x_k from rows r > k (__syncwarp only:
// the column is this warp's; batching several columns per round trip spilled and was slower)
#define CL_UPDATE(X)                                                 \
  {                                                                  \
    double *const Xc = (X);                                          \
    const double xk = Xc[pv], xo = Xc[k];                            \
    double xv[CL_RS];                                                \
    _Pragma("unroll") for (int j = 0; j < CL_RS; j++) {              \
      const int r = k + 1 + lane + 32 * j;                           \
      xv[j] = r < n ? (r == pv ? xo : Xc[r]) : 0.0;                  \
    }                                                                \
    __syncwarp();                                                    \
    if (lane == 0) Xc[k] = xk;                                       \
    _Pragma("unroll") for (int j = 0; j < CL_RS; j++) {              \
      const int r = k + 1 + lane + 32 * j;                           \
      if (r < n) Xc[r] = xv[j] - l[j] * xk;                          \
    }                                                                \
    __syncwarp();                                                    \
  }
    if (warp == 0) pivot(0);
    __syncthreads();
    // Step k needs column k (multipliers) and s_piv[k], final once its owner has run
    // pivot(k); every other column is written by its own warp only.  So the hand-off is
    // split: the owner of column k+1 ARRIVES at a named barrier right after pivot(k+1) and
    // only then updates its other columns; the other warps wait for it at the top of step
    // k+1.  The step chain is update(column k+1) + pivot(k+1), not the slowest warp's
    // whole trailing update (blockDim.x = 512: 15 warps sync, the owner arrives).
    const bool split = blockDim.x == 512;
    for (int k = 0; k < n; k++) {
      if (split && k > 0 && (k % nw) != warp) nb_sync512(1 + (k & 1));
      if (s_bad) break;
      const int pv = s_piv[k];
      double l[CL_RS];
#pragma unroll
      for (int j = 0; j < CL_RS; j++) {
        const int r = k + 1 + lane + 32 * j;
        l[j] = r < n ? sQ[r + n * k] : 0.0;
      }
      int c = k + 1 + ((warp - (k + 1)) % nw + nw) % nw;  // first owned column > k
      if (c == k + 1 && c < n) {
        CL_UPDATE(sQ + n * c);
        pivot(k + 1);
        __syncwarp();
        if (split) nb_arrive512(1 + ((k + 1) & 1));
        c += nw;
      }
      for (; c < n; c += nw) CL_UPDATE(sQ + n * c);
      if (!split) __syncthreads();
    }
    __syncthreads();
#undef CL_UPDATE
#ifdef KIOPS_PHASE_DEBUG
    if (threadIdx.x == 0) printf("cl_solve n=%d factor cycles %lld\n", n, clock64() - f0);
#endif
    // L into final row order: column c gets the swaps of the later steps k > c (thread
    // per column), so P Q = L U with P from the same swap sequence
    if (!s_bad)
      for (int c = threadIdx.x; c < n - 1; c += blockDim.x)
        for (int k = c + 1; k < n; k++) {
          const int pk = s_piv[k];
          if (pk != k) { const double t = sQ[k + n * c]; sQ[k + n * c] = sQ[pk + n * c]; sQ[pk + n * c] = t; }
        }
    __syncthreads();
    for (int c = warp; c < n; c += nw)
      for (int r = lane; r < n; r += 32) LUg[r + n * c] = sQ[r + n * c];
    if (threadIdx.x == 0) {  // row i of P Q is row perm[i] of Q
      for (int i = 0; i < n; i++) piv[i] = i;
      for (int k = 0; k < n; k++) { const int pk = s_piv[k], t = piv[k]; piv[k] = piv[pk]; piv[pk] = t; }
      *flag = s_bad;
    }
  }
#ifdef KIOPS_PHASE_DEBUG
  const long long s0 = clock64();
#endif
  cl_sync();
  if (__ldcg(flag)) return -1;
#ifdef KIOPS_PHASE_DEBUG
  const long long s1 = clock64();
#endif
  const int cb = (n + CTRL_CL - 1) / CTRL_CL, c0 = rank * cb, c1 = min(n, c0 + cb);
  if (c0 < n) {
    for (int c = warp; c < n; c += nw)
      for (int r = lane; r < n; r += 32) sQ[r + n * c] = __ldcg(LUg + r + n * c);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s_piv[k] = __ldcg(piv + k);
  }
  __syncthreads();
#ifdef KIOPS_PHASE_DEBUG
  const long long s2 = clock64();
#endif
  // 1/U(k,k) for the back substitution
  double *s_rdg = sm + (size_t)n * n;
  if (c0 < n)
    for (int k = threadIdx.x; k < n; k += blockDim.x) s_rdg[k] = 1.0 / sQ[k + n * k];
  __syncthreads();
  static_assert(CL_RS == 5, "row slots");
  for (int c = c0 + warp; c < c1; c += nw) {
    double x[CL_RS];
#pragma unroll
    for (int j = 0; j < CL_RS; j++) {  // P b
      const int r = lane + 32 * j;
      x[j] = r < n ? __ldcg(R + s_piv[r] + (size_t)LDH * c) : 0.0;
    }
    // forward: L y = P b (unit lower); row block kb of the pivots is register x[kb]
#pragma unroll
    for (int kb = 0; kb < CL_RS; kb++)
      for (int kk = 0; kk < 32; kk++) {
        const int k = 32 * kb + kk;
        if (k >= n) break;
        const double xk = __shfl_sync(0xffffffffu, x[kb], kk);
        const double *Lk = sQ + n * k;
#pragma unroll
        for (int j = kb; j < CL_RS; j++) {
          const int r = lane + 32 * j;
          if (r > k && r < n) x[j] -= Lk[r] * xk;
        }
      }
    // back: U x = y
#pragma unroll
    for (int kb = CL_RS - 1; kb >= 0; kb--)
      for (int kk = 31; kk >= 0; kk--) {
        const int k = 32 * kb + kk;
        if (k >= n) continue;
        const double xk = __shfl_sync(0xffffffffu, x[kb], kk) * s_rdg[k];
        const double *Uk = sQ + n * k;
        if (lane == kk) x[kb] = xk;
#pragma unroll
        for (int j = 0; j <= kb; j++) {
          const int r = lane + 32 * j;
          if (r < k) x[j] -= Uk[r] * xk;
        }
      }
#pragma unroll
    for (int j = 0; j < CL_RS; j++) {
      const int r = lane + 32 * j;
      if (r < n) R[r + (size_t)LDH * c] = x[j];
    }
  }
#ifdef KIOPS_PHASE_DEBUG
  const long long s3 = clock64();
  if (threadIdx.x == 0 && (rank == 0 || rank == CTRL_CL - 1))
    printf("cl_solve n=%d rank %d: wait %lld copy %lld trsv %lld\n", n, rank, s1 - s0, s2 - s1, s3 - s2);
#endif
  cl_sync();
  return 0;
}

// ---------------------------------------------------------------------------
// Storage / synchronisation policies for the Pade exponential:
//  * ClusterBk: matrices in global scratch (ld = LDH), work split over the cluster;
//  * SmemBk:    n <= SMALL_N, every matrix in ONE CTA's shared memory (ld = SM_LD),
//               __syncthreads only (used by CTA 0 alone for the small projected
//               matrices of configs 1-3, where cluster barriers would dominate).
// ---------------------------------------------------------------------------
#define SMALL_N 48

struct ClusterBk {
  double *scr, *sm;
  __device__ int ld() const { return LDH; }
  __device__ double *mat(int i) const { return scr + (size_t)i * LDH * LDH; }
  __device__ int gid() const { return cl_gtid(); }
  __device__ int gsz() const { return cl_gsize(); }
  __device__ void sync() const { cl_sync(); }
  // elementwise loops: e in [0, ecount) -> (i, j); false: not an element
  __device__ int ecount(int n) const { return n * n; }
  __device__ bool eindex(int n, int e, int &i, int &j) const { j = e / n; i = e - j * n; return true; }
  __device__ void matmul(int n, const double *A, const double *B, double *C) const { cl_matmul(n, A, B, C, sm); }
  __device__ double norm1(int n, const double *A) const { return cta_norm1(n, A, sm); }
  __device__ int solve(int n, const double *Q, double *R) const {
    return cl_solve(n, Q, R, scr + 10 * (size_t)LDH * LDH, reinterpret_cast<int *>(scr + 11 * (size_t)LDH * LDH),
                    reinterpret_cast<int *>(scr + 11 * (size_t)LDH * LDH) + LDH, sm);
  }
};

// Single-CTA policy (n <= SMALL_N): column-major matrices with leading dimension
// SM_LD = 52 (= 4 mod 16: the m8n8k4 fragment loads below are bank-conflict free),
// zero-padded to NP = n rounded up to 8 (products of zero-padded operands keep the
// padding zero, so the elementwise steps may stay on the n x n part).
#define SM_LD 52
#ifndef KIOPS_LU1W_MAXN
#define KIOPS_LU1W_MAXN 24  // n <= this: the LU by one warp (full-row swaps, no block barrier per
                            // step): 34.1 vs 38.6 k cycles per exponential at n = 12, 55 vs 59 k at
                            // n = 20, slower from n ~ 36 (scripts/mb_expm.cu)
#endif
#ifndef KIOPS_SMALL_MM_INLINE
#define KIOPS_SMALL_MM_INLINE __noinline__  // one copy of the small product for the 10+ call sites of
                                            // pade_expm (instruction-cache footprint)
#endif
#ifndef KIOPS_SOLVE3
#define KIOPS_SOLVE3 1  // small-n solve with the augmented matrix in registers (solve3 below)
#endif
#ifndef KIOPS_SOLVE2
#define KIOPS_SOLVE2 1  // small-n substitution: unit upper U', two right-hand sides per warp
                        // (114.7 vs 122.1 k cycles per exponential at n = 36)
#endif
struct SmemBk {
  double *base;   // 10 matrices of SM_LD x SMALL_N (ld = SM_LD) + reduction scratch
  int n_;
  __device__ int ld() const { return SM_LD; }
  __device__ double *mat(int i) const { return base + (size_t)i * SM_LD * SMALL_N; }
  __device__ int gid() const { return threadIdx.x; }
  __device__ int gsz() const { return blockDim.x; }
  __device__ void sync() const { __syncthreads(); }
  // elementwise loops run over the stored columns (constant leading dimension: no
  // runtime integer division per element); padding rows are skipped
  __device__ int ecount(int n) const { return SM_LD * n; }
  __device__ bool eindex(int n, int e, int &i, int &j) const { j = e / SM_LD; i = e - j * SM_LD; return i < n; }
  // zero the 10 matrices (padding included); call before the first use for this n
  __device__ void clear() const {
    for (int e = threadIdx.x; e < 10 * SM_LD * SMALL_N; e += blockDim.x) base[e] = 0.0;
    __syncthreads();
  }
  // C = A B on the FP64 tensor cores: one warp per 8 x 8 output tile (up to 3 tiles
  // per warp interleaved), k in steps of 4.  Fragments (PTX m8n8k4 .f64): A row
  // g = lane/4, col t = lane%4; B row t, col g; C row g, cols 2t, 2t+1.
  __device__ KIOPS_SMALL_MM_INLINE void matmul(int n, const double *A, const double *B, double *C) const {
    const int np = (n + 7) & ~7, nt = np >> 3, ntile = nt * nt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int g = lane >> 2, tq = lane & 3;
    for (int t0 = warp; t0 < ntile; t0 += 3 * nw) {
      double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      int ti[3], tj[3];
      bool on[3];
      const float rnt = __frcp_rn((float)nt);
#pragma unroll
      for (int u = 0; u < 3; u++) {
        const int tt = t0 + u * nw;
        on[u] = tt < ntile;
        // tt / nt for tt < 64, nt <= 8 without an integer division: (tt + 1/2) / nt is at
        // least 1 / (2 nt) away from an integer
        const int qd = __float2int_rz(((float)tt + 0.5f) * rnt);
        ti[u] = on[u] ? (tt - qd * nt) * 8 : 0;
        tj[u] = on[u] ? qd * 8 : 0;
      }
      for (int k0 = 0; k0 < np; k0 += 4) {
#pragma unroll
        for (int u = 0; u < 3; u++)
          if (on[u]) {
            const double a = A[(ti[u] + g) + SM_LD * (k0 + tq)];
            const double b = B[(k0 + tq) + SM_LD * (tj[u] + g)];
            dmma_8x8x4(c[u], a, b);
          }
      }
#pragma unroll
      for (int u = 0; u < 3; u++)
        if (on[u]) {
          C[(ti[u] + g) + SM_LD * (tj[u] + 2 * tq)] = c[u][0];
          C[(ti[u] + g) + SM_LD * (tj[u] + 2 * tq + 1)] = c[u][1];
        }
    }
    __syncthreads();
  }
  // (column sums in ascending row order, as the oracle's: the degree / scaling decision
  // compares this norm with the theta thresholds)
  __device__ double norm1(int n, const double *A) const {
    double *red = base + 10 * (size_t)SM_LD * SMALL_N;
    double best = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double s = 0.0;
#pragma unroll 8
      for (int i = 0; i < n; i++) s += fabs(A[i + SM_LD * j]);
      best = (s > best || s != s) ? s : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, best, o);
      best = (x > best || x != x) ? x : best;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) red[warp] = best;
    __syncthreads();
    double bb = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, bb, o);
      bb = (x > bb || x != x) ? x : bb;
    }
    __syncthreads();
    return bb;
  }
  // Register-resident solve (KIOPS_SOLVE3, the default): Gaussian elimination with
  // partial pivoting of the augmented matrix [Q | R], columns dealt to the warps (Q
  // column c and R column c in warp c mod 16, up to 3 + 3 per warp for n <= 48),
  // lane = row (rows lane, lane + 32), every entry in registers.  Rows are never moved:
  // each lane knows the step at which its rows were pivoted (implicit pivoting: the
  // maximal |value| among the rows not yet pivoted; exactly equal |values| -- which a
  // swapped scheme would break by position -- are broken by the lowest row index).  Step k: the owner of column k
  // updates that column first, finds the pivot (one 32-bit max reduction in the common
  // case), publishes the multipliers by row and the pivot row in shared memory and
  // ARRIVES at a named barrier (bar.arrive, non-blocking); the other warps bar.sync on
  // it, read the multipliers and update all their columns with one shuffle (the pivot
  // row's entry) per column, branch free (finished columns and finished rows see zero
  // multipliers).  So the dependency chain of a step is the owner's column update +
  // search only; the remaining updates overlap the next step's chain.  Eliminating
  // [Q | R] together is the forward substitution L y = P b.  Then U is scaled to unit
  // diagonal and written to shared memory (over Q), and every warp back substitutes
  // its right-hand-side columns from registers (one shuffle + one fma per step and
  // column on the dependency chain).  Same operations as LU + substitution.
  // Q is destroyed.  Returns 0 or -1 (zero / non-finite pivot column), all threads.
  // Requires 16 warps (CTRL_THREADS = 512).
  static __device__ __forceinline__ void nb_sync(int id) { nb_sync512(id); }
  static __device__ __forceinline__ void nb_arrive(int id) { nb_arrive512(id); }
  // shared-memory accesses by 32-bit shared address (the step chain carries no generic
  // address arithmetic)
  static __device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
  }
  static __device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
  }
  static __device__ __forceinline__ void sts_f64(unsigned a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
  }
  static __device__ __forceinline__ void sts_s32(unsigned a, int v) {
    asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
  }
  __device__ __noinline__ int solve3(int n, double *Q, double *R) const {
    constexpr int NS = 3, NW = 16;
    // per-step publication, double buffered: [buf][0..63] multipliers by row, [buf][64] pivot row
    __shared__ __align__(16) double s_pub[2][66];
    __shared__ double s_rd3[SMALL_N];
    __shared__ int s_prow[SMALL_N];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool r0ok = lane < n, r1ok = lane + 32 < n;
    unsigned pub0 = (unsigned)__cvta_generic_to_shared(&s_pub[0][0]);
    asm volatile("" : "+r"(pub0));  // (opaque: not rematerialised inside the step chain)
    const unsigned pubsz = 66 * 8;
    double q0[NS], q1[NS], y0[NS], y1[NS];  // Q and R columns warp + 16 i, rows lane / lane + 32
#pragma unroll
    for (int i = 0; i < NS; i++) {
      const int c = warp + NW * i;
      q0[i] = (c < n && r0ok) ? Q[lane + SM_LD * c] : 0.0;
      q1[i] = (c < n && r1ok) ? Q[lane + 32 + SM_LD * c] : 0.0;
      y0[i] = (c < n && r0ok) ? R[lane + SM_LD * c] : 0.0;
      y1[i] = (c < n && r1ok) ? R[lane + 32 + SM_LD * c] : 0.0;
    }
    // live0/1: my rows not yet pivoted (rows >= n never are); ps0/1: their pivot steps
    bool live0 = r0ok, live1 = r1ok;
    int ps0 = 0x7fffffff, ps1 = 0x7fffffff;
    // pivot search of step k on column values x0, x1 (owner warp): first maximal |value|
    // among the live rows (ties: the lowest row), published into buffer k & 1
    auto search = [&](int k, double x0, double x1) {
      const double v0 = live0 ? fabs(x0) : -1.0, v1 = live1 ? fabs(x1) : -1.0;
      const bool useb = v1 > v0;
      const double v = useb ? v1 : v0;
      const bool ok = v >= 0.0;  // (false for NaN and for rows already pivoted)
      const unsigned hi = ok ? (unsigned)__double2hiint(v) : 0u;
      const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
      bool cand = ok && hi == mhi;
      unsigned m = __ballot_sync(0xffffffffu, cand);
      if (m & (m - 1)) {  // several lanes share the high word
        const unsigned lo = cand ? (unsigned)__double2loint(v) : 0u;
        const unsigned mlo = __reduce_max_sync(0xffffffffu, lo);
        cand = cand && lo == mlo;
        m = __ballot_sync(0xffffffffu, cand);
        const unsigned ma = __ballot_sync(0xffffffffu, cand && !useb);  // equal |values|: rows < 32 first
        if (ma) m = ma;
      }
      const int wl = m ? __ffs(m) - 1 : 0;
      const double piv = __shfl_sync(0xffffffffu, useb ? x1 : x0, wl);
      const int rp = wl + (__shfl_sync(0xffffffffu, (int)useb, wl) ? 32 : 0);
      const bool good = m != 0 && fabs(piv) > 0.0 && fabs(piv) <= 1.7976931348623157e308;
      const double rpiv = __drcp_rn(piv);
      const unsigned pb = pub0 + (k & 1) * pubsz;
      sts_f64(pb + lane * 8, (live0 && lane != rp) ? x0 * rpiv : 0.0);
      sts_f64(pb + (lane + 32) * 8, (live1 && lane + 32 != rp) ? x1 * rpiv : 0.0);
      if (lane == 0) sts_s32(pb + 64 * 8, good ? rp : -1);
      __syncwarp();
      nb_arrive(1 + (k & 1));
      if (lane == 0) {
        s_rd3[k] = rpiv;
        s_prow[k] = rp;
      }
    };
    if (warp == 0) search(0, q0[0], q1[0]);
    int bad = 0;
    // step k (k1 = k + 1); IO = k1 / 16, the register slot of column k1 in its owner warp
    auto step = [&](int k1, auto iotag) {
      constexpr int IO = decltype(iotag)::value;
      const int k = k1 - 1;
      if ((k & (NW - 1)) != warp) nb_sync(1 + (k & 1));  // (the owner published L_k itself)
      const unsigned pb = pub0 + (k & 1) * pubsz;
      const int rp = lds_s32(pb + 64 * 8);
      const double l0 = lds_f64(pb + lane * 8), l1 = lds_f64(pb + (lane + 32) * 8);
      if (rp < 0) { bad = 1; return; }
      const int sl = rp & 31;
      const bool hi = rp >= 32;
      if (lane == sl) {
        if (hi) { live1 = false; ps1 = k; } else { live0 = false; ps0 = k; }
      }
      if (k1 < n && (k1 & (NW - 1)) == warp) {  // column k1 first, then its pivot search
        const double xp = __shfl_sync(0xffffffffu, hi ? q1[IO] : q0[IO], sl);
        search(k1, fma(-l0, xp, q0[IO]), fma(-l1, xp, q1[IO]));
      }
#pragma unroll
      for (int i = 0; i < NS; i++) {
        const double xq = __shfl_sync(0xffffffffu, hi ? q1[i] : q0[i], sl);
        const double xy = __shfl_sync(0xffffffffu, hi ? y1[i] : y0[i], sl);
        // (a column c <= k keeps its U entries: their rows were pivoted, l = 0)
        q0[i] = fma(-l0, xq, q0[i]);
        q1[i] = fma(-l1, xq, q1[i]);
        y0[i] = fma(-l0, xy, y0[i]);
        y1[i] = fma(-l1, xy, y1[i]);
      }
    };
    for (int k1 = 1; k1 <= n && k1 < NW && !bad; k1++) step(k1, std::integral_constant<int, 0>{});
    for (int k1 = NW; k1 <= n && k1 < 2 * NW && !bad; k1++) step(k1, std::integral_constant<int, 1>{});
    for (int k1 = 2 * NW; k1 <= n && !bad; k1++) step(k1, std::integral_constant<int, 2>{});
    __syncthreads();
    if (bad) return -1;
    // unit-diagonal U' = D^-1 U (row scaling by the reciprocal pivot of the row's step) to
    // shared memory over Q; y' = D^-1 y stays in registers
    const double d0 = r0ok ? s_rd3[ps0] : 0.0, d1 = r1ok ? s_rd3[ps1] : 0.0;
#pragma unroll
    for (int i = 0; i < NS; i++) {
      const int c = warp + NW * i;
      y0[i] *= d0;
      y1[i] *= d1;
      if (c < n) {
        if (r0ok) Q[lane + SM_LD * c] = q0[i] * d0;
        if (r1ok) Q[lane + 32 + SM_LD * c] = q1[i] * d1;
      }
    }
    __syncthreads();
    // back substitution, column oriented: x_k = y'(row of step k); rows of earlier steps
    // subtract U'(row, k) x_k
#pragma unroll 4
    for (int k = n - 1; k >= 0; k--) {
      const int rp = s_prow[k], sl = rp & 31;
      const bool hi = rp >= 32;
      const double u0 = ps0 < k ? Q[lane + SM_LD * k] : 0.0, u1 = ps1 < k ? Q[lane + 32 + SM_LD * k] : 0.0;
#pragma unroll
      for (int i = 0; i < NS; i++) {
        const double xk = __shfl_sync(0xffffffffu, hi ? y1[i] : y0[i], sl);
        y0[i] = fma(-u0, xk, y0[i]);
        y1[i] = fma(-u1, xk, y1[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < NS; i++) {
      const int c = warp + NW * i;
      if (c < n) {
        if (r0ok) R[ps0 + SM_LD * c] = y0[i];
        if (r1ok) R[ps1 + SM_LD * c] = y1[i];
      }
    }
    __syncthreads();
    return 0;
  }
  __device__ int solve(int n, double *Q, double *R) const {
#if KIOPS_SOLVE3
    if (blockDim.x == 512 && n <= SMALL_N) return solve3(n, Q, R);
#endif
    __shared__ int s_bad, s_piv[SMALL_N], s_perm[SMALL_N];
    __shared__ double s_rd[SMALL_N];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) s_bad = 0;
    auto pivot = [&](int k) {  // owner warp of column k (up to date)
      double *C = Q + SM_LD * k;
      const int ra = k + lane, rb = ra + 32;
      const double va = ra < n ? fabs(C[ra]) : -1.0, vb = rb < n ? fabs(C[rb]) : -1.0;
      const bool useb = vb > va;  // (equal: the lower row ra wins)
      const double v = useb ? vb : va;
      const int rv = useb ? rb : ra;
      const unsigned long long bits = v >= 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
      const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
      const unsigned mhi = __reduce_max_sync(0xffffffffu, v >= 0.0 ? hi : 0u);
      const bool onhi = v >= 0.0 && hi == mhi;
      const unsigned mlo = __reduce_max_sync(0xffffffffu, onhi ? lo : 0u);
      const bool top = onhi && lo == mlo;
      const int bi = (int)__reduce_min_sync(0xffffffffu, top ? (unsigned)rv : 0x7fffffffu);
      const double best = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
      if (!(best > 0.0) || bi >= n) {
        if (lane == 0) s_bad = 1;
        return;
      }
      const double piv = C[bi], ck = C[k];
      __syncwarp();
      if (lane == 0) { C[bi] = ck; C[k] = piv; }
      __syncwarp();
      const double rp = __drcp_rn(piv);
      if (ra > k && ra < n) C[ra] *= rp;  // multipliers l_r
      if (rb < n) C[rb] *= rp;
      if (lane == 0) { s_piv[k] = bi; s_rd[k] = rp; }
      __syncwarp();
    };
if (n <= KIOPS_LU1W_MAXN) {
    // one warp, everything in shared memory, no block barrier per step: pivot search (first
    // maximal |pivot|, as the block version), LAPACK-style swap of the FULL rows k and pivot
    // (L's columns included, so no reordering afterwards), multipliers by the reciprocal
    // pivot, rank-1 update of the trailing block with each lane owning rows r, r + 32
    if (warp == 0) {
      for (int k = 0; k < n; k++) {
        const double *C = Q + SM_LD * k;
        const int ra = k + lane, rb = ra + 32;
        const double va = ra < n ? fabs(C[ra]) : -1.0, vb = rb < n ? fabs(C[rb]) : -1.0;
        const bool useb = vb > va;
        const double v = useb ? vb : va;
        const int rv = useb ? rb : ra;
        const unsigned long long bits = v >= 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
        const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, v >= 0.0 ? hi : 0u);
        const bool onhi = v >= 0.0 && hi == mhi;
        const unsigned mlo = __reduce_max_sync(0xffffffffu, onhi ? lo : 0u);
        const bool top = onhi && lo == mlo;
        const int bi = (int)__reduce_min_sync(0xffffffffu, top ? (unsigned)rv : 0x7fffffffu);
        const double best = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
        if (!(best > 0.0) || bi >= n) {
          if (lane == 0) s_bad = 1;
          break;
        }
        if (bi != k)
          for (int c = lane; c < n; c += 32) {
            const double t = Q[k + SM_LD * c];
            Q[k + SM_LD * c] = Q[bi + SM_LD * c];
            Q[bi + SM_LD * c] = t;
          }
        __syncwarp();
        const double rp = __drcp_rn(Q[k + SM_LD * k]);
        const int r0 = k + 1 + lane, r1 = r0 + 32;
        const double l0 = r0 < n ? Q[r0 + SM_LD * k] * rp : 0.0, l1 = r1 < n ? Q[r1 + SM_LD * k] * rp : 0.0;
        if (r0 < n) Q[r0 + SM_LD * k] = l0;
        if (r1 < n) Q[r1 + SM_LD * k] = l1;
        if (lane == 0) { s_piv[k] = bi; s_rd[k] = rp; }
#pragma unroll 4
        for (int c = k + 1; c < n; c++) {
          double *Xc = Q + SM_LD * c;
          const double u = Xc[k];
          if (r0 < n) Xc[r0] = fma(-l0, u, Xc[r0]);
          if (r1 < n) Xc[r1] = fma(-l1, u, Xc[r1]);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (s_bad) return -1;
    if (threadIdx.x == 0) {  // row i of P Q is row perm[i] of Q
      for (int i = 0; i < n; i++) s_perm[i] = i;
      for (int k = 0; k < n; k++) { const int pk = s_piv[k], t = s_perm[k]; s_perm[k] = s_perm[pk]; s_perm[pk] = t; }
    }
    __syncthreads();
} else {
    if (warp == 0) pivot(0);
    __syncthreads();
    for (int k = 0; k < n; k++) {
      if (s_bad) return -1;
      const int pv = s_piv[k];
      const int r0 = k + 1 + lane, r1 = r0 + 32;
      const double l0 = r0 < n ? Q[r0 + SM_LD * k] : 0.0, l1 = r1 < n ? Q[r1 + SM_LD * k] : 0.0;
      int c = k + 1 + ((warp - (k + 1)) % nw + nw) % nw;  // first owned column > k
#define SB_UPDATE(X)                                                   \
  {                                                                    \
    double *const Xc = (X);                                            \
    const double xk = Xc[pv], xo = Xc[k];                              \
    const double x0 = r0 < n ? (r0 == pv ? xo : Xc[r0]) : 0.0;         \
    const double x1 = r1 < n ? (r1 == pv ? xo : Xc[r1]) : 0.0;         \
    __syncwarp();                                                      \
    if (lane == 0) Xc[k] = xk;                                         \
    if (r0 < n) Xc[r0] = x0 - l0 * xk;                                 \
    if (r1 < n) Xc[r1] = x1 - l1 * xk;                                 \
    __syncwarp();                                                      \
  }
      if (c == k + 1 && c < n) {
        SB_UPDATE(Q + SM_LD * c);
        pivot(k + 1);
        c += nw;
      }
      for (; c < n; c += nw) SB_UPDATE(Q + SM_LD * c);
#undef SB_UPDATE
      __syncthreads();
    }
    // L into final row order (thread per column), permutation of the right-hand sides
    for (int c = threadIdx.x; c < n - 1; c += blockDim.x)
      for (int k = c + 1; k < n; k++) {
        const int pk = s_piv[k];
        if (pk != k) { const double t = Q[k + SM_LD * c]; Q[k + SM_LD * c] = Q[pk + SM_LD * c]; Q[pk + SM_LD * c] = t; }
      }
    if (threadIdx.x == 0) {
      for (int i = 0; i < n; i++) s_perm[i] = i;
      for (int k = 0; k < n; k++) { const int pk = s_piv[k], t = s_perm[k]; s_perm[k] = s_perm[pk]; s_perm[pk] = t; }
    }
    __syncthreads();
}
#if KIOPS_SOLVE2
    // U' = D^-1 U: row k of U scaled by 1/u_kk (the reciprocal pivots), so the back
    // substitution is unit upper triangular and no multiply sits on its dependency chain
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int r = e % n, c = e / n;
      if (c > r) Q[r + SM_LD * c] *= s_rd[r];
    }
    __syncthreads();
    // two right-hand-side columns per warp (two independent substitution chains);
    // operands loaded as zeros where the triangle has none, so the updates are branch free
    for (int c0 = 2 * warp; c0 < n; c0 += 2 * nw) {
      const bool two = c0 + 1 < n;
      double *Ra = R + SM_LD * c0, *Rb = R + SM_LD * (two ? c0 + 1 : c0);
      double a0 = lane < n ? Ra[s_perm[lane]] : 0.0, a1 = lane + 32 < n ? Ra[s_perm[lane + 32]] : 0.0;
      double b0 = lane < n ? Rb[s_perm[lane]] : 0.0, b1 = lane + 32 < n ? Rb[s_perm[lane + 32]] : 0.0;
#pragma unroll 4
      for (int k = 0; k < n; k++) {  // L y = P b (unit lower)
        const double *Lk = Q + SM_LD * k;
        const double l0 = (lane > k && lane < n) ? Lk[lane] : 0.0;
        const double l1 = (lane + 32 > k && lane + 32 < n) ? Lk[lane + 32] : 0.0;
        const double ya = __shfl_sync(0xffffffffu, k < 32 ? a0 : a1, k & 31);
        const double yb = __shfl_sync(0xffffffffu, k < 32 ? b0 : b1, k & 31);
        a0 = fma(-l0, ya, a0); a1 = fma(-l1, ya, a1);
        b0 = fma(-l0, yb, b0); b1 = fma(-l1, yb, b1);
      }
      const double d0 = lane < n ? s_rd[lane] : 0.0, d1 = lane + 32 < n ? s_rd[lane + 32] : 0.0;
      a0 *= d0; a1 *= d1; b0 *= d0; b1 *= d1;
#pragma unroll 4
      for (int k = n - 1; k >= 0; k--) {  // U' x = D^-1 y (unit upper)
        const double *Uk = Q + SM_LD * k;
        const double u0 = lane < k ? Uk[lane] : 0.0, u1 = lane + 32 < k ? Uk[lane + 32] : 0.0;
        const double xa = __shfl_sync(0xffffffffu, k < 32 ? a0 : a1, k & 31);
        const double xb = __shfl_sync(0xffffffffu, k < 32 ? b0 : b1, k & 31);
        a0 = fma(-u0, xa, a0); a1 = fma(-u1, xa, a1);
        b0 = fma(-u0, xb, b0); b1 = fma(-u1, xb, b1);
      }
      __syncwarp();
      if (lane < n) Ra[lane] = a0;
      if (lane + 32 < n) Ra[lane + 32] = a1;
      if (two) {
        if (lane < n) Rb[lane] = b0;
        if (lane + 32 < n) Rb[lane + 32] = b1;
      }
    }
#else
    for (int c = warp; c < n; c += nw) {
      double *Rc = R + SM_LD * c;
      double x0 = lane < n ? Rc[s_perm[lane]] : 0.0, x1 = lane + 32 < n ? Rc[s_perm[lane + 32]] : 0.0;
      for (int k = 0; k < n; k++) {  // L y = P b (unit lower)
        const double xk = __shfl_sync(0xffffffffu, k < 32 ? x0 : x1, k & 31);
        const double *Lk = Q + SM_LD * k;
        if (lane > k && lane < n) x0 -= Lk[lane] * xk;
        if (lane + 32 > k && lane + 32 < n) x1 -= Lk[lane + 32] * xk;
      }
      for (int k = n - 1; k >= 0; k--) {  // U x = y
        const double xk = __shfl_sync(0xffffffffu, k < 32 ? x0 : x1, k & 31) * s_rd[k];
        const double *Uk = Q + SM_LD * k;
        if (lane == (k & 31)) { if (k < 32) x0 = xk; else x1 = xk; }
        if (lane < k) x0 -= Uk[lane] * xk;
        if (lane + 32 < k) x1 -= Uk[lane + 32] * xk;
      }
      __syncwarp();
      if (lane < n) Rc[lane] = x0;
      if (lane + 32 < n) Rc[lane + 32] = x1;
    }
#endif
    __syncthreads();
    return 0;
  }
};

// [m/m] Pade numerator coefficients p_m(x) = sum b_j x^j, b_j proportional to
// (2m-j)! m! / ((2m)! j! (m-j)!), integer-scaled as tabulated by Higham (2005);
// rows m = 3, 5, 7, 9, 13.
__constant__ double kPade[5][14] = {
    {120.0, 60.0, 12.0, 1.0},
    {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0},
    {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0},
    {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0, 2162160.0, 110880.0, 3960.0, 90.0, 1.0},
    {64764752532480000.0, 32382376266240000.0, 7771770303897600.0, 1187353796428800.0, 129060195264000.0,
     10559470521600.0, 670442572800.0, 33522128640.0, 1323241920.0, 40840800.0, 960960.0, 16380.0, 182.0, 1.0}};

// F = exp(scale * M) for n <= KMAXM+1: diagonal Pade approximant with scaling and
// squaring ("[47]" = Higham 2005, Algorithm 2.3; R17).  Degree cascade
// {3,5,7,9,13} by the 1-norm thresholds theta_m of Higham's Table 2.3; above
// theta_13, X is scaled by 2^-s and squared back s times.  M and F use the
// policy's leading dimension.  Every participant must call it with identical
// arguments.  Returns the number of dense products (or -1 on a zero pivot /
// non-finite norm).
template <class Bk>
__device__ int pade_expm(const Bk &bk, int n, const double *M, double scale, double *F) {
  const int ld = bk.ld();
  double *X = bk.mat(0), *X2 = bk.mat(1), *X4 = bk.mat(2), *X6 = bk.mat(3), *X8 = bk.mat(4), *U = bk.mat(5),
         *V = bk.mat(6), *T = bk.mat(7);
  // [m/m] Pade numerator coefficients (kPade, constant memory: a per-thread local
  // table indexed through a runtime pointer costs local-memory round trips).
  const int g0 = bk.gid(), gs = bk.gsz(), cnt = bk.ecount(n);
  // f(i, j, q) on every element (q = i + ld j), then a barrier
  auto each = [&](auto f) {
    for (int e = g0; e < cnt; e += gs) {
      int i, j;
      if (bk.eindex(n, e, i, j)) f(i, j, (size_t)i + (size_t)ld * j);
    }
    bk.sync();
  };
#ifdef KIOPS_PHASE_DEBUG
  const long long c0 = clock64();
#endif
  each([&](int, int, size_t q) { X[q] = scale * M[q]; });
  const double nrm = bk.norm1(n, X);
  if (!isfinite(nrm)) return -1;
  int deg, s = 0;
  if (nrm <= 1.495585217958292e-2) deg = 3;
  else if (nrm <= 2.539398330063230e-1) deg = 5;
  else if (nrm <= 9.504178996162932e-1) deg = 7;
  else if (nrm <= 2.097847961257068e0) deg = 9;
  else {
    deg = 13;
    s = ceil_log2_exact(nrm / 5.371920351148152e0);
    if (s < 0) s = 0;
    const double f = ldexp(1.0, -s);
    each([&](int, int, size_t q) { X[q] *= f; });
  }
  int mult = 0;
#ifdef KIOPS_PHASE_DEBUG
  const long long cA = clock64();
#endif
  bk.matmul(n, X, X, X2); mult++;
#ifdef KIOPS_PHASE_DEBUG
  const long long cB = clock64();
#endif
  if (deg >= 5) { bk.matmul(n, X2, X2, X4); mult++; }
  if (deg >= 7) { bk.matmul(n, X2, X4, X6); mult++; }
  if (deg == 9) { bk.matmul(n, X4, X4, X8); mult++; }
  if (deg < 13) {
    const double *b = kPade[deg == 3 ? 0 : deg == 5 ? 1 : deg == 7 ? 2 : 3];
    each([&](int i, int j, size_t q) {
      const double id = (i == j) ? 1.0 : 0.0;
      double odd = b[1] * id + b[3] * X2[q], even = b[0] * id + b[2] * X2[q];
      if (deg >= 5) { odd += b[5] * X4[q]; even += b[4] * X4[q]; }
      if (deg >= 7) { odd += b[7] * X6[q]; even += b[6] * X6[q]; }
      if (deg >= 9) { odd += b[9] * X8[q]; even += b[8] * X8[q]; }
      T[q] = odd;
      V[q] = even;
    });
    bk.matmul(n, X, T, U); mult++;   // U = X * odd part
    // (V - U) F = (V + U)
    each([&](int, int, size_t q) {
      T[q] = V[q] - U[q];
      F[q] = V[q] + U[q];
    });
  } else {
    const double *b = kPade[4];
    each([&](int, int, size_t q) {
      T[q] = b[13] * X6[q] + b[11] * X4[q] + b[9] * X2[q];
      X8[q] = b[12] * X6[q] + b[10] * X4[q] + b[8] * X2[q];
    });
    bk.matmul(n, X6, T, U); mult++;
    bk.matmul(n, X6, X8, V); mult++;
    each([&](int i, int j, size_t q) {
      const double id = (i == j) ? 1.0 : 0.0;
      U[q] += b[7] * X6[q] + b[5] * X4[q] + b[3] * X2[q] + b[1] * id;
      V[q] += b[6] * X6[q] + b[4] * X4[q] + b[2] * X2[q] + b[0] * id;
    });
    bk.matmul(n, X, U, X8); mult++;   // odd part: X [ ... ]
    // (V - U) F = (V + U)
    each([&](int, int, size_t q) {
      T[q] = V[q] - X8[q];
      F[q] = V[q] + X8[q];
    });
  }
#ifdef KIOPS_PHASE_DEBUG
  const long long c1 = clock64();
#endif
  if (bk.solve(n, T, F) != 0) return -1;
#ifdef KIOPS_PHASE_DEBUG
  const long long c2 = clock64();
#endif
  for (int k = 0; k < s; k++) {
    double *src = (k & 1) ? T : F, *dst = (k & 1) ? F : T;
    bk.matmul(n, src, src, dst); mult++;
  }
  if (s & 1) {  // result in T
    each([&](int, int, size_t q) { F[q] = T[q]; });
  }
#ifdef KIOPS_PHASE_DEBUG
  if (bk.gid() == 0)
    printf("expm n=%d deg=%d s=%d mult=%d cycles: pade %lld (setup+norm %lld, first product %lld) solve %lld squaring %lld\n",
           n, deg, s, mult, c1 - c0, cA - c0, cB - cA, c2 - c1, clock64() - c2);
#endif
  return mult;
}

// F (global, ld LDH) = exp(scale M), M global (ld LDH).  n > SMALL_N: the whole
// cluster; otherwise CTA 0 alone in shared memory (the others wait at the barrier).
__device__ int cl_expm(int n, const double *M, double scale, double *F, double *scr, double *sm) {
  if (n > SMALL_N) {
    ClusterBk bk{scr, sm};
    return pade_expm(bk, n, M, scale, F);
  }
  if (cl_rank() == 0) {
    SmemBk bk{sm, n};
    double *Ms = bk.mat(8), *Fs = bk.mat(9);
    bk.clear();
    for (int j = threadIdx.x >> 6; j < n; j += blockDim.x >> 6)
      for (int i = threadIdx.x & 63; i < n; i += 64) Ms[i + SM_LD * j] = M[i + (size_t)LDH * j];
    __syncthreads();
    const int r = pade_expm(bk, n, Ms, scale, Fs);
    for (int j = threadIdx.x >> 6; j < n; j += blockDim.x >> 6)
      for (int i = threadIdx.x & 63; i < n; i += 64) F[i + (size_t)LDH * j] = Fs[i + SM_LD * j];
    if (threadIdx.x == 0) reinterpret_cast<int *>(scr + 11 * (size_t)LDH * LDH)[LDH + 1] = r;
  }
  cl_sync();
  return reinterpret_cast<int *>(scr + 11 * (size_t)LDH * LDH)[LDH + 1];
}

// The same with the matrix given by fill(r, c) (every participant, identical values):
// n <= SMALL_N assembles it directly in CTA 0's shared memory (no global round trip, no
// cluster barrier before the exponential); larger n through the global scratch Mh.
template <class Fill>
__device__ int cl_expm_fill(int n, Fill fill, double *Mh, double scale, double *F, double *scr, double *sm) {
  if (n > SMALL_N) {
    for (int e = cl_gtid(); e < n * n; e += cl_gsize()) {
      const int c = e / n, r = e - c * n;
      Mh[r + (size_t)LDH * c] = fill(r, c);
    }
    cl_sync();
    ClusterBk bk{scr, sm};
    return pade_expm(bk, n, Mh, scale, F);
  }
  if (cl_rank() == 0) {
    SmemBk bk{sm, n};
    double *Ms = bk.mat(8), *Fs = bk.mat(9);
    bk.clear();
    for (int j = threadIdx.x >> 6; j < n; j += blockDim.x >> 6)
      for (int i = threadIdx.x & 63; i < n; i += 64) Ms[i + SM_LD * j] = fill(i, j);
    __syncthreads();
    const int r = pade_expm(bk, n, Ms, scale, Fs);
    for (int j = threadIdx.x >> 6; j < n; j += blockDim.x >> 6)
      for (int i = threadIdx.x & 63; i < n; i += 64) F[i + (size_t)LDH * j] = Fs[i + SM_LD * j];
    if (threadIdx.x == 0) reinterpret_cast<int *>(scr + 11 * (size_t)LDH * LDH)[LDH + 1] = r;
  }
  cl_sync();
  return reinterpret_cast<int *>(scr + 11 * (size_t)LDH * LDH)[LDH + 1];
}

// ---------------------------------------------------------------------------
// Alg. 4 with readings R4-R10.  Thread 0 only.
// ---------------------------------------------------------------------------
__device__ int alg4_adapt(bool happy, bool accept, int j, int m, int m_min, int m_max, double tau,
                          double omega, double t_now, double t_end, const DevState *st, double *tau_new) {
  const double gam = 0.9, gam_max = 0.6, delta = 1.4;
  const double rem = accept ? t_end - (t_now + tau) : t_end - t_now;  // R8
  const double om = fmax(omega, 1e-300);
  double ord = (double)j / 4.0;  // R4: model exponent, q + 1 with q = m/4 - 1
  double kap = 2.0;
  if (st->hist_valid) {          // only the preceding rejected attempt of this substep (R5)
    const double omo = fmax(st->omega_old, 1e-300);
    if (j == st->j_old && tau != st->tau_old) {  // Eq. 43 un-inverted (R4)
      const double o = log(om / omo) / log(tau / st->tau_old);
      if (isfinite(o) && o > 0.0) ord = fmax(o, 1.0);
    } else if (j != st->j_old && tau == st->tau_old) {  // Eq. 45 (R6)
      double kk = pow(om / omo, 1.0 / (double)(st->j_old - j));
      if (!(kk >= 1.1)) kk = 1.1;
      if (!(kk <= 10.0)) kk = 10.0;
      kap = kk;
    }
  }
  if (happy) {                   // Alg. 4 l.4-8
    *tau_new = fmin(tau, rem);
    return m;
  }
  if (j == m_max) {
    if (omega > delta) {         // l.10-13
      const double t = fmax(tau / 5.0, tau * pow(gam_max / om, 1.0 / ord));
      *tau_new = fmin(rem, t);
      return j;
    }
    // l.15 -> Sec. 3.6.1, Eq. 44 with gamma = 0.9, clip [tau/5, 5 tau]
    const double t = fmax(tau / 5.0, fmin(5.0 * tau, tau * pow(gam / om, 1.0 / ord)));
    *tau_new = fmin(rem, t);
    return m;
  }
  // l.18 -> Sec. 3.6.2, Eq. 46 with the -25%/+33% clip of P:510 (R7)
  const double x = (double)j + log(om / gam) / log(kap);
  int lo = (3 * j) / 4, hi = (4 * j + 2) / 3;
  lo = lo < m_min ? m_min : lo;
  hi = hi > m_max ? m_max : hi;
  lo = lo > hi ? hi : lo;
  int mn = x >= (double)hi ? hi : (x <= (double)lo ? lo : (int)ceil(x));
  mn = mn < lo ? lo : (mn > hi ? hi : mn);
  *tau_new = fmin(tau, rem);
  return mn;
}

// ---------------------------------------------------------------------------
// The controller: one thread-block cluster per attempt (Alg. 1 l.17-29 + Alg. 3
// bookkeeping).  Every CTA takes part in the dense exponentials; CTA 0 thread 0
// runs the scalar logic and broadcasts its decisions through global memory +
// cluster barriers, so all CTAs follow the same control flow.
// ---------------------------------------------------------------------------
__global__ void __cluster_dims__(CTRL_CL, 1, 1) __launch_bounds__(CTRL_THREADS, 1) k_ctrl(KParams P) {
  extern __shared__ double sm[];
  DevState *st = P.st;
  const CallBlock *call = P.call;
  double *Mh = P.scratch + 8 * (size_t)LDH * LDH;  // H~ / H_j input
  double *F = P.scratch + 9 * (size_t)LDH * LDH;   // exponential output
  double *scr = P.scratch;                          // work matrices
  const unsigned rank = cl_rank();
  const bool lead = rank == 0 && threadIdx.x == 0;
  const unsigned long long t_start = gtimer();
#ifdef KIOPS_PHASE_DEBUG
  unsigned long long tph[8] = {t_start, 0, 0, 0, 0, 0, 0, 0};
#define CTRL_STAMP(i) tph[i] = gtimer()
#else
#define CTRL_STAMP(i) do { } while (0)
#endif

  // phase 0: every thread reads the same state
  const int stop = (st->status != 0 || st->npass < 1) ? 1 : (st->zero_start ? 2 : 0);
  const double t_now = st->t_now, t_end = st->t_end, beta = st->beta;
  const double rem0 = t_end - t_now;  // R11: never step past T_end
  const bool final_ = st->tau >= rem0;
  const double tau = final_ ? rem0 : st->tau;
  const int j = st->npass - 1, happy = st->happy, l0 = st->l;
  cl_sync();  // nobody writes the state before everyone has read it
  CTRL_STAMP(1);

  if (stop == 1) {
    if (lead) {
      if (st->status == 0) st->status = KIOPS_ERR_CUDA;
      set_cond(P, COND_OUTER, 0u); set_cond(P, COND_INNER, 0u); set_cond(P, COND_ACCEPT, 0u);
    }
    return;
  }
  if (stop == 2) {  // R27: zero start vector => every remaining output is 0
    if (lead) {
      int o = 0;
      for (int l = st->l; l < call->n_out; l++) st->gemv_out[o++] = call->w[l];
      st->gemv_nout = o;
      st->gemv_j = 0;
      st->gemv_x1 = st->x1;
      st->l = call->n_out - 1;
      st->t_now = st->t_end;
      // (no attempt took place: counters and trace stay as the oracle's, R27)
      set_cond(P, COND_OUTER, 0u); set_cond(P, COND_INNER, 0u); set_cond(P, COND_ACCEPT, 1u);
    }
    return;
  }
  const int n1 = j + 1;
  // R1 / Eq. 37: H~ = [[H(1:j,1:j), e_1],[0, 0]] from the IOP band (rows c-q+1 .. c+1)
  auto htilde = [&](int r, int c) -> double {
    double v = 0.0;
    if (r < j && c < j && r >= c - P.q + 1 && r <= c + 1) v = P.H[r + (size_t)LDH * c];  // IOP band
    if (r == 0 && c == j) v = 1.0;
    return v;
  };
  CTRL_STAMP(2);
  const unsigned long long t_e0 = gtimer();
  const int nm = cl_expm_fill(n1, htilde, Mh, tau, F, scr, sm);  // Alg. 1 l.18
  CTRL_STAMP(3);
  if (lead) {
    st->ns_expm += gtimer() - t_e0;
    st->tau = tau;
    st->expm_calls++;
    double eps = 0.0, omega = 0.0, h_next = 0.0;
    if (nm < 0) st->status = KIOPS_ERR_NONFINITE;
    if (!happy) {  // Eq. 36 via Eq. 38: entry (j, j+1); Eq. 39
      h_next = P.H[j + (size_t)LDH * (j - 1)];
      eps = beta * h_next * fabs(F[(j - 1) + (size_t)LDH * j]);
      omega = t_end * eps / (tau * P.tol);
    }
    if (!isfinite(omega)) st->status = KIOPS_ERR_NONFINITE;
    const long long att = st->attempt;
    const bool forced = att < call->n_forced;
    const bool acc = forced ? (call->forced_acc[att] != 0) : (omega <= 1.4);  // P:425 (R10)
    double tau_new = tau;
    int m_new = st->m;
    if (!forced)
      m_new = alg4_adapt(happy, acc, j, st->m, P.m_min, P.m_max, tau, omega, t_now, t_end, st, &tau_new);
    if (att < KIOPS_TRACE_CAP) {
      kiops_trace_row &tr = P.trace[att];
      tr.attempt = att; tr.j = j; tr.happy = happy; tr.accept = acc; tr.m_new = m_new;
      tr.t_now = t_now; tr.tau = tau; tr.beta = beta; tr.h_next = h_next; tr.eps = eps;
      tr.omega = omega; tr.tau_new = tau_new;
    }
    const bool accept = acc && st->status == 0;
    // Alg. 3 l.2-9: outputs crossed by this substep (strict <, R16; all tasks, R15)
    int n_tau = 0;
    if (accept) {
      const double T_next = t_now + tau;
      for (int k = l0; k < call->n_out; k++)
        if (fabs(call->T[k]) < fabs(T_next)) n_tau++;
      st->substeps++;
      if (happy) st->happy_count++;
      st->hist_valid = 0;
    } else if (st->status == 0) {
      st->rejections++;
      st->hist_valid = 1;
      st->omega_old = omega; st->tau_old = tau; st->j_old = j;
    }
    st->attempt = att + 1;
    if (att + 1 < call->n_forced) {
      tau_new = call->forced_tau[att + 1];
      const int fm = call->forced_m[att + 1];
      m_new = fm < 1 ? 1 : (fm > P.m_max ? P.m_max : fm);
    }
    st->tau = tau_new;
    st->m = m_new;
    st->final_m = m_new;
    st->bc_accept = accept;
    st->bc_ntau = n_tau;
  }
  CTRL_STAMP(4);
  cl_sync();
  const int accept = st->bc_accept, n_tau = st->bc_ntau;
  CTRL_STAMP(5);
  if (accept) {
    // Alg. 3: coefficients of the one-pass GEMV.  Rows 0..n_tau-1 are the crossed
    // T_{l+k} (F2 = exp((T_{l+k} - T_now) H_j), l.13-15); the last row is the
    // running solution (F, l.20).  coef[o][c-1] = beta F(c,1) / s_c.
    // Saad's corrected scheme (options.corrected): the extra basis vector x_{j+1}
    // (stored by the closing pass) with beta h_{j+1,j} F(j, j+1) / s_{j+1}; F2 then comes
    // from exp(tt H~) (size j+1, H~ as in Alg. 1 l.17-18) for its entry (j, j+1).
    const bool corr = P.corrected && !happy;
    const double h_corr = corr ? P.H[j + (size_t)LDH * (j - 1)] : 0.0;
    const double sc_final = P.task1 ? pow(1.0 / call->T[call->n_out - 1], (double)P.p) : 1.0;
    if (rank == 0) {
      for (int c = threadIdx.x; c < j; c += blockDim.x) {
        const double sg = (c == 0) ? beta : P.sig[c + 1];
        P.coef[(size_t)n_tau * LDH + c] = beta * F[c] / sg * (final_ ? sc_final : 1.0);
      }
      if (corr && threadIdx.x == 0)
        P.coef[(size_t)n_tau * LDH + j] = beta * (h_corr * F[(j - 1) + (size_t)LDH * j]) / P.sig[j + 1] *
                                          (final_ ? sc_final : 1.0);
    }
    cl_sync();
    const int nf = corr ? j + 1 : j;
    for (int k = 0; k < n_tau; k++) {
      auto hj = [&](int r, int c) -> double {  // H_j, or H~ for the corrected scheme
        double v = 0.0;
        if (r < j && c < j && r >= c - P.q + 1 && r <= c + 1) v = P.H[r + (size_t)LDH * c];
        if (corr && r == 0 && c == j) v = 1.0;
        return v;
      };
      const double tt = call->T[l0 + k] - t_now;
      const int nm2 = cl_expm_fill(nf, hj, Mh, tt, F, scr, sm);
      const double sc = P.task1 ? pow(1.0 / call->T[l0 + k], (double)P.p) : 1.0;
      if (rank == 0) {
        for (int c = threadIdx.x; c < j; c += blockDim.x) {
          const double sg = (c == 0) ? beta : P.sig[c + 1];
          P.coef[(size_t)k * LDH + c] = beta * F[c] / sg * sc;
        }
        if (corr && threadIdx.x == 0)
          P.coef[(size_t)k * LDH + j] = beta * (h_corr * F[(j - 1) + (size_t)LDH * j]) / P.sig[j + 1] * sc;
      }
      if (lead) {
        st->expm_calls++;
        if (nm2 < 0) st->status = KIOPS_ERR_NONFINITE;
      }
      cl_sync();
    }
    if (lead) {
      for (int k = 0; k < n_tau; k++) st->gemv_out[k] = call->w[l0 + k];
      st->gemv_out[n_tau] = final_ ? call->w[call->n_out - 1] : P.V;  // V slot 1 = running solution
      st->gemv_nout = n_tau + 1;
      st->gemv_j = corr ? j + 1 : j;
      st->gemv_x1 = st->x1;
      st->x1 = P.V;
      st->l = l0 + n_tau;
      st->t_now = final_ ? t_end : t_now + tau;  // Alg. 1 l.24, R11
      st->npass = 0;                             // l.25
      st->happy = 0;
      write_exact_tail(P, st->t_now, st->mu, P.tails + 1 * KMAXP);  // next substep's exact tail (Eq. 47)
    }
  }
  CTRL_STAMP(6);
  if (lead) {
    const bool more = st->status == 0 && st->t_now < st->t_end;
    const bool cont = more && st->attempt < P.max_attempts;
    if (more && !cont) st->status = KIOPS_ERR_NO_CONVERGENCE;
    set_cond(P, COND_OUTER, cont ? 1u : 0u);
    set_cond(P, COND_INNER, (cont && st->npass < st->m + 1) ? 1u : 0u);
    set_cond(P, COND_ACCEPT, accept ? 1u : 0u);
    st->ns_ctrl += gtimer() - t_start;
#ifdef KIOPS_PHASE_DEBUG
    CTRL_STAMP(7);
    printf("CTRL j=%d accept=%d ns: read+sync %llu assemble+sync %llu expm %llu lead %llu sync %llu accept-path %llu tail %llu total %llu\n",
           j, accept, tph[1] - tph[0], tph[2] - tph[1], tph[3] - tph[2], tph[4] - tph[3], tph[5] - tph[4], tph[6] - tph[5],
           tph[7] - tph[6], tph[7] - tph[0]);
#endif
  }
#undef CTRL_STAMP
}

// ---------------------------------------------------------------------------
// Alg. 3 l.15 and l.20 (Eq. 33): out_o = sum_c coef[o][c] x_c, all outputs of an
// accepted substep in ONE pass over the basis.  The running-solution row (which
// may overwrite x_1 in place) is the last chunk.
// ---------------------------------------------------------------------------
// Row a8 in padded mode (Alg. 3 l.15, l.20): one pass over the padded basis; the
// running solution (basis slot 1) is written on the whole padded grid -- its ghosts
// are the same combination of the basis ghosts, i.e. again the periodic images -- and
// the caller's outputs on the interior points only, in their natural layout.
// TEST HOOK (kiops_debug_expm): F = exp(scale M) by the controller's own exponential
// (cl_expm: the single-CTA shared-memory path for n <= SMALL_N, the cluster path above),
// on the ctx's scratch.  M, F: global, n x n column-major with leading dimension n.
__global__ void __cluster_dims__(CTRL_CL, 1, 1) __launch_bounds__(CTRL_THREADS, 1)
    k_debug_expm(KParams P, int n, const double *M, double scale, double *Fout, int *rc) {
  extern __shared__ double sm[];
  double *Mh = P.scratch + 8 * (size_t)LDH * LDH, *F = P.scratch + 9 * (size_t)LDH * LDH;
  for (int e = cl_gtid(); e < n * n; e += cl_gsize()) Mh[(e % n) + (size_t)LDH * (e / n)] = M[e];
  cl_sync();
  const int nm = cl_expm(n, Mh, scale, F, P.scratch, sm);
  cl_sync();
  for (int e = cl_gtid(); e < n * n; e += cl_gsize()) Fout[e] = F[(e % n) + (size_t)LDH * (e / n)];
  if (cl_gtid() == 0) *rc = nm;
}

__device__ __forceinline__ void gemv_padded(const KParams &P, int j, int nout, const double *x1) {
  DevState *st = P.st;
  __shared__ double sc[GEMV_OCHUNK * LDH];
  __shared__ double *outp[GEMV_OCHUNK];
  const int Xp = P.Xp, Yp = P.Yp, nx = (int)P.nx, ny = (int)P.ny;
  const long long npair = P.Np / 2, ld2 = P.ldN / 2;
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x, gsz = (long long)gridDim.x * blockDim.x;
  for (int o0 = 0; o0 < nout; o0 += GEMV_OCHUNK) {
    const int no = min(GEMV_OCHUNK, nout - o0);
    __syncthreads();
    for (int e = threadIdx.x; e < no * j; e += blockDim.x) sc[(e / j) * LDH + e % j] = P.coef[(size_t)(o0 + e / j) * LDH + e % j];
    if (threadIdx.x < no) outp[threadIdx.x] = st->gemv_out[o0 + threadIdx.x];
    __syncthreads();
    for (long long q = gt; q < npair; q += gsz) {
      double2 acc[GEMV_OCHUNK];
#pragma unroll
      for (int o = 0; o < GEMV_OCHUNK; o++) acc[o] = make_double2(0.0, 0.0);
      if (j > 0) {
        const double2 x = __ldg(reinterpret_cast<const double2 *>(x1) + q);
#pragma unroll
        for (int o = 0; o < GEMV_OCHUNK; o++) {
          acc[o].x = fma(sc[o * LDH], x.x, acc[o].x);
          acc[o].y = fma(sc[o * LDH], x.y, acc[o].y);
        }
      }
      const double2 *vp = reinterpret_cast<const double2 *>(P.V + P.ldN) + q;  // slot 2
      int c = 1;
      for (; c + 3 < j; c += 4) {
        const double2 xa = __ldg(vp), xb = __ldg(vp + ld2), xc = __ldg(vp + 2 * ld2), xd = __ldg(vp + 3 * ld2);
        vp += 4 * ld2;
#pragma unroll
        for (int o = 0; o < GEMV_OCHUNK; o++) {
          if (o < no) {
            const double *cf = sc + o * LDH + c;
            acc[o].x = fma(cf[0], xa.x, acc[o].x); acc[o].y = fma(cf[0], xa.y, acc[o].y);
            acc[o].x = fma(cf[1], xb.x, acc[o].x); acc[o].y = fma(cf[1], xb.y, acc[o].y);
            acc[o].x = fma(cf[2], xc.x, acc[o].x); acc[o].y = fma(cf[2], xc.y, acc[o].y);
            acc[o].x = fma(cf[3], xd.x, acc[o].x); acc[o].y = fma(cf[3], xd.y, acc[o].y);
          }
        }
      }
      for (; c < j; c++) {
        const double2 xa = __ldg(vp);
        vp += ld2;
#pragma unroll
        for (int o = 0; o < GEMV_OCHUNK; o++)
          if (o < no) {
            acc[o].x = fma(sc[o * LDH + c], xa.x, acc[o].x);
            acc[o].y = fma(sc[o * LDH + c], xa.y, acc[o].y);
          }
      }
      // padded pair q -> (xp, yp, z); interior pairs map to the natural index
      const long long i = 2 * q, row = i / Xp;
      const int xp = (int)(i - row * Xp);
      const long long z = row / Yp;
      const int yp = (int)(row - z * Yp);
      const bool inner = xp >= 2 && xp < nx + 2 && yp >= 2 && yp < ny + 2;
      const long long ui = (xp - 2) + (long long)nx * ((yp - 2) + (long long)ny * z);
#ifdef KIOPS_BOUNDS_CHECK
      assert(xp % 2 == 0 && (!inner || (ui >= 0 && ui + 1 < P.N)) && 2 * q + 1 < P.Np);
#endif
#pragma unroll
      for (int o = 0; o < GEMV_OCHUNK; o++)
        if (o < no) {
          double *out = outp[o];
          if (out == P.V) {
            reinterpret_cast<double2 *>(out)[q] = acc[o];
          } else if (inner) {
            if ((((uintptr_t)(out + ui)) & 15) == 0) {
              *reinterpret_cast<double2 *>(out + ui) = acc[o];
            } else {
              out[ui] = acc[o].x;
              out[ui + 1] = acc[o].y;
            }
          }
        }
    }
  }
}

__global__ void __launch_bounds__(256) k_gemv(KParams P) {
  DevState *st = P.st;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->t_gemv0 = gtimer();
  const int j = st->gemv_j, nout = st->gemv_nout;
  const double *x1 = st->gemv_x1;
  const long long N = P.padded ? 0 : P.N;  // padded mode: gemv_padded below
  if (P.padded) gemv_padded(P, j, nout, x1);
  __shared__ double sc[GEMV_OCHUNK * LDH];
  __shared__ double *outp[GEMV_OCHUNK];
  // 16-byte path when every stream is 16-byte aligned (V slots always are)
  bool vec = ((uintptr_t)x1 & 15) == 0;
  for (int o = 0; o < nout; o++) vec = vec && (((uintptr_t)st->gemv_out[o] & 15) == 0);
  const long long npair = vec ? N / 2 : 0;
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x, gsz = (long long)gridDim.x * blockDim.x;
  for (int o0 = 0; o0 < nout; o0 += GEMV_OCHUNK) {
    const int no = min(GEMV_OCHUNK, nout - o0);
    __syncthreads();
    for (int e = threadIdx.x; e < no * j; e += blockDim.x) sc[(e / j) * LDH + e % j] = P.coef[(size_t)(o0 + e / j) * LDH + e % j];
    if (threadIdx.x < no) outp[threadIdx.x] = st->gemv_out[o0 + threadIdx.x];
    __syncthreads();
    for (long long q = gt; q < npair; q += gsz) {
      double2 acc[GEMV_OCHUNK];
#pragma unroll
      for (int o = 0; o < GEMV_OCHUNK; o++) acc[o] = make_double2(0.0, 0.0);
      if (j > 0) {
        const double2 x = __ldg(reinterpret_cast<const double2 *>(x1) + q);
#pragma unroll
        for (int o = 0; o < GEMV_OCHUNK; o++) {
          acc[o].x = fma(sc[o * LDH], x.x, acc[o].x);
          acc[o].y = fma(sc[o * LDH], x.y, acc[o].y);
        }
      }
      const double2 *vp = reinterpret_cast<const double2 *>(P.V + P.ldN) + q;  // slot 2
      const long long ld2 = P.ldN / 2;
      int c = 1;
      for (; c + 3 < j; c += 4) {
        const double2 xa = __ldg(vp), xb = __ldg(vp + ld2), xc = __ldg(vp + 2 * ld2), xd = __ldg(vp + 3 * ld2);
        vp += 4 * ld2;
#pragma unroll
        for (int o = 0; o < GEMV_OCHUNK; o++) {
          if (o < no) {
            const double *cf = sc + o * LDH + c;
            acc[o].x = fma(cf[0], xa.x, acc[o].x); acc[o].y = fma(cf[0], xa.y, acc[o].y);
            acc[o].x = fma(cf[1], xb.x, acc[o].x); acc[o].y = fma(cf[1], xb.y, acc[o].y);
            acc[o].x = fma(cf[2], xc.x, acc[o].x); acc[o].y = fma(cf[2], xc.y, acc[o].y);
            acc[o].x = fma(cf[3], xd.x, acc[o].x); acc[o].y = fma(cf[3], xd.y, acc[o].y);
          }
        }
      }
      for (; c < j; c++) {
        const double2 xa = __ldg(vp);
        vp += ld2;
#pragma unroll
        for (int o = 0; o < GEMV_OCHUNK; o++)
          if (o < no) {
            acc[o].x = fma(sc[o * LDH + c], xa.x, acc[o].x);
            acc[o].y = fma(sc[o * LDH + c], xa.y, acc[o].y);
          }
      }
#pragma unroll
      for (int o = 0; o < GEMV_OCHUNK; o++)
        if (o < no) reinterpret_cast<double2 *>(outp[o])[q] = acc[o];
    }
    // scalar path: odd tail element or unaligned streams
    for (long long i = 2 * npair + gt; i < N; i += gsz) {
      double acc[GEMV_OCHUNK];
#pragma unroll
      for (int o = 0; o < GEMV_OCHUNK; o++) acc[o] = 0.0;
      for (int cc = 0; cc < j; cc++) {
        const double x = (cc == 0) ? x1[i] : P.V[(size_t)cc * P.ldN + i];
#pragma unroll
        for (int o = 0; o < GEMV_OCHUNK; o++)
          if (o < no) acc[o] = fma(sc[o * LDH + cc], x, acc[o]);
      }
#pragma unroll
      for (int o = 0; o < GEMV_OCHUNK; o++)
        if (o < no) outp[o][i] = acc[o];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&st->gemv_ticket, 1u) == gridDim.x - 1) {
      st->ns_gemv += gtimer() - st->t_gemv0;
      st->gemv_ticket = 0;
    }
  }
}
