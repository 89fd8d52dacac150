// epirk.cuh -- SURVEY 8(f) row f1: EPIRK4s3 (Eq. 50) / EPIRK4s3A (Eq. 51) with the
// two-call "mixed implementation" of Sec. 2 (Eqs. 9-11), and the fifth-order EPIRK5P1
// (Eq. 52, Table 1, reading E8) / EXPRB5s3 (Eq. 53) with three calls (reading E9), on
// top of kiops_apply, for u' = L u + R(u) (periodic 5-point L, cubic pointwise R;
// Allen-Cahn).
// Included at the end of kiops.cu (one translation unit).  sm_100a, fp64.
//
// Per step (all on the ctx stream):
//   k_ep_f      f_n = L u + R(u), d = h R'(u) (the diagonal of the KIOPS operator h J_n,
//               whose stencil part h L is fixed at create), b1 = h f_n
//   kiops_apply Task I, p = 1: phi_1(c h J_n) h f_n at the two nodes (T ascending, 1/T)
//   k_ep_stage  U_i = u + c_i w_i; r_i = R(U_i) - R(u) - R'(u)(U_i - u) (the remainder
//               of P:85 with the linear part cancelled exactly); b3, b4 as Eq. 11 / Eq. 51
//   kiops_apply Task II, p = 4, T = 1: phi_1 b1 + phi_3 b3 + phi_4 b4
//   k_ep_update u += w
#pragma once

struct EpProblem {
  long long nx, ny;
  double w[5];  // {W, E, S, N, C}
  double c[4];  // R(u) = c0 + c1 u + c2 u^2 + c3 u^3
  double h;
  // general linear part (kiops_rd_problem.L_*): CSR, NULL for the periodic stencil
  const long long *rp;
  const int *ci;
  const double *lv;
};

__device__ __forceinline__ double ep_R(const EpProblem &q, double u) {
  return q.c[0] + u * (q.c[1] + u * (q.c[2] + u * q.c[3]));
}
__device__ __forceinline__ double ep_dR(const EpProblem &q, double u) {
  return q.c[1] + u * (2.0 * q.c[2] + u * 3.0 * q.c[3]);
}

__global__ void __launch_bounds__(256) k_ep_f(EpProblem q, const double *__restrict__ u, double *__restrict__ d,
                                              double *__restrict__ b1) {
  const long long N = q.nx * q.ny;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const long long x = i % q.nx, y = i / q.nx, b = i - x;
    const double uW = u[b + (x == 0 ? q.nx - 1 : x - 1)], uE = u[b + (x == q.nx - 1 ? 0 : x + 1)];
    const double uS = u[x + q.nx * (y == 0 ? q.ny - 1 : y - 1)], uN = u[x + q.nx * (y == q.ny - 1 ? 0 : y + 1)];
    const double uc = u[i];
    const double Lu = q.w[0] * uW + q.w[1] * uE + q.w[2] * uS + q.w[3] * uN + q.w[4] * uc;
    const double f = Lu + ep_R(q, uc);
    d[i] = q.h * ep_dR(q, uc);
    b1[i] = q.h * f;
  }
}

// CSR linear part: f_n = L u + R(u), b1 = h f_n, and the values of the KIOPS operator
// h J_n = h (L + diag R'(u_n)) on L's pattern (jv), one row per thread (row sums in
// storage order, as the oracle's).  bad: counts rows without a diagonal entry.
__global__ void __launch_bounds__(256) k_ep_f_csr(EpProblem q, const double *__restrict__ u, double *__restrict__ jv,
                                                  double *__restrict__ b1, int *__restrict__ bad) {
  const long long N = q.nx * q.ny;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double uc = u[i], hd = q.h * ep_dR(q, uc);
    double Lu = 0.0;
    bool has = false;
    for (long long e = q.rp[i]; e < q.rp[i + 1]; e++) {
      const int c = q.ci[e];
      const double v = q.lv[e];
      Lu += v * u[c];
      const bool dg = c == (int)i;
      has = has || dg;
      if (jv) jv[e] = dg ? q.h * v + hd : q.h * v;
    }
    if (b1) b1[i] = q.h * (Lu + ep_R(q, uc));
    if (!has && bad) atomicAdd(bad, 1);
  }
}

__global__ void __launch_bounds__(256) k_ep_stage(EpProblem q, int scheme, double c2, double c3,
                                                  const double *__restrict__ u, const double *__restrict__ w2,
                                                  const double *__restrict__ w3, double *__restrict__ b3,
                                                  double *__restrict__ b4) {
  const long long N = q.nx * q.ny;
  const double h = q.h;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double un = u[i], Rn = ep_R(q, un), dRn = ep_dR(q, un);
    const double U2 = un + c2 * w2[i], U3 = un + c3 * w3[i];
    const double r2 = ep_R(q, U2) - Rn - dRn * (U2 - un);
    const double r3 = ep_R(q, U3) - Rn - dRn * (U3 - un);
    if (scheme == KIOPS_EPIRK4S3) {  // Eq. 11
      const double dd = r3 - 2.0 * r2;
      b3[i] = 1892.0 * h * r2 + 1458.0 * h * dd;
      b4[i] = -42336.0 * h * r2 - 34992.0 * h * dd;
    } else {  // Eq. 51
      b3[i] = 32.0 * h * r2 - 13.5 * h * r3;
      b4[i] = -144.0 * h * r2 + 81.0 * h * r3;
    }
  }
}

__global__ void __launch_bounds__(256) k_ep_update(long long N, const double *__restrict__ w, double *__restrict__ u) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    u[i] += w[i];
}

// fifth-order stage kernels (oracle/epirk.py step5, operand for operand)
#define EP_A11 0.3512959269505819
#define EP_A21 0.8440547201165712
#define EP_A22 1.690589160956896
#define EP_B1 1.0
#define EP_B2 1.272712731735689
#define EP_B3 2.271459926542262
__device__ __forceinline__ double ep_rem(const EpProblem &q, double un, double U) {
  return ep_R(q, U) - ep_R(q, un) - ep_dR(q, un) * (U - un);
}
// EPIRK5P1 after call 1: t = h r(U2), U2 = u + a11 phi_1(g11 hJ) hf
__global__ void __launch_bounds__(256) k_ep5p1_a(EpProblem q, const double *__restrict__ u, const double *__restrict__ o10,
                                                 double *__restrict__ t) {
  const long long N = q.nx * q.ny;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double un = u[i], U2 = un + EP_A11 * o10[i];
    t[i] = q.h * ep_rem(q, un, U2);
  }
}
// after call 2: U3 = u + a21 phi_1(g21 hJ) hf + a22 phi_1(g22 hJ) h r2; t = h (-2 r2 + r3)
__global__ void __launch_bounds__(256) k_ep5p1_b(EpProblem q, const double *__restrict__ u, const double *__restrict__ o10,
                                                 const double *__restrict__ o11, const double *__restrict__ o21,
                                                 double *__restrict__ t) {
  const long long N = q.nx * q.ny;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double un = u[i];
    const double r2 = ep_rem(q, un, un + EP_A11 * o10[i]);
    const double U3 = un + EP_A21 * o11[i] + EP_A22 * o21[i];
    t[i] = q.h * (-2.0 * r2 + ep_rem(q, un, U3));
  }
}
// after call 3: u = u + b1 phi_1(g31 hJ) hf + b2 phi_1(g32 hJ) h r2 + b3 phi_3(g33 hJ) h(-2 r2 + r3)
__global__ void __launch_bounds__(256) k_ep5p1_c(long long N, const double *__restrict__ o12,
                                                 const double *__restrict__ o20, const double *__restrict__ o3,
                                                 double *__restrict__ u) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    u[i] = u[i] + EP_B1 * o12[i] + EP_B2 * o20[i] + EP_B3 * o3[i];
}
// EXPRB5s3 after call 1: t = h r(U2), U2 = u + 1/2 phi_1(hJ/2) hf
__global__ void __launch_bounds__(256) k_ex5_a(EpProblem q, const double *__restrict__ u, const double *__restrict__ o10,
                                               double *__restrict__ t) {
  const long long N = q.nx * q.ny;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double un = u[i];
    t[i] = q.h * ep_rem(q, un, un + 0.5 * o10[i]);
  }
}
// after call 2: U3 = u + 9/10 phi_1(9hJ/10) hf + 27/25 phi_3(hJ/2) h r2 + 729/125 phi_3(9hJ/10) h r2;
// b3 = 18 h r2 - 250/81 h r3, b4 = -60 h r2 + 500/27 h r3 (Eq. 53)
__global__ void __launch_bounds__(256) k_ex5_b(EpProblem q, const double *__restrict__ u, const double *__restrict__ o10,
                                               const double *__restrict__ o11, const double *__restrict__ o20,
                                               const double *__restrict__ o21, double *__restrict__ b3,
                                               double *__restrict__ b4) {
  const long long N = q.nx * q.ny;
  const double h = q.h;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const double un = u[i];
    const double r2 = ep_rem(q, un, un + 0.5 * o10[i]);
    const double U3 = un + 0.9 * o11[i] + (27.0 / 25.0) * o20[i] + (729.0 / 125.0) * o21[i];
    const double r3 = ep_rem(q, un, U3);
    b3[i] = 18.0 * h * r2 - (250.0 / 81.0) * h * r3;
    b4[i] = -60.0 * h * r2 + (500.0 / 27.0) * h * r3;
  }
}

struct kiops_epirk_s {
  kiops_ctx kA = nullptr;        // p = 1, Task I (phi_1 at several T)
  kiops_ctx kB = nullptr;        // p = 4, Task II at tau = 1      (4s3, 4s3A, EXPRB5s3)
  kiops_ctx kC = nullptr;        // p = 3, Task I (phi_3)          (EPIRK5P1, EXPRB5s3)
  EpProblem q{};
  int scheme = 0;
  double c2 = 0.0, c3 = 0.0;     // fourth order: stage nodes of U_{n2}, U_{n3}
  cudaStream_t stream = nullptr;
  double *d = nullptr, *b1 = nullptr, *zero = nullptr, *o1[3] = {}, *o2[2] = {}, *o3 = nullptr, *t1 = nullptr,
         *t2 = nullptr;
  double *jv = nullptr;          // CSR linear part: the values of h J_n (L_nnz doubles)
  int m[3] = {0, 0, 0};          // warm start of calls 1-3 (Sec. 3.6, reading E1)
  bool record = false;           // kiops_epirk_record_history
  struct Forced {
    int step, call;
    std::vector<double> tau;
    std::vector<int32_t> m, acc;
  };
  std::vector<Forced> forced;    // kiops_epirk_set_forced_schedule (test hook)
  std::vector<kiops_epirk_call_record> hist;  // per-call records of the last kiops_epirk_step
  std::string err;
};

namespace {
constexpr int EP_VECS = 11;  // d, b1, zero, o1[3], o2[2], o3, t1, t2

kiops_operator_desc ep_desc(const kiops_rd_problem *pb, double h, const double *d, const double *jv = nullptr) {
  kiops_operator_desc o{};
  if (pb->L_row_ptr) {  // h J_n as a CSR operator on L's pattern; the driver rewrites jv every step
    o.kind = KIOPS_OP_CSR;
    o.periodic = 1;
    o.nx = pb->nx * pb->ny; o.ny = 1; o.nz = 1;
    o.row_ptr = pb->L_row_ptr; o.col_idx = pb->L_col_idx; o.vals = jv ? jv : pb->L_vals; o.nnz = pb->L_nnz;
    return o;
  }
  o.kind = KIOPS_OP_STENCIL2D5;
  o.periodic = 1;
  o.nx = pb->nx; o.ny = pb->ny; o.nz = 1;
  for (int i = 0; i < 5; i++) o.w[i] = h * pb->w[i];  // the matrix argument is h J_n
  o.diag = d;
  return o;
}

size_t ep_jv_bytes(const kiops_rd_problem *pb) {
  return pb->L_row_ptr ? (((size_t)pb->L_nnz * sizeof(double) + 255) & ~(size_t)255) : 0;
}

bool ep_uses(int scheme, int which) {  // 0: kA, 1: kB, 2: kC
  if (which == 0) return true;
  if (which == 1) return scheme != KIOPS_EPIRK5P1;
  return scheme == KIOPS_EPIRK5P1 || scheme == KIOPS_EXPRB5S3;
}

kiops_status ep_sizes(const kiops_rd_problem *pb, int scheme, const kiops_options *o, size_t b[3], size_t *vec) {
  if (!pb || !o || pb->nx < 1 || pb->ny < 1) return KIOPS_ERR_INVALID_ARG;
  if (pb->L_row_ptr && (!pb->L_col_idx || !pb->L_vals || pb->L_nnz < pb->nx * pb->ny)) return KIOPS_ERR_INVALID_ARG;
  const double fake = 0.0;
  kiops_operator_desc dsc = ep_desc(pb, 1.0, &fake);
  const int pk[3] = {1, 4, 3}, t1[3] = {1, 0, 1};
  for (int i = 0; i < 3; i++) {
    b[i] = 0;
    if (!ep_uses(scheme, i)) continue;
    kiops_options oi = *o;
    oi.task1 = t1[i];
    oi.host_staging = 0;
    const kiops_status s = kiops_workspace_bytes(&dsc, pk[i], &oi, &b[i]);
    if (s != KIOPS_OK) return s;
    b[i] = (b[i] + 255) & ~(size_t)255;
  }
  *vec = ((size_t)pb->nx * (size_t)pb->ny * sizeof(double) + 255) & ~(size_t)255;
  return KIOPS_OK;
}
}  // namespace

kiops_status kiops_epirk_workspace_bytes(const kiops_rd_problem *pb, int scheme, const kiops_options *o,
                                         size_t *bytes) {
  if (!bytes || scheme < KIOPS_EPIRK4S3 || scheme > KIOPS_EXPRB5S3) return KIOPS_ERR_INVALID_ARG;
  size_t b[3], vec;
  const kiops_status s = ep_sizes(pb, scheme, o, b, &vec);
  if (s != KIOPS_OK) return s;
  *bytes = b[0] + b[1] + b[2] + EP_VECS * vec + ep_jv_bytes(pb);
  return KIOPS_OK;
}

kiops_status kiops_epirk_create(const kiops_rd_problem *pb, int scheme, double h, const kiops_options *o,
                                void *cuda_stream, void *workspace, size_t workspace_bytes, kiops_epirk_ctx *out) {
  if (!out) return KIOPS_ERR_INVALID_ARG;
  *out = nullptr;
  if (scheme < KIOPS_EPIRK4S3 || scheme > KIOPS_EXPRB5S3) return KIOPS_ERR_INVALID_ARG;
  if (!(h > 0.0) || !std::isfinite(h)) return KIOPS_ERR_INVALID_ARG;
  size_t b[3], vec;
  kiops_status s = ep_sizes(pb, scheme, o, b, &vec);
  if (s != KIOPS_OK) return s;
  const size_t kb = b[0] + b[1] + b[2];
  if (!workspace || ((uintptr_t)workspace & 255) || workspace_bytes < kb + EP_VECS * vec + ep_jv_bytes(pb))
    return KIOPS_ERR_WORKSPACE;
  kiops_epirk_ctx e = new (std::nothrow) kiops_epirk_s();
  if (!e) return KIOPS_ERR_WORKSPACE;
  e->scheme = scheme;
  e->stream = (cudaStream_t)cuda_stream;
  e->q.nx = pb->nx; e->q.ny = pb->ny; e->q.h = h;
  for (int i = 0; i < 5; i++) e->q.w[i] = pb->w[i];
  for (int i = 0; i < 4; i++) e->q.c[i] = pb->c[i];
  if (scheme == KIOPS_EPIRK4S3) { e->c2 = 1.0 / 8.0; e->c3 = 1.0 / 9.0; }        // Eq. 50
  else if (scheme == KIOPS_EPIRK4S3A) { e->c2 = 1.0 / 2.0; e->c3 = 2.0 / 3.0; }  // Eq. 51
  unsigned char *ws = (unsigned char *)workspace;
  double **vp[EP_VECS] = {&e->d, &e->b1, &e->zero, &e->o1[0], &e->o1[1], &e->o1[2], &e->o2[0], &e->o2[1],
                          &e->o3, &e->t1, &e->t2};
  for (int i = 0; i < EP_VECS; i++) *vp[i] = (double *)(ws + kb + (size_t)i * vec);
  if (pb->L_row_ptr) {  // general linear part: check the diagonals, give jv valid values (h L)
    e->q.rp = (const long long *)pb->L_row_ptr;
    e->q.ci = (const int *)pb->L_col_idx;
    e->q.lv = pb->L_vals;
    e->jv = (double *)(ws + kb + (size_t)EP_VECS * vec);
    const long long N = pb->nx * pb->ny;
    const int grid = (int)std::min<long long>((N + 255) / 256, SM_COUNT_HINT * 8);
    int *bad = (int *)e->t1, hbad = -1;
    cudaError_t ce = cudaMemsetAsync(e->zero, 0, vec, e->stream);  // (u = 0 for this pass)
    if (ce == cudaSuccess) ce = cudaMemsetAsync(bad, 0, sizeof(int), e->stream);
    if (ce == cudaSuccess) {
      k_ep_f_csr<<<grid, 256, 0, e->stream>>>(e->q, e->zero, e->jv, nullptr, bad);
      ce = cudaGetLastError();
    }
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, e->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->stream);
    if (ce != cudaSuccess || hbad != 0) {
      delete e;
      return ce != cudaSuccess ? KIOPS_ERR_CUDA : KIOPS_ERR_INVALID_ARG;  // a row of L without its diagonal
    }
  }
  const kiops_operator_desc dsc = ep_desc(pb, h, e->d, e->jv);
  const int pk[3] = {1, 4, 3}, t1[3] = {1, 0, 1};
  kiops_ctx *kc[3] = {&e->kA, &e->kB, &e->kC};
  size_t off = 0;
  for (int i = 0; i < 3 && s == KIOPS_OK; i++) {
    if (!ep_uses(scheme, i)) continue;
    kiops_options oi = *o;
    oi.task1 = t1[i];
    oi.host_staging = 0;
    s = kiops_create(&dsc, pk[i], &oi, cuda_stream, ws + off, b[i], kc[i]);
    off += b[i];
  }
  if (s == KIOPS_OK) {
    const cudaError_t ce = cudaMemsetAsync(e->zero, 0, vec, e->stream);
    if (ce != cudaSuccess) { e->err = cudaGetErrorString(ce); s = KIOPS_ERR_CUDA; }
  }
  if (s != KIOPS_OK) {
    kiops_epirk_destroy(e);
    return s;
  }
  *out = e;
  return KIOPS_OK;
}

namespace {
// one kiops_apply of the step with warm start; accumulates the stats
kiops_status ep_call(kiops_epirk_ctx e, kiops_ctx k, int call, int step, const double *const *u, const double *T,
                     int n_out, double *const *w, kiops_epirk_stats *acc) {
  kiops_stats st{};
  kiops_set_m_init(k, e->m[call]);
  {  // test hook: replay a forced schedule on this call, else free-running
    const kiops_epirk_s::Forced *f = nullptr;
    for (const auto &x : e->forced)
      if (x.step == step && x.call == call) f = &x;
    const kiops_status fs = f ? kiops_set_forced_schedule(k, f->tau.data(), f->m.data(), f->acc.data(), (int)f->tau.size())
                              : kiops_set_forced_schedule(k, nullptr, nullptr, nullptr, 0);
    if (fs != KIOPS_OK) {
      e->err = "forced schedule rejected";
      return fs;
    }
  }
  const kiops_status s = kiops_apply(k, u, T, n_out, w, &st);
  if (s != KIOPS_OK) {
    e->err = "step " + std::to_string(step) + ", call " + std::to_string(call + 1) + ": " + kiops_last_error(k);
    return s;
  }
  e->m[call] = st.final_m;
  if (e->record) {  // the decision history of this call (kiops_apply has synchronised)
    kiops_epirk_call_record r{};
    r.step = step;
    r.call = call;
    r.final_m = st.final_m;
    r.krylov_vectors = st.krylov_vectors;
    r.substeps = st.substeps;
    r.rejections = st.rejections;
    kiops_trace_row tr[KIOPS_EPIRK_HIST_ATTEMPTS];
    int64_t rows = 0;
    const kiops_status ts = kiops_get_trace(k, tr, sizeof(tr), &rows);
    if (ts != KIOPS_OK) {
      e->err = "history: kiops_get_trace failed";
      return ts;
    }
    r.n_attempts = (int32_t)rows;
    for (int64_t a = 0; a < rows && a < KIOPS_EPIRK_HIST_ATTEMPTS; a++) {
      r.j[a] = (int16_t)tr[a].j;
      r.m_new[a] = (int16_t)tr[a].m_new;
      r.accept[a] = (int8_t)tr[a].accept;
      r.omega[a] = tr[a].omega;
    }
    e->hist.push_back(r);
  }
  acc->krylov_vectors += st.krylov_vectors;
  acc->passes += st.passes;
  acc->substeps += st.substeps;
  acc->rejections += st.rejections;
  acc->expm_calls += st.expm_calls;
  acc->kiops_ms += st.pass_ms + st.ctrl_ms + st.gemv_ms;
  return KIOPS_OK;
}
}  // namespace

kiops_status kiops_epirk_step(kiops_epirk_ctx e, double *u, int nsteps, kiops_epirk_stats *stats) {
  if (!e || !u || nsteps < 0) return KIOPS_ERR_INVALID_ARG;
  const long long N = e->q.nx * e->q.ny;
  const int grid = (int)std::min<long long>((N + 255) / 256, SM_COUNT_HINT * 8);
  kiops_epirk_stats acc{};
  e->hist.clear();
  const double *z = e->zero;
#define EP_LAUNCHED(name) \
  if (cudaGetLastError() != cudaSuccess) { e->err = name " launch"; return KIOPS_ERR_CUDA; }
  for (int n = 0; n < nsteps; n++) {
    kiops_status s;
    if (e->jv) {  // CSR linear part: new values of h J_n, then the SELL copies of the contexts
      k_ep_f_csr<<<grid, 256, 0, e->stream>>>(e->q, u, e->jv, e->b1, nullptr);
      EP_LAUNCHED("k_ep_f_csr");
      kiops_ctx kc[3] = {e->kA, e->kB, e->kC};
      for (int i = 0; i < 3; i++)
        if (kc[i] && (s = kiops_refresh_operator(kc[i])) != KIOPS_OK) {
          e->err = std::string("operator refresh: ") + kiops_last_error(kc[i]);
          return s;
        }
    } else {
      k_ep_f<<<grid, 256, 0, e->stream>>>(e->q, u, e->d, e->b1);
      EP_LAUNCHED("k_ep_f");
    }
    const double *uf[2] = {z, e->b1};
    if (e->scheme == KIOPS_EPIRK4S3 || e->scheme == KIOPS_EPIRK4S3A) {
      const bool asc = e->c2 < e->c3;  // call-1 outputs come in ascending T
      const double T1[2] = {asc ? e->c2 : e->c3, asc ? e->c3 : e->c2};
      if ((s = ep_call(e, e->kA, 0, n, uf, T1, 2, e->o1, &acc)) != KIOPS_OK) return s;
      k_ep_stage<<<grid, 256, 0, e->stream>>>(e->q, e->scheme, e->c2, e->c3, u, asc ? e->o1[0] : e->o1[1],
                                              asc ? e->o1[1] : e->o1[0], e->t1, e->t2);
      EP_LAUNCHED("k_ep_stage");
      const double *u2[5] = {z, e->b1, z, e->t1, e->t2};
      const double T2[1] = {1.0};
      if ((s = ep_call(e, e->kB, 1, n, u2, T2, 1, &e->o3, &acc)) != KIOPS_OK) return s;
      k_ep_update<<<grid, 256, 0, e->stream>>>(N, e->o3, u);
      EP_LAUNCHED("k_ep_update");
    } else if (e->scheme == KIOPS_EPIRK5P1) {  // Eq. 52, Table 1
      const double T1[3] = {0.3512959269505819, 0.8440547201165712, 1.0};  // g11, g21, g31
      if ((s = ep_call(e, e->kA, 0, n, uf, T1, 3, e->o1, &acc)) != KIOPS_OK) return s;
      k_ep5p1_a<<<grid, 256, 0, e->stream>>>(e->q, u, e->o1[0], e->t1);
      EP_LAUNCHED("k_ep5p1_a");
      const double *u2[2] = {z, e->t1};
      const double T2[2] = {0.71111109536436687, 1.0};  // g32, g22
      if ((s = ep_call(e, e->kA, 1, n, u2, T2, 2, e->o2, &acc)) != KIOPS_OK) return s;
      k_ep5p1_b<<<grid, 256, 0, e->stream>>>(e->q, u, e->o1[0], e->o1[1], e->o2[1], e->t1);
      EP_LAUNCHED("k_ep5p1_b");
      const double *u3[4] = {z, z, z, e->t1};
      const double T3[1] = {0.6237811195337149};  // g33
      if ((s = ep_call(e, e->kC, 2, n, u3, T3, 1, &e->o3, &acc)) != KIOPS_OK) return s;
      k_ep5p1_c<<<grid, 256, 0, e->stream>>>(N, e->o1[2], e->o2[0], e->o3, u);
      EP_LAUNCHED("k_ep5p1_c");
    } else {  // EXPRB5s3, Eq. 53
      const double T1[2] = {0.5, 0.9};
      if ((s = ep_call(e, e->kA, 0, n, uf, T1, 2, e->o1, &acc)) != KIOPS_OK) return s;
      k_ex5_a<<<grid, 256, 0, e->stream>>>(e->q, u, e->o1[0], e->t1);
      EP_LAUNCHED("k_ex5_a");
      const double *u2[4] = {z, z, z, e->t1};
      if ((s = ep_call(e, e->kC, 1, n, u2, T1, 2, e->o2, &acc)) != KIOPS_OK) return s;
      k_ex5_b<<<grid, 256, 0, e->stream>>>(e->q, u, e->o1[0], e->o1[1], e->o2[0], e->o2[1], e->t1, e->t2);
      EP_LAUNCHED("k_ex5_b");
      const double *u3[5] = {z, e->b1, z, e->t1, e->t2};
      const double T3[1] = {1.0};
      if ((s = ep_call(e, e->kB, 2, n, u3, T3, 1, &e->o3, &acc)) != KIOPS_OK) return s;
      k_ep_update<<<grid, 256, 0, e->stream>>>(N, e->o3, u);
      EP_LAUNCHED("k_ep_update");
    }
    acc.steps++;
  }
#undef EP_LAUNCHED
  const cudaError_t ce = cudaStreamSynchronize(e->stream);
  if (ce != cudaSuccess) { e->err = cudaGetErrorString(ce); return KIOPS_ERR_CUDA; }
  for (int i = 0; i < 3; i++) acc.final_m[i] = e->m[i];
  if (stats) *stats = acc;
  return KIOPS_OK;
}

kiops_status kiops_epirk_record_history(kiops_epirk_ctx e, int on) {
  if (!e) return KIOPS_ERR_INVALID_ARG;
  e->record = on != 0;
  return KIOPS_OK;
}

kiops_status kiops_epirk_set_forced_schedule(kiops_epirk_ctx e, int step, int call, const double *tau,
                                            const int32_t *m, const int32_t *accept, int n) {
  if (!e) return KIOPS_ERR_INVALID_ARG;
  if (n == 0 && step < 0) {
    e->forced.clear();
    return KIOPS_OK;
  }
  if (step < 0 || call < 0 || call > 2 || n < 1 || n > KIOPS_MAX_FORCED || !tau || !m) return KIOPS_ERR_INVALID_ARG;
  kiops_epirk_s::Forced f{step, call, std::vector<double>(tau, tau + n), std::vector<int32_t>(m, m + n),
                          std::vector<int32_t>(n, 1)};
  if (accept)
    for (int i = 0; i < n; i++) f.acc[i] = accept[i] != 0;
  e->forced.push_back(f);
  return KIOPS_OK;
}

kiops_status kiops_epirk_history(kiops_epirk_ctx e, kiops_epirk_call_record *buf, int64_t cap, int64_t *rows) {
  if (!e || !rows || cap < 0 || (cap > 0 && !buf)) return KIOPS_ERR_INVALID_ARG;
  *rows = (int64_t)e->hist.size();
  for (int64_t i = 0; i < cap && i < *rows; i++) buf[i] = e->hist[(size_t)i];
  return KIOPS_OK;
}

kiops_status kiops_epirk_destroy(kiops_epirk_ctx e) {
  if (!e) return KIOPS_ERR_INVALID_ARG;
  if (e->kA) kiops_destroy(e->kA);
  if (e->kB) kiops_destroy(e->kB);
  if (e->kC) kiops_destroy(e->kC);
  delete e;
  return KIOPS_OK;
}

const char *kiops_epirk_last_error(kiops_epirk_ctx e) { return e ? e->err.c_str() : "NULL ctx"; }
