// epirk.cuh -- SURVEY 8(f) row f1: EPIRK4s3 (Eq. 50) / EPIRK4s3A (Eq. 51) with the
// two-call "mixed implementation" of Sec. 2 (Eqs. 9-11) on top of kiops_apply, for
// u' = L u + R(u) (periodic 5-point L, cubic pointwise R; Allen-Cahn).
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

struct kiops_epirk_s {
  kiops_ctx k1 = nullptr, k2 = nullptr;
  EpProblem q{};
  int scheme = 0;
  double c2 = 0.0, c3 = 0.0;   // stage nodes of U_{n2}, U_{n3}
  cudaStream_t stream = nullptr;
  double *d = nullptr, *b1 = nullptr, *zero = nullptr, *wa = nullptr, *wb = nullptr, *b3 = nullptr, *b4 = nullptr,
         *w = nullptr;
  int m1 = 0, m2 = 0;          // warm start of call 1 / call 2 (Sec. 3.6, reading E1)
  std::string err;
};

namespace {
constexpr int EP_VECS = 8;

kiops_operator_desc ep_desc(const kiops_rd_problem *pb, double h, const double *d) {
  kiops_operator_desc o{};
  o.kind = KIOPS_OP_STENCIL2D5;
  o.periodic = 1;
  o.nx = pb->nx; o.ny = pb->ny; o.nz = 1;
  for (int i = 0; i < 5; i++) o.w[i] = h * pb->w[i];  // the matrix argument is h J_n
  o.diag = d;
  return o;
}

kiops_status ep_sizes(const kiops_rd_problem *pb, const kiops_options *o, size_t *b1, size_t *b2, size_t *vec) {
  if (!pb || !o || pb->nx < 1 || pb->ny < 1) return KIOPS_ERR_INVALID_ARG;
  kiops_options o1 = *o, o2 = *o;
  o1.task1 = 1; o1.host_staging = 0;
  o2.task1 = 0; o2.host_staging = 0;
  const double fake = 0.0;
  kiops_operator_desc dsc = ep_desc(pb, 1.0, &fake);
  kiops_status s = kiops_workspace_bytes(&dsc, 1, &o1, b1);
  if (s != KIOPS_OK) return s;
  s = kiops_workspace_bytes(&dsc, 4, &o2, b2);
  if (s != KIOPS_OK) return s;
  *b1 = (*b1 + 255) & ~(size_t)255;
  *b2 = (*b2 + 255) & ~(size_t)255;
  *vec = ((size_t)pb->nx * (size_t)pb->ny * sizeof(double) + 255) & ~(size_t)255;
  return KIOPS_OK;
}
}  // namespace

kiops_status kiops_epirk_workspace_bytes(const kiops_rd_problem *pb, const kiops_options *o, size_t *bytes) {
  if (!bytes) return KIOPS_ERR_INVALID_ARG;
  size_t b1, b2, vec;
  const kiops_status s = ep_sizes(pb, o, &b1, &b2, &vec);
  if (s != KIOPS_OK) return s;
  *bytes = b1 + b2 + EP_VECS * vec;
  return KIOPS_OK;
}

kiops_status kiops_epirk_create(const kiops_rd_problem *pb, int scheme, double h, const kiops_options *o,
                                void *cuda_stream, void *workspace, size_t workspace_bytes, kiops_epirk_ctx *out) {
  if (!out) return KIOPS_ERR_INVALID_ARG;
  *out = nullptr;
  if (scheme != KIOPS_EPIRK4S3 && scheme != KIOPS_EPIRK4S3A) return KIOPS_ERR_INVALID_ARG;
  if (!(h > 0.0) || !std::isfinite(h)) return KIOPS_ERR_INVALID_ARG;
  size_t b1, b2, vec;
  kiops_status s = ep_sizes(pb, o, &b1, &b2, &vec);
  if (s != KIOPS_OK) return s;
  if (!workspace || ((uintptr_t)workspace & 255) || workspace_bytes < b1 + b2 + EP_VECS * vec)
    return KIOPS_ERR_WORKSPACE;
  kiops_epirk_ctx e = new (std::nothrow) kiops_epirk_s();
  if (!e) return KIOPS_ERR_WORKSPACE;
  e->scheme = scheme;
  e->stream = (cudaStream_t)cuda_stream;
  e->q.nx = pb->nx; e->q.ny = pb->ny; e->q.h = h;
  for (int i = 0; i < 5; i++) e->q.w[i] = pb->w[i];
  for (int i = 0; i < 4; i++) e->q.c[i] = pb->c[i];
  if (scheme == KIOPS_EPIRK4S3) { e->c2 = 1.0 / 8.0; e->c3 = 1.0 / 9.0; }   // Eq. 50
  else { e->c2 = 1.0 / 2.0; e->c3 = 2.0 / 3.0; }                             // Eq. 51
  unsigned char *ws = (unsigned char *)workspace;
  double **vp[EP_VECS] = {&e->d, &e->b1, &e->zero, &e->wa, &e->wb, &e->b3, &e->b4, &e->w};
  for (int i = 0; i < EP_VECS; i++) *vp[i] = (double *)(ws + b1 + b2 + (size_t)i * vec);
  kiops_options o1 = *o, o2 = *o;
  o1.task1 = 1; o1.host_staging = 0;
  o2.task1 = 0; o2.host_staging = 0;
  const kiops_operator_desc dsc = ep_desc(pb, h, e->d);
  s = kiops_create(&dsc, 1, &o1, cuda_stream, ws, b1, &e->k1);
  if (s == KIOPS_OK) s = kiops_create(&dsc, 4, &o2, cuda_stream, ws + b1, b2, &e->k2);
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

kiops_status kiops_epirk_step(kiops_epirk_ctx e, double *u, int nsteps, kiops_epirk_stats *stats) {
  if (!e || !u || nsteps < 0) return KIOPS_ERR_INVALID_ARG;
  const long long N = e->q.nx * e->q.ny;
  const int grid = (int)std::min<long long>((N + 255) / 256, SM_COUNT_HINT * 8);
  kiops_epirk_stats acc{};
  const bool asc = e->c2 < e->c3;  // call-1 outputs come in ascending T
  const double T1[2] = {asc ? e->c2 : e->c3, asc ? e->c3 : e->c2};
  double *w1[2] = {e->wa, e->wb};
  const double *w2 = asc ? e->wa : e->wb, *w3 = asc ? e->wb : e->wa;
  for (int n = 0; n < nsteps; n++) {
    k_ep_f<<<grid, 256, 0, e->stream>>>(e->q, u, e->d, e->b1);
    if (cudaGetLastError() != cudaSuccess) { e->err = "k_ep_f launch"; return KIOPS_ERR_CUDA; }
    kiops_stats s1{}, s2{};
    const double *u1[2] = {e->zero, e->b1};
    kiops_set_m_init(e->k1, e->m1);
    kiops_status s = kiops_apply(e->k1, u1, T1, 2, w1, &s1);
    if (s != KIOPS_OK) { e->err = "step " + std::to_string(n) + ", call 1: " + kiops_last_error(e->k1); return s; }
    e->m1 = s1.final_m;
    k_ep_stage<<<grid, 256, 0, e->stream>>>(e->q, e->scheme, e->c2, e->c3, u, w2, w3, e->b3, e->b4);
    if (cudaGetLastError() != cudaSuccess) { e->err = "k_ep_stage launch"; return KIOPS_ERR_CUDA; }
    const double *u2[5] = {e->zero, e->b1, e->zero, e->b3, e->b4};
    const double T2[1] = {1.0};
    double *wo[1] = {e->w};
    kiops_set_m_init(e->k2, e->m2);
    s = kiops_apply(e->k2, u2, T2, 1, wo, &s2);
    if (s != KIOPS_OK) { e->err = "step " + std::to_string(n) + ", call 2: " + kiops_last_error(e->k2); return s; }
    e->m2 = s2.final_m;
    k_ep_update<<<grid, 256, 0, e->stream>>>(N, e->w, u);
    if (cudaGetLastError() != cudaSuccess) { e->err = "k_ep_update launch"; return KIOPS_ERR_CUDA; }
    acc.steps++;
    acc.krylov_vectors += s1.krylov_vectors + s2.krylov_vectors;
    acc.passes += s1.passes + s2.passes;
    acc.substeps += s1.substeps + s2.substeps;
    acc.rejections += s1.rejections + s2.rejections;
    acc.expm_calls += s1.expm_calls + s2.expm_calls;
    acc.kiops_ms += s1.pass_ms + s1.ctrl_ms + s1.gemv_ms + s2.pass_ms + s2.ctrl_ms + s2.gemv_ms;
  }
  const cudaError_t ce = cudaStreamSynchronize(e->stream);
  if (ce != cudaSuccess) { e->err = cudaGetErrorString(ce); return KIOPS_ERR_CUDA; }
  acc.final_m[0] = e->m1;
  acc.final_m[1] = e->m2;
  if (stats) *stats = acc;
  return KIOPS_OK;
}

kiops_status kiops_epirk_destroy(kiops_epirk_ctx e) {
  if (!e) return KIOPS_ERR_INVALID_ARG;
  if (e->k1) kiops_destroy(e->k1);
  if (e->k2) kiops_destroy(e->k2);
  delete e;
  return KIOPS_OK;
}

const char *kiops_epirk_last_error(kiops_epirk_ctx e) { return e ? e->err.c_str() : "NULL ctx"; }
