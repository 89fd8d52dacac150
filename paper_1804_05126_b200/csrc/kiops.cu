// kiops.cu -- host side of the C ABI declared in include/kiops.h, plus the single
// translation unit that instantiates every device kernel (sm_100a).
//
// One kiops_apply = one H2D copy of the call block, ONE cudaGraphLaunch, one D2H
// copy of the device state, one stream synchronisation.  The graph is
//
//   k_setup                                  a1 (Eqs. 48-49), Alg. 1 l.2-8
//   WHILE (outer)                            Alg. 1 l.9   T_now < T_end
//     WHILE (inner)                          Alg. 2 l.2   j < m and not happy
//       k_pass_*  (CSR: k_csr_form, k_sell_spmv)     a2-a4
//     k_ctrl                                 a5-a7, Alg. 3 bookkeeping (one CTA)
//     IF (accept)
//       k_gemv                               a8, Alg. 3 l.15, l.20
//
// with the three conditional handles set from device code (no host round trip per
// step, no CPU fallback).
#include <cuda.h>  // CUtensorMap (encoded through cudaGetDriverEntryPoint: no libcuda link)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "controller.cuh"
#include "passq.cuh"
#include "kiops_internal.cuh"
#include "passes.cuh"
#include "inner.cuh"
#include "passrc.cuh"

namespace {

constexpr int SM_COUNT_HINT = 148;  // only if the device query fails

// SMs of the current device (grids of the persistent and one-wave kernels)
int sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      sms < 1) {
    cudaGetLastError();
    return SM_COUNT_HINT;
  }
  return sms;
}

// Padded mode: the 3D variable-kappa operator with an even nx runs
// the recompute pass (rc3d.cuh) on ghost-padded vectors.  KIOPS_3D=lazy keeps the lazy
// pair pass (A/B switch).
bool use_padded(const kiops_operator_desc *op, int p, const kiops_options *o) {
  if (op->kind != KIOPS_OP_STENCIL3D7_VARKAPPA || o->iop_q != 2) return false;
  if (op->nx % 2 != 0 || op->nx < 4 || op->ny < 4 || p > 4) return false;
  const char *e = getenv("KIOPS_3D");
  return !(e && strcmp(e, "lazy") == 0);
}

// v1 stencil tiles
#define T1D 1, 256, 1, 1
#define T2D 2, 64, 16, 1
#define T3D 3, 32, 8, 4
#ifndef L2YC
#define L2YC 8
#endif
#ifndef Q3Y
#define Q3Y 7   // lock-step 3D pass: max tile rows (config 4 bands: 6-7 rows)
#endif
#ifndef Q3D
#define Q3D 2   // planes in flight (p <= 2; p = 3, 4 use 1 to fit 2 CTAs/SM)
#endif
#define M3X 32   // one-point-per-thread 3D pass (odd nx / p > 4)
#define M3Y 8
#define M3Z 32   // z-planes per CTA chunk

struct Layout {
  size_t V, r, staging, state, call, H, sig, R2, tails, partials, recs, npart, scratch, coef, trace, sell_off, sell_col,
      sell_val, qa, gram, qpart, tmaps, total;
  bool padded = false;
  int Xp = 0, Yp = 0, rc_ntx = 0, rc_nb = 0, rc_zs = 0, nslots = 0;
  long long Np = 0;
  long long sell_entries;
  long long ldN;
  int grid_pass, grid_setup, grid_gemv, grid_form, grid_max;
  int block_pass;
  int nh3 = 1;  // 3D pair pass: z-parts per CTA
  int w2d = 8;  // 2D async pass: warps per CTA
  int yc2d = L2YC;  // 2D lazy pass: rows a warp's strip marches (8; 4 / 2 for small grids)
  size_t smem_pass;
};

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

long long op_n(const kiops_operator_desc *op) { return op->nx * op->ny * op->nz; }

kiops_status validate(const kiops_operator_desc *op, int p, const kiops_options *o, std::string &err) {
  if (!op || !o) { err = "NULL operator or options"; return KIOPS_ERR_INVALID_ARG; }
  if (op->nx < 1 || op->ny < 1 || op->nz < 1) { err = "grid extents must be >= 1"; return KIOPS_ERR_INVALID_ARG; }
  if (p < 0 || p > KIOPS_MAX_P) { err = "p must be in [0, KIOPS_MAX_P]"; return KIOPS_ERR_INVALID_ARG; }
  if (!(o->tol > 0.0) || !std::isfinite(o->tol)) { err = "tol must be > 0"; return KIOPS_ERR_INVALID_ARG; }
  if (o->m_min < 1 || o->m_min > o->m_max) { err = "need 1 <= m_min <= m_max"; return KIOPS_ERR_INVALID_ARG; }
  if (o->m_max > KIOPS_MAX_M) { err = "m_max > KIOPS_MAX_M (single-CTA exponential of (m_max+1)^2)"; return KIOPS_ERR_UNSUPPORTED; }
  if (o->m_init < 1) { err = "m_init must be >= 1"; return KIOPS_ERR_INVALID_ARG; }
  if (o->iop_q < 1 || o->iop_q > o->m_max) { err = "need 1 <= iop_q <= m_max"; return KIOPS_ERR_INVALID_ARG; }
  if (o->max_attempts < 1) { err = "max_attempts must be >= 1"; return KIOPS_ERR_INVALID_ARG; }
  if (o->corrected != 0 && o->corrected != 1) { err = "corrected must be 0 or 1"; return KIOPS_ERR_INVALID_ARG; }
  if (o->host_staging && (o->max_outputs < 1 || o->max_outputs > KIOPS_MAX_OUT)) {
    err = "max_outputs must be in [1, KIOPS_MAX_OUT]"; return KIOPS_ERR_INVALID_ARG;
  }
  switch (op->kind) {
    case KIOPS_OP_STENCIL1D3:
      if (op->ny != 1 || op->nz != 1) { err = "1D stencil needs ny = nz = 1"; return KIOPS_ERR_INVALID_ARG; }
      break;
    case KIOPS_OP_STENCIL2D5:
      if (op->nz != 1) { err = "2D stencil needs nz = 1"; return KIOPS_ERR_INVALID_ARG; }
      break;
    case KIOPS_OP_STENCIL3D7_VARKAPPA:
      if (!op->kappa) { err = "3D stencil needs kappa"; return KIOPS_ERR_INVALID_ARG; }
      if (op->nx * op->ny > 2147483647LL) { err = "3D stencil planes must have < 2^31 points"; return KIOPS_ERR_UNSUPPORTED; }
      break;
    case KIOPS_OP_CSR:
      if (op->ny != 1 || op->nz != 1) { err = "CSR needs ny = nz = 1 (nx = rows)"; return KIOPS_ERR_INVALID_ARG; }
      if (!op->row_ptr || !op->col_idx || !op->vals) { err = "CSR arrays must be non-NULL"; return KIOPS_ERR_INVALID_ARG; }
      if (op_n(op) > 2147483647LL) { err = "CSR with more than 2^31-1 rows (int32 col_idx)"; return KIOPS_ERR_UNSUPPORTED; }
      break;
    default:
      err = "unknown operator kind";
      return KIOPS_ERR_INVALID_ARG;
  }
  if (op->kind != KIOPS_OP_CSR && op->periodic != 1) { err = "stencils are periodic only"; return KIOPS_ERR_UNSUPPORTED; }
  return KIOPS_OK;
}

// SELL-32 slice offsets from the (device) CSR row pointer; host computation, done at
// workspace sizing / create time only (not on the apply path).
static std::vector<long long> sell_offsets(const kiops_operator_desc *op) {
  const long long N = op_n(op), ns = (N + 31) / 32;
  std::vector<long long> rp(N + 1), off(ns + 1, 0);
  if (cudaMemcpy(rp.data(), op->row_ptr, sizeof(long long) * (N + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
    return {};
  for (long long s = 0; s < ns; s++) {
    long long mx = 0;
    for (long long r = 32 * s; r < std::min(N, 32 * s + 32); r++) mx = std::max(mx, rp[r + 1] - rp[r]);
    off[s + 1] = off[s] + 32 * mx;
  }
  return off;
}
static long long sell_size(const kiops_operator_desc *op) {
  std::vector<long long> off = sell_offsets(op);
  return off.empty() ? -1 : off.back();
}

Layout layout(const kiops_operator_desc *op, int p, const kiops_options *o) {
  Layout L{};
  const long long N = op_n(op);
  L.ldN = (N + 31) & ~31LL;
  L.block_pass = 256;
  const long long blocks256 = (N + 255) / 256;
  L.grid_setup = (int)std::min<long long>(blocks256, sm_count() * 8);
  L.grid_gemv = (int)std::min<long long>((N / 2 + 255) / 256 + 1, sm_count() * 8);
  L.grid_form = L.grid_gemv;
  switch (op->kind) {
    case KIOPS_OP_STENCIL1D3:
    case KIOPS_OP_STENCIL2D5:
      if (op->nx % 2 == 0 && p <= 4) {  // warp-strip lazy kernel (16-byte pairs)
        // strip height: 8 rows; small grids take 4 or 2 so that more warps march shorter strips (the
        // pass of a small grid is the latency of one warp's march: config 2 passes 0.120 -> 0.091 ms
        // per call with 2 rows; from ~2^19 points the halo rows' extra loads cost more than they gain,
        // and 1024^2 needs 8 to stay one co-resident grid).  KIOPS_2D_YC=2|4|8 forces.
        const char *ey = getenv("KIOPS_2D_YC");
        const int yc = (ey && (atoi(ey) == 2 || atoi(ey) == 4 || atoi(ey) == 8)) ? atoi(ey)
                     : (N <= (1LL << 17) ? 2 : N <= (1LL << 19) ? 4 : L2YC);
        L.yc2d = yc;
        const long long strips = (op->nx + 59) / 60 * ((op->ny + yc - 1) / yc);
        const char *ev = getenv("KIOPS_2D_ASYNC");  // 0: register-prefetch body (A/B switch)
        // warps per CTA: 16 (one 512-thread CTA per SM: half the per-CTA dot records to gather
        // per pass) when that still fills >= 128 SMs -- config 3: 144 CTAs, pass 14.8 -> 13.6 us
        // (measured); else 8.  KIOPS_2D_WARPS=8|16 forces (async body only).
        const char *ew = getenv("KIOPS_2D_WARPS");
        L.w2d = (ew && (atoi(ew) == 8 || atoi(ew) == 16)) ? atoi(ew) : ((strips + 15) / 16 >= 128 ? 16 : 8);
        if (ev && ev[0] == '0') L.w2d = 8;
        L.block_pass = 32 * L.w2d;
        L.grid_pass = (int)((strips + L.w2d - 1) / L.w2d);
        L.smem_pass = (ev && ev[0] == '0') ? 0
                    : RING_SLACK + (L.w2d / 8) * (p == 0 ? Ring2<0, 2>::smem_bytes : p == 1 ? Ring2<1, 2>::smem_bytes
                                   : p == 2 ? Ring2<2, 2>::smem_bytes : p == 3 ? Ring2<3, 2>::smem_bytes
                                                                          : Ring2<4, 2>::smem_bytes);
      } else if (op->kind == KIOPS_OP_STENCIL1D3) {
        L.grid_pass = (int)((op->nx + 255) / 256);
        L.smem_pass = stencil_smem_bytes<T1D>();
      } else {
        L.grid_pass = (int)(((op->nx + 63) / 64) * ((op->ny + 15) / 16));
        L.smem_pass = stencil_smem_bytes<T2D>();
      }
      break;
    case KIOPS_OP_STENCIL3D7_VARKAPPA:
      if (use_padded(op, p, o)) {  // recompute pass on the padded layout (rc3d.cuh)
        const int sms = sm_count();
        L.padded = true;
        L.Xp = (int)op->nx + 4;
        L.Yp = (int)op->ny + 4;
        L.Np = (long long)L.Xp * L.Yp * op->nz;
        L.ldN = (L.Np + 31) & ~31LL;
        rc3::tiles((int)op->nx, (int)op->ny, (int)op->nz, sms, RC_HM, &L.rc_ntx, &L.rc_nb, &L.rc_zs);
        L.grid_pass = std::min(L.rc_ntx * L.rc_nb * L.rc_zs, sms);
        L.block_pass = RcCfg<0>::NT;
        L.smem_pass = p == 0 ? RcCfg<0>::smem_bytes : p == 1 ? RcCfg<1>::smem_bytes : p == 2 ? RcCfg<2>::smem_bytes
                    : p == 3 ? RcCfg<3>::smem_bytes : RcCfg<4>::smem_bytes;
      } else if (op->nx % 2 == 0 && op->nx >= 2 && p >= 1 && p <= 4) {  // lock-step persistent pair pass
        using Q = LazyQ<2, Q3Y, 2>;
        int ntx, nb;
        rc_tiles(op->nx, op->ny, Q::TILES, Q3Y, &ntx, &nb);
        const int zs = rc_zsplit(op->nx, op->ny, op->nz, Q::TILES, Q3Y, Q::CTAS);
        const char *ev = getenv("KIOPS_3D_NH");  // 1: one z-part per CTA (A/B switch)
        L.nh3 = (zs % 2 == 0 && !(ev && ev[0] == '1')) ? 2 : 1;
        L.grid_pass = ntx * nb * zs / L.nh3;
        L.smem_pass = RING_SLACK + L.nh3 * (p == 1 ? LazyQ<1, Q3Y, 2, Q3D>::half_bytes : p == 2 ? LazyQ<2, Q3Y, 2, Q3D>::half_bytes
                               : p == 3 ? LazyQ<3, Q3Y, 2, 1>::half_bytes : LazyQ<4, Q3Y, 2, 1>::half_bytes);
        L.block_pass = L.nh3 * Q::NT;
      } else {
        L.grid_pass = (int)(((op->nx + M3X - 1) / M3X) * ((op->ny + M3Y - 1) / M3Y) * ((op->nz + M3Z - 1) / M3Z));
        L.smem_pass = sizeof(double) * (p <= 2 ? Lazy3<M3X, M3Y, 2>::smem_doubles
                                       : p <= 4 ? Lazy3<M3X, M3Y, 4>::smem_doubles : Lazy3<M3X, M3Y, 8>::smem_doubles);
        L.block_pass = Lazy3<M3X, M3Y, 2>::NT;
      }
      break;
    default:  // CSR (SELL-32): thread per row, 8 CTAs of 256 per SM
      L.grid_pass = (int)std::min<long long>((N + 255) / 256, sm_count() * 8);
      L.smem_pass = 0;
  }
  L.grid_max = std::max(L.grid_pass, L.grid_setup);
  size_t off = 0;
  const size_t vec = (size_t)L.ldN * sizeof(double);
  // padded mode: basis slots 1..m_max+1, then copies of B's p columns and of kappa, one
  // 4-D tensor for the TMA maps; no r buffers (the recompute pass never stores r)
  L.nslots = (o->m_max + 1) + (L.padded ? p + 1 : 0);
  L.V = off; off += al((size_t)L.nslots * vec);
  L.r = off; off += L.padded ? 0 : 2 * al(vec);  // r_k ping-pong (lazy passes; CSR uses the first)
  L.staging = off; off += o->host_staging ? al((size_t)(p + 1 + o->max_outputs) * vec) : 0;
  L.state = off; off += al(sizeof(DevState));
  L.call = off; off += al(sizeof(CallBlock));
  L.H = off; off += al(sizeof(double) * LDH * LDH);
  L.sig = off; off += al(sizeof(double) * (LDH + 2));
  L.R2 = off; off += al(sizeof(double) * (LDH + 2));
  L.tails = off; off += al(sizeof(double) * (LDH + 2) * KMAXP);
  L.partials = off; off += al(sizeof(double) * NDOT * (size_t)L.grid_max);
  L.recs = off; off += al(sizeof(double) * 2 * 8 * (size_t)L.grid_max);
  L.npart = off; off += al(sizeof(double) * KMAXP * (size_t)L.grid_max);
  L.scratch = off; off += al(sizeof(double) * NSCR * (size_t)LDH * LDH);
  L.coef = off; off += al(sizeof(double) * (KMAXO + 1) * (size_t)LDH);
  L.trace = off; off += al(sizeof(kiops_trace_row) * (size_t)KIOPS_TRACE_CAP);
  L.qa = off; off += al(sizeof(double) * (size_t)LDH);                          // generic-q path
  L.gram = off; off += al(sizeof(double) * (size_t)LDH * LDH);
  L.qpart = off; off += al(sizeof(double) * (2 * (size_t)LDH + 2) * QG);
  L.tmaps = off; off += L.padded ? al(2 * sizeof(CUtensorMap)) : 0;
  L.sell_entries = 0;
  if (op->kind == KIOPS_OP_CSR) {  // SELL-32 copy: exact size from the row lengths
    const long long ns = (N + 31) / 32;
    L.sell_entries = sell_size(op);
    L.sell_off = off; off += al(sizeof(long long) * (size_t)(ns + 1));
    L.sell_col = off; off += al(sizeof(int) * (size_t)L.sell_entries);
    L.sell_val = off; off += al(sizeof(double) * (size_t)L.sell_entries);
  }
  L.total = off;
  return L;
}

size_t ctrl_smem_bytes() {
  const size_t n = KMAXM + 1, cb = (n + CTRL_CL - 1) / CTRL_CL;
  const size_t solve = sizeof(double) * (n * n + n * cb);
  const size_t np = (n + 7) & ~(size_t)7;
  const size_t mm = sizeof(double) * MM_LD * (np + 8 * ((np / 8 + CTRL_CL - 1) / CTRL_CL));  // A + B panels
  const size_t small = sizeof(double) * (10 * (size_t)SM_LD * SMALL_N + 64);  // single-CTA path
  return std::max(std::max(solve, mm), small);
}

}  // namespace

struct kiops_ctx_s {
  KParams P{};
  Layout L{};
  kiops_operator_desc op{};
  kiops_options o{};
  int p = 0;
  cudaStream_t stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  CallBlock *h_call = nullptr;   // pinned
  DevState *h_state = nullptr;   // pinned
  unsigned char *ws = nullptr;
  int n_forced = 0;
  double forced_tau[KIOPS_MAX_FORCED];
  int forced_m[KIOPS_MAX_FORCED];
  int forced_acc[KIOPS_MAX_FORCED];
  long long last_attempts = 0;
  int m_init_call = 0;           // kiops_set_m_init (0: options.m_init)
  int align16 = 0;               // the chosen pass kernels read u, diag, kappa as 16-byte pairs
  void *fpass = nullptr;         // stencil pass kernel (NULL for CSR)
  void *finner = nullptr;        // persistent inner-loop kernel (inner.cuh), NULL if not used
  std::string err;
};

static kiops_status cuda_fail(kiops_ctx c, cudaError_t e, const char *what) {
  if (c) {
    c->err = std::string(what) + ": " + cudaGetErrorString(e);
  }
  return KIOPS_ERR_CUDA;
}

#define CK(call, what)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, what); \
  } while (0)

static cudaError_t add_kernel(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, size_t nd,
                              void *func, int grid, int block, size_t smem, KParams *P, int grid_y = 1) {
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeKernel;
  void *args[] = {P};
  np.kernel.func = func;
  np.kernel.gridDim = dim3(grid, grid_y);
  np.kernel.blockDim = dim3(block);
  np.kernel.sharedMemBytes = (unsigned)smem;
  np.kernel.kernelParams = args;
  return cudaGraphAddNode(node, g, deps, nd, &np);
}

static cudaError_t add_cond(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, size_t nd,
                            cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type, cudaGraph_t *body) {
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = type;
  np.conditional.size = 1;
  cudaError_t e = cudaGraphAddNode(node, g, deps, nd, &np);
  if (e == cudaSuccess) *body = np.conditional.phGraph_out[0];
  return e;
}

// TMA tensor maps of the padded 4-D tensor [Xp][Yp][nz][nslots] (basis slots, B copies,
// kappa copy; slot stride ldN doubles): box 68 x (HM+4) (halo-2 operands x_{k-1},
// kappa) and 68 x (HM+2) (halo-1 operands x_{k-2}, B).  Encoded on the host once per
// ctx, stored in the workspace (the kernels pass their global address to the TMA unit).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static kiops_status encode_tmaps(kiops_ctx c) {
  const Layout &L = c->L;
  EncodeTiledFn enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &qr), "driver entry point");
  if (!enc || qr != cudaDriverEntryPointSuccess) {
    c->err = "cuTensorMapEncodeTiled unavailable";
    return KIOPS_ERR_CUDA;
  }
  CUtensorMap maps[2];
  const cuuint64_t gdim[4] = {(cuuint64_t)L.Xp, (cuuint64_t)L.Yp, (cuuint64_t)c->op.nz, (cuuint64_t)L.nslots};
  const cuuint64_t gstr[3] = {(cuuint64_t)L.Xp * 8, (cuuint64_t)L.Xp * L.Yp * 8, (cuuint64_t)L.ldN * 8};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  for (int m = 0; m < 2; m++) {
    const cuuint32_t box[4] = {(cuuint32_t)RcCfg<0>::W, (cuuint32_t)(m == 0 ? RcCfg<0>::RA : RcCfg<0>::RB), 1, 1};
    const CUresult r = enc(&maps[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, c->P.V, gdim, gstr, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      c->err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
      return KIOPS_ERR_CUDA;
    }
  }
  CK(cudaMemcpyAsync((void *)c->P.tmapA, maps, sizeof(maps), cudaMemcpyHostToDevice, c->stream), "H2D tensor maps");
  CK(cudaStreamSynchronize(c->stream), "tensor maps");
  return KIOPS_OK;
}

static kiops_status build_graph(kiops_ctx c) {
  KParams &P = c->P;
  CK(cudaGraphCreate(&c->graph, 0), "cudaGraphCreate");
  CK(cudaGraphConditionalHandleCreate(&P.h_outer, c->graph, 1, cudaGraphCondAssignDefault), "handle outer");
  CK(cudaGraphConditionalHandleCreate(&P.h_accept, c->graph, 0, cudaGraphCondAssignDefault), "handle accept");

  void *fpass = nullptr;
  const bool lazy2d = c->op.nx % 2 == 0 && c->p <= 4;
// a 2D kernel instantiation by p (0..4) and strip height (Layout::yc2d); VA: the remaining template arguments
#define SEL2D_P(FN, YC, ...)                                                                                         \
  (c->p == 0 ? (void *)FN<YC, 0, __VA_ARGS__> : c->p == 1 ? (void *)FN<YC, 1, __VA_ARGS__>                           \
   : c->p == 2 ? (void *)FN<YC, 2, __VA_ARGS__> : c->p == 3 ? (void *)FN<YC, 3, __VA_ARGS__> : (void *)FN<YC, 4, __VA_ARGS__>)
#define SEL2D(FN, ...)                                                                                               \
  (c->L.yc2d == 2 ? SEL2D_P(FN, 2, __VA_ARGS__) : c->L.yc2d == 4 ? SEL2D_P(FN, 4, __VA_ARGS__) : SEL2D_P(FN, L2YC, __VA_ARGS__))
  switch (c->op.kind) {
    case KIOPS_OP_STENCIL1D3:
    case KIOPS_OP_STENCIL2D5:
      if (lazy2d && c->L.smem_pass == 0)  // strip height 8, 2 CTAs/SM: measured best of YC 4/8/16 and 2-3 CTAs/SM
        fpass = SEL2D(k_pass_2d_lazy, 2);
      else if (lazy2d && c->L.w2d == 16)
        fpass = SEL2D(k_pass_2d_lazy, 1, 2, 512);
      else if (lazy2d)  // cp.async ring, 2 rows in flight per warp
        fpass = SEL2D(k_pass_2d_lazy, 2, 2);
      else
        fpass = c->op.kind == KIOPS_OP_STENCIL1D3 ? (void *)k_pass_stencil<T1D> : (void *)k_pass_stencil<T2D>;
      break;
    case KIOPS_OP_STENCIL3D7_VARKAPPA:
      if (c->L.padded)
        fpass = c->p == 0 ? (void *)k_pass_3d_rc<0> : c->p == 1 ? (void *)k_pass_3d_rc<1> : c->p == 2 ? (void *)k_pass_3d_rc<2>
              : c->p == 3 ? (void *)k_pass_3d_rc<3> : (void *)k_pass_3d_rc<4>;
      else if (c->op.nx % 2 == 0 && c->op.nx >= 2 && c->p >= 1 && c->p <= 4)
        fpass = c->L.nh3 == 2
                    ? (c->p == 1 ? (void *)k_pass_3d_lazyq<1, Q3Y, 2, Q3D, 2> : c->p == 2 ? (void *)k_pass_3d_lazyq<2, Q3Y, 2, Q3D, 2>
                       : c->p == 3 ? (void *)k_pass_3d_lazyq<3, Q3Y, 2, 1, 2> : (void *)k_pass_3d_lazyq<4, Q3Y, 2, 1, 2>)
                    : (c->p == 1 ? (void *)k_pass_3d_lazyq<1, Q3Y, 2, Q3D> : c->p == 2 ? (void *)k_pass_3d_lazyq<2, Q3Y, 2, Q3D>
                       : c->p == 3 ? (void *)k_pass_3d_lazyq<3, Q3Y, 2, 1> : (void *)k_pass_3d_lazyq<4, Q3Y, 2, 1>);
      else
        fpass = c->p <= 2 ? (void *)k_pass_3d_lazy<M3X, M3Y, M3Z, 2, 3>
              : c->p <= 4 ? (void *)k_pass_3d_lazy<M3X, M3Y, M3Z, 4, 3>
                          : (void *)k_pass_3d_lazy<M3X, M3Y, M3Z, 8, 2>;
      break;
    default: break;
  }
  c->fpass = fpass;
  if (fpass && c->L.smem_pass > 0)
    CK(cudaFuncSetAttribute(fpass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->L.smem_pass), "smem attr pass");

  // persistent inner loop (inner.cuh) for the fused q = 2 stencil passes, when the whole
  // pass grid is co-resident; KIOPS_PERSIST=0 in the environment keeps one launch per pass
  void *finner = nullptr;
  const char *pe = getenv("KIOPS_PERSIST");
  if (P.q == 2 && !(pe && pe[0] == '0')) {
    if (lazy2d && (c->op.kind == KIOPS_OP_STENCIL1D3 || c->op.kind == KIOPS_OP_STENCIL2D5) && c->L.smem_pass == 0)
      finner = SEL2D(k_inner_2d_lazy, 2);
    else if (lazy2d && (c->op.kind == KIOPS_OP_STENCIL1D3 || c->op.kind == KIOPS_OP_STENCIL2D5) && c->L.w2d == 16)
      finner = SEL2D(k_inner_2d_lazy, 1, 2, 512);
    else if (lazy2d && (c->op.kind == KIOPS_OP_STENCIL1D3 || c->op.kind == KIOPS_OP_STENCIL2D5))
      finner = SEL2D(k_inner_2d_lazy, 2, 2);
    else if (c->L.padded)
      finner = c->p == 0 ? (void *)k_inner_3d_rc<0> : c->p == 1 ? (void *)k_inner_3d_rc<1> : c->p == 2 ? (void *)k_inner_3d_rc<2>
             : c->p == 3 ? (void *)k_inner_3d_rc<3> : (void *)k_inner_3d_rc<4>;
    else if (c->op.kind == KIOPS_OP_STENCIL3D7_VARKAPPA && c->op.nx % 2 == 0 && c->op.nx >= 2 && c->p >= 1 &&
             c->p <= 4)
      finner = c->L.nh3 == 2
                   ? (c->p == 1 ? (void *)k_inner_3d_lazyq<1, Q3Y, 2, Q3D, 2> : c->p == 2 ? (void *)k_inner_3d_lazyq<2, Q3Y, 2, Q3D, 2>
                      : c->p == 3 ? (void *)k_inner_3d_lazyq<3, Q3Y, 2, 1, 2> : (void *)k_inner_3d_lazyq<4, Q3Y, 2, 1, 2>)
                   : (c->p == 1 ? (void *)k_inner_3d_lazyq<1, Q3Y, 2, Q3D> : c->p == 2 ? (void *)k_inner_3d_lazyq<2, Q3Y, 2, Q3D>
                      : c->p == 3 ? (void *)k_inner_3d_lazyq<3, Q3Y, 2, 1> : (void *)k_inner_3d_lazyq<4, Q3Y, 2, 1>);
    if (finner) {
      if (c->L.smem_pass > 0)
        CK(cudaFuncSetAttribute(finner, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->L.smem_pass),
           "smem attr inner");
      int dev = 0, sms = 0, per_sm = 0;
      CK(cudaGetDevice(&dev), "cudaGetDevice");
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, finner, c->L.block_pass, c->L.smem_pass),
         "occupancy inner");
      if ((long long)per_sm * sms < c->L.grid_pass) finner = nullptr;  // not co-resident: per-pass launches
    }
  }
  // CSR: the persistent loop for small matrices only (inner.cuh, k_inner_csr); KIOPS_CSR_PERSIST=0|1
  // forces per-pass launches / the persistent loop
  if (P.q == 2 && c->op.kind == KIOPS_OP_CSR && !(pe && pe[0] == '0')) {
    const char *ce = getenv("KIOPS_CSR_PERSIST");
    // default: matrices whose pass streams <= 64 MB (12 bytes per nonzero + 8 vectors), i.e. a pass of at
    // most ~15 us, the order of the per-pass launch overhead it removes
    const long long pass_bytes = 12LL * (long long)c->op.nnz + 64LL * c->P.N;
    const bool want = ce ? ce[0] != '0' : (pass_bytes <= (64LL << 20));
    if (want) {
      int dev = 0, sms = 0, per_sm = 0;
      CK(cudaGetDevice(&dev), "cudaGetDevice");
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (void *)k_inner_csr, 256, 0), "occupancy csr");
      if (per_sm >= 1) {
        finner = (void *)k_inner_csr;
        // few CTAs: every pass ends in two grid barriers and every CTA reads every CTA's dot record
        // (measured, EPIRK4s3 steps: ADR 400^2 1.14 / 1.02 / 1.26 ms and Allen-Cahn 500^2 5.99 / 4.46 / 5.14 ms
        // with 1 / 2 / 4 CTAs per SM; per-pass launches: 1.43 and 5.84)
        const char *ge = getenv("KIOPS_CSR_CPS");  // CTAs per SM of the persistent CSR loop (default 2)
        const int cps = std::max(1, std::min(per_sm, ge ? atoi(ge) : 2));
        c->L.grid_pass = (int)std::min<long long>(c->L.grid_pass, (long long)cps * sms);
        c->L.block_pass = 256;
        c->L.smem_pass = 0;
      }
    }
  }
  c->finner = finner;
  CK(cudaFuncSetAttribute((void *)k_ctrl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctrl_smem_bytes()),
     "smem attr ctrl");

  // (set before any node is added: every kernel node copies P)
  const char *fe = getenv("KIOPS_FLAT");  // 0: keep the inner WHILE node around the persistent kernel (A/B switch)
  const bool flat = finner && P.q == 2 && !(fe && fe[0] == '0');
  P.flat_inner = flat ? 1 : 0;
  if (!flat) CK(cudaGraphConditionalHandleCreate(&P.h_inner, c->graph, 1, cudaGraphCondAssignDefault), "handle inner");
  cudaGraphNode_t n_setup, n_outer, n_inner, n_ctrl, n_if, n_a, n_b, n_gemv;
  cudaGraph_t b_outer, b_inner, b_if;
  CK(add_kernel(c->graph, &n_setup, nullptr, 0, (void *)k_setup, c->L.grid_setup, 256, 0, &P), "node setup");
  CK(add_cond(c->graph, &n_outer, &n_setup, 1, P.h_outer, cudaGraphCondTypeWhile, &b_outer), "node outer");
  // persistent inner loop: ONE launch runs every pass of the attempt, so the kernel is a plain
  // node of the outer loop's body (it returns at once when the attempt needs no pass); the other
  // paths launch per pass inside an inner WHILE node
  if (flat) {
    CK(add_kernel(b_outer, &n_a, nullptr, 0, finner, c->L.grid_pass, c->L.block_pass, c->L.smem_pass, &P), "node inner");
    cudaLaunchAttributeValue av = {};
    av.cooperative = 1;
    CK(cudaGraphKernelNodeSetAttribute(n_a, cudaLaunchAttributeCooperative, &av), "cooperative attr");
    n_inner = n_a;
  } else {
  CK(add_cond(b_outer, &n_inner, nullptr, 0, P.h_inner, cudaGraphCondTypeWhile, &b_inner), "node inner");
  if (P.q != 2) {  // generic IOP window (passq.cuh): form, apply, window dots, finalise
    cudaGraphNode_t n_c, n_d;
    CK(add_kernel(b_inner, &n_a, nullptr, 0, (void *)k_q_form, c->L.grid_form, 256, 0, &P), "node q form");
    CK(add_kernel(b_inner, &n_b, &n_a, 1, (void *)k_q_apply, QG, 256, 0, &P), "node q apply");
    CK(add_kernel(b_inner, &n_c, &n_b, 1, (void *)k_q_dots, QG, 256, 0, &P, P.q), "node q dots");
    CK(add_kernel(b_inner, &n_d, &n_c, 1, (void *)k_q_finalize, 1, 256, 0, &P), "node q finalize");
  } else if (finner) {  // the WHILE body runs once: the kernel loops over the passes itself
    CK(add_kernel(b_inner, &n_a, nullptr, 0, finner, c->L.grid_pass, c->L.block_pass, c->L.smem_pass, &P),
       "node inner");
    cudaLaunchAttributeValue av = {};
    av.cooperative = 1;
    CK(cudaGraphKernelNodeSetAttribute(n_a, cudaLaunchAttributeCooperative, &av), "cooperative attr");
  } else if (c->op.kind == KIOPS_OP_CSR) {
    CK(add_kernel(b_inner, &n_a, nullptr, 0, (void *)k_csr_form, c->L.grid_form, 256, 0, &P), "node form");
    CK(add_kernel(b_inner, &n_b, &n_a, 1, (void *)k_sell_spmv, c->L.grid_pass, 256, 0, &P), "node spmv");
  } else {
    CK(add_kernel(b_inner, &n_a, nullptr, 0, fpass, c->L.grid_pass, c->L.block_pass, c->L.smem_pass, &P), "node pass");
  }
  }
  CK(add_kernel(b_outer, &n_ctrl, &n_inner, 1, (void *)k_ctrl, CTRL_CL, CTRL_THREADS, ctrl_smem_bytes(), &P), "node ctrl");
  CK(add_cond(b_outer, &n_if, &n_ctrl, 1, P.h_accept, cudaGraphCondTypeIf, &b_if), "node if");
  CK(add_kernel(b_if, &n_gemv, nullptr, 0, (void *)k_gemv, c->L.grid_gemv, 256, 0, &P), "node gemv");
  CK(cudaGraphInstantiate(&c->exec, c->graph, 0), "cudaGraphInstantiate");
  return KIOPS_OK;
}

extern "C" {

void kiops_options_default(kiops_options *o) {
  if (!o) return;
  o->tol = 1e-7;
  o->m_init = 10;
  o->m_min = 10;
  o->m_max = 128;
  o->iop_q = 2;
  o->task1 = 0;
  o->max_attempts = 10000;
  o->host_staging = 0;
  o->max_outputs = 4;
  o->corrected = 0;
}

kiops_status kiops_workspace_bytes(const kiops_operator_desc *op, int p, const kiops_options *o, size_t *bytes) {
  std::string err;
  kiops_status s = validate(op, p, o, err);
  if (s != KIOPS_OK) return s;
  if (!bytes) return KIOPS_ERR_INVALID_ARG;
  const Layout L = layout(op, p, o);
  if (op->kind == KIOPS_OP_CSR && L.sell_entries < 0) return KIOPS_ERR_CUDA;  // row_ptr not readable
  *bytes = L.total;
  return KIOPS_OK;
}

kiops_status kiops_create(const kiops_operator_desc *op, int p, const kiops_options *o, void *cuda_stream,
                          void *workspace, size_t workspace_bytes, kiops_ctx *out) {
  if (!out) return KIOPS_ERR_INVALID_ARG;
  *out = nullptr;
  std::string err;
  kiops_status s = validate(op, p, o, err);
  if (s != KIOPS_OK) return s;
  const Layout L = layout(op, p, o);
  if (!workspace || ((uintptr_t)workspace & 255) || workspace_bytes < L.total) return KIOPS_ERR_WORKSPACE;
  kiops_ctx c = new (std::nothrow) kiops_ctx_s();
  if (!c) return KIOPS_ERR_CUDA;
  c->op = *op;
  c->o = *o;
  c->p = p;
  c->L = L;
  c->stream = (cudaStream_t)cuda_stream;
  c->ws = (unsigned char *)workspace;
  KParams &P = c->P;
  P.kind = op->kind;
  P.nx = op->nx; P.ny = op->ny; P.nz = op->nz;
  P.N = op_n(op);
  P.ldN = L.ldN;
  for (int i = 0; i < 5; i++) P.w[i] = P.w5[i] = op->w[i];
  if (op->kind == KIOPS_OP_STENCIL1D3) {  // 1D {W, C, E} -> {W, E, 0, 0, C}
    P.w5[0] = op->w[0]; P.w5[1] = op->w[2]; P.w5[2] = 0.0; P.w5[3] = 0.0; P.w5[4] = op->w[1];
  }
  if (op->kind == KIOPS_OP_STENCIL1D3 && op->nx % 2 == 0 && p <= 4) {
    // the 1D operator runs on the 2D warp-strip kernel (ny = 1): {W, E, S, N, C} = {W, E, 0, 0, C}
    P.w[0] = op->w[0]; P.w[1] = op->w[2]; P.w[2] = 0.0; P.w[3] = 0.0; P.w[4] = op->w[1];
  }
  P.diag = op->diag;
  P.kappa = op->kappa;
  P.inv_h2 = op->inv_h2;
  P.row_ptr = (const long long *)op->row_ptr;
  P.col_idx = op->col_idx;
  P.vals = op->vals;
  P.p = p;
  P.tol = o->tol;
  P.m_init = o->m_init; P.m_min = o->m_min; P.m_max = o->m_max;
  P.task1 = o->task1;
  P.corrected = o->corrected;
  P.max_attempts = o->max_attempts;
  unsigned char *w = c->ws;
  P.V = (double *)(w + L.V);
  P.r = (double *)(w + L.r);
  P.st = (DevState *)(w + L.state);
  P.call = (CallBlock *)(w + L.call);
  P.H = (double *)(w + L.H);
  P.sig = (double *)(w + L.sig);
  P.R2 = (double *)(w + L.R2);
  P.tails = (double *)(w + L.tails);
  P.partials = (double *)(w + L.partials);
  P.recs = (double *)(w + L.recs);
  P.npart = (double *)(w + L.npart);
  P.scratch = (double *)(w + L.scratch);
  P.coef = (double *)(w + L.coef);
  P.trace = (kiops_trace_row *)(w + L.trace);
  P.qa = (double *)(w + L.qa);
  P.gram = (double *)(w + L.gram);
  P.qpart = (double *)(w + L.qpart);
  P.q = o->iop_q;
  if (op->kind == KIOPS_OP_CSR) {
    P.sell_off = (const long long *)(w + L.sell_off);
    P.sell_col = (const int *)(w + L.sell_col);
    P.sell_val = (const double *)(w + L.sell_val);
  }
  P.grid_pass = L.grid_pass;
  P.grid_max = L.grid_max;
  if (L.padded) {
    P.padded = 1;
    P.Xp = L.Xp; P.Yp = L.Yp; P.Np = L.Np;
    P.rc_ntx = L.rc_ntx; P.rc_nb = L.rc_nb; P.rc_zs = L.rc_zs;
    P.slot_B = o->m_max + 1;
    P.slot_kappa = o->m_max + 1 + p;
    P.r = nullptr;
    P.tmapA = w + L.tmaps;
    P.tmapB = w + L.tmaps + sizeof(CUtensorMap);
  }
  kiops_status st = KIOPS_OK;
  cudaError_t e = cudaMallocHost((void **)&c->h_call, sizeof(CallBlock));
  if (e == cudaSuccess) e = cudaMallocHost((void **)&c->h_state, sizeof(DevState));
  if (e != cudaSuccess) st = cuda_fail(c, e, "cudaMallocHost");
  if (st == KIOPS_OK) {
    memset(c->h_call, 0, sizeof(CallBlock));
    e = cudaMemsetAsync(P.st, 0, sizeof(DevState), c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(P.H, 0, sizeof(double) * LDH * LDH, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) st = cuda_fail(c, e, "workspace init");
  }
  // the lazy pair kernels (1D/2D with even nx, 3D lazy with even nx) read u, diag and kappa
  // with 16-byte loads: a misaligned device pointer would fault (sticky CUDA error), so it
  // is rejected here and in check_call instead (kiops.h, "alignment")
  c->align16 = (o->iop_q == 2 && op->nx % 2 == 0 && !L.padded &&
                ((op->kind == KIOPS_OP_STENCIL1D3 || op->kind == KIOPS_OP_STENCIL2D5) && p <= 4 ||
                 (op->kind == KIOPS_OP_STENCIL3D7_VARKAPPA && p >= 1 && p <= 4)))
                   ? 1 : 0;
  if (st == KIOPS_OK && c->align16 && (((uintptr_t)op->diag & 15) || ((uintptr_t)op->kappa & 15))) {
    c->err = "diag / kappa must be 16-byte aligned for this operator (even nx: 16-byte pair loads)";
    st = KIOPS_ERR_INVALID_ARG;
  }
  if (st == KIOPS_OK && L.padded) st = encode_tmaps(c);
  if (st == KIOPS_OK && op->kind == KIOPS_OP_CSR) {  // build the SELL-32 copy once
    std::vector<long long> off = sell_offsets(op);
    if (off.empty() || off.back() != L.sell_entries) {
      c->err = "SELL sizing failed (row_ptr changed between kiops_workspace_bytes and kiops_create?)";
      st = KIOPS_ERR_WORKSPACE;
    } else {
      e = cudaMemcpy((void *)P.sell_off, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) {
        k_sell_build<<<sm_count() * 8, 256, 0, c->stream>>>(P.N, P.row_ptr, P.col_idx, P.vals, P.sell_off,
                                                               (int *)P.sell_col, (double *)P.sell_val);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
      if (e != cudaSuccess) st = cuda_fail(c, e, "SELL build");
    }
  }
  if (st == KIOPS_OK) st = build_graph(c);
  if (st != KIOPS_OK) {
    fprintf(stderr, "kiops_create: %s\n", c->err.c_str());
    kiops_destroy(c);
    return st;
  }
  *out = c;
  return KIOPS_OK;
}

static kiops_status check_call(kiops_ctx c, const double *const *u, const double *T, int n_out, double *const *w) {
  if (!c || !u || !T || !w) return KIOPS_ERR_INVALID_ARG;
  if (n_out < 1 || n_out > KIOPS_MAX_OUT) { c->err = "n_out must be in [1, KIOPS_MAX_OUT]"; return KIOPS_ERR_INVALID_ARG; }
  for (int l = 0; l < n_out; l++) {
    if (!std::isfinite(T[l]) || !(T[l] > 0.0) || (l > 0 && !(T[l] > T[l - 1]))) {
      c->err = "output times must satisfy 0 < T_1 < ... < T_n (R21)";
      return KIOPS_ERR_INVALID_ARG;
    }
    if (!w[l]) { c->err = "NULL output pointer"; return KIOPS_ERR_INVALID_ARG; }
  }
  for (int k = 0; k <= c->p; k++) {
    if (!u[k]) { c->err = "NULL input vector"; return KIOPS_ERR_INVALID_ARG; }
    if (c->align16 && ((uintptr_t)u[k] & 15)) {  // 16-byte pair loads (kiops.h: alignment)
      c->err = "input vectors must be 16-byte aligned for this operator (even nx: 16-byte pair loads)";
      return KIOPS_ERR_INVALID_ARG;
    }
  }
  return KIOPS_OK;
}

static kiops_status launch_and_finish(kiops_ctx c, kiops_stats *stats) {
  CK(cudaMemcpyAsync(c->P.call, c->h_call, sizeof(CallBlock), cudaMemcpyHostToDevice, c->stream), "H2D call block");
  CK(cudaGraphLaunch(c->exec, c->stream), "cudaGraphLaunch");
  CK(cudaMemcpyAsync(c->h_state, c->P.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream), "D2H state");
  return KIOPS_OK;
}

static kiops_status finish(kiops_ctx c, kiops_stats *stats) {
  CK(cudaStreamSynchronize(c->stream), "stream sync");
  CK(cudaGetLastError(), "kernel error");
  const DevState &S = *c->h_state;
  c->last_attempts = S.attempt;
  if (stats) {
    stats->substeps = S.substeps;
    stats->rejections = S.rejections;
    stats->krylov_vectors = S.kv;
    stats->expm_calls = S.expm_calls;
    stats->passes = S.passes;
    stats->final_m = S.final_m;
    stats->happy_breakdowns = (int)S.happy_count;
    stats->t_reached = S.t_now;
    stats->nu = S.nu;
    stats->mu = S.mu;
    stats->pass_ms = S.ns_pass * 1e-6;
    stats->ctrl_ms = S.ns_ctrl * 1e-6;
    stats->gemv_ms = S.ns_gemv * 1e-6;
    stats->expm_ms = S.ns_expm * 1e-6;
    stats->pass_launches = (int64_t)S.launches;
  }
  if (S.status == KIOPS_ERR_NONFINITE) { c->err = "non-finite value in the Krylov recurrence or estimate"; return KIOPS_ERR_NONFINITE; }
  if (S.status == KIOPS_ERR_NO_CONVERGENCE) { c->err = "max_attempts exceeded"; return KIOPS_ERR_NO_CONVERGENCE; }
  if (S.status != 0) { c->err = "device status"; return (kiops_status)S.status; }
  return KIOPS_OK;
}

static void fill_call(kiops_ctx c, const double *const *u, const double *T, int n_out, double *const *w) {
  CallBlock &B = *c->h_call;
  for (int k = 0; k <= KMAXP; k++) B.u[k] = k <= c->p ? u[k] : nullptr;
  for (int l = 0; l < KMAXO; l++) {
    B.w[l] = l < n_out ? w[l] : nullptr;
    B.T[l] = l < n_out ? T[l] : 0.0;
  }
  B.n_out = n_out;
  B.m_init = c->m_init_call;
  B.n_forced = c->n_forced;
  for (int i = 0; i < c->n_forced; i++) {
    B.forced_tau[i] = c->forced_tau[i];
    B.forced_m[i] = c->forced_m[i];
    B.forced_acc[i] = c->forced_acc[i];
  }
}

kiops_status kiops_apply(kiops_ctx c, const double *const *u, const double *tau_out, int n_out, double *const *w,
                         kiops_stats *stats) {
  kiops_status s = check_call(c, u, tau_out, n_out, w);
  if (s != KIOPS_OK) return s;
  fill_call(c, u, tau_out, n_out, w);
  s = launch_and_finish(c, stats);
  if (s != KIOPS_OK) return s;
  return finish(c, stats);
}

kiops_status kiops_apply_host(kiops_ctx c, const double *const *u, const double *tau_out, int n_out, double *const *w,
                              kiops_stats *stats) {
  kiops_status s = check_call(c, u, tau_out, n_out, w);
  if (s != KIOPS_OK) return s;
  if (!c->o.host_staging || n_out > c->o.max_outputs) {
    c->err = "kiops_apply_host needs host_staging and n_out <= max_outputs";
    return KIOPS_ERR_WORKSPACE;
  }
  const size_t vb = (size_t)c->P.N * sizeof(double);
  double *stg = (double *)(c->ws + c->L.staging);
  const double *ud[KMAXP + 1];
  double *wd[KMAXO];
  for (int k = 0; k <= c->p; k++) {
    ud[k] = stg + (size_t)k * c->L.ldN;
    CK(cudaMemcpyAsync((void *)ud[k], u[k], vb, cudaMemcpyHostToDevice, c->stream), "H2D u");
  }
  bool direct[KMAXO];
  for (int l = 0; l < n_out; l++) {
    // pinned + device-mapped host output: the GEMV writes it over the host link
    cudaPointerAttributes pa{};
    direct[l] = cudaPointerGetAttributes(&pa, w[l]) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                pa.devicePointer != nullptr;
    if (!direct[l]) cudaGetLastError();  // clear a "not a CUDA pointer" error of the query
    wd[l] = direct[l] ? (double *)pa.devicePointer : stg + (size_t)(c->p + 1 + l) * c->L.ldN;
  }
  fill_call(c, ud, tau_out, n_out, wd);
  s = launch_and_finish(c, stats);
  if (s != KIOPS_OK) return s;
  for (int l = 0; l < n_out; l++)
    if (!direct[l]) CK(cudaMemcpyAsync(w[l], wd[l], vb, cudaMemcpyDeviceToHost, c->stream), "D2H w");
  return finish(c, stats);
}

static kiops_status launch_plain(kiops_ctx c, void *f, int grid, int block, size_t smem, KParams *P) {
  void *args[] = {P};
  CK(cudaLaunchKernel(f, dim3(grid), dim3(block), args, smem, c->stream), "cudaLaunchKernel");
  return KIOPS_OK;
}

static kiops_status read_conds(kiops_ctx c, unsigned *cond) {
  CK(cudaMemcpyAsync(cond, c->P.st->cond, sizeof(unsigned) * 3, cudaMemcpyDeviceToHost, c->stream), "D2H cond");
  CK(cudaStreamSynchronize(c->stream), "sync cond");
  return KIOPS_OK;
}

kiops_status kiops_apply_hostloop(kiops_ctx c, const double *const *u, const double *tau_out, int n_out,
                                  double *const *w, kiops_stats *stats) {
  kiops_status s = check_call(c, u, tau_out, n_out, w);
  if (s != KIOPS_OK) return s;
  fill_call(c, u, tau_out, n_out, w);
  KParams P = c->P;
  P.no_cond = 1;
  unsigned *cond = (unsigned *)(c->h_state);  // scratch in pinned memory, overwritten below
  CK(cudaMemcpyAsync(c->P.call, c->h_call, sizeof(CallBlock), cudaMemcpyHostToDevice, c->stream), "H2D call block");
  if ((s = launch_plain(c, (void *)k_setup, c->L.grid_setup, 256, 0, &P)) != KIOPS_OK) return s;
  if ((s = read_conds(c, cond)) != KIOPS_OK) return s;
  while (cond[COND_OUTER]) {
    while (cond[COND_INNER]) {
      if (P.q != 2) {
        void *args[] = {&P};
        if ((s = launch_plain(c, (void *)k_q_form, c->L.grid_form, 256, 0, &P)) != KIOPS_OK) return s;
        if ((s = launch_plain(c, (void *)k_q_apply, QG, 256, 0, &P)) != KIOPS_OK) return s;
        CK(cudaLaunchKernel((void *)k_q_dots, dim3(QG, P.q), dim3(256), args, 0, c->stream), "k_q_dots");
        if ((s = launch_plain(c, (void *)k_q_finalize, 1, 256, 0, &P)) != KIOPS_OK) return s;
      } else if (c->finner) {
        void *args[] = {&P};
        CK(cudaLaunchCooperativeKernel(c->finner, dim3(c->L.grid_pass), dim3(c->L.block_pass), args, c->L.smem_pass,
                                       c->stream),
           "cudaLaunchCooperativeKernel inner");
      } else if (c->op.kind == KIOPS_OP_CSR) {
        if ((s = launch_plain(c, (void *)k_csr_form, c->L.grid_form, 256, 0, &P)) != KIOPS_OK) return s;
        if ((s = launch_plain(c, (void *)k_sell_spmv, c->L.grid_pass, 256, 0, &P)) != KIOPS_OK) return s;
      } else {
        if ((s = launch_plain(c, c->fpass, c->L.grid_pass, c->L.block_pass, c->L.smem_pass, &P)) != KIOPS_OK) return s;
      }
      if ((s = read_conds(c, cond)) != KIOPS_OK) return s;
    }
    if ((s = launch_plain(c, (void *)k_ctrl, CTRL_CL, CTRL_THREADS, ctrl_smem_bytes(), &P)) != KIOPS_OK) return s;
    if ((s = read_conds(c, cond)) != KIOPS_OK) return s;
    if (cond[COND_ACCEPT])
      if ((s = launch_plain(c, (void *)k_gemv, c->L.grid_gemv, 256, 0, &P)) != KIOPS_OK) return s;
  }
  CK(cudaMemcpyAsync(c->h_state, c->P.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream), "D2H state");
  return finish(c, stats);
}

kiops_status kiops_get_trace(kiops_ctx c, void *host_buf, size_t bytes, int64_t *rows) {
  if (!c || !rows) return KIOPS_ERR_INVALID_ARG;
  const long long avail = std::min<long long>(c->last_attempts, KIOPS_TRACE_CAP);
  *rows = avail;
  const size_t n = std::min<size_t>((size_t)avail, bytes / sizeof(kiops_trace_row));
  if (n && host_buf) {
    CK(cudaMemcpyAsync(host_buf, c->P.trace, n * sizeof(kiops_trace_row), cudaMemcpyDeviceToHost, c->stream), "D2H trace");
    CK(cudaStreamSynchronize(c->stream), "stream sync");
  }
  return KIOPS_OK;
}

kiops_status kiops_set_m_init(kiops_ctx c, int m_init) {
  if (!c || m_init < 0) return KIOPS_ERR_INVALID_ARG;
  c->m_init_call = m_init;
  return KIOPS_OK;
}

kiops_status kiops_set_forced_schedule(kiops_ctx c, const double *tau, const int32_t *m, const int32_t *accept,
                                       int n) {
  if (!c || n < 0 || n > KIOPS_MAX_FORCED || (n > 0 && (!tau || !m))) return KIOPS_ERR_INVALID_ARG;
  for (int i = 0; i < n; i++) {
    if (!(tau[i] > 0.0)) return KIOPS_ERR_INVALID_ARG;
    c->forced_tau[i] = tau[i];
    c->forced_m[i] = m[i];
    c->forced_acc[i] = accept ? (accept[i] != 0) : 1;
  }
  c->n_forced = n;
  return KIOPS_OK;
}

kiops_status kiops_debug_basis(kiops_ctx c, double *h, double *sig, int32_t *npass) {
  if (!c) return KIOPS_ERR_INVALID_ARG;
  if (h) CK(cudaMemcpyAsync(h, c->P.H, sizeof(double) * LDH * LDH, cudaMemcpyDeviceToHost, c->stream), "D2H H");
  if (sig) CK(cudaMemcpyAsync(sig, c->P.sig + 1, sizeof(double) * LDH, cudaMemcpyDeviceToHost, c->stream), "D2H sig");
  CK(cudaMemcpyAsync(c->h_state, c->P.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream), "D2H state");
  CK(cudaStreamSynchronize(c->stream), "stream sync");
  if (npass) *npass = c->h_state->npass;
  return KIOPS_OK;
}

kiops_status kiops_debug_expm(kiops_ctx c, int n, const double *m, double scale, double *f, int32_t *products) {
  if (!c || !m || !f || n < 1 || n > KMAXM + 1) return KIOPS_ERR_INVALID_ARG;
  double *dm = nullptr;
  int *drc = nullptr;
  const size_t nb = sizeof(double) * (size_t)n * n;
  CK(cudaMalloc(&dm, 2 * nb + 16), "debug alloc");
  drc = (int *)((unsigned char *)dm + 2 * nb);
  kiops_status s = KIOPS_OK;
  int hrc = -1;
  cudaError_t e = cudaMemcpyAsync(dm, m, nb, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((void *)k_debug_expm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctrl_smem_bytes());
  if (e == cudaSuccess) {
    k_debug_expm<<<CTRL_CL, CTRL_THREADS, ctrl_smem_bytes(), c->stream>>>(c->P, n, dm, scale, dm + (size_t)n * n, drc);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(f, dm + (size_t)n * n, nb, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hrc, drc, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) s = cuda_fail(c, e, "debug expm");
  cudaFree(dm);
  if (products) *products = hrc;
  if (s == KIOPS_OK && hrc < 0) return KIOPS_ERR_NONFINITE;
  return s;
}

kiops_status kiops_refresh_operator(kiops_ctx c) {
  if (!c) return KIOPS_ERR_INVALID_ARG;
  if (c->op.kind != KIOPS_OP_CSR) return KIOPS_OK;  // stencil kinds read diag / kappa at every apply
  const KParams &P = c->P;
  k_sell_build<<<sm_count() * 8, 256, 0, c->stream>>>(P.N, P.row_ptr, P.col_idx, P.vals, P.sell_off, (int *)P.sell_col,
                                                         (double *)P.sell_val);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c, e, "SELL rebuild");
  return KIOPS_OK;
}

kiops_status kiops_destroy(kiops_ctx c) {
  if (!c) return KIOPS_ERR_INVALID_ARG;
  if (c->exec) cudaGraphExecDestroy(c->exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->h_call) cudaFreeHost(c->h_call);
  if (c->h_state) cudaFreeHost(c->h_state);
  delete c;
  return KIOPS_OK;
}

const char *kiops_status_string(kiops_status s) {
  switch (s) {
    case KIOPS_OK: return "KIOPS_OK";
    case KIOPS_ERR_INVALID_ARG: return "KIOPS_ERR_INVALID_ARG";
    case KIOPS_ERR_UNSUPPORTED: return "KIOPS_ERR_UNSUPPORTED";
    case KIOPS_ERR_CUDA: return "KIOPS_ERR_CUDA";
    case KIOPS_ERR_NO_CONVERGENCE: return "KIOPS_ERR_NO_CONVERGENCE";
    case KIOPS_ERR_NONFINITE: return "KIOPS_ERR_NONFINITE";
    case KIOPS_ERR_WORKSPACE: return "KIOPS_ERR_WORKSPACE";
  }
  return "KIOPS_ERR_UNKNOWN";
}

const char *kiops_last_error(kiops_ctx c) { return c ? c->err.c_str() : "NULL ctx"; }

}  // extern "C"
#include "epirk.cuh"
