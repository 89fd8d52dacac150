// Microbenchmark + self-check of the recompute-form TMA pass body (csrc/rc3d.cuh) on a
// synthetic padded 3-D grid, outside the KIOPS engine: one pass = one launch of 148
// (SM count) CTAs running rc3::body once, block partials added with atomics.  Checks
// x_k (interior and ghost images) and the five dots against naive per-point kernels.
// Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o mb_rc3d scripts/mb_rc3d.cu -lcuda
//   ./mb_rc3d [nx ny nz] [reps]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1804_05126_b200/csrc/rc3d.cuh"

#ifndef MB_XALIGN
#define MB_XALIGN 1   // padded row pitch rounded up to a multiple of this many doubles
#endif
#define XPITCH(nx) (((nx) + 4 + MB_XALIGN - 1) / MB_XALIGN * MB_XALIGN)
#ifndef MB_L2PROMO
#define MB_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
#ifndef MB_CPS
#define MB_CPS 1  // CTAs per SM (2 for the 32-point-wide tile prototype, profiles/r02_kernel_evolution.md)
#endif
#ifndef MB_HM
#define MB_HM 7
#endif
#ifndef MB_ROT
#define MB_ROT 0
#endif
#ifndef MB_QREG
#define MB_QREG 0
#endif
#ifndef MB_GRID
#define MB_GRID 0
#endif
#ifndef MB_D
#define MB_D 3
#endif
constexpr int PM = 2, HM = MB_HM, DD = MB_D;
using C = rc3::Cfg<PM, HM, DD>;

#define CKR(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

__host__ __device__ inline double hval(int slot, long long i) {
  unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull + (unsigned long long)(slot + 1) * 0xD1B54A32D192ED03ull;
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 29;
  const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
  return slot == 2 ? 0.2 + 3.0 * u : 2.0 * u - 1.0;  // slot 2: kappa > 0
}

// fill slot s over the padded grid: value of the periodic image (ghosts = copies)
__global__ void k_fill(double *V, long long ldN, int s, int nx, int ny, int nz) {
  const int Xp = XPITCH(nx), Yp = ny + 4;
  const long long np = (long long)Xp * Yp * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < np; i += (long long)gridDim.x * blockDim.x) {
    const int xp = (int)(i % Xp), yp = (int)((i / Xp) % Yp), z = (int)(i / ((long long)Xp * Yp));
    const int x = (xp - 2 + nx) % nx, y = (yp - 2 + ny) % ny;
    V[(size_t)s * ldN + i] = hval(s, x + (long long)nx * (y + (long long)ny * z));
  }
}

__global__ void k_scale(double *a, long long n, double f) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) a[i] *= f;
}

__device__ __forceinline__ double at(const double *V, long long ldN, int s, int nx, int ny, int nz, int x, int y, int z) {
  x = (x % nx + nx) % nx;
  y = (y % ny + ny) % ny;
  z = (z % nz + nz) % nz;
  return V[(size_t)s * ldN + (x + 2) + (long long)XPITCH(nx) * ((y + 2) + (long long)(ny + 4) * z)];
}
__device__ double Aop(const double *V, long long ldN, int s, int nx, int ny, int nz, int x, int y, int z, double hh,
                      const double *U, long long ldU) {
  // U: if non-null, the operand is the unpadded array U (x_k reference), else slot s of V
  auto u = [&](int a, int b, int c) -> double {
    if (U) {
      a = (a % nx + nx) % nx; b = (b % ny + ny) % ny; c = (c % nz + nz) % nz;
      return U[a + (long long)nx * (b + (long long)ny * c)];
    }
    return at(V, ldN, s, nx, ny, nz, a, b, c);
  };
  auto kap = [&](int a, int b, int c) { return at(V, ldN, 2, nx, ny, nz, a, b, c); };
  const double xc = u(x, y, z), kc = kap(x, y, z);
  double r = 0.0;
  const int d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
  for (int q = 0; q < 6; q++) r += (kc + kap(x + d[q][0], y + d[q][1], z + d[q][2])) * (u(x + d[q][0], y + d[q][1], z + d[q][2]) - xc);
  return r * hh;
}
__global__ void k_ref_xk(const double *V, long long ldN, int nx, int ny, int nz, double hh, double a0, double a1, double a2,
                         double bp0, double bp1, double *XK) {
  const long long N = (long long)nx * ny * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((long long)nx * ny));
    const double bt = at(V, ldN, 3, nx, ny, nz, x, y, z) * bp0 + at(V, ldN, 4, nx, ny, nz, x, y, z) * bp1;
    const double r = Aop(V, ldN, 0, nx, ny, nz, x, y, z, hh, nullptr, 0) + bt;
    XK[i] = a0 * r - a1 * at(V, ldN, 0, nx, ny, nz, x, y, z) - a2 * at(V, ldN, 1, nx, ny, nz, x, y, z);
  }
}
__global__ void k_ref_dots(const double *V, long long ldN, int nx, int ny, int nz, double hh, double bc0, double bc1,
                           const double *XK, double *dots) {
  const long long N = (long long)nx * ny * nz;
  double s[5] = {0, 0, 0, 0, 0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((long long)nx * ny));
    const double bt = at(V, ldN, 3, nx, ny, nz, x, y, z) * bc0 + at(V, ldN, 4, nx, ny, nz, x, y, z) * bc1;
    const double r = Aop(V, ldN, 0, nx, ny, nz, x, y, z, hh, XK, 0) + bt;
    const double xk = XK[i], xp = at(V, ldN, 0, nx, ny, nz, x, y, z);
    s[0] += xk * xk; s[1] += xp * xk; s[2] += xp * r; s[3] += xk * r; s[4] += r * r;
  }
  for (int q = 0; q < 5; q++) atomicAdd(dots + q, s[q]);
}
__global__ void k_check(const double *XO, const double *XK, int nx, int ny, int nz, double *err) {
  const int Xp = XPITCH(nx), Yp = ny + 4;
  const long long np = (long long)Xp * Yp * nz;
  double e1 = 0.0, e2 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < np; i += (long long)gridDim.x * blockDim.x) {
    const int xp = (int)(i % Xp), yp = (int)((i / Xp) % Yp), z = (int)(i / ((long long)Xp * Yp));
    if (xp >= nx + 4) continue;  // pitch padding
    const int x = (xp - 2 + nx) % nx, y = (yp - 2 + ny) % ny;
    const double ref = XK[x + (long long)nx * (y + (long long)ny * z)];
    const double d = fabs(XO[i] - ref);
    const bool ghost = xp < 2 || xp >= nx + 2 || yp < 2 || yp >= ny + 2;
    if (ghost) e2 = fmax(e2, d); else e1 = fmax(e1, d);
  }
  atomicMax((unsigned long long *)err, __double_as_longlong(e1));
  atomicMax((unsigned long long *)(err + 1), __double_as_longlong(e2));
}

__device__ unsigned long long mb_count;  // grid barrier (MB_GRID): monotonic arrivals

__device__ rc3::Geom mb_G;
__device__ rc3::PassArgs<PM> mb_Q;
#if MB_QREG  // geometry and pass scalars in registers (as in the product), not kernel parameters
__global__ void __launch_bounds__(C::NT, MB_CPS) k_mb(rc3::Geom G0, rc3::PassArgs<PM> Q0, double *dots, int reps) {
#if MB_QREG == 1
  rc3::Geom G;
  memcpy(&G, (const void *)&mb_G, sizeof(G));
#else
  const rc3::Geom &G = G0;
#endif
  rc3::PassArgs<PM> Q;
  memcpy(&Q, (const void *)&mb_Q, sizeof(Q));
#else
__global__ void __maxnreg__(200) k_mb(rc3::Geom G, rc3::PassArgs<PM> Q, double *dots, int reps) {
#endif
  rc3::init<PM, HM, DD>(G);
  unsigned nl = 0;
  int pre = 0;
  double v[5] = {0, 0, 0, 0, 0};
  __shared__ double red0[5][32];
  unsigned long long target = 0;
  if (threadIdx.x == 0) target = *(volatile unsigned long long *)&mb_count;
  auto slots = [&](int r, int &sp, int &spp, double *&xo) {
    sp = Q.slot_prev; spp = Q.slot_pp; xo = Q.xout;
#if MB_ROT  // rotate x_{k-1}, x_{k-2}, x_k through the basis slots like consecutive passes
    if (reps > 1) { sp = 5 + (r + 1) % 8; spp = 5 + r % 8; xo = G.V + (size_t)(5 + (r + 2) % 8) * G.ldN; }
#endif
  };
  for (int r = 0; r < reps; r++) {
    Q.k = r + 3;  // alternate the march direction like consecutive passes
    slots(r, Q.slot_prev, Q.slot_pp, Q.xout);
    rc3::body<PM, HM, DD>(G, Q, v, nl, pre);
#if MB_GRID  // the persistent loop's pass boundary: block sums, grid barrier, (prefetch)
    for (int q = 0; q < 5; q++) {
      double x = v[q];
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) == 0) red0[q][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&mb_count, 1ull);
      target += gridDim.x;
      while (*(volatile unsigned long long *)&mb_count < target) {
      }
      __threadfence();
    }
    __syncthreads();
#endif
  }
  __shared__ double red[5][32];
  for (int q = 0; q < 5; q++) {
    double x = v[q];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double x = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) x += red[threadIdx.x][w];
    atomicAdd(dots + threadIdx.x, x);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  int nx = 256, ny = 256, nz = 256, reps = 20;
  if (argc >= 4) { nx = atoi(argv[1]); ny = atoi(argv[2]); nz = atoi(argv[3]); }
  if (argc >= 5) reps = atoi(argv[4]);
  int dev = 0, sms = 0;
  CKR(cudaSetDevice(dev));
  CKR(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int Xp = XPITCH(nx), Yp = ny + 4;
  const long long ldN = ((long long)Xp * Yp * nz + 31) / 32 * 32;
  const int nslot = MB_ROT ? 13 : 6;  // 0 x_{k-1}, 1 x_{k-2}, 2 kappa, 3-4 B, 5 x_k (MB_ROT: 5..12 basis ring)
  double *V;
  CKR(cudaMalloc(&V, sizeof(double) * ldN * nslot));
  for (int s = 0; s < nslot; s++)
    if (s != 5) k_fill<<<1184, 256>>>(V, ldN, s, nx, ny, nz);
  CKR(cudaMemset(V + 5 * ldN, 0, sizeof(double) * ldN));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CKR(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &qr));
  CUtensorMap maps[2];
  cuuint64_t gdim[4] = {(cuuint64_t)Xp, (cuuint64_t)Yp, (cuuint64_t)nz, (cuuint64_t)nslot};
  cuuint64_t gstr[3] = {(cuuint64_t)Xp * 8, (cuuint64_t)Xp * Yp * 8, (cuuint64_t)ldN * 8};
  cuuint32_t es[4] = {1, 1, 1, 1};
  for (int m = 0; m < 2; m++) {
    cuuint32_t box[4] = {(cuuint32_t)C::W, (cuuint32_t)(m == 0 ? C::RA : C::RB), 1, 1};
    CUresult r = enc(&maps[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, V, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, MB_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { fprintf(stderr, "encode failed %d\n", (int)r); return 1; }
  }
  void *dmaps;
  CKR(cudaMalloc(&dmaps, sizeof(maps)));
  CKR(cudaMemcpy(dmaps, maps, sizeof(maps), cudaMemcpyHostToDevice));
  rc3::Geom G{};
  G.nx = nx; G.ny = ny; G.nz = nz; G.Xp = Xp; G.Yp = Yp; G.ldN = ldN;
  const int ctas = sms * MB_CPS;
  rc3::tiles(nx, ny, nz, ctas, HM, &G.ntx, &G.nb, &G.zsplit);
  G.slot_kappa = 2; G.slot_B = 3;
  G.mapA = dmaps; G.mapB = (char *)dmaps + sizeof(CUtensorMap);
  G.V = V;
  const double h = 1.0 / nx;
  G.hh = 0.5 / (h * h);
#if RC3_KSCALED  // the kappa slot holds hh kappa; the references then use hh = 1
  k_scale<<<1184, 256>>>(V + 2 * (size_t)ldN, (long long)XPITCH(nx) * (ny + 4) * nz, G.hh);
  const double hh_ref = 1.0;
#else
  const double hh_ref = G.hh;
#endif
  rc3::PassArgs<PM> Q{};
  Q.k = 3; Q.slot_prev = 0; Q.slot_pp = 1; Q.xout = V + 5 * ldN;
  Q.a0 = 1.0 / 3000.0; Q.a1 = 0.3; Q.a2 = 0.2; Q.btp[0] = 0.7; Q.btp[1] = -0.4; Q.btc[0] = 0.25; Q.btc[1] = 0.6; Q.use_r = 1;
  const int grid = std::min(ctas, G.ntx * G.nb * G.zsplit);
  CKR(cudaMemcpyToSymbol(mb_G, &G, sizeof(G)));
  CKR(cudaMemcpyToSymbol(mb_Q, &Q, sizeof(Q)));
  CKR(cudaFuncSetAttribute(k_mb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
  double *dots, *rdots, *err, *XK;
  CKR(cudaMalloc(&dots, 5 * sizeof(double)));
  CKR(cudaMalloc(&rdots, 5 * sizeof(double)));
  CKR(cudaMalloc(&err, 2 * sizeof(double)));
  CKR(cudaMalloc(&XK, sizeof(double) * (size_t)nx * ny * nz));
  printf("grid %d x %d threads, smem %zu B, tiles %d x %d x %d, HM %d D %d\n", grid, C::NT, C::smem_bytes, G.ntx, G.nb,
         G.zsplit, HM, DD);
  // correctness: one pass (k = 3)
  CKR(cudaMemset(dots, 0, 5 * sizeof(double)));
  k_mb<<<grid, C::NT, C::smem_bytes>>>(G, Q, dots, 1);
  CKR(cudaGetLastError());
  CKR(cudaDeviceSynchronize());
  // k = 3 is odd: parts with part ^ 1 odd march down -- same values either way up to rounding order of r
  k_ref_xk<<<1184, 256>>>(V, ldN, nx, ny, nz, hh_ref, Q.a0, Q.a1, Q.a2, Q.btp[0], Q.btp[1], XK);
  CKR(cudaMemset(rdots, 0, 5 * sizeof(double)));
  k_ref_dots<<<1184, 256>>>(V, ldN, nx, ny, nz, hh_ref, Q.btc[0], Q.btc[1], XK, rdots);
  CKR(cudaMemset(err, 0, 2 * sizeof(double)));
  k_check<<<1184, 256>>>(V + 5 * ldN, XK, nx, ny, nz, err);
  CKR(cudaDeviceSynchronize());
  double hd[5], hr[5], he[2];
  CKR(cudaMemcpy(hd, dots, sizeof(hd), cudaMemcpyDeviceToHost));
  CKR(cudaMemcpy(hr, rdots, sizeof(hr), cudaMemcpyDeviceToHost));
  CKR(cudaMemcpy(he, err, sizeof(he), cudaMemcpyDeviceToHost));
  double worst = 0;
  for (int q = 0; q < 5; q++) {
    const double rel = fabs(hd[q] - hr[q]) / fabs(hr[q]);
    worst = fmax(worst, rel);
    printf("dot %d: %.15e ref %.15e rel %.2e\n", q, hd[q], hr[q], rel);
  }
  printf("x_k max abs err interior %.3e ghosts %.3e\n", he[0], he[1]);
  const bool ok = worst < 1e-10 && he[0] < 1e-9 && he[1] < 1e-9;
  printf("CHECK %s\n", ok ? "OK" : "FAIL");
  // timing: reps passes inside one launch (mimics the persistent loop minus the grid reduction)
  cudaEvent_t e0, e1;
  CKR(cudaEventCreate(&e0));
  CKR(cudaEventCreate(&e1));
  k_mb<<<grid, C::NT, C::smem_bytes>>>(G, Q, dots, 2);
  CKR(cudaEventRecord(e0));
  k_mb<<<grid, C::NT, C::smem_bytes>>>(G, Q, dots, reps);
  CKR(cudaEventRecord(e1));
  CKR(cudaEventSynchronize(e1));
  float ms;
  CKR(cudaEventElapsedTime(&ms, e0, e1));
  const double us = ms * 1e3 / reps;
  const double N = (double)nx * ny * nz, minb = (2 + 1 + PM + 1) * 8.0 * N;
  printf("RESULT us_per_pass %.2f  algorithmic_GBps %.1f (min bytes %.1f MB)\n", us, minb / (us * 1e-6) / 1e9, minb / 1e6);
  return ok ? 0 : 2;
}
