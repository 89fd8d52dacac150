// Microbenchmark (not product code): DRAM streaming rate of the config-4 pass's access
// pattern without its arithmetic, to separate the memory-pattern ceiling from the
// compute / barrier cost of k_inner_3d_lazyq.  256^3 doubles, 6 read + 2 write vectors.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/mb_stream3d.cu && ./mb
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int NX = 256, NY = 256, NZ = 256;
constexpr long long NXY = (long long)NX * NY, N = NXY * NZ;

__device__ __forceinline__ void cpa16(void *dst, const void *src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }
__device__ __forceinline__ long long wr(long long g, long long n) { return g < 0 ? g + n : (g >= n ? g - n : g); }

// V0: plain grid-stride 16-byte streaming of 6 inputs -> 2 outputs
__global__ void __launch_bounds__(640) k_flat(const double2 *a, const double2 *b, const double2 *c, const double2 *d,
                                               const double2 *e, const double2 *f, double2 *o1, double2 *o2, double *acc) {
  double s = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N / 2; i += (long long)gridDim.x * blockDim.x) {
    const double2 x = a[i], y = b[i], z = c[i], w = d[i], u = e[i], v = f[i];
    double2 r1 = {x.x + y.x + z.x, x.y + y.y + z.y}, r2 = {w.x + u.x + v.x, w.y + u.y + v.y};
    o1[i] = r1;
    o2[i] = r2;
    s += r1.x;
  }
  if (s == 12345.0) acc[0] = s;
}

// V1/V2: the pass's tile pattern: 148 CTAs x (2 halves x 320 threads), 64x7 tiles (4 x 37),
// 2 z-parts, halo-1 pairs (34 x 9) load 4 arrays, interior pairs 2 more (B), DD planes
// in flight, one __syncthreads per plane (SYNC), x/kappa published to a shared ring and
// the 4 in-plane neighbours read back (SMEMNB), 2 outputs per interior pair.
template <int DD, int SYNC, int SMEMNB, int HEAVY = 0>
__global__ void __launch_bounds__(640, 1) k_tile(const double *r, const double *xp, const double *xpp, const double *kap,
                                                 const double *b0, const double *b1, double *o1, double *o2, double *acc) {
  constexpr int PX = 34, NPAIR = 34 * 9, NIN = 32 * 7, NT = 320, RD = DD + 1, SLOT = 4 * NPAIR + 2 * NIN;
  extern __shared__ double2 sm[];
  const int h = threadIdx.x / NT, t = threadIdx.x % NT;
  double2 *sX = sm + (size_t)h * (4 * NPAIR + RD * SLOT), *sK = sX + 2 * NPAIR, *sOp = sX + 4 * NPAIR;
  const int tile = blockIdx.x, ntx = 4, nb = 37;
  const long long ox = (long long)(tile % ntx) * 64, band = tile / ntx;
  const long long oy = band * NY / nb, hb = (band + 1) * NY / nb - oy;
  const int part = h;
  const long long zlo = part * NZ / 2, zhi = (part + 1) * NZ / 2;
  const int nzc = (int)(zhi - zlo);
  const int px = t % PX, py = t / PX;
  const bool act = py < hb + 2;
  const long long o1x = act ? (wr(ox - 2 + 2 * px, NX) + NX * wr(oy - 1 + py, NY)) : 0;
  const bool pin = act && py >= 1 && py <= hb && px >= 1 && px <= 32;
  const long long oo = (ox - 2 + 2 * px) + NX * (oy - 1 + py);
  const int ib = (py - 1) * 32 + (px - 1);
  long long zoL = wr(zlo - 1, NZ) * NXY;
  auto issue = [&](int slot) {
    if (act) {
      double2 *d = sOp + slot * SLOT + t;
      const long long g = zoL + o1x;
      cpa16(d, r + g);
      cpa16(d + NPAIR, xp + g);
      cpa16(d + 2 * NPAIR, xpp + g);
      cpa16(d + 3 * NPAIR, kap + g);
      if (pin) {
        cpa16(sOp + slot * SLOT + 4 * NPAIR + ib, b0 + g);
        cpa16(sOp + slot * SLOT + 4 * NPAIR + NIN + ib, b1 + g);
      }
    }
    zoL += NXY;
    if (zoL >= N) zoL -= N;
  };
  for (int q = 0; q < DD; q++) {
    issue(q);
    commit();
  }
  double s = 0;
  double2 prev = {0, 0}, kprev = {0, 0}, xmm = {0, 0}, km = {0, 0};
  double d0 = 0, d1 = 0, d2 = 0, d3 = 0;
  long long zo = zlo * NXY;
  int rs = 0, ri = DD;
  for (int i = 0; i <= nzc + 1; i++) {
    if (i + DD <= nzc + 1) issue(ri);
    commit();
    waitg<DD>();
    const double2 *o = sOp + rs * SLOT + t;
    const double2 a = o[0], b = o[NPAIR], c = o[2 * NPAIR], k = o[3 * NPAIR];
    double2 x = {a.x - b.x - c.x, a.y - b.y - c.y};
    double2 bt = {0, 0};
    if (pin) {
      const double2 u = sOp[rs * SLOT + 4 * NPAIR + ib], w = sOp[rs * SLOT + 4 * NPAIR + NIN + ib];
      bt = {u.x + w.x, u.y + w.y};
    }
    if (SYNC) __syncthreads();
    if (SMEMNB && act) {
      sX[(i & 1) * NPAIR + t] = x;
      sK[(i & 1) * NPAIR + t] = k;
    }
    if (i >= 2 && pin) {
      double2 rr = {prev.x + bt.x, prev.y + bt.y};
      if (HEAVY) {  // the pass's 7-point variable-kappa pair stencil + 5 dots, same operand count
        const double2 *X0 = sX + ((i + 1) & 1) * NPAIR, *K0 = sK + ((i + 1) & 1) * NPAIR;
        const double2 xc = prev, kc = kprev, xs = X0[t - PX], xn = X0[t + PX], ks = K0[t - PX], kn = K0[t + PX];
        const double xl = X0[t - 1].y, xr = X0[t + 1].x, kl = K0[t - 1].y, kr = K0[t + 1].x;
        double ra = (kc.x + kl) * (xl - xc.x), rb = (kc.y + kr) * (xr - xc.y);
        ra = fma(kc.x + kc.y, xc.y - xc.x, ra); rb = fma(kc.y + kc.x, xc.x - xc.y, rb);
        ra = fma(kc.x + ks.x, xs.x - xc.x, ra); rb = fma(kc.y + ks.y, xs.y - xc.y, rb);
        ra = fma(kc.x + kn.x, xn.x - xc.x, ra); rb = fma(kc.y + kn.y, xn.y - xc.y, rb);
        ra = fma(kc.x + km.x, xmm.x - xc.x, ra); rb = fma(kc.y + km.y, xmm.y - xc.y, rb);
        ra = fma(kc.x + k.x, x.x - xc.x, ra); rb = fma(kc.y + k.y, x.y - xc.y, rb);
        rr = make_double2(fma(ra, 0.5, bt.x), fma(rb, 0.5, bt.y));
        d0 = fma(xc.x, xc.x, fma(xc.y, xc.y, d0)); d1 = fma(b.x, xc.x, fma(b.y, xc.y, d1));
        d2 = fma(b.x, rr.x, fma(b.y, rr.y, d2)); d3 = fma(xc.x, rr.x, fma(xc.y, rr.y, d3));
      } else if (SMEMNB) {
        const double2 *X0 = sX + ((i + 1) & 1) * NPAIR;
        rr.x += X0[t - 1].y + X0[t + PX].x + X0[t - PX].x;
        rr.y += X0[t + 1].x + X0[t + PX].y + X0[t - PX].y;
      }
      s = fma(rr.x, rr.x, s);
      *reinterpret_cast<double2 *>(o1 + zo + oo) = prev;
      *reinterpret_cast<double2 *>(o2 + zo + oo) = rr;
    }
    if (i >= 2) zo += NXY;
    xmm = prev; km = kprev;
    prev = x; kprev = k;
    rs = rs + 1 == RD ? 0 : rs + 1;
    ri = ri + 1 == RD ? 0 : ri + 1;
  }
  waitg<0>();
  if (s + d0 + d1 + d2 + d3 == 12345.0) acc[0] = s;
}

__global__ void k_fill(double *p, long long n, unsigned seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = (unsigned long long)i * 0x9E3779B97F4A7C15ull + seed;
    z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
    p[i] = (double)(z >> 11) * 0x1.0p-53 - 0.5;
  }
}

template <class F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; i++) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; i++) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main() {
  double *v[9];
  const bool rnd = getenv("MB_RANDOM") != nullptr;
  for (int i = 0; i < 9; i++) {
    cudaMalloc(&v[i], N * 8 + 4096);
    cudaMemset(v[i], 0, N * 8 + 4096);
    if (rnd) k_fill<<<1184, 256>>>(v[i], N, 17u * i + 1);
  }
  cudaDeviceSynchronize();
  printf("data: %s\n", rnd ? "random" : "zeros");
  const double bytes = 8.0 * N * 8;  // 6 reads + 2 writes
  double *acc = v[8];
  {
    for (int g : {148, 296, 592, 1184}) {
      const float us = timeit([&] { k_flat<<<g, 640>>>((double2 *)v[0], (double2 *)v[1], (double2 *)v[2], (double2 *)v[3], (double2 *)v[4], (double2 *)v[5], (double2 *)v[6], (double2 *)v[7], acc); });
      printf("flat grid %5d x 640: %7.1f us  %6.0f GB/s\n", g, us, bytes / us * 1e-3);
    }
  }
#define RUN(DD, SY, NB, HV)                                                                                          \
  {                                                                                                              \
    const size_t smem = 2 * 16 * (4 * 306 + (DD + 1) * (4 * 306 + 2 * 224));                                     \
    cudaFuncSetAttribute(k_tile<DD, SY, NB, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);           \
    const float us = timeit([&] { k_tile<DD, SY, NB, HV><<<148, 640, smem>>>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], acc); }); \
    printf("tile DD=%d sync=%d smemnb=%d heavy=%d smem %zu: %7.1f us  %6.0f GB/s  err=%s\n", DD, SY, NB, HV, smem, us, bytes / us * 1e-3, \
           cudaGetErrorString(cudaGetLastError()));                                                              \
  }
  RUN(2, 1, 1, 0) RUN(2, 1, 1, 1) RUN(2, 1, 1, 0) RUN(2, 1, 1, 1)
  return 0;
}
