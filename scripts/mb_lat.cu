// Single-warp dependent-chain latencies on sm_100a (debug aid, not product):
// DFMA / DADD / DMUL / DSETP+FSEL / SHFL(64-bit) / REDUX / MUFU.RCP64H+Newton / LDS / named-barrier hand-off.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_lat scripts/mb_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
#define N 512
__global__ void k_lat(double *out, long long *cyc, double a, double b, int nwarps_active) {
  __shared__ double sm[64];
  __shared__ int hand;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x = a + lane;
  long long t[16];
  int q = 0;
  if (warp == 0) {
    t[q++] = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = fma(x, b, a);
    t[q++] = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x + a;
    t[q++] = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x * b;
    t[q++] = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = (x > a) ? x - 1.0 : x + 1.0;  // DSETP + select + DADD
    t[q++] = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    t[q++] = clock64();
    unsigned u = (unsigned)__double2hiint(x);
#pragma unroll 16
    for (int i = 0; i < N; i++) u = __reduce_max_sync(0xffffffffu, u ^ lane) + 1;
    t[q++] = clock64();
    x += u;
#pragma unroll 16
    for (int i = 0; i < N; i++) x = __drcp_rn(x) + 1.5;
    t[q++] = clock64();
    sm[lane] = x;
    __syncwarp();
    int idx = lane;
#pragma unroll 16
    for (int i = 0; i < N; i++) idx = ((int)sm[idx] + lane + i) & 31;
    t[q++] = clock64();
    x += idx;
#pragma unroll 16
    for (int i = 0; i < N; i++) { unsigned m = __ballot_sync(0xffffffffu, x > (double)i); x += __popc(m); }
    t[q++] = clock64();
    if (lane == 0) for (int i = 0; i + 1 < q; i++) cyc[i] = (t[i + 1] - t[i]);
  }
  __syncthreads();
  // named-barrier hand-off ring: warp w arrives on barrier 1+(i&1) for warp (w+1): measure round trip
  // simple version: two warps ping-pong N times with bar.arrive / bar.sync (64 threads each barrier)
  if (warp < 2) {
    long long t0 = clock64();
    for (int i = 0; i < N; i++) {
      const int id = 1 + (i & 1);
      if ((i & 1) == warp) {
        if (lane == 0) sm[32] = x + i;
        __syncwarp();
        asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
      } else {
        asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
        x += sm[32];
      }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[15] = t1 - t0;
  }
  out[threadIdx.x] = x;
}
int main() {
  double *o; long long *c, h[16] = {0};
  cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 16 * 8); cudaMemset(c, 0, 128);
  k_lat<<<1, 512>>>(o, c, 1.000001, 0.999999, 1);
  cudaDeviceSynchronize();
  cudaMemcpy(h, c, 128, cudaMemcpyDeviceToHost);
  const char *nm[] = {"DFMA", "DADD", "DMUL", "DSETP+sel+DADD", "SHFL64", "REDUX+xor+add", "DRCP+DADD", "LDS.64+cvt+idx", "DSETP+VOTE+POPC+I2F+DADD"};
  for (int i = 0; i < 9; i++) printf("%-28s %.1f cycles / op\n", nm[i], h[i] / (double)N);
  printf("%-28s %.1f cycles / hand-off\n", "bar.arrive -> bar.sync", h[15] / (double)N);
  return 0;
}
