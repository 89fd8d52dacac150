// DMMA m8n8k4 (fp64 mma.sync) latency / throughput on sm_100a (debug aid, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_dmma scripts/mb_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double *out, long long *cyc, int iters, double a, double b) {
  double c[CH][2];
  for (int i = 0; i < CH; i++) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) dmma(c[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; i++) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void kf(double *out, long long *cyc, int iters, double a, double b) {  // DFMA throughput, 8 chains
  double c[8];
  for (int i = 0; i < 8; i++) c[i] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) c[i] = fma(c[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; i++) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o; long long *c, h;
  cudaMalloc(&o, 8 * 4096); cudaMalloc(&c, 8);
  const int it = 2000;
#define RUN(K, CH, thr, label) { K<<<1, thr>>>(o, c, it, 1.0000001, 0.9999999); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
  printf("%-44s %.1f cycles per instruction per warp; %.2f cycles per instr per SM sub-partition\n", label, h / (double)(it * CH), h / (double)(it * CH) / ((thr + 127) / 128)); }
  RUN(k<1>, 1, 32, "DMMA 1 warp, 1 chain (latency)");
  RUN(k<4>, 4, 32, "DMMA 1 warp, 4 chains");
  RUN(k<8>, 8, 32, "DMMA 1 warp, 8 chains");
  RUN(k<2>, 2, 512, "DMMA 16 warps x 2 chains");
  RUN(k<4>, 4, 512, "DMMA 16 warps x 4 chains");
  RUN(kf, 8, 32, "DFMA 1 warp, 8 chains");
  RUN(kf, 8, 512, "DFMA 16 warps x 8 chains");
  return 0;
}
