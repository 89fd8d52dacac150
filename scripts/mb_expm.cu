// Microbenchmark of the controller's small-n exponential (pade_expm<SmemBk>, one CTA of
// CTRL_THREADS threads, n <= SMALL_N): cycles per exponential of a config-3-like H~
// (IOP band + the e_1 column, ||tau H~||_1 ~ 90 -> s = 4) for n = 12..48, with a
// checksum against the first variant built.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_expm scripts/mb_expm.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1804_05126_b200/csrc/kiops.cu"

__global__ void __launch_bounds__(CTRL_THREADS, 1) k_mbexpm(int n, const double *M, double scale, double *F, int reps,
                                                           long long *cyc) {
  extern __shared__ double sm[];
  SmemBk bk{sm, n};
  double *Ms = bk.mat(8), *Fs = bk.mat(9);
  bk.clear();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) Ms[(e % n) + SM_LD * (e / n)] = M[e];
  __syncthreads();
  long long t0 = clock64();
  int r = 0;
  for (int i = 0; i < reps; i++) r = pade_expm(bk, n, Ms, scale, Fs);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) F[e] = Fs[(e % n) + SM_LD * (e / n)];
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps, cyc[1] = r;
}

int main() {
  const size_t smem = ctrl_smem_bytes();
  cudaFuncSetAttribute(k_mbexpm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double *dM, *dF;
  long long *dc, hc[2];
  cudaMalloc(&dM, 64 * 64 * 8);
  cudaMalloc(&dF, 64 * 64 * 8);
  cudaMalloc(&dc, 16);
  srand(7);
  for (int n : {12, 20, 28, 36, 40, 44, 48}) {
    std::vector<double> M((size_t)n * n, 0.0), F((size_t)n * n);
    const int j = n - 1;
    for (int c = 0; c < j; c++)
      for (int r = c > 0 ? c - 1 : 0; r <= c + 1 && r < j; r++) M[r + (size_t)n * c] = (rand() / (double)RAND_MAX - 0.5) * 40.0 - (r == c ? 40.0 : 0.0);
    M[0 + (size_t)n * j] = 1.0;
    cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice);
    k_mbexpm<<<1, CTRL_THREADS, smem>>>(n, dM, 1.0, dF, 10, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hc, dc, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(F.data(), dF, F.size() * 8, cudaMemcpyDeviceToHost);
    double cs = 0.0;
    for (double x : F) cs += x;
    printf("n %2d: %7lld cycles per expm (products %lld) checksum %.15e %s\n", n, hc[0], hc[1], cs,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
