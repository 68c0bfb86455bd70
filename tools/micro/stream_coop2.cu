// Micro-benchmark: the x / r update inside a cooperative kernel with grid barriers (as the
// h-multigrid CG), 296 blocks of 256 threads, with and without a stencil-like phase in between.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(256, 2) coop(long long n, int iters, int stencil, double a, double* X, double* pv,
                                                double* q, double* R, unsigned long long* stamps) {
  cg::grid_group grid = cg::this_grid();
  const long long T = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    if (stencil) {   // q = 7-point stencil of pv (neighbours from L1 / L2)
      const long long s2 = 257, s3 = 257 * 257;
      for (long long i = t0; i < n; i += T) {
        const long long im = i >= s3 ? i : s3, ip = i + s3 < n ? i : n - 1 - s3;
        q[i] = 6.0 * pv[i] - pv[im - 1] - pv[ip + 1] - pv[im - s2] - pv[ip + s2] - pv[im - s3] - pv[ip + s3];
      }
      grid.sync();
    }
    unsigned long long t;
    if (blockIdx.x == 0 && threadIdx.x == 0) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); stamps[2 * it] = t; }
    for (long long i = t0; i < n; i += 4 * T) {
      double xv[4], pvv[4], qv[4], rv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long ik = i + k * T < n ? i + k * T : i;
        xv[k] = X[ik]; pvv[k] = pv[ik]; qv[k] = q[ik]; rv[k] = R[ik];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (i + k * T >= n) break;
        X[i + k * T] = fma(a, pvv[k], xv[k]);
        R[i + k * T] = fma(-a, qv[k], rv[k]);
      }
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); stamps[2 * it + 1] = t; }
  }
}
int main() {
  const long long n = 257LL * 257 * 257;
  double *X, *P, *Q, *R;
  unsigned long long* st;
  cudaMalloc(&X, n * 8); cudaMalloc(&P, n * 8); cudaMalloc(&Q, n * 8); cudaMalloc(&R, n * 8);
  cudaMalloc(&st, 2 * 64 * 8);
  cudaMemset(X, 0x3F, n * 8); cudaMemset(P, 0x3E, n * 8); cudaMemset(Q, 0x3D, n * 8); cudaMemset(R, 0x3C, n * 8);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coop, 256, 0);
  for (int stencil = 0; stencil < 2; ++stencil) {
    int nb = per_sm * 148, iters = 16;
    double a = 0.5;
    void* args[] = {(void*)&n, &iters, &stencil, &a, &X, &P, &Q, &R, &st};
    cudaLaunchCooperativeKernel((void*)coop, nb, 256, args, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[128];
    cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 4; i < iters; ++i) s += (h[2 * i + 1] - h[2 * i]) / 1e3;
    printf("per_sm %d blocks %d stencil %d: update phase %.1f us (%s)\n", per_sm, nb, stencil, s / (iters - 4), cudaGetErrorString(e));
  }
  return 0;
}
