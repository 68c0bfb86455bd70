// Micro-benchmark: the h-multigrid CG's x / r update pattern (4 loads, 2 stores per point) over
// 17M points, grid-stride, as a cooperative-sized grid vs a full grid; unroll 1 vs 4.
#include <cstdio>
#include <cuda_runtime.h>
template <int U>
__global__ void __launch_bounds__(256) upd(long long n, double a, double* X, const double* pv, const double* q, double* R) {
  const long long T = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long i = t0; i < n; i += U * T) {
    double xv[U], pvv[U], qv[U], rv[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const long long ik = i + k * T < n ? i + k * T : i;
      xv[k] = X[ik]; pvv[k] = pv[ik]; qv[k] = q[ik]; rv[k] = R[ik];
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (i + k * T >= n) break;
      X[i + k * T] = fma(a, pvv[k], xv[k]);
      R[i + k * T] = fma(-a, qv[k], rv[k]);
    }
  }
}
int main() {
  const long long n = 257LL * 257 * 257;
  double *X, *P, *Q, *R;
  cudaMalloc(&X, n * 8); cudaMalloc(&P, n * 8); cudaMalloc(&Q, n * 8); cudaMalloc(&R, n * 8);
  cudaMemset(X, 0x3F, n * 8); cudaMemset(P, 0x3E, n * 8); cudaMemset(Q, 0x3D, n * 8); cudaMemset(R, 0x3C, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grids[] = {296, 444, 592, 1184, 2368, 8192};
  for (int g : grids)
    for (int u = 0; u < 2; ++u) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (u == 0) upd<1><<<g, 256>>>(n, 0.5, X, P, Q, R); else upd<4><<<g, 256>>>(n, 0.5, X, P, Q, R);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("grid %5d unroll %d: %8.1f us  %7.0f GB/s\n", g, u ? 4 : 1, ms * 1e3, 48.0 * n / (ms * 1e-3) / 1e9);
      }
    }
  return 0;
}
