// Step-0 box facts: sustained FP64 FFMA (DFMA) and FP64 DMMA (mma.sync m8n8k4 f64)
// throughput, FP64 copy bandwidth, and device limits on the B200 we run on.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  // per iteration: 8 DMMA (2048 FMA per warp) and 64 DFMA per thread (2048 FMA per warp)
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  double ma = 1.0 + threadIdx.x * 1e-3, mb = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(ma), "d"(mb));
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int smemOptin = 0; cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%d,\"smem_per_sm\":%zu,\"clock_khz\":%d,\"regs_per_sm\":%d}\n",
         pr.name, pr.multiProcessorCount, pr.l2CacheSize, smemOptin, pr.sharedMemPerMultiprocessor, clk, pr.regsPerMultiprocessor);
  double* out; CK(cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = pr.multiProcessorCount;
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 2000;
    dfma_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
    float best = 1e30;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("{\"test\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bpsm, flops / best / 1e9);
  }
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 128, iters = 2000;
    dmma_kernel<<<blocks, threads>>>(out, 10); CK(cudaDeviceSynchronize());
    float best = 1e30;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"test\":\"dmma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bpsm, flops / best / 1e9);
  }
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 128, iters = 2000;
    mixed_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
    float best = 1e30;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); mixed_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * (8.0 * 256 + 64.0 * 32) * (double)iters * blocks * (threads / 32);
    printf("{\"test\":\"dmma+dfma mixed\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bpsm, flops / best / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 2^27 double2 = 2 GiB per buffer
  double2 *a, *b; CK(cudaMalloc(&a, n * sizeof(double2))); CK(cudaMalloc(&b, n * sizeof(double2)));
  cudaMemset(a, 0, n * sizeof(double2));
  copy_kernel<<<sms * 8, 512>>>(a, b, n); CK(cudaDeviceSynchronize());
  float best = 1e30;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); copy_kernel<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("{\"test\":\"copy_fp64\",\"gbs\":%.1f}\n", 2.0 * n * sizeof(double2) / best / 1e6);
  return 0;
}
