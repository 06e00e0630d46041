// Dependent-chain latency of FP64 and FP32 ops on one warp (cycles/op).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_dadd(double* out, double a, int n, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + a;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_ffma(float* out, float a, float b, int n, long long* cyc) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fmaf(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// 8 independent chains on one warp: throughput-limited rate
__global__ void ilp_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 4096); cudaMalloc(&c, 8);
  const int n = 4096;
  chain_dfma<<<1, 32>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  chain_dfma<<<1, 32>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA: %.2f cyc/op\n", double(h) / n);
  chain_dadd<<<1, 32>>>(d, 1e-3, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent DADD: %.2f cyc/op\n", double(h) / n);
  chain_ffma<<<1, 32>>>((float*)d, 0.999f, 1e-3f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent FFMA: %.2f cyc/op\n", double(h) / n);
  ilp_dfma<<<1, 32>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("8 independent DFMA chains, one warp: %.2f cyc/op\n", double(h) / n / 8);
  return 0;
}
