// Does the FP64 tensor pipe (DMMA m8n8k4) run concurrently with the FP64
// CUDA-core pipe (DFMA)? Each warp runs `iters` trips of ND independent DMMAs
// and NF independent DFMAs per lane; FMA throughput for DMMA-only,
// DFMA-only and mixed loops tells whether the two add up.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NF>
__global__ void mix(double* out, int iters, double x) {
  double d[ND > 0 ? ND : 1][2];
  double f[NF > 0 ? NF : 1];
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) d[i][0] = d[i][1] = threadIdx.x;
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = threadIdx.x + i;
  const double a = x + threadIdx.x * 1e-9, b = x - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ND; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) s += d[i][0] + d[i][1];
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += f[i];
  if (s == 1.2345) out[0] = s;
}

template <int ND, int NF>
void run(int warps_per_sm, int sms) {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096;
  mix<ND, NF><<<sms, 32 * warps_per_sm>>>(out, 16, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<ND, NF><<<sms, 32 * warps_per_sm>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma_dmma = double(sms) * warps_per_sm * iters * ND * 256.0;
  const double fma_dfma = double(sms) * warps_per_sm * iters * NF * 32.0;
  printf("ND=%2d NF=%2d warps/SM=%2d: %.3f ms, DMMA %.1f TFLOP/s + DFMA %.1f TFLOP/s = %.1f TFLOP/s\n", ND, NF,
         warps_per_sm, ms, 2 * fma_dmma / ms / 1e9, 2 * fma_dfma / ms / 1e9, 2 * (fma_dmma + fma_dfma) / ms / 1e9);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run<8, 0>(w, sms);
    run<0, 16>(w, sms);
    run<8, 16>(w, sms);
    run<8, 32>(w, sms);
    run<4, 16>(w, sms);
  }
  return 0;
}
