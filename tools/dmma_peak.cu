// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput probe next to the
// DFMA peak of tools/fma_peak.cu: can a DMMA consumer loop beat the
// shared-memory-bound DFMA loop of the MTTKRP kernel? Each warp runs 8
// independent accumulator chains; grid covers every SM several times.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, double a, double b) {
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = threadIdx.x + j;
  double av = a + threadIdx.x * 1e-9, bv = b;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[j], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wpb : {4, 8, 16}) {
    const int blocks = sms * 4, threads = 32 * wpb;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double flops = 2.0 * 256 * 8 * double(ITERS) * blocks * wpb;  // 256 FMA per warp-level m8n8k4
    printf("{\"warps_per_block\": %d, \"dmma_tflops\": %.2f, \"err\": \"%s\"}\n", wpb, flops / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
