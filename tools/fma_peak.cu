// CUDA-core FMA peak microbenchmark for the roofline denominators that
// MEASURED_PEAKS.json does not carry (FP64 DFMA, FP32 FFMA, FP32x2 FFMA2).
// Each thread runs 8 independent FMA chains for ITERS steps; the grid covers
// every SM several times over. Timed with CUDA events, best of 5.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void dfma_kernel(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x + j;
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
  float2 x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = make_float2(threadIdx.x + j, threadIdx.x - j);
  float2 av = make_float2(a, a), bv = make_float2(b, b);
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      unsigned long long xr = *reinterpret_cast<unsigned long long*>(&x[j]);
      unsigned long long ar = *reinterpret_cast<unsigned long long*>(&av);
      unsigned long long br = *reinterpret_cast<unsigned long long*>(&bv);
      asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(xr) : "l"(ar), "l"(br));
      x[j] = *reinterpret_cast<float2*>(&xr);
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j].x + x[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8;
  const double n = double(blocks) * threads * ITERS;
  void* buf;
  cudaMalloc(&buf, size_t(blocks) * threads * 8);
  double ms = best_ms([&] { dfma_kernel<<<blocks, threads>>>((double*)buf, 0.999, 1e-3); });
  printf("{\"sms\": %d, \"dfma_tflops\": %.2f", sms, n * 8 * 2 / ms / 1e9);
  ms = best_ms([&] { ffma_kernel<<<blocks, threads>>>((float*)buf, 0.999f, 1e-3f); });
  printf(", \"ffma_tflops\": %.2f", n * 16 * 2 / ms / 1e9);
  ms = best_ms([&] { ffma2_kernel<<<blocks, threads>>>((float*)buf, 0.999f, 1e-3f); });
  printf(", \"ffma2_tflops\": %.2f}\n", n * 16 * 2 / ms / 1e9);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
