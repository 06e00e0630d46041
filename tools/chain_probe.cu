// Per-step cost of the AHALS column recurrence on one warp per SM
// sub-partition: dependent (DFMA + clip) chain with P independent pushes per
// step, and the latency of a shuffle / shared load on the chain.
#include <cstdio>
#include <cuda_runtime.h>

template <int P>
__global__ void step_chain(double* out, const double* __restrict__ h, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3, lo = -1e300;
  double u[P > 0 ? P : 1];
  double hh[P > 0 ? P : 1];
#pragma unroll
  for (int p = 0; p < (P > 0 ? P : 1); ++p) { u[p] = p; hh[p] = h[p]; }
  const double hd = h[40];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double v = fma(-hd, x, u[0]);
    x = v < lo ? 0.0 : v;
#pragma unroll
    for (int p = 1; p < P; ++p) u[p] = fma(-x, hh[p], u[p]);
    if (P > 0) u[0] = u[P > 1 ? 1 : 0] * 0.5 + 1e-9;
  }
  long long t1 = clock64();
  double s = x;
#pragma unroll
  for (int p = 0; p < (P > 0 ? P : 1); ++p) s += u[p];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void shfl_chain(double* out, int n, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lds_chain(double* out, int n, long long* cyc) {
  __shared__ double s[64];
  s[threadIdx.x] = 0.0;
  s[threadIdx.x + 32] = 0.0;
  __syncwarp();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) idx = int(s[idx]) + (threadIdx.x);
  long long t1 = clock64();
  out[threadIdx.x] = idx;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int P>
void run(double* d, double* h, long long* c, int warps) {
  const int n = 4096;
  long long hc;
  step_chain<P><<<1, 32 * warps>>>(d, h, n, c);
  step_chain<P><<<1, 32 * warps>>>(d, h, n, c);
  cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
  printf("step chain + %2d pushes, %d warps/CTA: %.1f cyc/step\n", P > 0 ? P - 1 : 0, warps, double(hc) / n);
}

int main() {
  double *d, *h;
  long long* c;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&h, 4096);
  cudaMemset(h, 0, 4096);
  cudaMalloc(&c, 8);
  for (int w : {1, 4, 8}) {
    run<0>(d, h, c, w);
    run<2>(d, h, c, w);
    run<6>(d, h, c, w);
    run<11>(d, h, c, w);
    run<20>(d, h, c, w);
  }
  long long hc;
  const int n = 4096;
  shfl_chain<<<1, 32>>>(d, n, c);
  shfl_chain<<<1, 32>>>(d, n, c);
  cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent SHFL + DADD: %.1f cyc\n", double(hc) / n);
  lds_chain<<<1, 32>>>(d, n, c);
  lds_chain<<<1, 32>>>(d, n, c);
  cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent LDS.64 + cvt + add: %.1f cyc\n", double(hc) / n);
  return 0;
}
