// FP64 chain latencies on one warp per SM (diagnostic for the AHALS column chain):
//  a) dependent DFMA chain, b) DFMA + sign-mask clip (SHF + LOP3) chain,
//  c) 8 independent DFMA streams (issue cost per DFMA), d) chain + 8 side DFMAs per step.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/chain_probe tools/chain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double clip(double v) {
  const int hi = __double2hiint(v), lo = __double2loint(v);
  int h2, l2;
  asm("{\n\t.reg .b32 m;\n\tshr.s32 m, %2, 31;\n\tlop3.b32 %0, %2, m, %4, 0x70;\n\tlop3.b32 %1, %3, m, %4, 0x70;\n\t}"
      : "=r"(h2), "=r"(l2) : "r"(hi), "r"(lo), "r"(-1));
  return __hiloint2double(h2, l2);
}

template <int MODE>
__global__ void probe(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-9, s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] = b + i;
  const long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (MODE == 0) x = fma(x, a, b);
      if (MODE == 1) x = clip(fma(x, a, b));
      if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = fma(s[i], a, b);
      }
      if (MODE == 3) {
        x = clip(fma(x, a, b));
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = fma(s[i], a, x);
      }
      if (MODE == 4) {  // max via DSETP/FSEL style
        const double v = fma(x, a, b);
        x = v < 0.0 ? 0.0 : v;
      }
      if (MODE == 5) x = fmax(fma(x, a, b), 0.0);
    }
  }
  const long long t1 = clock64();
  double r = x;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 128 * 8); cudaMallocManaged(&cyc, 8);
  const int n = 256;
  const char* names[] = {"dfma chain", "dfma+clip(shr,lop3) chain", "8 indep dfma (per group of 8)", "chain+clip+8 side dfma", "dfma + (v<0?0:v)", "dfma + fmax"};
  for (int warps = 1; warps <= 2; ++warps) {
    for (int m = 0; m < 6; ++m) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (m) {
          case 0: probe<0><<<148, 32 * warps * (warps == 2 ? 4 : 1)>>>(out, cyc, 0.999, 1e-3, n); break;
          case 1: probe<1><<<148, 32 * warps * (warps == 2 ? 4 : 1)>>>(out, cyc, 0.999, 1e-3, n); break;
          case 2: probe<2><<<148, 32 * warps * (warps == 2 ? 4 : 1)>>>(out, cyc, 0.999, 1e-3, n); break;
          case 3: probe<3><<<148, 32 * warps * (warps == 2 ? 4 : 1)>>>(out, cyc, 0.999, 1e-3, n); break;
          case 4: probe<4><<<148, 32 * warps * (warps == 2 ? 4 : 1)>>>(out, cyc, 0.999, 1e-3, n); break;
          case 5: probe<5><<<148, 32 * warps * (warps == 2 ? 4 : 1)>>>(out, cyc, 0.999, 1e-3, n); break;
        }
        cudaDeviceSynchronize();
      }
      printf("warps/SM=%d  %-32s %.2f cycles per step\n", warps == 2 ? 8 : 1, names[m], double(*cyc) / (n * 16));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
