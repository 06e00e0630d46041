// Latency probes for the NNLS sweep design (one warp, dependent chains).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, int n, double x0) {
  __shared__ double sm[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
  __syncwarp();
  const int lane = threadIdx.x;
  double v = x0 + lane;
  long long t0, t1;
  // 1. dependent DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = fma(v, 0.999, 1e-3);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // 2. dependent SHFL.IDX of a double (src lane depends on nothing)
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, (lane & ~3) | (i & 3));
  t1 = clock64();
  cyc[1] = t1 - t0;
  // 3. dependent LDS (address from value)
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double w = sm[idx & 255];
    idx = int(w) + (idx & 7);
  }
  t1 = clock64();
  cyc[2] = t1 - t0;
  // 4. DFMA -> DSETP -> FSEL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double u = fma(v, -0.5, 0.25);
    v = u < 0.0 ? 0.0 : u;
  }
  t1 = clock64();
  cyc[3] = t1 - t0;
  // 5. select-form chain: v = c ? p : fma(...)
  bool c = false;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double u = c ? 0.25 : fma(v, -0.5, 0.25);
    c = u < 0.0;
    v = u;
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  // 6. empty loop with clock reads
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    long long z = clock64();
    v += double(z & 1);
  }
  t1 = clock64();
  cyc[5] = t1 - t0;
  // 7. butterfly sum of a double over the warp (5 steps)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    v *= 1e-3;
  }
  t1 = clock64();
  cyc[6] = t1 - t0;
  // 8. independent DFMA throughput (8 chains)
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = v + k;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999, 1e-3);
  t1 = clock64();
  cyc[7] = t1 - t0;
  for (int k = 0; k < 8; ++k) v += a[k];
  // 9. __syncwarp
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    __syncwarp();
    v = fma(v, 0.999, 1e-3);
  }
  t1 = clock64();
  cyc[8] = t1 - t0;
  out[lane] = v + double(idx);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) probe<<<1, 32>>>(out, cyc, n, 0.5);
  cudaDeviceSynchronize();
  const char* names[] = {"dep DFMA", "dep SHFL.IDX f64", "dep LDS.64", "DFMA+clip", "select chain", "clock64 loop",
                         "butterfly sum (5 steps)", "8 indep DFMA", "syncwarp+DFMA"};
  for (int i = 0; i < 9; ++i) printf("%-26s %7.2f cycles/iter\n", names[i], double(cyc[i]) / n);
  return 0;
}
