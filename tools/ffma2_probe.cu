// FFMA2 issue cadence with the FP32 consumer's operand pattern (diagnostic):
// acc[A][4] float2 += t[i][kk] (scalar broadcast) * wv[kk][q] (pair), operands
// in registers (MODE 0) or reloaded from shared memory every step like the
// kernel (MODE 1: A + 8 LDS.128 per 16 A FFMA2).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ffma2_probe tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  unsigned long long d;
  const float2 aa = make_float2(a, a);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d)
      : "l"(*reinterpret_cast<const unsigned long long*>(&aa)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

template <int A, int MODE>
__global__ void probe(float* out, long long* cyc, int n) {
  extern __shared__ float4 sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_float4(1e-3f * i, 1.f, 0.5f, 0.25f);
  __syncthreads();
  float2 acc[A][4];
  for (int i = 0; i < A; ++i)
    for (int q = 0; q < 4; ++q) acc[i][q] = make_float2(0.f, 0.f);
  float4 t[A], w[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < A; ++i) t[i] = sm[(lane % 8) * 8 + i];
  for (int i = 0; i < 8; ++i) w[i] = sm[64 + (lane / 8) * 8 + i];
  const long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    if (MODE == 1) {
      // the kernel's conflict-free pattern: T stage [rows][128 B] with the 128-byte swizzle, W rows [k][128 B]
      const unsigned char* ts = reinterpret_cast<const unsigned char*>(sm);
      const unsigned char* ws = ts + 32768;
      const int kq = it & 7, rg = lane % 8, cg = lane / 8;
#pragma unroll
      for (int i = 0; i < A; ++i) {
        const int row = warp * 8 * A % 256 + rg + 8 * i;
        t[i] = *reinterpret_cast<const float4*>(ts + row * 128 + (((kq ^ (row & 7)) & 7) << 4));
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        w[2 * kk] = *reinterpret_cast<const float4*>(ws + (4 * kq + kk) * 128 + cg * 32);
        w[2 * kk + 1] = *reinterpret_cast<const float4*>(ws + (4 * kq + kk) * 128 + cg * 32 + 16);
      }
    }
#pragma unroll
    for (int i = 0; i < A; ++i) {
      const float tk[4] = {t[i].x, t[i].y, t[i].z, t[i].w};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        acc[i][0] = ffma2(tk[kk], make_float2(w[2 * kk].x, w[2 * kk].y), acc[i][0]);
        acc[i][1] = ffma2(tk[kk], make_float2(w[2 * kk].z, w[2 * kk].w), acc[i][1]);
        acc[i][2] = ffma2(tk[kk], make_float2(w[2 * kk + 1].x, w[2 * kk + 1].y), acc[i][2]);
        acc[i][3] = ffma2(tk[kk], make_float2(w[2 * kk + 1].z, w[2 * kk + 1].w), acc[i][3]);
      }
    }
  }
  const long long t1 = clock64();
  float r = 0.f;
  for (int i = 0; i < A; ++i)
    for (int q = 0; q < 4; ++q) r += acc[i][q].x + acc[i][q].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int A, int MODE>
void run(const char* name, int warps, float* out, long long* cyc) {
  const int n = 2000;
  cudaFuncSetAttribute(probe<A, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int rep = 0; rep < 2; ++rep) {
    probe<A, MODE><<<148, 32 * warps, 65536>>>(out, cyc, n);
    cudaDeviceSynchronize();
  }
  const double per = double(*cyc) / (double(n) * A * 16);
  printf("%-28s warps/SM=%d  %.3f cycles per FFMA2 per warp  -> pipe use per SMSP %.2f\n", name, warps, per,
         2.0 * ((warps + 3) / 4) / per);
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4); cudaMallocManaged(&cyc, 8);
  for (int warps : {4, 8}) {
    if (warps == 4) { run<8, 0>("A=8 regs", warps, out, cyc); run<8, 1>("A=8 lds", warps, out, cyc); }
    run<4, 0>("A=4 regs", warps, out, cyc); run<4, 1>("A=4 lds", warps, out, cyc);
    if (warps == 8) { run<8, 0>("A=8 regs", warps, out, cyc); run<8, 1>("A=8 lds", warps, out, cyc); }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
