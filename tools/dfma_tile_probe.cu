// DFMA throughput of the MTTKRP consumer pattern: acc[A][B] += t[i] * w[b]
// with every operand a register (3 register pairs per DFMA), vs the peak
// pattern fma(x, a, b) with uniform a, b; and the same tile with t / w read
// from shared memory every k (the real consumer loop).
#include <cstdio>
#include <cuda_runtime.h>

template <int A, int B>
__global__ void tile_regs(double* out, int iters) {
  double acc[A][B], t[A], w[B];
#pragma unroll
  for (int i = 0; i < A; ++i) {
    t[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int b = 0; b < B; ++b) acc[i][b] = 0.0;
  }
#pragma unroll
  for (int b = 0; b < B; ++b) w[b] = b * 0.5;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int b = 0; b < B; ++b) acc[i][b] = fma(t[i], w[b], acc[i][b]);
#pragma unroll
    for (int i = 0; i < A; ++i) t[i] = t[i] * 0.999;  // keeps t live per k (A DMULs per A*B DFMAs)
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int b = 0; b < B; ++b) s += acc[i][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int A, int B>
__global__ void tile_smem(double* out, int iters) {
  __shared__ double ts[64 * 16 + 16];
  __shared__ double ws[16 * 16];
  for (int e = threadIdx.x; e < 64 * 16 + 16; e += blockDim.x) ts[e] = e * 1e-3;
  for (int e = threadIdx.x; e < 256; e += blockDim.x) ws[e] = e * 1e-2;
  __syncthreads();
  double acc[A][B];
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int b = 0; b < B; ++b) acc[i][b] = 0.0;
  const int lane = threadIdx.x & 31;
  const int rg = lane % 8, cg = lane / 8;
  for (int k = 0; k < iters; ++k) {
    const int kk = k & 15;
    double w[B];
#pragma unroll
    for (int b = 0; b < B; ++b) w[b] = ws[kk * 16 + cg * 4 + (b & 3)];
#pragma unroll
    for (int i = 0; i < A; ++i) {
      const double t = ts[(rg + 8 * i) * 16 + kk];
#pragma unroll
      for (int b = 0; b < B; ++b) acc[i][b] = fma(t, w[b], acc[i][b]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int b = 0; b < B; ++b) s += acc[i][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the ROW consumer loop of mttkrp_fast_impl.cuh without the pipeline: T in
// a [320][128 B] 128-byte-swizzled tile, W [16][24] (G = 4 groups of 5 + pad)
__global__ void tile_row(double* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ts = sm;
  double* ws = reinterpret_cast<double*>(sm + 320 * 128);
  for (int e = threadIdx.x; e < 320 * 16; e += blockDim.x) reinterpret_cast<double*>(ts)[e] = e * 1e-6;
  for (int e = threadIdx.x; e < 16 * 24; e += blockDim.x) ws[e] = e * 1e-3;
  __syncthreads();
  constexpr int A = 8, B = 5, BP = 6, RG = 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mw = warp % 5, kw = (warp / 5) & 1;
  const int rg = lane % RG, cg = lane / RG;
  double acc[A][B];
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int b = 0; b < B; ++b) acc[i][b] = 0.0;
  int off[A];
#pragma unroll
  for (int i = 0; i < A; ++i) off[i] = mw * 64 + rg + RG * i;
  const double* wsb = ws + cg * BP;
  for (int it = 0; it < iters; ++it) {
    for (int pc = kw; pc < 8; pc += 2) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        double w[BP];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double2 x = *reinterpret_cast<const double2*>(wsb + (pc * 2 + kk) * 24 + q * 2);
          w[2 * q] = x.x;
          w[2 * q + 1] = x.y;
        }
#pragma unroll
        for (int i = 0; i < A; ++i) {
          const int m = off[i];
          const double t = *reinterpret_cast<const double*>(ts + m * 128 + (((pc ^ m) & 7) << 4) + kk * 8);
#pragma unroll
          for (int b = 0; b < B; ++b) acc[i][b] = fma(t, w[b], acc[i][b]);
        }
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int b = 0; b < B; ++b) s += acc[i][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// generic ROW-loop variants: G column groups of B, A rows per lane; T2: read
// both k of a 16-byte chunk at once; PF: prefetch the next chunk's T / W
template <int G, int B, int A, bool T2, bool PF>
__global__ void tile_row_v(double* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ts = sm;
  constexpr int BP = (B + 1) / 2 * 2, WLD = G * BP, RG = 32 / G, RW = RG * A;
  double* ws = reinterpret_cast<double*>(sm + 320 * 128);
  for (int e = threadIdx.x; e < 320 * 16; e += blockDim.x) reinterpret_cast<double*>(ts)[e] = e * 1e-6;
  for (int e = threadIdx.x; e < 16 * WLD; e += blockDim.x) ws[e] = e * 1e-3;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5, half = nw / 2;
  const int mw = warp % half, kw = warp / half;
  const int rg = lane % RG, cg = lane / RG;
  double acc[A][B];
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int b = 0; b < B; ++b) acc[i][b] = 0.0;
  int off[A];
#pragma unroll
  for (int i = 0; i < A; ++i) off[i] = (mw * RW + rg + RG * i) % 320;
  const double* wsb = ws + cg * BP;
  auto loadT = [&](int pc, double2 (&t)[A]) {
#pragma unroll
    for (int i = 0; i < A; ++i) {
      const int m = off[i];
      t[i] = *reinterpret_cast<const double2*>(ts + m * 128 + (((pc ^ m) & 7) << 4));
    }
  };
  auto loadW = [&](int pc, double (&w)[2][BP]) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int q = 0; q < BP / 2; ++q) {
        const double2 x = *reinterpret_cast<const double2*>(wsb + (pc * 2 + kk) * WLD + q * 2);
        w[kk][2 * q] = x.x;
        w[kk][2 * q + 1] = x.y;
      }
  };
  for (int it = 0; it < iters; ++it) {
    if constexpr (T2) {
      double2 t[A];
      double w[2][BP];
      loadT(kw, t);
      loadW(kw, w);
      for (int pc = kw; pc < 8; pc += 2) {
        double2 tn[A];
        double wn[2][BP];
        if (PF && pc + 2 < 8) {
          loadT(pc + 2, tn);
          loadW(pc + 2, wn);
        }
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
#pragma unroll
          for (int i = 0; i < A; ++i) {
            const double tv = kk ? t[i].y : t[i].x;
#pragma unroll
            for (int b = 0; b < B; ++b) acc[i][b] = fma(tv, w[kk][b], acc[i][b]);
          }
        if (pc + 2 < 8) {
          if (PF) {
#pragma unroll
            for (int i = 0; i < A; ++i) t[i] = tn[i];
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
              for (int b = 0; b < BP; ++b) w[kk][b] = wn[kk][b];
          } else {
            loadT(pc + 2, t);
            loadW(pc + 2, w);
          }
        }
      }
    } else {
      for (int pc = kw; pc < 8; pc += 2) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          double w[BP];
#pragma unroll
          for (int q = 0; q < BP / 2; ++q) {
            const double2 x = *reinterpret_cast<const double2*>(wsb + (pc * 2 + kk) * WLD + q * 2);
            w[2 * q] = x.x;
            w[2 * q + 1] = x.y;
          }
#pragma unroll
          for (int i = 0; i < A; ++i) {
            const int m = off[i];
            const double tv = *reinterpret_cast<const double*>(ts + m * 128 + (((pc ^ m) & 7) << 4) + kk * 8);
#pragma unroll
            for (int b = 0; b < B; ++b) acc[i][b] = fma(tv, w[b], acc[i][b]);
          }
        }
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int b = 0; b < B; ++b) s += acc[i][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int G, int B, int A, bool T2, bool PF>
void run_v(double* d, int warps, const char* name) {
  auto k = tile_row_v<G, B, A, T2, PF>;
  const int smem = 320 * 128 + 16 * G * ((B + 1) / 2 * 2) * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int it = 1024;
  k<<<148, warps * 32, smem>>>(d, it);
  cudaEventRecord(e0);
  k<<<148, warps * 32, smem>>>(d, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 148 * warps * 32 * double(it) * 4 * 2 * A * B;
  printf("%-28s %2d warps: %.1f TFLOP/s (%s)\n", name, warps, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

template <typename K>
float time_ms(K kern, int grid, int threads, double* d, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, threads>>>(d, iters);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    kern<<<grid, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  double* d;
  cudaMalloc(&d, 148 * 1024 * 8);
  const int iters = 4096;
  for (int warps : {4, 8, 12}) {
    const int threads = warps * 32;
    float ms = time_ms(tile_regs<8, 5>, 148, threads, d, iters);
    double fl = 2.0 * 148 * threads * double(iters) * 40;
    printf("regs 8x5, %2d warps/SM: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    ms = time_ms(tile_regs<4, 10>, 148, threads, d, iters);
    printf("regs 4x10, %2d warps/SM: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    ms = time_ms(tile_smem<8, 5>, 148, threads, d, iters);
    printf("smem 8x5, %2d warps/SM: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  {
    cudaFuncSetAttribute(tile_row, cudaFuncAttributeMaxDynamicSharedMemorySize, 320 * 128 + 16 * 24 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int it = 1024;
    tile_row<<<148, 320, 320 * 128 + 16 * 24 * 8>>>(d, it);
    cudaEventRecord(e0);
    tile_row<<<148, 320, 320 * 128 + 16 * 24 * 8>>>(d, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per iteration a warp does 4 pc x 2 kk x 40 FMA per lane
    const double fl = 2.0 * 148 * 320 * double(it) * 4 * 2 * 40;
    printf("ROW consumer loop (10 warps, 8x5, swizzled T, no pipeline): %.1f TFLOP/s (%s)\n", fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  run_v<4, 5, 8, false, false>(d, 10, "8x5 base");
  run_v<4, 5, 8, true, false>(d, 10, "8x5 T2");
  run_v<4, 5, 8, true, true>(d, 10, "8x5 T2+PF");
  run_v<4, 5, 8, true, true>(d, 8, "8x5 T2+PF");
  run_v<2, 10, 4, true, false>(d, 10, "4x10 T2");
  run_v<2, 10, 4, true, true>(d, 10, "4x10 T2+PF");
  run_v<2, 10, 6, true, false>(d, 8, "6x10 T2");
  run_v<2, 10, 6, true, true>(d, 8, "6x10 T2+PF");
  run_v<2, 10, 8, true, false>(d, 8, "8x10 T2");
  run_v<4, 5, 12, true, false>(d, 8, "12x5 T2");
  return 0;
}
