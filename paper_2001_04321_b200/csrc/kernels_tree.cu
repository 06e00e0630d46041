// Dimension-tree MTTKRP reuse.
//
// Inside one HER / AO outer iteration, block n < N-1 contracts the tensor
// with A_{N-1} of the previous sweep (or its restart value): her.cpp:64-65
// uses the current sweep's blocks for j < n and the previous ones for j > n.
// So the partial contraction
//     Y[i_0..i_{N-2}][c] = sum_{i_{N-1}} T[i_0..i_{N-1}] * A_{N-1}[i_{N-1}][c]
// (a tall-skinny GEMM, computed by the fast MTTKRP kernel on the 2-way view
// (prod_{n<N-1} I_n) x I_{N-1}) is shared by blocks 0..N-2, and block n only
// needs
//     M_n[i][c] = sum_{l, rho} Y[l][i][rho][c] * wl[l][c] * wr[rho][c]
// with wl / wr the Khatri-Rao rows of the blocks before / after n among
// 0..N-2 (kernels.cpp:90-113). Y is |T| / I_{N-1} * r values — 14.4 MB at
// BASELINE config 2, L2-resident — so full tensor passes per iteration drop
// from N to 2. Results differ from the direct MTTKRP only by summation order.
//
// tree_mttkrp_kernel: CTA (chunk, tile) owns a contiguous range of the
// flattened reduction index q = l * R' + rho and a tile of (i, c) output
// pairs; it forms the chunk's Khatri-Rao rows in shared memory, streams Y
// and writes a partial [chunk][I][r] slab; the fixed-order slab reduction
// (reduce_partials_kernel) follows. No atomics: bit-reproducible.
#include "ntf_internal.h"

namespace ntfb {
namespace {

constexpr int kTreeThreads = 256;
constexpr int kTreePPT = 4;  // output pairs per thread per tile
constexpr int kTreeTile = kTreeThreads * kTreePPT;
constexpr int kTreeQB = 8;  // q steps per load batch

__global__ void __launch_bounds__(kTreeThreads) tree_mttkrp_kernel(const double* __restrict__ Y, TreeView v,
                                                                   const DevFactors* __restrict__ F,
                                                                   double* __restrict__ partial, int qpc) {
  extern __shared__ double wsh[];  // [qpc][r]
  __shared__ const double* fac[kMaxOrder];
  const int r = v.rank;
  // factor pointers of the current roles: one round trip (sel and both
  // candidate pointers in flight together), then shared by the CTA
  if (threadIdx.x < unsigned(v.order)) {
    const int j = threadIdx.x;
    const int sel = F->sel[j];
    const double* x0 = F->x[j][0];
    const double* x1 = F->x[j][1];
    fac[j] = sel ? x1 : x0;
  }
  __syncthreads();
  // every index below fits 32 bits (checked by the launcher)
  const int Q = int(v.L * v.R);
  const int q0 = int(blockIdx.x) * qpc;
  const int q1 = q0 + qpc < Q ? q0 + qpc : Q;
  const int I = int(v.I), R = int(v.R);
  const int pairs = I * r;
  const int p0 = int(blockIdx.y) * kTreeTile;

  // Khatri-Rao rows of the chunk: rho digits over the blocks after n (last
  // fastest), l digits over the blocks before n (block 0 carries the slab
  // offset on a multi-GPU context).
  for (int e = threadIdx.x; e < (q1 - q0) * r; e += blockDim.x) {
    const int q = q0 + e / r;
    const int c = e % r;
    int l = q / R, rho = q - (q / R) * R;
    double w = 1.0;
    for (int j = v.order - 1; j > v.mode; --j) {
      const int d = rho % v.dims[j];
      rho /= v.dims[j];
      w *= fac[j][(long long)d * r + c];
    }
    for (int j = v.mode - 1; j >= 0; --j) {
      const int d = l % v.dims[j];
      l /= v.dims[j];
      w *= fac[j][((long long)d + (j == 0 ? v.row0 : 0)) * r + c];
    }
    wsh[e] = w;
  }
  __syncthreads();

  double acc[kTreePPT];
  long long yoff[kTreePPT];
  int col[kTreePPT];
  bool ok[kTreePPT];
#pragma unroll
  for (int k = 0; k < kTreePPT; ++k) {
    const int p = p0 + int(threadIdx.x) + k * kTreeThreads;
    ok[k] = p < pairs;
    const int i = ok[k] ? p / r : 0;
    col[k] = ok[k] ? p - i * r : 0;
    yoff[k] = (long long)i * R * r + col[k];
    acc[k] = 0.0;
  }
  const long long istride = (long long)I * R * r;  // one step of l
  // (l, rho) of q advance by counting, no division in the loop;
  // kTreeQB steps per batch keep kTreeQB * kTreePPT loads in flight
  int l = q0 / R, rho = q0 - (q0 / R) * R;
  int q = q0;
  for (; q + kTreeQB <= q1; q += kTreeQB) {
    double y[kTreeQB][kTreePPT];
#pragma unroll
    for (int b = 0; b < kTreeQB; ++b) {
      const double* yq = Y + l * istride + (long long)rho * r;
#pragma unroll
      for (int k = 0; k < kTreePPT; ++k) y[b][k] = ok[k] ? __ldg(yq + yoff[k]) : 0.0;
      if (++rho == R) {
        rho = 0;
        ++l;
      }
    }
#pragma unroll
    for (int b = 0; b < kTreeQB; ++b) {
      const double* wq = wsh + (q + b - q0) * r;
#pragma unroll
      for (int k = 0; k < kTreePPT; ++k) acc[k] = fma(y[b][k], wq[col[k]], acc[k]);
    }
  }
  {
    // tail: up to kTreeQB - 1 steps, loads first
    double y[kTreeQB][kTreePPT];
    const int nt = q1 - q;
#pragma unroll
    for (int b = 0; b < kTreeQB; ++b) {
      if (b < nt) {
        const double* yq = Y + l * istride + (long long)rho * r;
#pragma unroll
        for (int k = 0; k < kTreePPT; ++k) y[b][k] = ok[k] ? __ldg(yq + yoff[k]) : 0.0;
        if (++rho == R) {
          rho = 0;
          ++l;
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kTreeQB; ++b) {
      if (b < nt) {
        const double* wq = wsh + (q + b - q0) * r;
#pragma unroll
        for (int k = 0; k < kTreePPT; ++k) acc[k] = fma(y[b][k], wq[col[k]], acc[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kTreePPT; ++k) {
    const int p = p0 + int(threadIdx.x) + k * kTreeThreads;
    if (ok[k]) partial[(long long)blockIdx.x * pairs + p] = acc[k];
  }
}

}  // namespace

int tree_chunks(const TreeView& v, int sms) {
  const long long pairs = v.I * v.rank;
  const long long tiles = (pairs + kTreeTile - 1) / kTreeTile;
  const long long Q = v.L * v.R;
  long long chunks = (2LL * sms + tiles - 1) / tiles;
  // a chunk's Khatri-Rao rows live in shared memory (<= 192 KB)
  const long long min_chunks = (Q * v.rank * (long long)sizeof(double) + 192 * 1024 - 1) / (192 * 1024);
  chunks = std::max(1LL, std::min(std::max(chunks, min_chunks), Q));
  return int(chunks);
}

void launch_tree_mttkrp(const double* Y, const TreeView& v, const DevFactors* dF, double* partial, int chunks,
                        double* out, cudaStream_t s) {
  const long long pairs = v.I * v.rank;
  const long long Q = v.L * v.R;
  if (Q >= (1LL << 31) || pairs >= (1LL << 31)) throw Unsupported("dimension tree: view too large for 32-bit indexing");
  const long long qpc = (Q + chunks - 1) / chunks;
  const int nchunk = int((Q + qpc - 1) / qpc);
  const size_t smem = size_t(qpc) * v.rank * sizeof(double);
  if (smem > 200 * 1024) throw Unsupported("dimension tree: chunk too large");
  if (smem > 48 * 1024)
    NTF_CUDA(cudaFuncSetAttribute(tree_mttkrp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const dim3 grid(unsigned(nchunk), unsigned((pairs + kTreeTile - 1) / kTreeTile));
  tree_mttkrp_kernel<<<grid, kTreeThreads, smem, s>>>(Y, v, dF, partial, int(qpc));
  NTF_CUDA(cudaGetLastError());
  launch_reduce_partials(partial, nchunk, pairs, out, s);
}

}  // namespace ntfb
