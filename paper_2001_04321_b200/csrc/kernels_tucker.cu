// TuckerProvider MTTKRP on the device (tucker.hpp:60-73, tucker.cpp:62-77):
//
//   M_n = U_n * ( core_(n) * KR_{l != n}(U_l^T A_l) )
//
// = U_n times the MTTKRP of the small core with the projected factors
// P_l = U_l^T A_l (r_l x r). The core MTTKRP runs on the dense kernels
// (MttkrpEngine on the core); the two thin matrix products here are short
// fixed-order sums, one thread per output (the factors are at most a few
// thousand rows; the products are a few MFLOP).
#include <algorithm>

#include "ntf_internal.h"

namespace ntfb {

namespace {

// P_l[a][c] = sum_i U_l[i][a] * A_l[i][c] for every l != skip (blockIdx.y = l),
// A_l = the X-role buffer of mode l.
__global__ void tucker_project_kernel(TuckerDev td, const DevFactors* __restrict__ F, int skip, int r) {
  const int l = blockIdx.y;
  if (l == skip) return;
  const int I = td.rows[l], R = td.ranks[l];
  const double* U = td.bases + td.base_off[l];
  const double* A = F->x[l][F->sel[l]];
  double* P = td.proj + td.proj_off[l];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * r; e += gridDim.x * blockDim.x) {
    const int a = e / r, c = e % r;
    double s = 0.0;
    for (int i = 0; i < I; ++i) s += U[(long long)i * R + a] * A[(long long)i * r + c];
    P[e] = s;
  }
}

// out[i][c] = sum_a U_n[i][a] * Mc[a][c]
__global__ void tucker_expand_kernel(TuckerDev td, int n, int r, const double* __restrict__ Mc,
                                     double* __restrict__ out) {
  const int I = td.rows[n], R = td.ranks[n];
  const double* U = td.bases + td.base_off[n];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)I * r;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / r;
    const int c = int(e % r);
    double s = 0.0;
    for (int a = 0; a < R; ++a) s += U[i * R + a] * Mc[(long long)a * r + c];
    out[e] = s;
  }
}

}  // namespace

void launch_tucker_project(const TuckerDev& td, const DevFactors* dF, int skip, int order, int rank, cudaStream_t s) {
  int maxe = 1;
  for (int l = 0; l < order; ++l) maxe = std::max(maxe, td.ranks[l] * rank);
  const dim3 grid(unsigned((maxe + 127) / 128), unsigned(order));
  tucker_project_kernel<<<grid, 128, 0, s>>>(td, dF, skip, rank);
  NTF_CUDA(cudaGetLastError());
}

void launch_tucker_expand(const TuckerDev& td, int mode, int rank, const double* Mc, double* out, cudaStream_t s) {
  const long long n = (long long)td.rows[mode] * rank;
  const unsigned blocks = unsigned(std::min<long long>((n + 255) / 256, 4096));
  tucker_expand_kernel<<<blocks, 256, 0, s>>>(td, mode, rank, Mc, out);
  NTF_CUDA(cudaGetLastError());
}

}  // namespace ntfb
