// FP64 instantiations of the fast MTTKRP kernel (DFMA on CUDA cores).
#include "mttkrp_fast_impl.cuh"
#include "mttkrp_fast_launch.h"

namespace ntfb {
namespace fast {

template <typename T, int G, int B, int A, int LAYOUT>
void launch_impl(const CUtensorMap& map, const Params& p, int grid, int threads, size_t smem, cudaStream_t s) {
  auto fn = mttkrp_fast_kernel<T, G, B, A, LAYOUT>;
  NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  fn<<<grid, threads, smem, s>>>(map, p);
  NTF_CUDA(cudaGetLastError());
}

#define NTF_CFG(T, G, B, A) KernelCfg{G, B, A, launch_impl<T, G, B, A, kRow>, launch_impl<T, G, B, A, kCol>}

bool lookup_f64(int r, long long rows, KernelCfg* out) {
  if (r <= 4) *out = NTF_CFG(double, 2, 2, 2);
  else if (r <= 8) *out = NTF_CFG(double, 2, 4, 2);
  else if (r <= 10) *out = NTF_CFG(double, 2, 5, 2);
  else if (r <= 12) *out = NTF_CFG(double, 2, 6, 2);
  else if (r <= 16) *out = (rows > 64 && rows <= 112) ? NTF_CFG(double, 4, 4, 14) : NTF_CFG(double, 2, 8, 2);
  else if (r <= 20) *out = NTF_CFG(double, 4, 5, 4);
  else if (r <= 24) *out = NTF_CFG(double, 4, 6, 4);
  else if (r <= 32) *out = NTF_CFG(double, 4, 8, 4);
  else if (r <= 64) *out = NTF_CFG(double, 8, 8, 8);
  else return false;
  return true;
}

bool lookup(int dtype, int rank, long long rows, KernelCfg* out) {
  return dtype == NTF_DTYPE_F32 ? lookup_f32(rank, rows, out) : lookup_f64(rank, rows, out);
}

}  // namespace fast
}  // namespace ntfb
