// FP32 instantiations of the fast MTTKRP kernel (FFMA on CUDA cores; the
// per-CTA partials are written in FP64 and reduced in FP64).
#include <cstdlib>

#include "mttkrp_fast_impl.cuh"
#include "mttkrp_fast_launch.h"

namespace ntfb {
namespace fast {

template <typename T, int G, int B, int A, int LAYOUT>
void launch_impl32(const CUtensorMap& map, const Params& p, int grid, int threads, size_t smem, cudaStream_t s) {
  auto fn = mttkrp_fast_kernel<T, G, B, A, LAYOUT>;
  NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  // cooperative: the in-kernel slab reduction waits for every CTA
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = p.counter ? 1 : 0;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  NTF_CUDA(cudaLaunchKernelEx(&cfg, fn, map, p));
}

#define NTF_CFG32(G, B, A) KernelCfg{G, B, A, launch_impl32<float, G, B, A, kRow>, launch_impl32<float, G, B, A, kCol>}

bool lookup_f32(int r, long long, KernelCfg* out) {
  if (const char* e = std::getenv("NTF_FAST_ALT")) {  // tuning: alternative blockings
    const int alt = std::atoi(e);
    if (r > 20 && r <= 32 && alt == 1) return *out = NTF_CFG32(4, 8, 8), true;
    if (r > 20 && r <= 32 && alt == 2) return *out = NTF_CFG32(2, 16, 8), true;
    if (r > 20 && r <= 32 && alt == 3) return *out = NTF_CFG32(4, 8, 6), true;
  }
  if (r <= 4) *out = NTF_CFG32(2, 2, 4);
  else if (r <= 8) *out = NTF_CFG32(2, 4, 4);
  else if (r <= 12) *out = NTF_CFG32(2, 6, 4);
  else if (r <= 16) *out = NTF_CFG32(2, 8, 4);
  else if (r <= 20) *out = NTF_CFG32(4, 5, 4);
  else if (r <= 32) *out = NTF_CFG32(2, 16, 8);  // r01 C4 sweep: best of 4x8x4, 4x8x8, 2x16x8, 4x8x6
  else if (r <= 64) *out = NTF_CFG32(8, 8, 8);
  else return false;
  return true;
}

}  // namespace fast
}  // namespace ntfb
