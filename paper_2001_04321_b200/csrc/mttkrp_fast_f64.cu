// FP64 instantiations of the fast MTTKRP kernel (DFMA on CUDA cores).
#include <cstdlib>

#include "mttkrp_fast_impl.cuh"
#include "mttkrp_fast_launch.h"

namespace ntfb {
namespace fast {

template <typename T, int G, int B, int A, int LAYOUT>
void launch_impl(const CUtensorMap& map, const Params& p, int grid, int threads, size_t smem, cudaStream_t s) {
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

// DMMA consumers exist for blockings whose warp rows form 8-row fragments
template <typename T, int G, int B, int A, int L>
constexpr LaunchFn mma_launch() {
  if constexpr (((32 / G) * A) % 8 == 0)
    return launch_impl<T, G, B, A, L>;
  else
    return nullptr;
}

#define NTF_CFG(T, G, B, A)                                                                          \
  KernelCfg{G, B, A, launch_impl<T, G, B, A, kRow>, launch_impl<T, G, B, A, kCol>, 4,                 \
            mma_launch<T, G, B, A, kRowMma>(), mma_launch<T, G, B, A, kColMma>()}

// Blocking per rank. Shared-memory bytes per DFMA are 8 (A + B) / (A B)
// (T and W values delivered per lane), and the SM moves 128 B/clk against 64
// DFMA/clk, so the shapes keep A*B/(A+B) near 3-5 and split k across warps
// to keep four (or, with smaller tiles, eight) consumer warps.
bool lookup_f64(int r, long long rows, KernelCfg* out) {
  if (const char* e = std::getenv("NTF_FAST_ALT")) {  // tuning: alternative blockings
    const int alt = std::atoi(e);
    if (r > 16 && r <= 20 && alt == 1) return *out = NTF_CFG(double, 2, 10, 5), true;
    if (r > 16 && r <= 20 && alt == 2) return *out = NTF_CFG(double, 4, 5, 8), true;
    if (r > 12 && r <= 16 && alt == 1) return *out = NTF_CFG(double, 2, 8, 4), true;
  }
  if (r <= 4) *out = NTF_CFG(double, 2, 2, 2);
  else if (r <= 8) *out = NTF_CFG(double, 2, 4, 4);
  else if (r <= 10) *out = NTF_CFG(double, 2, 5, 4);
  else if (r <= 12) *out = NTF_CFG(double, 2, 6, 6);
  else if (r <= 16) {
    *out = (rows > 64 && rows <= 112) ? NTF_CFG(double, 2, 8, 7) : NTF_CFG(double, 2, 8, 8);
    // DMMA consumers (r01f sweep, C3): eight consumer warps, 1432 -> 1466 iters/s
    const char* me = std::getenv("NTF_FAST_MMA");
    if (!(me && std::atoi(me) == 0)) out->cons = 8;
  }
  else if (r <= 20) {
    // measured (r01, C2): 8 consumer warps of 8 x 5 tiles beat 4 of 10 x 10
    // on every mode, and the COL layout most (80 vs 100 us)
    *out = NTF_CFG(double, 4, 5, 8);
    out->cons = 8;
  }
  else if (r <= 24) *out = NTF_CFG(double, 2, 12, 8);
  else if (r <= 32) *out = NTF_CFG(double, 4, 8, 8);
  else if (r <= 64) *out = NTF_CFG(double, 8, 8, 8);
  else return false;
  return true;
}

bool lookup(int dtype, int rank, long long rows, KernelCfg* out) {
  return dtype == NTF_DTYPE_F32 ? lookup_f32(rank, rows, out) : lookup_f64(rank, rows, out);
}

}  // namespace fast
}  // namespace ntfb
