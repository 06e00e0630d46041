// Fast sm_100a MTTKRP paths — see mttkrp_fast.h.
#include "mttkrp_fast.h"

namespace ntfb {

bool fast_mttkrp_supported(const ModeView&, int) { return false; }
int fast_mttkrp_kernels(const ModeView&, int) { return 2; }
size_t fast_mttkrp_partial_len(const ModeView&, int, int) { return 0; }
void fast_mttkrp(const void*, int, const ModeView&, const DevFactors*, double*, double*, int, cudaStream_t) {
  throw Unsupported("fast MTTKRP path not available");
}

}  // namespace ntfb
