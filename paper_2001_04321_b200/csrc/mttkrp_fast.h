// Fast sm_100a MTTKRP paths (TMA-staged tensor tiles, on-the-fly Khatri-Rao
// rows, register-blocked CUDA-core FMA, deterministic split-K reduction).
#pragma once

#include <vector>

#include "ntf_internal.h"

namespace ntfb {

// True when the view/dtype/rank has a fast kernel on this build.
bool fast_mttkrp_supported(const ModeView& v, int dtype);
// Kernel launches per MTTKRP call on the fast path.
int fast_mttkrp_kernels(const ModeView& v, int dtype);
// Doubles of split-K workspace the fast path needs for this view.
size_t fast_mttkrp_partial_len(const ModeView& v, int dtype, int sms);
// out = MTTKRP (I x r, FP64) of the local view.
// Host-built per-unit table of the fast path (see mttkrp_fast_launch.h);
// empty when the view has no fast plan. Depends only on shape and dtype.
std::vector<int> fast_mttkrp_unit_table(const ModeView& v, int dtype, int sms);
// `counter` (zeroed device word owned by the caller, used by one stream at a
// time) enables the in-kernel split-K reduction; nullptr: separate kernel.
// pdl: launch as a programmatic dependent of the previous kernel in the
// stream (it may start while that kernel runs, on the SMs it leaves free).
void fast_mttkrp(const void* t, int dtype, const ModeView& v, const DevFactors* dF, const int* unit_table,
                 double* partial, double* out, int sms, cudaStream_t s, unsigned* counter = nullptr, bool pdl = false);

}  // namespace ntfb
