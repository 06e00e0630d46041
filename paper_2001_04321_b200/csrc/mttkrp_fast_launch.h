// Dispatch table of the fast MTTKRP kernel instantiations.
#pragma once

#include <cuda.h>

#include <string>

#include "ntf_internal.h"

namespace ntfb {
namespace fast {

enum { kRow = 0, kCol = 1 };

struct Params {
  ModeView v;
  const DevFactors* F;
  double* partial;  // [ctas_per_mtile][I][r]
  long long units;  // per m-tile
  long long nbox_r; // ROW: rho boxes per l
  int kbox;         // reduction indices per unit
  int m_box, n_mbox, m_cta, ctas_per_mtile;
  int MW, KW, NP, stages, wld;  // consumer m-warps, k-warps, producer warps
  unsigned t_stage_bytes, w_stage_bytes, tx_bytes;
};
using LaunchFn = void (*)(const CUtensorMap& map, const Params& p, int grid, int threads, size_t smem,
                          cudaStream_t s);

// One register-blocking shape: G column groups x B columns, A rows per lane.
struct KernelCfg {
  int G, B, A;
  LaunchFn row, col;
};

// Picks the blocking for (dtype, rank, rows); false when no instantiation
// covers the rank.
bool lookup(int dtype, int rank, long long rows, KernelCfg* out);
bool lookup_f64(int rank, long long rows, KernelCfg* out);
bool lookup_f32(int rank, long long rows, KernelCfg* out);

}  // namespace fast

std::string fast_mttkrp_describe(const ModeView& v, int dtype, int sms);

}  // namespace ntfb
