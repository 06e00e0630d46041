// Stream-K FP64 DMMA MTTKRP (mttkrp_sk.cu): plan, tables and launch.
#pragma once

#include <string>
#include <vector>

#include "mttkrp_fast_launch.h"
#include "ntf_internal.h"

namespace ntfb {
namespace sk {
constexpr int kMaxNP = 4;  // producer warps
constexpr int kMaxMW = 8;  // consumer warps
}  // namespace sk

struct SkParams {
  ModeView v;
  const DevFactors* F;
  double* partial;  // [2 * grid][m_cta][r] split-tile slabs
  double* out;
  unsigned* counter;  // grid barrier [arrivals, generation]
  const int* utab;    // unit table, then [n_tiles][2] contributor CTAs, then the split-tile list
  long long U;        // units per m-tile
  long long W;        // n_tiles * U
  int n_tiles, n_split;
  int align;  // 1: CTA ranges are whole tiles (tall views: no split tiles, no grid barrier)
  int lpo;    // split-tile reduction: lanes per output (1, or 8 for wide fan-in)
  int direct_b;  // no base modes: DMMA B operand = the bulk-copied factor rows (no W formation)
  int naw;       // W formation: aq slots per producer warp
  int flush_units;  // FP32: FP64 flush every flush_units units (0: at segment ends only)
  int pdl;       // host only: launch as a programmatic dependent
  int m_box, n_mbox, m_cta, m_pitch;
  int MW, NP, stages, wld;
  unsigned t_stage_bytes, w_stage_bytes, aq_stage_bytes, tx_bytes;
  int nb, bq[fast::kMaxBase], qL, rowL_wrap;
};

struct SkPlan {
  SkParams p{};
  int grid = 0, threads = 0, layout = 0, nmf = 0, nnf = 0;
  bool f32 = false;
  size_t smem = 0;
  std::vector<int> tile_ctas;  // [n_tiles][2]: first / last CTA touching the tile
  std::vector<int> split;      // tiles with more than one contributor
};

// The stream-K plan of an FP64 view (false: the view stays on the fast kernel).
bool sk_choose(const ModeView& v, int dtype, int sms, SkPlan* out);
size_t sk_partial_len(const ModeView& v, int dtype, int sms);
void sk_append_tables(const SkPlan& pl, std::vector<int>* tab);
void sk_mttkrp(const void* t, const ModeView& v, const SkPlan& pl, const DevFactors* dF, const int* unit_table,
               double* partial, double* out, cudaStream_t s, unsigned* counter, const fast::Params& modes,
               bool pdl = false);
std::string sk_describe(const SkPlan& pl);

}  // namespace ntfb
