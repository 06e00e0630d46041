// Dispatch table of the fast MTTKRP kernel instantiations.
#pragma once

#include <cuda.h>

#include <string>

#include "ntf_internal.h"

namespace ntfb {
namespace fast {

enum { kRow = 0, kCol = 1, kRowMma = 2, kColMma = 3 };
// DMMA consumer scratch per warp (doubles): rows x (8 * column fragments + 1)
constexpr int mma_scratch_doubles(int G, int B, int A) { return (32 / G) * A * (((G * B + 7) / 8) * 8 + 1); }

// Unit table: per unit, ints
//   [0] ROW: rho0 / COL: l0 (TMA coordinate along the reduction)
//   [1] ROW: l (TMA coordinate of the outer modes)
//   [2] row of the last varying mode's factor at k = 0 (slab offset included)
//   [3] valid k count, [4] rows before the wrap of that digit, [5] first k
//   after the wrap (>= KB when none)
//   [6, 6+kMaxBase) base rows at k = 0, [6+kMaxBase, 6+2*kMaxBase) after the wrap
constexpr int kMaxBase = 2;  // fast path: tensors of order <= 4 (others: generic kernel)
constexpr int kUnitInts = 6 + 2 * kMaxBase;
// prof slots: [0] producer total, [1] producer waiting for a free stage,
// [2] producer waiting for its copies, [3] consumer total, [4] consumer
// waiting for a full stage, [5] units, [6] globaltimer at kernel start,
// [7] globaltimer at the end of the consumer loop
constexpr int kProfSlots = 12;

struct Params {
  ModeView v;
  const DevFactors* F;
  double* partial;  // [ctas_per_mtile][I][r]
  // in-kernel slab reduction (ctas_per_mtile > 1): every CTA is resident
  // (cooperative launch); after a grid-wide arrival count each CTA sums its
  // share of the outputs over the slabs in slab order into `out`
  double* out;
  unsigned* counter;  // [arrivals, generation] of the grid barrier (zeroed once)
  long long units;  // per m-tile
  long long nbox_r; // ROW: rho boxes per l
  int kbox;         // reduction indices per unit
  int m_box, n_mbox, m_cta, ctas_per_mtile;
  // COL: shared-memory row pitch of a box (>= m_box); the DMMA consumers
  // read 4 k rows per half-warp, so the pitch is m_box + 4 doubles (32 B off
  // a bank period; the 4 extra rows are real neighbouring rows, unused)
  int m_pitch;
  int MW, KW, NP, stages, wld;  // consumer m-warps, k-warps, producer warps
  unsigned t_stage_bytes, w_stage_bytes, aq_stage_bytes, tx_bytes;
  const int* utab;       // units x kUnitInts (device)
  int nb;                // base factors per W row
  int bq[kMaxBase];      // their modes
  int qL, rowL_wrap;     // last varying mode; its row after a wrap
  unsigned long long* prof;  // optional per-CTA cycle counters (diagnostics), kProfSlots each
  // FP32 tensors with long reductions: every flush_units units (KW == 1 only)
  // each consumer lane adds its FP32 accumulators into its rows of the
  // CTA's FP64 slab and restarts them, so no FP32 sum runs over more than
  // flush_units * kbox terms (0: accumulate the whole range in registers)
  int flush_units;
  int pdl;  // host only: launch as a programmatic dependent
};
using LaunchFn = void (*)(const CUtensorMap& map, const Params& p, int grid, int threads, size_t smem,
                          cudaStream_t s);

// One register-blocking shape: G column groups x B columns, A rows per lane.
struct KernelCfg {
  int G, B, A;
  LaunchFn row, col;
  int cons = 4;
  LaunchFn row_mma = nullptr, col_mma = nullptr;  // FP64 DMMA consumers (null: none)  // target consumer warps per CTA (8: two per SM sub-partition)
};

// Thread cap of an instantiation: small accumulator tiles allow 16 warps
// (<= 128 registers), medium ones 12 warps (<= 168), large 8 (<= 255).
constexpr int max_threads(int A, int B) { return A * B <= 24 ? 512 : (A * B <= 50 ? 384 : 256); }
// FP32 accumulators take one register instead of two.
constexpr int max_threads_es(int A, int B, int es) { return es == 4 ? max_threads(A, (B + 1) / 2) : max_threads(A, B); }

// Picks the blocking for (dtype, rank, rows); false when no instantiation
// covers the rank.
bool lookup(int dtype, int rank, long long rows, KernelCfg* out);
bool lookup_f64(int rank, long long rows, KernelCfg* out);
bool lookup_f32(int rank, long long rows, KernelCfg* out);

}  // namespace fast

std::string fast_mttkrp_describe(const ModeView& v, int dtype, int sms);

}  // namespace ntfb
