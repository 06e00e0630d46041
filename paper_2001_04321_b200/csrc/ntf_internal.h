// Internal declarations shared by the CUDA kernels and the host runtime of
// libntf_b200.so. Nothing here crosses the C ABI (include/ntf_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only; a no-op unless a profiler injects itself

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/ntf_b200.h"

namespace ntfb {

// NVTX range for the host-side phases (per-mode / per-kernel
// ranges for ncu / Nsight timelines): "ntf:upload", "ntf:session", "ntf:mttkrp m",
// "ntf:nnls m", "ntf:graph", "ntf:run".
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* name, int mode) {
    char buf[48];
    snprintf(buf, sizeof buf, "%s %d", name, mode);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace ntfb

namespace ntfb {

constexpr int kMaxOrder = NTF_MAX_ORDER;
constexpr int kMaxRank = 64;  // largest r served by the fused NNLS kernels
constexpr int kMaxTallRank = 128;  // largest r of the grid-kernel block update (kernels_nnls_tall.cu)
constexpr int kMaxNnlsRows = 16 * 256;  // largest factor height it serves (one 16-CTA cluster)
constexpr int kNnlsReserveSms = 16;      // SMs a concurrent pass leaves to the NNLS cluster

// ---- errors ----------------------------------------------------------------
// Host code throws these; the C ABI maps them to status codes.
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct LogicError : std::logic_error {
  using std::logic_error::logic_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define NTF_CUDA(x)                                                   \
  do {                                                                \
    cudaError_t e__ = (x);                                            \
    if (e__ != cudaSuccess) ::ntfb::cuda_fail(e__, #x, __FILE__, __LINE__); \
  } while (0)

// ---- device-resident solver state ------------------------------------------
// Two FP64 buffers per mode. Role X_i = x[i][sel[i]] holds the accepted
// factor (== the extrapolated twin at the start of an outer iteration);
// role S_i = x[i][sel[i]^1] receives the NNLS solution. A restart flips sel
// (X := S for every mode) instead of copying (her.cpp:76-80). gram[i][b] is
// always the Gram of buffer x[i][b]; x32 are FP32 mirrors for FP32 tensors.
struct DevFactors {
  double* x[kMaxOrder][2];
  float* x32[kMaxOrder][2];
  double* gram[kMaxOrder][2];
  int sel[kMaxOrder];
  int rows[kMaxOrder];
  int order, rank;
};

// HER/AO scalars (her.hpp:25-31) plus run bookkeeping, all on the device.
struct RunState {
  double beta, beta_bar, f_prev, f_last, f0, nsq;
  double beta0, gamma, gamma_bar, eta;
  double max_time_s;
  double tol;
  unsigned long long t_start_ns;
  int k, done, max_iters, inner_max_iters;
  int algo;  // 0 = HER, 1 = AO
  int last_sweeps[kMaxOrder];
  // multi-GPU time budget: the last-mode kernel only records its elapsed
  // time; the ranks all-reduce (max) it and apply the budget together
  // (launch_apply_time_budget), so every rank stops at the same iteration
  int collective_time;
  double elapsed_s;
  int error;  // first inner-solver failure (solver_error_message), 0 = none
};

struct TraceEntry {
  double f, beta, time_s;
  int restarted, sweeps;
};

// Mode view (L, I, R) of the LOCAL slab (kernels.cpp:10-27); dims[0] is the
// local slab height and row0 its offset in the full mode-1 factor.
struct ModeView {
  int order, mode, rank;
  int dims[kMaxOrder];
  long long L, I, R;
  long long row0;
  // dimension-tree views whose dim 0 is a merged row index: view dims q >= 1
  // contract with factor q + fshift (Y_L = T x_h A_h ... x_{N-1} A_{N-1})
  int fshift = 0;
};

// Dimension tree: a partial Y_L (modes 0..h-1 of T, r trailing) or Y_R
// (modes h..N-1) viewed around block `mode` as (L, I, R, r); see
// kernels_tree.cu.
struct TreeView {
  int order, mode, rank;  // order = number of tensor modes in the partial
  int dims[kMaxOrder];
  long long L, I, R;
  long long row0;
  int foff = 0;  // view dim j contracts with factor j + foff (Y_R of a split tree)
};
int tree_chunks(const TreeView& v, int sms);
int tree_tiles(const TreeView& v);
// out (I x r) = block `mode`'s MTTKRP from Y; partial holds chunks * I * r doubles.
void launch_tree_mttkrp(const double* Y, const TreeView& v, const DevFactors* dF, double* partial, int chunks,
                        unsigned* arrivals, double* out, cudaStream_t s);

// TuckerProvider (tucker.hpp:60-73) on the device: the bases U_l (I_l x r_l,
// row-major, concatenated) and the projected factors P_l = U_l^T A_l
// (r_l x r, concatenated) of one MTTKRP (kernels_tucker.cu).
struct TuckerDev {
  const double* bases;
  double* proj;
  long long base_off[kMaxOrder], proj_off[kMaxOrder];
  int rows[kMaxOrder], ranks[kMaxOrder];
};
// P_l for every l != skip from the X-role factors of dF
void launch_tucker_project(const TuckerDev& td, const DevFactors* dF, int skip, int order, int rank, cudaStream_t s);
// out (I_mode x r) = U_mode * Mc (r_mode x r)
void launch_tucker_expand(const TuckerDev& td, int mode, int rank, const double* Mc, double* out, cudaStream_t s);

// ---- kernel launchers (CUDA translation units) ------------------------------
struct MttkrpPlan;

// Generic MTTKRP (any shape / rank): partial[seg][I][r] in FP64.
void launch_mttkrp_generic(const void* t, int dtype, const ModeView& v, const DevFactors* dF,
                           double* partial, int segs, cudaStream_t s);
// Deterministic fixed-order sum of `segs` partial slabs of n values.
void launch_reduce_partials(const double* partial, int segs, long long n, double* out, cudaStream_t s);
// Fixed-order FP64 sum of squares of a device array.
void launch_norm_sq(const void* t, int dtype, long long n, double* scratch, int scratch_len, double* out,
                    cudaStream_t s);
// gram[i][b] = x[i][b]^T x[i][b] for every mode (b = sel) and FP32 mirrors.
void launch_init_factors(DevFactors* dF, const DevFactors& hF, double* scratch, size_t scratch_len, cudaStream_t s);
size_t init_factors_scratch(const DevFactors& hF);  // doubles of scratch launch_init_factors wants
// cheap objective at pivot: 0.5 nsq - <A,C> + 0.5 <A^T A, G>, G = hadamard of
// the X-role Grams except `pivot` (kernels.cpp:298-311). Writes *out.
void launch_objective(const DevFactors* dF, int order, int rank, int pivot, int rows, const double* C,
                      const double* nsq_dev, double* out, cudaStream_t s);
void launch_stamp_start(RunState* st, cudaStream_t s);
// done := elapsed_s >= max_time_s (after the ranks' max-allreduce of elapsed_s)
void launch_apply_time_budget(RunState* st, cudaStream_t s);
void launch_compact_rows(const double* gathered, long long maxrows, const long long* begins,
                         const long long* counts, int world, int rank_cols, double* out, cudaStream_t s);

// Fused AHALS + extrapolate/project + Grams + objective/decision kernel.
struct NnlsLaunch {
  int mode, order, rows, rank;
  int role;  // 0 = HER driver, 1 = AO driver, 2 = standalone solve
  int last;  // mode == order-1 in a driver
  const double* C;
  DevFactors* F;      // drivers
  RunState* st;       // drivers
  TraceEntry* trace;  // drivers
  // standalone solve
  const double* gram_in;
  const double* w0;
  double* w_out;
  int* sweeps_out;
  int max_iters;
  double tol;
  double* scratch;  // >= grid * (kMaxRank*kMaxRank + 64) doubles
  unsigned int* counter;
  // drivers: the buffers behind F (fixed for a session), so the kernel only
  // loads the role bits sel[] from device memory (hF: host copy of *F)
  const DevFactors* hF;
  DevFactors bufs;
  int has_bufs;
  // drivers with another inner solver: the block's rows come from w0 (the
  // solver's result) and no AHALS sweep runs; the kernel only extrapolates,
  // writes, forms the Grams and (last mode) decides
  int zero_sweeps;
  int solver;        // NTF_SOLVER_* (launch_nnls_solver)
  double* work;      // solver: >= 3 * rows * rank doubles of per-row state
  int* error;        // solver: first failure code (0 = none), see solver_error_message
  // workspace of the tall-factor path (kernels_nnls_tall.cu): >= nnls_tall_workspace(rows, rank)
  // doubles, or null (factors beyond one cluster are then refused)
  double* tall;
};
void launch_nnls(const NnlsLaunch& a, cudaStream_t s);
// Factors too tall for one cluster (or NTF_NNLS_TALL=1): the same update as plain grid kernels.
size_t nnls_tall_workspace(int rows, int rank);
void launch_nnls_tall(const NnlsLaunch& a, cudaStream_t s, int max_iters_host);
bool nnls_needs_tall(int rows, int rank);
// PGD / Nesterov / ADMM / active-set (nnls.cpp:51-211) on one thread-block
// cluster: reads G (Hadamard of the other modes' X-role Grams, or gram_in),
// C and the warm start (X, or w0), writes the result rows to w_out.
void launch_nnls_solver(const NnlsLaunch& a, cudaStream_t s);
// message of a solver failure code (the reference's std::runtime_error texts)
const char* solver_error_message(int code);
// diagnostics: {sweep-loop cycles, reduction cycles, sweeps, calls} of CTA 0
void nnls_prof_read(unsigned long long out[8 + 384], bool reset);

int device_sm_count();
// Small host -> device upload carried in kernel parameters (no copy engine: it does not queue
// behind a large transfer in flight); asynchronous on `s`, the host buffer may be reused at once.
void dev_upload(void* dst, const void* src, size_t bytes, cudaStream_t s);
void dev_zero(void* dst, size_t bytes, cudaStream_t s);  // zero fill by a kernel (same reason)

}  // namespace ntfb
