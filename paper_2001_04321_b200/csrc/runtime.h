// Host runtime of libntf_b200.so: contexts, device tensors, the MTTKRP
// engine (kernel choice + deterministic reduction + NCCL exchange) and the
// GPU-resident HER / AO sessions behind ntf_her_run / ntf_ao_run.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "ntf_internal.h"

struct ntf_ctx;
struct ntf_tensor;

namespace ntfb {

// ---- datagen / metrics (datagen.cpp) ---------------------------------------
uint64_t stream_seed(uint64_t base, uint64_t stream);
void random_init(const int* shape, int order, int rank, uint64_t seed, double* out);
void generate(const int* shape, int order, int rank, double sigma, int ill, int collinear, uint64_t seed,
              int dtype, void* tensor, double* truth, long long slab_b = -1, long long slab_e = -1);
double factor_error(const double* est, const double* truth, const int* shape, int order, int rank);

// ---- NTFT container (tensor.cpp:56-96; ntft_io.cpp) -----------------------------
struct NtftHeader {
  int order = 0;
  int64_t shape[kMaxOrder] = {};
  int64_t payload_offset = 0;  // bytes
};
NtftHeader ntft_read_header(const std::string& path);
// TuckerFormat container "NTFK" (tucker.cpp:106-165)
struct NtfkHeader {
  int order = 0;
  int64_t shape[kMaxOrder] = {};  // full dims
  int64_t ranks[kMaxOrder] = {};  // core dims
  int64_t payload_offset = 0;
};
NtfkHeader ntfk_read_header(const std::string& path);
void ntfk_read(const std::string& path, double* core, double* bases);
void ntfk_write(const std::string& path, const double* core, const double* bases, int order, const int64_t* shape,
                const int64_t* ranks);
void ntft_write(const std::string& path, const void* data, int dtype, int order, const int64_t* shape);
void ntft_read_slab(const std::string& path, int dtype, int64_t slab_begin, int64_t slab_end, void* out);
void ntft_stream_to_device(const std::string& path, const NtftHeader& h, long long first, long long count,
                           int dtype, void* dst, cudaStream_t s);

// ---- device memory ------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n);
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// ---- collectives ---------------------------------------------------------------
struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int rank = 0, world = 1;
  // collectives run whenever a communicator exists -- also for a 1-rank
  // world created through ntf_ctx_create_dist (the NCCL path on one GPU)
  bool active() const { return nccl != nullptr; }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) const;
  void allgather(double* buf, size_t n_per_rank, cudaStream_t s) const;  // in place
  void allreduce_max(double* buf, size_t n, cudaStream_t s) const;
  ~Comm();
};

void slab_range(long long dim0, int rank, int world, long long* begin, long long* end);
// Keep freed DevBuf memory in the device's pool (called by context creation).
void retain_pool_memory(int device);

// ---- MTTKRP engine -------------------------------------------------------------
// Owns the split-K partial workspace; produces the FULL I_mode x r FP64
// MTTKRP (identical on every rank) in `out`.
class MttkrpEngine {
 public:
  MttkrpEngine(const ntf_ctx* ctx, const ntf_tensor* t, int rank, unsigned flags);
  // Enqueue on `s`. With kernel timing on, the main kernel of each call is
  // bracketed by events ev[0], ev[1] (may be null).
  void run(int mode, const DevFactors* dF, double* out, cudaStream_t s, cudaEvent_t ev0 = nullptr,
           cudaEvent_t ev1 = nullptr);
  int kernels_per_call(int mode) const;
  // Work enqueued after block `mode`'s NNLS kernel: with the overlapped
  // 3-way tree (below) the partial P_0 = T x_0 A_0 of block 2 after block
  // 1's NNLS, as a programmatic dependent launch (pdl) so it runs on the SMs
  // the NNLS leaves free. ev0/ev1 (timing) bracket it when launched.
  void after_block(int mode, const DevFactors* dF, cudaStream_t s, bool pdl, cudaEvent_t ev0 = nullptr,
                   cudaEvent_t ev1 = nullptr);
  bool overlap() const { return overlap_; }
  // timing slots that hold full tensor passes (Y_L at block 0; the second
  // pass: P_0 after block 1 when overlapped, else block h's)
  int second_pass_slot() const { return overlap_ ? 1 : split_; }
  ModeView view(int mode) const;
  std::string describe(int mode) const;
  // Dimension tree (NTF_RUN_DIMTREE, order >= 3, fast plans for the partials):
  // run(0) first forms Y_L = T x_h A_h .. x_{N-1} A_{N-1} and blocks 0..h-1
  // contract it; run(h) forms Y_R = T x_0 A_0 .. x_{h-1} A_{h-1} for blocks
  // h..N-1 (h = N-1: Y_R is block N-1's MTTKRP, computed directly).
  bool tree() const { return tree_; }

 private:
  const ntf_ctx* ctx_;
  const ntf_tensor* t_;
  int rank_;
  unsigned flags_;
  int segs_[kMaxOrder];
  DevBuf partial_;
  DevBuf gather_;                // padded rows for the mode-1 allgather
  DevBuf slab_meta_;             // begins/counts (long long) per rank
  DevBuf unit_tab_[kMaxOrder];   // fast-path unit tables (empty: generic kernel)
  long long maxrows_ = 0;
  bool tree_ = false;
  int split_ = 0;                // dimension-tree split h (blocks < h contract Y_L, the rest Y_R)
  ModeView ttm_view_{};          // Y_L view: (prod_{n<h} I_n) x I_h x ... x I_{N-1}
  DevBuf ttm_tab_, ybuf_;        // its unit table; Y_L (local rows x r, FP64)
  ModeView ttmr_view_{};         // Y_R view (h < N-1): I_0 x ... x I_{h-1} x (prod_{n>=h} I_n)
  DevBuf ttmr_tab_, yrbuf_;      // its unit table; Y_R (partial over the local slab, FP64)
  int order_ = 0;
  int last_mode_ = -1;           // previous run() block (a tree partial is reused only in sweep order)
  bool tree_mode(int mode) const {
    return tree_ && (mode < split_ || split_ < order_ - 1 || (overlap_ && mode == order_ - 1));
  }
  // Overlapped 3-way tree: blocks 0 and 1 contract Y_L = T x_2 A_2 as before;
  // block 2 contracts P_0 = T x_0 A_0 (rows (i1, i2)) with A_1. P_0 needs only
  // block 0's new factor, so its full tensor pass runs beside block 1's NNLS
  // (16 SMs) on the other SMs instead of on the critical path.
  bool overlap_ = false;
  bool p0_ready_ = false;
  int p0_sms_ = 0;
  ModeView p0_view_{};
  DevBuf p0_tab_, p0buf_;
  DevBuf counter_;               // arrival counter of the in-kernel split-K reduction
  int tree_chunks_[kMaxOrder] = {};
  int tree_tiles_max_ = 1;
  DevBuf tree_arrivals_;         // per-tile arrival counters of the tree kernel (self-resetting)
  TreeView tree_view(int mode) const;
  // TuckerProvider (t->kind == kTucker): P_l = U_l^T A_l, the core's MTTKRP
  // with P on the dense kernels, then U_mode times it (tucker.cpp:62-77)
  bool tucker_ = false;
  std::unique_ptr<MttkrpEngine> core_eng_;
  TuckerDev td_{};
  DevFactors core_hF_{};
  DevBuf proj_, core_dF_, mc_;
};

// Per-tensor workspace of the per-call provider entry points (ntf_mttkrp,
// ntf_mttkrp_all, ntf_objective): the engine (unit tables, partial slabs) and
// the factor buffers of the last (rank, flags), reused while they match.
struct CallCache {
  int rank = 0;
  unsigned flags = 0;
  std::unique_ptr<MttkrpEngine> eng;
  DevBuf fac, fac32, grams, dF, C, gscratch;
  DevFactors h{};
};

// ---- GPU-resident solver session ---------------------------------------------
class Session {
 public:
  Session(ntf_ctx* ctx, const ntf_tensor* t, int algo, const double* init, int rank, const ntf_ao_config& cfg,
          const ntf_her_params* params);
  ~Session();
  void step(int iters);
  void sync();
  int iterations();
  bool done();
  void factors(double* out);
  void trace(double* f0, ntf_trace_record* out, int cap, int* n);
  bool last_record(ntf_trace_record* out);  // the newest trace record (false: none yet)
  void check_error();  // throws the inner solver's failure (std::runtime_error in the reference)
  // after an iteration of an observed run: done flag, iteration count, the newest trace record and
  // (factors_out != null) the accepted factors, in one staged download and one synchronisation
  void snapshot(double* factors_out, ntf_trace_record* last, int* k, bool* done);
  // error check + accepted factors + trace in one staged download (the drivers' epilogue)
  void finish(double* out_factors, double* f0, ntf_trace_record* out, int cap, int* n);
  void set_kernel_timing(bool on);
  void kernel_times(double* ms_per_mode, int* launches, int* total_kernels);
  cudaStream_t stream() const { return stream_; }
  // timing slots (per-mode) holding the iteration's full tensor passes
  int pass_slots(int* slots) const {
    if (!eng_->tree()) {
      for (int i = 0; i < order_; ++i) slots[i] = i;
      return order_;
    }
    slots[0] = 0;
    slots[1] = eng_->second_pass_slot();
    return 2;
  }
  int order() const { return order_; }

 private:
  void enqueue_iteration(bool timed);
  void build_graph();

  ntf_ctx* ctx_;
  const ntf_tensor* t_;
  int algo_, rank_, order_;
  int rows_[kMaxOrder];
  long long total_factor_len_ = 0;
  ntf_ao_config cfg_;
  cudaStream_t stream_ = nullptr;
  std::unique_ptr<MttkrpEngine> eng_;
  DevFactors hF_{};
  DevBuf dF_, fac_, fac32_, grams_, C_, state_, trace_, scratch_, counter_;
  DevBuf solve_buf_, solve_work_;  // another inner solver: its result rows and per-row state
  DevBuf tall_work_;               // block update of factors beyond one cluster (kernels_nnls_tall.cu)
  DevBuf init_scratch_;            // partial Grams of the constructor's setup kernels (kept: no host sync there)
  int trace_cap_ = 0;
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
  bool graph_failed_ = false;
  bool timing_ = false;
  std::vector<cudaEvent_t> ev_;
  std::vector<int> ev_mode_;
  double kernel_ms_[kMaxOrder] = {};
  int kernel_n_[kMaxOrder] = {};
  int host_iters_ = 0;  // iterations enqueued
  int done_host_ = 0;  // host mirror of RunState::done
  bool collective_time_ = false;  // a communicator and a time budget
};

}  // namespace ntfb

// Opaque ABI objects.
struct ntf_ctx {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t setup = nullptr;  // table uploads of the engines (idle otherwise: never behind a tensor upload)
  // page-locked staging of a run's results (one download, one synchronisation); grows on demand
  mutable void* pinned = nullptr;
  mutable size_t pinned_bytes = 0;
  void* staging(size_t bytes) const;
  ntfb::Comm comm;
  ntfb::DevBuf scratch;  // small shared scratch (norms, standalone NNLS)
  ~ntf_ctx();
};

struct ntf_tensor {
  ntf_ctx* ctx = nullptr;
  int dtype = NTF_DTYPE_F64;
  int order = 0;
  long long shape[NTF_MAX_ORDER] = {};  // full shape
  long long row0 = 0, rows = 0;         // local mode-1 slab
  long long n_local = 0;
  ntfb::DevBuf data;
  ntfb::DevBuf nsq_dev;  // ||T||^2 (global, FP64) on the device
  mutable double nsq = 0.0;       // host copy, valid once nsq_valid (ntfb::host_nsq fetches it lazily)
  mutable bool nsq_valid = true;  // false after an asynchronous upload until the first host read
  cudaEvent_t ready = nullptr;    // recorded on ctx->stream after the upload and the ||T||^2 reduction
  bool rows_only = false;  // a caller-chosen row slab on a 1-GPU context (ntf_tensor_upload_rows)
  mutable std::unique_ptr<ntfb::CallCache> cache;
  // TuckerProvider (kind == 1): the core as a dense device tensor, the bases
  // (I_l x r_l row-major, concatenated); nsq = ||core||^2 (provider ctor,
  // tucker.cpp:94-95). `data` is empty: the full tensor never exists.
  int kind = 0;
  std::unique_ptr<ntf_tensor> core;
  ntfb::DevBuf bases;
  long long ranks[NTF_MAX_ORDER] = {};
  ~ntf_tensor();
};
