/*
 * ntf_b200.h — C ABI of the B200-native HER-AHALS hot path.
 *
 * This is the drop-in boundary for the reference toolkit's dense NTF inner
 * loop (arXiv 2001.04321 implementation, /root/reference/proj). Every entry
 * point below names the reference interface it replaces (file:line under
 * proj/). Conventions:
 *
 *   * plain pointers and sizes only; no C++ or torch types cross the ABI;
 *   * every call returns an int status (NTF_OK or an NTF_ERR_* code) and
 *     never throws; ntf_last_error() returns the message of the last failure
 *     on the calling thread. The codes mirror the reference's exception
 *     classes: std::invalid_argument -> NTF_ERR_INVALID_ARGUMENT,
 *     std::logic_error -> NTF_ERR_LOGIC, std::runtime_error -> NTF_ERR_RUNTIME;
 *   * tensors are row-major with the last index fastest (tensor.hpp:11-13);
 *   * factor models are row-major I_n x r matrices, modes concatenated in
 *     mode order (total sum_n I_n * r doubles);
 *   * a context is single-owner and not thread-safe;
 *   * host buffers are borrowed for the duration of a call only.
 *
 * There is no CPU fallback: a context cannot be created without a CUDA
 * device, and every compute entry point runs hand-written sm_100a kernels.
 */
#ifndef NTF_B200_H_
#define NTF_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTF_OK 0
#define NTF_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define NTF_ERR_LOGIC 2            /* std::logic_error (e.g. her.cpp:34-35)   */
#define NTF_ERR_RUNTIME 3          /* std::runtime_error                      */
#define NTF_ERR_CUDA 4             /* CUDA runtime/driver failure             */
#define NTF_ERR_NCCL 5             /* NCCL failure                            */
#define NTF_ERR_UNSUPPORTED 6      /* valid request this build does not serve */

#define NTF_MAX_ORDER 8

typedef enum { NTF_DTYPE_F64 = 0, NTF_DTYPE_F32 = 1 } ntf_dtype;

/* NnlsSolver (include/ntf/nnls.hpp:53). Only AHALS runs on the GPU path; the
 * others return NTF_ERR_UNSUPPORTED. */
typedef enum {
  NTF_SOLVER_AHALS = 0,
  NTF_SOLVER_ADMM = 1,
  NTF_SOLVER_NESTEROV = 2,
  NTF_SOLVER_PGD = 3,
  NTF_SOLVER_ACTIVE_SET = 4
} ntf_solver;

/* InnerStop (include/ntf/nnls.hpp:20-23). */
typedef struct {
  int max_iters;         /* default 50   */
  double rel_change_tol; /* default 1e-2 */
} ntf_inner_stop;

/* Performance options of the GPU drivers (no reference counterpart). */
/* The drivers use the dimension tree by default: two full tensor passes per
 * outer iteration (Y_L, Y_R) plus small contractions instead of N full
 * passes -- the same algorithm, only the summation order of the MTTKRPs
 * differs. NTF_RUN_DIMTREE is accepted for compatibility (it is the default);
 * NTF_RUN_DIRECT selects the reference's loop shape (one full MTTKRP pass per
 * block, kernels.cpp:161-191). */
#define NTF_RUN_DIMTREE 1u  /* default; kept for compatibility                */
#define NTF_RUN_NO_GRAPH 2u /* launch kernels directly instead of a CUDA graph */
#define NTF_RUN_GENERIC 4u  /* force the generic MTTKRP kernel (testing)     */
#define NTF_RUN_DIRECT 8u   /* N full MTTKRP passes per iteration (no tree)   */
#define NTF_RUN_NO_OVERLAP 16u /* 3-way: keep block N-1's pass on the critical
                                  path instead of beside block 1's NNLS      */

/* AoConfig (include/ntf/ao.hpp:15-24). `ground_truth` is a concatenated
 * factor model (same shape and rank as the init) and is required when
 * record_factor_error is set. */
typedef struct {
  int solver;
  ntf_inner_stop inner_stop;
  int max_outer_iters; /* 0 = no iteration cap */
  double max_time_s;   /* 0 = no time cap      */
  int record_factor_error;
  const double* ground_truth;
  unsigned flags; /* NTF_RUN_* */
} ntf_ao_config;

/* HerParams (include/ntf/her.hpp:13-21). */
typedef struct {
  double beta0;     /* 0.5  */
  double gamma;     /* 1.05 */
  double gamma_bar; /* 1.01 */
  double eta;       /* 1.5  */
} ntf_her_params;

/* TraceRecord (include/ntf/trace.hpp:11-18); has_* flags encode the
 * std::optional fields. */
typedef struct {
  int iter;
  int has_e;
  int has_restarted;
  int restarted;
  int has_beta;
  int inner_sweeps; /* AHALS passes summed over the modes of the iteration */
  double time_s;
  double f;
  double e;
  double beta;
} ntf_trace_record;

/* HerIterationInfo (include/ntf/her.hpp:50-57). Factor pointers are host
 * copies valid during the callback only. */
typedef struct {
  int iter;
  double f_hat;
  int restarted;
  double beta_used;
  const double* factors;
  const double* hat_factors;
} ntf_her_iteration_info;
typedef void (*ntf_her_observer)(const ntf_her_iteration_info* info, void* user);

typedef struct ntf_ctx ntf_ctx;
typedef struct ntf_tensor ntf_tensor;
typedef struct ntf_session ntf_session;

/* ---- errors / defaults ---------------------------------------------------- */
const char* ntf_version(void);
int ntf_last_error(char* buf, size_t n);
void ntf_her_params_default(ntf_her_params* p);
void ntf_ao_config_default(ntf_ao_config* c);
/* HerParams::validate (src/her.cpp:10-14). */
int ntf_her_params_validate(const ntf_her_params* p);
/* AoConfig::validate (src/ao.cpp:10-15). */
int ntf_ao_config_validate(const ntf_ao_config* c);

/* ---- synthetic data (src/datagen.cpp:13-80; host, bit-exact) ------------- */
/* stream_seed (datagen.cpp:30-35). */
uint64_t ntf_stream_seed(uint64_t base, uint64_t stream);
/* random_init (datagen.cpp:72-80). out: sum(shape)*rank doubles. */
int ntf_random_init(const int* shape, int order, int rank, uint64_t seed, double* out);
/* generate (datagen.cpp:48-70). `collinear` selects the build's BASELINE
 * config-4 factor rule. tensor_out: prod(shape) values of `dtype` (F32 is
 * the FP64 instance rounded to nearest); truth_out: sum(shape)*rank doubles. */
int ntf_generate(const int* shape, int order, int rank, double sigma, int ill_conditioned,
                 int collinear, uint64_t seed, int dtype, void* tensor_out, double* truth_out);
/* generate restricted to the mode-1 slab [slab_begin, slab_end) (the rows a
 * rank of a sharded context owns, ntf_slab_range): tensor_out receives
 * (slab_end - slab_begin) * prod(shape[1:]) values, bit-identical to that
 * slab of ntf_generate's tensor (the noise stream is entered at the slab's
 * first entry); truth_out is the full truth. No reference counterpart: the
 * reference generates whole instances (datagen.cpp:48-70). */
int ntf_generate_slab(const int* shape, int order, int rank, double sigma, int ill_conditioned,
                      int collinear, uint64_t seed, int dtype, int64_t slab_begin, int64_t slab_end,
                      void* tensor_out, double* truth_out);
/* NTFT container on the host (tensor.cpp:56-96; README "File formats").
 * info: order and dims (shape has room for 8). read: rows [slab_begin,
 * slab_end) of mode 1 (-1, -1: all) as dtype (FP32 = round to nearest of the
 * FP64 payload). write = DenseTensor::save (FP32 data is written exactly
 * upcast). Errors as DenseTensor::load: NTF_ERR_RUNTIME with the same text
 * ("cannot open", "not a tensor container", "unsupported version",
 * "bad order", "truncated payload"). */
int ntf_ntft_info(const char* path, int* order, int64_t* shape);
int ntf_ntft_read(const char* path, int dtype, int64_t slab_begin, int64_t slab_end, void* out);
int ntf_ntft_write(const char* path, const void* data, int dtype, int order, const int64_t* shape);
/* factor_error (src/metrics.cpp:79-111). */
int ntf_factor_error(const double* est, const double* truth, const int* shape, int order, int rank,
                     double* out);

/* ---- context ---------------------------------------------------------------- */
int ntf_device_count(int* n);
/* One GPU; fails with NTF_ERR_CUDA when no device is present. */
int ntf_ctx_create(int device, ntf_ctx** out);
/* NCCL unique id for ntf_ctx_create_dist (128 bytes, rank 0 creates it). */
int ntf_nccl_unique_id(unsigned char out[128]);
/* One rank of a world of `world` GPUs on one node; the mode-1 slab of the
 * tensor lives on this rank. world = 1 creates a one-rank
 * communicator: the drivers then run the sharded code path (allgather +
 * row compaction for mode 1, allreduce for the other modes, collective time
 * budget) on one GPU. */
int ntf_ctx_create_dist(int device, int rank, int world, const unsigned char id[128], ntf_ctx** out);
int ntf_ctx_info(const ntf_ctx* ctx, int* device, int* rank, int* world);
int ntf_ctx_destroy(ntf_ctx* ctx);

/* ---- dense tensor provider (include/ntf/provider.hpp:14-34) --------------- */
/* Rows [begin, end) of mode 1 owned by `rank` of `world` (contiguous slabs;
 * the first I_1 % world ranks hold one extra row). */
int ntf_slab_range(int64_t dim0, int rank, int world, int64_t* begin, int64_t* end);
/* DenseTensor -> device. `shape` is the FULL tensor shape; `host` holds this
 * rank's mode-1 slab (the whole tensor on a 1-GPU context). Computes ||T||^2
 * once in FP64 (DenseProvider ctor, provider.cpp:7; tensor.cpp:43-47). */
int ntf_tensor_upload(ntf_ctx* ctx, const void* host, int dtype, int order, const int64_t* shape,
                      ntf_tensor** out);
/* The same without blocking the host: returns once the copy and the ||T||^2
 * reduction are ENQUEUED on the context's stream, so the caller's next calls
 * (ntf_her_run / ntf_ao_run / ntf_session_create: engine tables, buffers,
 * first launches, CUDA-graph capture) overlap the transfer; every consumer is
 * ordered after it on the device. Contract: `host` must stay valid and
 * unmodified until ntf_tensor_wait(t) returns or a later call on this handle
 * has returned tensor-derived data to the host (ntf_tensor_norm_sq, ntf_mttkrp*,
 * a driver run). With pageable memory the CUDA runtime stages the copy
 * synchronously and nothing is gained; use pinned memory (cudaHostAlloc /
 * cudaHostRegister). DenseProvider takes its tensor by reference too
 * (provider.hpp:24-33: "does not own it"). */
int ntf_tensor_upload_async(ntf_ctx* ctx, const void* host, int dtype, int order, const int64_t* shape,
                            ntf_tensor** out);
/* Blocks until the upload of `t` (and its ||T||^2) has completed. */
int ntf_tensor_wait(const ntf_tensor* t);
/* Page-locked host memory for ntf_tensor_upload_async (cudaHostAlloc /
 * cudaFreeHost), so a host program needs no CUDA headers of its own. */
int ntf_pinned_alloc(size_t bytes, void** out);
int ntf_pinned_free(void* p);
/* Same, from a device buffer of this context's GPU (copied). Ordering: the
 * copy runs on the context's own stream, so the caller's producer work must
 * be complete -- this entry point synchronises the device before copying.
 * ntf_tensor_upload_device_async instead orders the copy after all work
 * enqueued so far on `caller_stream` (a cudaStream_t as void*, NULL = the
 * legacy default stream) without blocking the host. */
int ntf_tensor_upload_device(ntf_ctx* ctx, const void* dev, int dtype, int order,
                             const int64_t* shape, ntf_tensor** out);
int ntf_tensor_upload_device_async(ntf_ctx* ctx, const void* dev, int dtype, int order,
                                   const int64_t* shape, void* caller_stream, ntf_tensor** out);
/* A caller-chosen mode-1 row slab [row_begin, row_end) of a tensor of FULL
 * shape `shape` on a 1-GPU context (`host` holds only those rows). This is
 * the per-rank piece of the sharded path made callable on
 * one GPU: ntf_mttkrp / ntf_mttkrp_all then return this slab's
 * contribution -- for mode 1 the slab's rows (the other rows zero), for the
 * other modes the slab's partial I_n x r sum -- so the MTTKRP of the whole
 * tensor is the sum over a row partition. ||T||^2 is the slab's. Driver
 * runs (her/ao/session) reject such a tensor. */
int ntf_tensor_upload_rows(ntf_ctx* ctx, const void* host, int dtype, int order, const int64_t* shape,
                           int64_t row_begin, int64_t row_end, ntf_tensor** out);
/* ObjectiveProvider::shape / norm_sq (provider.hpp:16-17). */
int ntf_tensor_shape(const ntf_tensor* t, int* order, int64_t* shape);
int ntf_tensor_norm_sq(const ntf_tensor* t, double* out);
int ntf_tensor_destroy(ntf_tensor* t);
/* DenseTensor::load from the reference's binary container (tensor.cpp:73-96,
 * magic "NTFT", u32 version 1, u32 order, u64 dims, FP64 payload): this
 * rank's mode-1 slab is read (one seek) and streamed to the device through
 * pinned staging buffers, rounded to FP32 when dtype is NTF_DTYPE_F32. */
int ntf_tensor_upload_ntft(ntf_ctx* ctx, const char* path, int dtype, ntf_tensor** out);
/* TuckerProvider (include/ntf/tucker.hpp:60-73, src/tucker.cpp:62-77, 94-95):
 * a TuckerFormat -- the dense core (order N, dims core_shape, row-major) and
 * one basis per mode, U_l (full_shape[l] x core_shape[l], row-major,
 * orthonormal columns), concatenated in mode order -- as a provider handle.
 * ntf_mttkrp / ntf_mttkrp_all / ntf_objective / the drivers accept it; the
 * MTTKRP runs in the compressed space (P_l = U_l^T A_l, the core's MTTKRP
 * with P on the dense kernels, then U_mode times it) and ||T||^2 is
 * ||core||^2. Validation as TuckerFormat::validate (tucker.cpp:16-26):
 * NTF_ERR_INVALID_ARGUMENT "basis columns are not orthonormal" (|U^T U - I|
 * > 1e-10), "basis column count does not match the core shape". One GPU
 * (NTF_ERR_UNSUPPORTED on an NCCL context). */
int ntf_tucker_upload(ntf_ctx* ctx, const double* core, int order, const int64_t* core_shape,
                      const double* bases, const int64_t* full_shape, ntf_tensor** out);
/* TuckerFormat::save / load (tucker.cpp:106-165): container "NTFK" (magic,
 * u32 version 1, u32 order, u64 full dims, u64 core dims, FP64 core, the
 * bases row-major in mode order). info: order and both shapes; read: core
 * and concatenated bases into caller buffers. Errors as TuckerFormat::load
 * (NTF_ERR_RUNTIME: "cannot open", "not a tucker container", "unsupported
 * version", "bad order", "truncated payload"). */
int ntf_ntfk_info(const char* path, int* order, int64_t* full_shape, int64_t* core_shape);
int ntf_ntfk_read(const char* path, double* core, double* bases);
int ntf_ntfk_write(const char* path, const double* core, const double* bases, int order,
                   const int64_t* full_shape, const int64_t* core_shape);
int ntf_tensor_upload_ntfk(ntf_ctx* ctx, const char* path, ntf_tensor** out);
/* ObjectiveProvider::mttkrp (provider.hpp:18; kernels.cpp:161-191): out is
 * the I_mode x rank MTTKRP (row-major, FP64), identical on every rank. The
 * tensor keeps the kernel plan and device workspaces of its last (rank)
 * between calls, so a provider loop pays the factor upload and one kernel
 * per call. */
int ntf_mttkrp(ntf_ctx* ctx, const ntf_tensor* t, const double* factors, int rank, int mode,
               double* out);
/* Every mode's MTTKRP at one fixed model, in sweep order 0..N-1, written
 * concatenated (mode n at offset sum_{m<n} I_m * rank). flags: 0 = the
 * dimension tree the drivers use (two full passes + contractions),
 * NTF_RUN_DIRECT = N full passes, NTF_RUN_GENERIC = the generic kernel.
 * Repeated calls on one tensor reuse its plan and device workspaces. */
int ntf_mttkrp_all(ntf_ctx* ctx, const ntf_tensor* t, const double* factors, int rank, unsigned flags,
                   double* out);
/* objective(t, m, cache, pivot) (kernels.cpp:305-311): one MTTKRP at `pivot`
 * (-1 = last mode) plus the cheap objective. */
int ntf_objective(ntf_ctx* ctx, const ntf_tensor* t, const double* factors, int rank, int pivot,
                  double* out);

/* Diagnostics: the kernel plan ntf_mttkrp uses for (rank, mode) on this
 * tensor ("generic" or the fast-path blocking), NUL-terminated into buf. */
int ntf_mttkrp_plan(ntf_ctx* ctx, const ntf_tensor* t, int rank, int mode, char* buf, size_t n);

/* ---- inner solver (include/ntf/nnls.hpp:12-55) --------------------------- */
/* solve_nnls(solver, {gram, target, init}, stop) on the GPU. gram: r x r,
 * target/init/out: rows x r (row-major). `sweeps` (optional) receives the
 * number of HALS passes run. */
int ntf_solve_nnls(ntf_ctx* ctx, int solver, const double* gram, const double* target,
                   const double* init, int rows, int rank, const ntf_inner_stop* stop, double* out,
                   int* sweeps);

/* ---- drivers (src/her.cpp:40-110, src/ao.cpp:17-52) ---------------------- */
/* her_run: returns the accepted model in out_factors, f0 and up to
 * trace_cap records; n_records receives the number of outer iterations. */
int ntf_her_run(ntf_ctx* ctx, const ntf_tensor* t, const double* init, int rank,
                const ntf_ao_config* cfg, const ntf_her_params* params, ntf_her_observer observer,
                void* user, double* out_factors, double* f0, ntf_trace_record* trace, int trace_cap,
                int* n_records);
int ntf_ao_run(ntf_ctx* ctx, const ntf_tensor* t, const double* init, int rank,
               const ntf_ao_config* cfg, double* out_factors, double* f0, ntf_trace_record* trace,
               int trace_cap, int* n_records);

/* ---- stepping sessions (benchmarking / incremental use) ------------------ */
/* A session holds a GPU-resident her_run (algo 0) or ao_run (algo 1) state
 * after f0 has been computed. ntf_session_step enqueues `iters` outer
 * iterations on the session stream without synchronising. */
int ntf_session_create(ntf_ctx* ctx, const ntf_tensor* t, int algo, const double* init, int rank,
                       const ntf_ao_config* cfg, const ntf_her_params* params, ntf_session** out);
int ntf_session_step(ntf_session* s, int iters);
int ntf_session_sync(ntf_session* s);
/* The cudaStream_t the session launches on (as void*). */
void* ntf_session_stream(ntf_session* s);
int ntf_session_iterations(ntf_session* s, int* done);
int ntf_session_factors(ntf_session* s, double* out);
int ntf_session_trace(ntf_session* s, double* f0, ntf_trace_record* trace, int cap, int* n);
/* Per-mode MTTKRP kernel timing (CUDA events on the session stream),
 * accumulated over steps taken with timing on (disables graph replay). */
int ntf_session_set_kernel_timing(ntf_session* s, int on);
int ntf_session_kernel_times(ntf_session* s, double* ms_per_mode, int* launches_per_mode,
                             int* kernel_launches_total);
/* Which per-mode timing slots of ntf_session_kernel_times hold the outer
 * iteration's full tensor passes (the rest are dimension-tree contractions):
 * slots[0..n), n <= order. */
int ntf_session_pass_slots(ntf_session* s, int* slots, int* n);
int ntf_session_destroy(ntf_session* s);

#ifdef __cplusplus
}
#endif

#endif /* NTF_B200_H_ */
