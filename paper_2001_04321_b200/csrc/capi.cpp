// extern "C" boundary (include/ntf_b200.h). Every entry point catches all
// exceptions and maps them to status codes; messages go to a thread-local
// buffer read by ntf_last_error().
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <cstring>
#include <string>
#include <vector>

#include "runtime.h"

using namespace ntfb;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return NTF_OK;
  } catch (const InvalidArgument& e) {
    g_last_error = e.what();
    return NTF_ERR_INVALID_ARGUMENT;
  } catch (const LogicError& e) {
    g_last_error = e.what();
    return NTF_ERR_LOGIC;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return NTF_ERR_CUDA;
  } catch (const NcclError& e) {
    g_last_error = e.what();
    return NTF_ERR_NCCL;
  } catch (const Unsupported& e) {
    g_last_error = e.what();
    return NTF_ERR_UNSUPPORTED;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return NTF_ERR_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return NTF_ERR_LOGIC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return NTF_ERR_RUNTIME;
  } catch (...) {
    g_last_error = "unknown error";
    return NTF_ERR_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw InvalidArgument(std::string(what) + " must not be null");
}

// HerParams::validate (her.cpp:10-14).
void validate_params(const ntf_her_params& p) {
  if (!(p.beta0 > 0.0 && p.beta0 < 1.0)) throw InvalidArgument("beta0 must lie in (0,1)");
  if (!(1.0 < p.gamma_bar && p.gamma_bar <= p.gamma && p.gamma <= p.eta))
    throw InvalidArgument("parameters must satisfy 1 < gamma_bar <= gamma <= eta");
}

// AoConfig::validate (ao.cpp:10-15).
void validate_cfg(const ntf_ao_config& c) {
  if (c.max_outer_iters <= 0 && c.max_time_s <= 0.0) throw InvalidArgument("set an iteration or time budget");
  if (c.record_factor_error && c.ground_truth == nullptr)
    throw InvalidArgument("factor error recording needs ground truth factors");
}

std::vector<int> int_shape(const ntf_tensor* t) {
  std::vector<int> s(static_cast<size_t>(t->order));
  for (int i = 0; i < t->order; ++i) s[size_t(i)] = int(t->shape[i]);
  return s;
}

long long model_len(const ntf_tensor* t, int rank) {
  long long n = 0;
  for (int i = 0; i < t->order; ++i) n += t->shape[i] * rank;
  return n;
}

// check_run_inputs (driver_common.hpp:14-25).
void check_run_inputs(const ntf_tensor* t, const double* init, int rank, const ntf_ao_config& cfg) {
  validate_cfg(cfg);
  if (rank < 1) throw InvalidArgument("rank must be >= 1");
  const long long n = model_len(t, rank);
  for (long long e = 0; e < n; ++e)
    if (init[e] < 0.0) throw InvalidArgument("initial model must be entrywise nonnegative");
  if (cfg.solver < NTF_SOLVER_AHALS || cfg.solver > NTF_SOLVER_ACTIVE_SET) throw LogicError("unknown solver");
  if (cfg.solver == NTF_SOLVER_ACTIVE_SET && rank > 32)
    throw Unsupported("the GPU active-set solver serves ranks up to 32");
  if (cfg.inner_stop.max_iters < 0) throw InvalidArgument("inner max_iters must be >= 0");
  // limits are refused up front, before the session is built. AHALS serves
  // any factor height (taller than one cluster: the grid-kernel path of
  // kernels_nnls_tall.cu); the other inner solvers keep a factor on one
  // thread-block cluster
  if (rank > kMaxTallRank) throw Unsupported("rank above the NNLS kernels' limit (128)");
  if (cfg.solver != NTF_SOLVER_AHALS && rank > kMaxRank)
    throw Unsupported("the PGD / Nesterov / ADMM / active-set kernels serve ranks up to 64 (AHALS: 128)");
  if (cfg.solver != NTF_SOLVER_AHALS)
    for (int i = 0; i < t->order; ++i)
      if (t->shape[i] > kMaxNnlsRows)
        throw Unsupported("mode " + std::to_string(i) + " has " + std::to_string(t->shape[i]) +
                          " rows; the " + "PGD / Nesterov / ADMM / active-set kernels hold at most " +
                          std::to_string(kMaxNnlsRows) + " rows per factor (AHALS has no such limit)");
}

// The tensor handle of this rank's mode-1 slab; `fill` copies the slab's
// n_local values into t->data on ctx->stream. ||T||^2 follows (FP64,
// all-reduced over the ranks).
// rows = {begin, end} picks a caller-chosen mode-1 slab on a 1-GPU context
// (ntf_tensor_upload_rows); {-1, -1} = this rank's slab_range.
// The host value of ||T||^2: fetched on first use after an asynchronous upload.
double host_nsq(const ntf_tensor* t) {
  if (!t->nsq_valid) {
    NTF_CUDA(cudaSetDevice(t->ctx->device));
    NTF_CUDA(cudaMemcpyAsync(&t->nsq, t->nsq_dev.p, sizeof(double), cudaMemcpyDeviceToHost, t->ctx->stream));
    NTF_CUDA(cudaStreamSynchronize(t->ctx->stream));
    t->nsq_valid = true;
  }
  return t->nsq;
}

// async: return once the copy and the ||T||^2 reduction are enqueued on
// ctx->stream (ntf_tensor_upload_async); `ready` marks their completion for
// consumers on other streams (Session).
template <typename Fill>
ntf_tensor* make_tensor_with(ntf_ctx* ctx, int dtype, int order, const int64_t* shape, Fill&& fill,
                             long long rows_b = -1, long long rows_e = -1, bool async = false) {
  need(ctx, "ctx");
  need(shape, "shape");
  if (dtype != NTF_DTYPE_F64 && dtype != NTF_DTYPE_F32) throw InvalidArgument("unknown dtype");
  if (order < 1 || order > NTF_MAX_ORDER) throw InvalidArgument("tensor order must lie in 1..8");
  NvtxRange nvtx("ntf:upload");
  auto* t = new ntf_tensor();
  try {
    t->ctx = ctx;
    t->dtype = dtype;
    t->order = order;
    for (int i = 0; i < order; ++i) {
      if (shape[i] < 1 || shape[i] > (1LL << 31) - 1) throw InvalidArgument("tensor dimensions must be positive");
      t->shape[i] = shape[i];
    }
    long long b = 0, e = shape[0];
    if (rows_b >= 0) {
      if (ctx->comm.active()) throw InvalidArgument("explicit row slabs need a 1-GPU context without NCCL");
      if (rows_e <= rows_b || rows_e > shape[0]) throw InvalidArgument("row slab outside the first mode");
      b = rows_b;
      e = rows_e;
      t->rows_only = (b != 0 || e != shape[0]);
    } else {
      slab_range(shape[0], ctx->comm.rank, ctx->comm.world, &b, &e);
    }
    t->row0 = b;
    t->rows = e - b;
    if (t->rows < 1) throw InvalidArgument("every rank needs at least one mode-1 row");
    t->n_local = t->rows;
    for (int i = 1; i < order; ++i) t->n_local *= shape[i];
    const size_t es = dtype == NTF_DTYPE_F32 ? 4 : 8;
    NTF_CUDA(cudaSetDevice(ctx->device));
    t->data = DevBuf(size_t(t->n_local) * es);
    fill(t);
    t->nsq_dev = DevBuf(sizeof(double));
    launch_norm_sq(t->data.p, dtype, t->n_local, ctx->scratch.as<double>(), int(ctx->scratch.bytes / 8),
                   t->nsq_dev.as<double>(), ctx->stream);
    ctx->comm.allreduce_sum(t->nsq_dev.as<double>(), 1, ctx->stream);
    NTF_CUDA(cudaEventCreateWithFlags(&t->ready, cudaEventDisableTiming));
    NTF_CUDA(cudaEventRecord(t->ready, ctx->stream));
    if (async) {
      t->nsq_valid = false;
    } else {
      NTF_CUDA(cudaMemcpyAsync(&t->nsq, t->nsq_dev.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      NTF_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

ntf_tensor* make_tensor(ntf_ctx* ctx, const void* src, bool src_on_device, int dtype, int order,
                        const int64_t* shape, long long rows_b = -1, long long rows_e = -1, bool async = false) {
  need(src, "tensor data");
  return make_tensor_with(
      ctx, dtype, order, shape,
      [&](ntf_tensor* t) {
        const size_t es = dtype == NTF_DTYPE_F32 ? 4 : 8;
        NTF_CUDA(cudaMemcpyAsync(t->data.p, src, size_t(t->n_local) * es,
                                 src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
      },
      rows_b, rows_e, async);
}

// The per-call provider workspace of tensor t for (rank, flags): engine,
// factor buffers (one buffer per mode, both roles alias it) and Grams /
// FP32 mirrors of `factors`, which are uploaded on ctx->stream.
CallCache& call_setup(ntf_ctx* ctx, const ntf_tensor* t, const double* factors, int rank, unsigned flags) {
  need(factors, "factors");
  if (rank < 1) throw InvalidArgument("rank must be >= 1");
  NTF_CUDA(cudaSetDevice(ctx->device));
  auto& c = t->cache;
  if (!c || c->rank != rank || c->flags != flags) {
    if (c) NTF_CUDA(cudaStreamSynchronize(ctx->stream));
    c.reset();
    auto n = std::make_unique<CallCache>();
    n->rank = rank;
    n->flags = flags;
    n->eng = std::make_unique<MttkrpEngine>(ctx, t, rank, flags);
    const long long len = model_len(t, rank);
    n->fac = DevBuf(size_t(len) * sizeof(double));
    if (t->dtype == NTF_DTYPE_F32) n->fac32 = DevBuf(size_t(len) * sizeof(float));
    n->grams = DevBuf(size_t(t->order) * rank * rank * sizeof(double));
    n->dF = DevBuf(sizeof(DevFactors));
    long long maxrows = 0;
    for (int i = 0; i < t->order; ++i) maxrows = std::max(maxrows, t->shape[i]);
    n->C = DevBuf(size_t(maxrows) * rank * sizeof(double));
    std::memset(&n->h, 0, sizeof n->h);
    n->h.order = t->order;
    n->h.rank = rank;
    long long off = 0;
    for (int i = 0; i < t->order; ++i) {
      n->h.x[i][0] = n->h.x[i][1] = n->fac.as<double>() + off;
      if (n->fac32.p) n->h.x32[i][0] = n->h.x32[i][1] = n->fac32.as<float>() + off;
      n->h.gram[i][0] = n->h.gram[i][1] = n->grams.as<double>() + size_t(i) * rank * rank;
      n->h.rows[i] = int(t->shape[i]);
      off += t->shape[i] * rank;
    }
    NTF_CUDA(cudaMemcpyAsync(n->dF.p, &n->h, sizeof n->h, cudaMemcpyHostToDevice, ctx->stream));
    c = std::move(n);
  }
  NTF_CUDA(cudaMemcpyAsync(c->fac.p, factors, c->fac.bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (c->gscratch.bytes < init_factors_scratch(c->h) * sizeof(double))
    c->gscratch = DevBuf(init_factors_scratch(c->h) * sizeof(double));
  launch_init_factors(c->dF.as<DevFactors>(), c->h, c->gscratch.as<double>(), c->gscratch.bytes / sizeof(double),
                      ctx->stream);
  return *c;
}

void run_driver(int algo, ntf_ctx* ctx, const ntf_tensor* t, const double* init, int rank,
                const ntf_ao_config* cfg, const ntf_her_params* params, ntf_her_observer observer, void* user,
                double* out_factors, double* f0, ntf_trace_record* trace, int trace_cap, int* n_records) {
  need(ctx, "ctx");
  need(t, "tensor");
  need(init, "init");
  need(cfg, "config");
  need(out_factors, "out_factors");
  need(n_records, "n_records");
  if (algo == 0) {
    need(params, "params");
    validate_params(*params);
  }
  check_run_inputs(t, init, rank, *cfg);
  NvtxRange nvtx(algo == 0 ? "ntf:her_run" : "ntf:ao_run");
  const auto shape = int_shape(t);
  // NTF_TIMING=1: host-side phase times of the driver on stderr (diagnostics)
  static const bool timing = std::getenv("NTF_TIMING") != nullptr;
  const auto now = [] { return std::chrono::steady_clock::now(); };
  const auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  Session s(ctx, t, algo, init, rank, *cfg, params);
  const auto t1 = now();
  const long long len = model_len(t, rank);
  const bool per_iteration = observer != nullptr || cfg->record_factor_error;
  std::vector<double> e_values;
  if (!per_iteration && cfg->max_time_s > 0.0) {
    // A time budget alone: the device decides (the last block's kernel sets
    // `done` once the run clock passes the budget, her.cpp:105 / ao.cpp:48,
    // and every later kernel of the run is a no-op that writes no record), so
    // the host only has to stop enqueuing: graph replays in batches of 8
    // with one synchronisation per batch instead of one per iteration.
    const int batch = 8;
    for (;;) {
      s.step(batch);
      s.sync();
      if (s.done()) break;
    }
  } else if (!per_iteration) {
    s.step(cfg->max_outer_iters);
    const auto t2 = now();
    s.sync();
    if (timing)
      fprintf(stderr, "[ntf timing] session %.2f ms, enqueue %.2f ms, device wait %.2f ms\n", ms(t0, t1), ms(t1, t2),
              ms(t2, now()));
  } else {
    std::vector<double> acc(static_cast<size_t>(len));
    while (true) {
      s.step(1);
      bool finished = false;
      int k = 0;
      ntf_trace_record last{};
      s.snapshot(acc.data(), observer ? &last : nullptr, &k, &finished);  // one download, one synchronisation
      if (cfg->record_factor_error)
        e_values.push_back(factor_error(acc.data(), cfg->ground_truth, shape.data(), t->order, rank));
      if (observer) {
        ntf_her_iteration_info info{};
        info.iter = k;
        info.f_hat = last.f;
        info.restarted = last.restarted;
        info.beta_used = last.beta;
        info.factors = acc.data();
        info.hat_factors = acc.data();  // equal after every decision (her.cpp:76-83)
        observer(&info, user);
      }
      if (finished) break;
    }
  }
  std::vector<ntf_trace_record> recs(size_t(std::max(trace_cap, 0)));
  int n = 0;
  s.finish(out_factors, f0, recs.data(), trace_cap, &n);
  *n_records = n;
  if (trace)
    for (int i = 0; i < std::min(n, trace_cap); ++i) {
      trace[i] = recs[size_t(i)];
      if (size_t(i) < e_values.size()) {
        trace[i].has_e = 1;
        trace[i].e = e_values[size_t(i)];
      }
    }
}

}  // namespace

extern "C" {

const char* ntf_version(void) { return "ntf_b200 0.1 (sm_100a)"; }

int ntf_last_error(char* buf, size_t n) {
  if (buf && n) {
    std::strncpy(buf, g_last_error.c_str(), n - 1);
    buf[n - 1] = '\0';
  }
  return int(g_last_error.size());
}

void ntf_her_params_default(ntf_her_params* p) {
  if (p) *p = ntf_her_params{0.5, 1.05, 1.01, 1.5};
}

void ntf_ao_config_default(ntf_ao_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->solver = NTF_SOLVER_AHALS;
  c->inner_stop.max_iters = 50;
  c->inner_stop.rel_change_tol = 1e-2;
}

int ntf_her_params_validate(const ntf_her_params* p) {
  return guarded([&] {
    need(p, "params");
    validate_params(*p);
  });
}

int ntf_ao_config_validate(const ntf_ao_config* c) {
  return guarded([&] {
    need(c, "config");
    validate_cfg(*c);
  });
}

uint64_t ntf_stream_seed(uint64_t base, uint64_t stream) { return stream_seed(base, stream); }

int ntf_random_init(const int* shape, int order, int rank, uint64_t seed, double* out) {
  return guarded([&] {
    need(shape, "shape");
    need(out, "out");
    random_init(shape, order, rank, seed, out);
  });
}

int ntf_generate(const int* shape, int order, int rank, double sigma, int ill_conditioned, int collinear,
                 uint64_t seed, int dtype, void* tensor_out, double* truth_out) {
  return guarded([&] {
    need(shape, "shape");
    need(tensor_out, "tensor_out");
    need(truth_out, "truth_out");
    generate(shape, order, rank, sigma, ill_conditioned, collinear, seed, dtype, tensor_out, truth_out);
  });
}

int ntf_generate_slab(const int* shape, int order, int rank, double sigma, int ill_conditioned, int collinear,
                      uint64_t seed, int dtype, int64_t slab_begin, int64_t slab_end, void* tensor_out,
                      double* truth_out) {
  return guarded([&] {
    need(shape, "shape");
    need(tensor_out, "tensor_out");
    need(truth_out, "truth_out");
    if (order < 1 || slab_begin < 0 || slab_end < slab_begin || slab_end > shape[0])
      throw InvalidArgument("slab outside the first mode");
    generate(shape, order, rank, sigma, ill_conditioned, collinear, seed, dtype, tensor_out, truth_out,
             (long long)slab_begin, (long long)slab_end);
  });
}

int ntf_factor_error(const double* est, const double* truth, const int* shape, int order, int rank, double* out) {
  return guarded([&] {
    need(est, "est");
    need(truth, "truth");
    need(shape, "shape");
    need(out, "out");
    *out = factor_error(est, truth, shape, order, rank);
  });
}

int ntf_device_count(int* n) {
  return guarded([&] {
    need(n, "n");
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *n = c;
  });
}

int ntf_ctx_create(int device, ntf_ctx** out) {
  return guarded([&] {
    need(out, "out");
    int n = 0;
    NTF_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw InvalidArgument("no such CUDA device");
    auto* c = new ntf_ctx();
    try {
      c->device = device;
      NTF_CUDA(cudaSetDevice(device));
      retain_pool_memory(device);
      NTF_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      NTF_CUDA(cudaStreamCreateWithFlags(&c->setup, cudaStreamNonBlocking));
      c->sms = device_sm_count();
      c->scratch = DevBuf(4096 * sizeof(double));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int ntf_nccl_unique_id(unsigned char out[128]) {
  return guarded([&] {
    need(out, "out");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out, &id, 128);
  });
}

int ntf_ctx_create_dist(int device, int rank, int world, const unsigned char id[128], ntf_ctx** out) {
  return guarded([&] {
    need(out, "out");
    need(id, "id");
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("rank must lie in [0, world)");
    ntf_ctx* c = nullptr;
    const int rc = ntf_ctx_create(device, &c);
    if (rc != NTF_OK) throw CudaError(g_last_error);
    try {
      c->comm.rank = rank;
      c->comm.world = world;
      {  // world 1 too: a 1-rank communicator runs the collective path on one GPU
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        ncclComm_t comm;
        const ncclResult_t r = ncclCommInitRank(&comm, world, uid, rank);
        if (r != ncclSuccess) throw NcclError(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        c->comm.nccl = comm;
      }
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int ntf_ctx_info(const ntf_ctx* ctx, int* device, int* rank, int* world) {
  return guarded([&] {
    need(ctx, "ctx");
    if (device) *device = ctx->device;
    if (rank) *rank = ctx->comm.rank;
    if (world) *world = ctx->comm.world;
  });
}

int ntf_ctx_destroy(ntf_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int ntf_slab_range(int64_t dim0, int rank, int world, int64_t* begin, int64_t* end) {
  return guarded([&] {
    need(begin, "begin");
    need(end, "end");
    long long b, e;
    slab_range(dim0, rank, world, &b, &e);
    *begin = b;
    *end = e;
  });
}

int ntf_tensor_upload(ntf_ctx* ctx, const void* host, int dtype, int order, const int64_t* shape, ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    *out = make_tensor(ctx, host, false, dtype, order, shape);
  });
}

int ntf_tensor_upload_async(ntf_ctx* ctx, const void* host, int dtype, int order, const int64_t* shape,
                            ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    *out = make_tensor(ctx, host, false, dtype, order, shape, -1, -1, true);
  });
}

int ntf_tensor_wait(const ntf_tensor* t) {
  return guarded([&] {
    need(t, "tensor");
    if (t->ready) NTF_CUDA(cudaEventSynchronize(t->ready));
  });
}

int ntf_pinned_alloc(size_t bytes, void** out) {
  return guarded([&] {
    need(out, "out");
    NTF_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
  });
}

int ntf_pinned_free(void* p) {
  return guarded([&] {
    if (p) NTF_CUDA(cudaFreeHost(p));
  });
}

int ntf_tensor_upload_ntft(ntf_ctx* ctx, const char* path, int dtype, ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    need(path, "path");
    const NtftHeader h = ntft_read_header(path);
    *out = make_tensor_with(ctx, dtype, h.order, h.shape, [&](ntf_tensor* t) {
      long long stride0 = 1;
      for (int i = 1; i < h.order; ++i) stride0 *= h.shape[i];
      ntft_stream_to_device(path, h, t->row0 * stride0, t->n_local, dtype, t->data.p, ctx->stream);
    });
  });
}

int ntf_ntft_info(const char* path, int* order, int64_t* shape) {
  return guarded([&] {
    need(path, "path");
    const NtftHeader h = ntft_read_header(path);
    if (order) *order = h.order;
    if (shape)
      for (int i = 0; i < h.order; ++i) shape[i] = h.shape[i];
  });
}

int ntf_ntft_read(const char* path, int dtype, int64_t slab_begin, int64_t slab_end, void* out) {
  return guarded([&] {
    need(path, "path");
    need(out, "out");
    ntft_read_slab(path, dtype, slab_begin, slab_end, out);
  });
}

int ntf_ntft_write(const char* path, const void* data, int dtype, int order, const int64_t* shape) {
  return guarded([&] {
    need(path, "path");
    need(data, "data");
    need(shape, "shape");
    ntft_write(path, data, dtype, order, shape);
  });
}

int ntf_tensor_upload_device(ntf_ctx* ctx, const void* dev, int dtype, int order, const int64_t* shape,
                             ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    need(ctx, "ctx");
    NTF_CUDA(cudaSetDevice(ctx->device));
    NTF_CUDA(cudaDeviceSynchronize());  // the producer of `dev` ran on some other stream
    *out = make_tensor(ctx, dev, true, dtype, order, shape);
  });
}

int ntf_tensor_upload_device_async(ntf_ctx* ctx, const void* dev, int dtype, int order, const int64_t* shape,
                                   void* caller_stream, ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    need(ctx, "ctx");
    NTF_CUDA(cudaSetDevice(ctx->device));
    cudaEvent_t ev;
    NTF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    const cudaError_t e1 = cudaEventRecord(ev, static_cast<cudaStream_t>(caller_stream));
    const cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(ctx->stream, ev, 0) : e1;
    cudaEventDestroy(ev);
    NTF_CUDA(e2);
    *out = make_tensor(ctx, dev, true, dtype, order, shape);
  });
}

int ntf_tensor_upload_rows(ntf_ctx* ctx, const void* host, int dtype, int order, const int64_t* shape,
                           int64_t row_begin, int64_t row_end, ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    if (row_begin < 0) throw InvalidArgument("row slab outside the first mode");
    *out = make_tensor(ctx, host, false, dtype, order, shape, (long long)row_begin, (long long)row_end);
  });
}

// TuckerFormat::validate (tucker.cpp:16-26) + TuckerProvider (tucker.hpp:60-73)
ntf_tensor* make_tucker(ntf_ctx* ctx, const double* core, int order, const int64_t* core_shape, const double* bases,
                        const int64_t* full_shape) {
  need(ctx, "ctx");
  need(core, "core");
  need(core_shape, "core_shape");
  need(bases, "bases");
  need(full_shape, "full_shape");
  if (ctx->comm.active()) throw Unsupported("a Tucker provider lives on one GPU (no NCCL context)");
  if (order < 1 || order > NTF_MAX_ORDER) throw InvalidArgument("basis count does not match the core order");
  long long off = 0;
  for (int l = 0; l < order; ++l) {
    if (full_shape[l] < 1 || core_shape[l] < 1 || full_shape[l] > (1LL << 31) - 1)
      throw InvalidArgument("basis column count does not match the core shape");
    const long long I = full_shape[l], R = core_shape[l];
    const double* U = bases + off;
    double defect = 0.0;  // max |U^T U - I|
    for (long long a = 0; a < R; ++a)
      for (long long b = 0; b < R; ++b) {
        double g = 0.0;
        for (long long i = 0; i < I; ++i) g += U[i * R + a] * U[i * R + b];
        defect = std::max(defect, std::abs(g - (a == b ? 1.0 : 0.0)));
      }
    if (!(defect <= 1e-10)) throw InvalidArgument("basis columns are not orthonormal");
    off += I * R;
  }
  ntf_tensor* c = make_tensor(ctx, core, false, NTF_DTYPE_F64, order, core_shape);
  auto* t = new ntf_tensor();
  try {
    t->core.reset(c);
    t->ctx = ctx;
    t->kind = 1;
    t->dtype = NTF_DTYPE_F64;
    t->order = order;
    for (int l = 0; l < order; ++l) {
      t->shape[l] = full_shape[l];
      t->ranks[l] = core_shape[l];
    }
    t->row0 = 0;
    t->rows = full_shape[0];
    t->n_local = 0;
    t->bases = DevBuf(size_t(off) * sizeof(double));
    NTF_CUDA(cudaMemcpyAsync(t->bases.p, bases, size_t(off) * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    t->nsq = c->nsq;  // ||core||^2 == ||T||^2 for orthonormal bases (tucker.cpp:94-95)
    t->nsq_dev = DevBuf(sizeof(double));
    NTF_CUDA(cudaMemcpyAsync(t->nsq_dev.p, c->nsq_dev.p, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    NTF_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

int ntf_tucker_upload(ntf_ctx* ctx, const double* core, int order, const int64_t* core_shape, const double* bases,
                      const int64_t* full_shape, ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    *out = make_tucker(ctx, core, order, core_shape, bases, full_shape);
  });
}

int ntf_ntfk_info(const char* path, int* order, int64_t* full_shape, int64_t* core_shape) {
  return guarded([&] {
    need(path, "path");
    const NtfkHeader h = ntfk_read_header(path);
    if (order) *order = h.order;
    for (int l = 0; l < h.order; ++l) {
      if (full_shape) full_shape[l] = h.shape[l];
      if (core_shape) core_shape[l] = h.ranks[l];
    }
  });
}

int ntf_ntfk_read(const char* path, double* core, double* bases) {
  return guarded([&] {
    need(path, "path");
    need(core, "core");
    need(bases, "bases");
    ntfk_read(path, core, bases);
  });
}

int ntf_ntfk_write(const char* path, const double* core, const double* bases, int order, const int64_t* full_shape,
                   const int64_t* core_shape) {
  return guarded([&] {
    need(path, "path");
    need(core, "core");
    need(bases, "bases");
    need(full_shape, "full_shape");
    need(core_shape, "core_shape");
    ntfk_write(path, core, bases, order, full_shape, core_shape);
  });
}

int ntf_tensor_upload_ntfk(ntf_ctx* ctx, const char* path, ntf_tensor** out) {
  return guarded([&] {
    need(out, "out");
    need(path, "path");
    const NtfkHeader h = ntfk_read_header(path);
    long long nc = 1, nb = 0;
    for (int l = 0; l < h.order; ++l) {
      nc *= h.ranks[l];
      nb += h.shape[l] * h.ranks[l];
    }
    std::vector<double> core(static_cast<size_t>(nc)), bases(static_cast<size_t>(nb));
    ntfk_read(path, core.data(), bases.data());
    *out = make_tucker(ctx, core.data(), h.order, h.ranks, bases.data(), h.shape);
  });
}

int ntf_tensor_shape(const ntf_tensor* t, int* order, int64_t* shape) {
  return guarded([&] {
    need(t, "tensor");
    if (order) *order = t->order;
    if (shape)
      for (int i = 0; i < t->order; ++i) shape[i] = t->shape[i];
  });
}

int ntf_tensor_norm_sq(const ntf_tensor* t, double* out) {
  return guarded([&] {
    need(t, "tensor");
    need(out, "out");
    *out = host_nsq(t);
  });
}

int ntf_tensor_destroy(ntf_tensor* t) {
  return guarded([&] {
    if (t && t->ctx) NTF_CUDA(cudaStreamSynchronize(t->ctx->stream));  // no work may still read it
    delete t;
  });
}

int ntf_mttkrp(ntf_ctx* ctx, const ntf_tensor* t, const double* factors, int rank, int mode, double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(t, "tensor");
    need(out, "out");
    if (mode < 0 || mode >= t->order) throw InvalidArgument("mode out of range");
    CallCache& c = call_setup(ctx, t, factors, rank, NTF_RUN_DIRECT);
    c.eng->run(mode, c.dF.as<DevFactors>(), c.C.as<double>(), ctx->stream);
    NTF_CUDA(cudaMemcpyAsync(out, c.C.p, size_t(t->shape[mode]) * rank * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    NTF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ntf_mttkrp_all(ntf_ctx* ctx, const ntf_tensor* t, const double* factors, int rank, unsigned flags,
                   double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(t, "tensor");
    need(out, "out");
    if (flags & ~(NTF_RUN_DIMTREE | NTF_RUN_DIRECT | NTF_RUN_GENERIC | NTF_RUN_NO_GRAPH | NTF_RUN_NO_OVERLAP))
      throw InvalidArgument("unknown NTF_RUN_* flags");
    CallCache& c = call_setup(ctx, t, factors, rank, flags & (NTF_RUN_DIRECT | NTF_RUN_GENERIC | NTF_RUN_NO_OVERLAP));
    long long off = 0;
    for (int m = 0; m < t->order; ++m) {  // sweep order: the tree forms Y_L at block 0, Y_R at block h
      c.eng->run(m, c.dF.as<DevFactors>(), c.C.as<double>(), ctx->stream);
      const size_t n = size_t(t->shape[m]) * rank;
      NTF_CUDA(cudaMemcpyAsync(out + off, c.C.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      off += (long long)n;
    }
    NTF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ntf_mttkrp_plan(ntf_ctx* ctx, const ntf_tensor* t, int rank, int mode, char* buf, size_t n) {
  return guarded([&] {
    need(ctx, "ctx");
    need(t, "tensor");
    need(buf, "buf");
    if (rank < 1) throw InvalidArgument("rank must be >= 1");
    if (mode < 0 || mode >= t->order) throw InvalidArgument("mode out of range");
    MttkrpEngine eng(ctx, t, rank, NTF_RUN_DIRECT);
    const std::string s = eng.describe(mode);
    if (n) {
      std::strncpy(buf, s.c_str(), n - 1);
      buf[n - 1] = '\0';
    }
  });
}

int ntf_objective(ntf_ctx* ctx, const ntf_tensor* t, const double* factors, int rank, int pivot, double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(t, "tensor");
    need(out, "out");
    const int p = pivot < 0 ? t->order - 1 : pivot;
    if (p >= t->order) throw InvalidArgument("mode out of range");
    if (t->rows_only) throw InvalidArgument("the objective needs the whole tensor, not a row slab");
    CallCache& c = call_setup(ctx, t, factors, rank, NTF_RUN_DIRECT);
    DevBuf res(sizeof(double));
    c.eng->run(p, c.dF.as<DevFactors>(), c.C.as<double>(), ctx->stream);
    launch_objective(c.dF.as<DevFactors>(), t->order, rank, p, int(t->shape[p]), c.C.as<double>(),
                     t->nsq_dev.as<double>(), res.as<double>(), ctx->stream);
    NTF_CUDA(cudaMemcpyAsync(out, res.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    NTF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int ntf_solve_nnls(ntf_ctx* ctx, int solver, const double* gram, const double* target, const double* init,
                   int rows, int rank, const ntf_inner_stop* stop, double* out, int* sweeps) {
  return guarded([&] {
    need(ctx, "ctx");
    need(gram, "gram");
    need(target, "target");
    need(init, "init");
    need(out, "out");
    if (solver < NTF_SOLVER_AHALS || solver > NTF_SOLVER_ACTIVE_SET) throw LogicError("unknown solver");
    if (rows < 1 || rank < 1) throw InvalidArgument("rows and rank must be >= 1");
    const ntf_inner_stop st = stop ? *stop : ntf_inner_stop{50, 1e-2};
    NTF_CUDA(cudaSetDevice(ctx->device));
    const size_t n = size_t(rows) * rank;
    DevBuf g(size_t(rank) * rank * 8), c(n * 8), w0(n * 8), w(n * 8), sw(sizeof(int));
    DevBuf scratch(size_t(3072 + 64 * kMaxRank * kMaxRank) * sizeof(double));
    NTF_CUDA(cudaMemcpyAsync(g.p, gram, g.bytes, cudaMemcpyHostToDevice, ctx->stream));
    NTF_CUDA(cudaMemcpyAsync(c.p, target, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    NTF_CUDA(cudaMemcpyAsync(w0.p, init, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    NnlsLaunch a{};
    a.rows = rows;
    a.rank = rank;
    a.role = 2;
    a.C = c.as<double>();
    a.gram_in = g.as<double>();
    a.w0 = w0.as<double>();
    a.w_out = w.as<double>();
    a.sweeps_out = sw.as<int>();
    a.max_iters = st.max_iters;
    a.tol = st.rel_change_tol;
    a.scratch = scratch.as<double>();
    DevBuf work, err, tall;
    if (solver == NTF_SOLVER_AHALS) {
      if (nnls_needs_tall(rows, rank)) {
        tall = DevBuf(nnls_tall_workspace(rows, rank) * sizeof(double));
        a.tall = tall.as<double>();
      }
      launch_nnls(a, ctx->stream);
    } else {
      work = DevBuf(2 * n * 8);
      err = DevBuf(sizeof(int));
      NTF_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), ctx->stream));
      a.solver = solver;
      a.work = work.as<double>();
      a.error = err.as<int>();
      launch_nnls_solver(a, ctx->stream);
      int e = 0;
      NTF_CUDA(cudaMemcpyAsync(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      NTF_CUDA(cudaStreamSynchronize(ctx->stream));
      if (e) throw std::runtime_error(solver_error_message(e));
    }
    int s = 0;
    NTF_CUDA(cudaMemcpyAsync(out, w.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    NTF_CUDA(cudaMemcpyAsync(&s, sw.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    NTF_CUDA(cudaStreamSynchronize(ctx->stream));
    if (sweeps) *sweeps = s;
  });
}

int ntf_her_run(ntf_ctx* ctx, const ntf_tensor* t, const double* init, int rank, const ntf_ao_config* cfg,
                const ntf_her_params* params, ntf_her_observer observer, void* user, double* out_factors,
                double* f0, ntf_trace_record* trace, int trace_cap, int* n_records) {
  return guarded([&] {
    run_driver(0, ctx, t, init, rank, cfg, params, observer, user, out_factors, f0, trace, trace_cap, n_records);
  });
}

int ntf_ao_run(ntf_ctx* ctx, const ntf_tensor* t, const double* init, int rank, const ntf_ao_config* cfg,
               double* out_factors, double* f0, ntf_trace_record* trace, int trace_cap, int* n_records) {
  return guarded([&] {
    run_driver(1, ctx, t, init, rank, cfg, nullptr, nullptr, nullptr, out_factors, f0, trace, trace_cap,
               n_records);
  });
}

int ntf_session_create(ntf_ctx* ctx, const ntf_tensor* t, int algo, const double* init, int rank,
                       const ntf_ao_config* cfg, const ntf_her_params* params, ntf_session** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(t, "tensor");
    need(init, "init");
    need(cfg, "config");
    need(out, "out");
    if (algo != 0 && algo != 1) throw InvalidArgument("algo must be 0 (HER) or 1 (AO)");
    if (algo == 0) {
      need(params, "params");
      validate_params(*params);
    }
    check_run_inputs(t, init, rank, *cfg);
    auto* sess = new Session(ctx, t, algo, init, rank, *cfg, params);
    try {
      sess->sync();  // `init` (possibly pinned) has been consumed and setup errors surface here;
                     // the drivers (ntf_her_run / ntf_ao_run) skip this to overlap an asynchronous upload
    } catch (...) {
      delete sess;
      throw;
    }
    *out = reinterpret_cast<ntf_session*>(sess);
  });
}

#define SESSION(s) reinterpret_cast<Session*>(s)

int ntf_session_step(ntf_session* s, int iters) {
  return guarded([&] {
    need(s, "session");
    SESSION(s)->step(iters);
  });
}

int ntf_session_sync(ntf_session* s) {
  return guarded([&] {
    need(s, "session");
    SESSION(s)->sync();
  });
}

void* ntf_session_stream(ntf_session* s) { return s ? static_cast<void*>(SESSION(s)->stream()) : nullptr; }

int ntf_session_iterations(ntf_session* s, int* done) {
  return guarded([&] {
    need(s, "session");
    need(done, "done");
    *done = SESSION(s)->iterations();
  });
}

int ntf_session_factors(ntf_session* s, double* out) {
  return guarded([&] {
    need(s, "session");
    need(out, "out");
    SESSION(s)->factors(out);
  });
}

int ntf_session_trace(ntf_session* s, double* f0, ntf_trace_record* trace, int cap, int* n) {
  return guarded([&] {
    need(s, "session");
    need(n, "n");
    std::vector<ntf_trace_record> tmp(size_t(std::max(cap, 0)));
    SESSION(s)->trace(f0, tmp.data(), cap, n);
    if (trace)
      for (int i = 0; i < std::min(*n, cap); ++i) trace[i] = tmp[size_t(i)];
  });
}

int ntf_session_set_kernel_timing(ntf_session* s, int on) {
  return guarded([&] {
    need(s, "session");
    SESSION(s)->set_kernel_timing(on != 0);
  });
}

int ntf_session_kernel_times(ntf_session* s, double* ms_per_mode, int* launches_per_mode, int* total) {
  return guarded([&] {
    need(s, "session");
    SESSION(s)->kernel_times(ms_per_mode, launches_per_mode, total);
  });
}

int ntf_session_pass_slots(ntf_session* s, int* slots, int* n) {
  return guarded([&] {
    need(s, "session");
    need(slots, "slots");
    need(n, "n");
    *n = SESSION(s)->pass_slots(slots);
  });
}

// Diagnostics (not part of the public header): CTA-0 cycle counters of the
// NNLS kernel {sweep-loop cycles, reduction cycles, sweeps, calls}.
int ntf_debug_nnls_prof(unsigned long long* out, int reset) {
  return guarded([&] {
    need(out, "out");
    nnls_prof_read(out, reset != 0);
  });
}

int ntf_session_destroy(ntf_session* s) {
  return guarded([&] { delete SESSION(s); });
}

}  // extern "C"
