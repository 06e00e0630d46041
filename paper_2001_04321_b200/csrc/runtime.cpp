#include <chrono>
#include <cstdio>
#include <cstdlib>
// Host runtime: device buffers, NCCL plumbing, the MTTKRP engine and the
// GPU-resident HER / AO sessions.
#include "runtime.h"

#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "mttkrp_fast.h"
#include "mttkrp_fast_launch.h"

namespace ntfb {

// Engine tables: small ones travel as kernel parameters on the context's
// setup stream (they must not queue behind a tensor upload in flight on the
// copy engine -- ntf_tensor_upload_async), large ones take the copy engine.
// Blocking either way: the table is visible to every stream on return.
static void table_upload(const ntf_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (bytes <= 2 * 1024 * 1024 && ctx->setup) {
    static const bool trace = std::getenv("NTF_TIMING_ALLOC") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    dev_upload(dst, src, bytes, ctx->setup);
    const auto t1 = std::chrono::steady_clock::now();
    NTF_CUDA(cudaStreamSynchronize(ctx->setup));
    if (trace) {
      const auto t2 = std::chrono::steady_clock::now();
      fprintf(stderr, "[ntf table] %zu bytes: launch %.2f ms, sync %.2f ms\n", bytes,
              std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
  } else {
    NTF_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  }
}

static void table_zero(const ntf_ctx* ctx, void* dst, size_t bytes) {
  if (ctx->setup) {
    dev_zero(dst, bytes, ctx->setup);
    NTF_CUDA(cudaStreamSynchronize(ctx->setup));
  } else {
    NTF_CUDA(cudaMemset(dst, 0, bytes));
  }
}

// ---- DevBuf ------------------------------------------------------------------
// Device buffers come from the device's stream-ordered memory pool, which
// the context configures to keep freed memory (release threshold = max):
// a run's workspaces and a re-uploaded tensor are then served without the
// driver unmapping and remapping hundreds of MB (cudaFree of a 216 MB
// tensor measured 1-800 ms on the B200 boxes). Owners synchronise the
// streams that used a buffer before it is destroyed.
// The pool's allocations and frees run on one private non-blocking stream per
// device. (The legacy default stream served before: synchronising it waited
// for an asynchronous tensor upload in flight on the context's stream --
// 3 ms of a session's setup at C2, NTF_TIMING_ALLOC=1 -- although that stream
// is non-blocking.)
static cudaStream_t alloc_stream() {
  static cudaStream_t streams[64] = {};
  int dev = 0;
  NTF_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return cudaStreamLegacy;
  if (!streams[dev]) NTF_CUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
  return streams[dev];
}

DevBuf::DevBuf(size_t n) : bytes(n) {
  if (n) {
    static const bool trace = std::getenv("NTF_TIMING_ALLOC") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t as = alloc_stream();
    NTF_CUDA(cudaMallocAsync(&p, n, as));
    const auto t1 = std::chrono::steady_clock::now();
    NTF_CUDA(cudaStreamSynchronize(as));  // usable from any stream
    if (trace) {
      const auto t2 = std::chrono::steady_clock::now();
      const double a = std::chrono::duration<double, std::milli>(t1 - t0).count();
      const double b = std::chrono::duration<double, std::milli>(t2 - t1).count();
      if (a + b > 0.1) fprintf(stderr, "[ntf alloc] %zu bytes: malloc %.2f ms, sync %.2f ms\n", n, a, b);
    }
  }
}
DevBuf::~DevBuf() {
  if (p) cudaFreeAsync(p, alloc_stream());
}
DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
  if (this != &o) {
    if (p) cudaFreeAsync(p, alloc_stream());
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    o.bytes = 0;
  }
  return *this;
}

// ---- NCCL ----------------------------------------------------------------------
static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string("NCCL failure in ") + what + ": " + ncclGetErrorString(r));
}

void Comm::allreduce_sum(double* buf, size_t n, cudaStream_t s) const {
  if (!nccl) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(nccl), s), "ncclAllReduce");
}

void Comm::allgather(double* buf, size_t n_per_rank, cudaStream_t s) const {
  if (!nccl) return;
  nccl_check(ncclAllGather(buf + size_t(rank) * n_per_rank, buf, n_per_rank, ncclDouble,
                           static_cast<ncclComm_t>(nccl), s),
             "ncclAllGather");
}

void Comm::allreduce_max(double* buf, size_t n, cudaStream_t s) const {
  if (!nccl) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclDouble, ncclMax, static_cast<ncclComm_t>(nccl), s), "ncclAllReduce(max)");
}

Comm::~Comm() {
  if (nccl) ncclCommDestroy(static_cast<ncclComm_t>(nccl));
}

void retain_pool_memory(int device) {
  cudaMemPool_t pool;
  NTF_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = ~0ull;
  NTF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
}

void slab_range(long long dim0, int rank, int world, long long* begin, long long* end) {
  if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("rank must lie in [0, world)");
  if (dim0 < 1) throw InvalidArgument("tensor dimensions must be positive");
  const long long base = dim0 / world, extra = dim0 % world;
  const long long b = rank < extra ? rank * (base + 1) : extra * (base + 1) + (rank - extra) * base;
  *begin = b;
  *end = b + base + (rank < extra ? 1 : 0);
}

// ---- MTTKRP engine -------------------------------------------------------------
ModeView MttkrpEngine::view(int mode) const {
  ModeView v{};
  v.order = t_->order;
  v.mode = mode;
  v.rank = rank_;
  for (int l = 0; l < t_->order; ++l) v.dims[l] = int(l == 0 ? t_->rows : t_->shape[l]);
  v.L = 1;
  v.R = 1;
  for (int l = 0; l < mode; ++l) v.L *= v.dims[l];
  v.I = v.dims[mode];
  for (int l = mode + 1; l < t_->order; ++l) v.R *= v.dims[l];
  v.row0 = t_->row0;
  return v;
}

MttkrpEngine::MttkrpEngine(const ntf_ctx* ctx, const ntf_tensor* t, int rank, unsigned flags)
    : ctx_(ctx), t_(t), rank_(rank), flags_(flags), order_(t->order) {
  if (t->kind == 1) {  // TuckerProvider: the core's engine plus the projections
    tucker_ = true;
    core_eng_ = std::make_unique<MttkrpEngine>(ctx, t->core.get(), rank, flags | NTF_RUN_DIRECT);
    long long boff = 0, poff = 0, maxr = 1;
    for (int l = 0; l < t->order; ++l) {
      td_.rows[l] = int(t->shape[l]);
      td_.ranks[l] = int(t->ranks[l]);
      td_.base_off[l] = boff;
      td_.proj_off[l] = poff;
      boff += t->shape[l] * t->ranks[l];
      poff += t->ranks[l] * rank;
      maxr = std::max(maxr, t->ranks[l]);
    }
    proj_ = DevBuf(size_t(poff) * sizeof(double));
    mc_ = DevBuf(size_t(maxr) * rank * sizeof(double));
    td_.bases = t->bases.as<double>();
    td_.proj = proj_.as<double>();
    std::memset(&core_hF_, 0, sizeof core_hF_);
    core_hF_.order = t->order;
    core_hF_.rank = rank;
    for (int l = 0; l < t->order; ++l) {
      core_hF_.x[l][0] = core_hF_.x[l][1] = proj_.as<double>() + td_.proj_off[l];
      core_hF_.rows[l] = td_.ranks[l];
    }
    core_dF_ = DevBuf(sizeof(DevFactors));
    table_upload(ctx_, core_dF_.p, &core_hF_, sizeof core_hF_);
    counter_ = DevBuf(2 * sizeof(unsigned));
    table_zero(ctx_, counter_.p, 2 * sizeof(unsigned));
    return;
  }
  size_t need = 0;
  for (int m = 0; m < t->order; ++m) {
    const ModeView v = view(m);
    const long long cgroups = (rank + 7) / 8;
    const long long plane = v.L * v.R;
    long long segs = (4LL * ctx->sms + v.I * cgroups - 1) / (v.I * cgroups);
    segs = std::max(1LL, std::min({segs, std::max(1LL, plane / 256), 1024LL}));
    segs_[m] = int(segs);
    need = std::max(need, size_t(segs) * size_t(v.I) * rank);
    need = std::max(need, fast_mttkrp_partial_len(v, t->dtype, ctx->sms));
  }
  // the dimension tree is the default; NTF_RUN_DIRECT asks for N full passes
  if (!(flags & (NTF_RUN_DIRECT | NTF_RUN_GENERIC)) && t->order >= 3 &&
      view(t->order - 1).L < (1LL << 31)) {
    // Split point h of the dimension tree: blocks 0..h-1 contract
    // Y_L = T x_h A_h ... x_{N-1} A_{N-1} (previous sweep), blocks h..N-1
    // contract Y_R = T x_0 A_0 ... x_{h-1} A_{h-1} (this sweep). h = N-1 is
    // the one-sided tree (Y_R is block N-1's MTTKRP itself); 4-way tensors
    // split in the middle so both partials are small (C3: 1.28 MB each
    // instead of one 128 MB Y).
    const int N = t->order;
    int h = N >= 4 ? N / 2 : N - 1;
    if (const char* e = std::getenv("NTF_TREE_SPLIT")) h = std::max(1, std::min(N - 1, std::atoi(e)));
    const ModeView full = view(0);
    const auto left_view = [&](int hh) {
      ModeView tv{};
      tv.order = 1 + (N - hh);
      tv.mode = 0;
      tv.rank = rank;
      long long rows = 1;
      for (int j = 0; j < hh; ++j) rows *= full.dims[j];
      tv.dims[0] = int(rows);
      for (int j = hh; j < N; ++j) tv.dims[1 + j - hh] = full.dims[j];
      tv.L = 1;
      tv.I = rows;
      tv.R = 1;
      for (int j = hh; j < N; ++j) tv.R *= full.dims[j];
      tv.row0 = 0;
      tv.fshift = hh - 1;
      return tv;
    };
    const auto right_view = [&](int hh) {
      ModeView rv{};
      rv.order = hh + 1;
      rv.mode = hh;
      rv.rank = rank;
      for (int j = 0; j < hh; ++j) rv.dims[j] = full.dims[j];
      long long cols = 1;
      for (int j = hh; j < N; ++j) cols *= full.dims[j];
      rv.dims[hh] = int(cols);
      rv.L = 1;
      for (int j = 0; j < hh; ++j) rv.L *= full.dims[j];
      rv.I = cols;
      rv.R = 1;
      rv.row0 = t->row0;
      return rv;
    };
    std::vector<int> tab, rtab;
    if (h < N - 1) {
      long long cols = 1;
      for (int j = h; j < N; ++j) cols *= full.dims[j];
      if (cols < (1LL << 31)) {
        tab = fast_mttkrp_unit_table(left_view(h), t->dtype, ctx->sms);
        rtab = fast_mttkrp_unit_table(right_view(h), t->dtype, ctx->sms);
      }
      if (tab.empty() || rtab.empty()) h = N - 1;  // no fast plan for a split view: one-sided tree
    }
    if (h == N - 1) tab = fast_mttkrp_unit_table(left_view(h), t->dtype, ctx->sms);
    if (!tab.empty()) {
      tree_ = true;
      split_ = h;
      ttm_view_ = left_view(h);
      ttm_tab_ = DevBuf(tab.size() * sizeof(int));
      table_upload(ctx_, ttm_tab_.p, tab.data(), tab.size() * sizeof(int));
      ybuf_ = DevBuf(size_t(ttm_view_.I) * rank * sizeof(double));
      need = std::max(need, fast_mttkrp_partial_len(ttm_view_, t->dtype, ctx->sms));
      if (N == 3 && h == N - 1 && !t->rows_only && !(flags & NTF_RUN_NO_OVERLAP)) {
        const char* oe = std::getenv("NTF_OVERLAP");
        if (!(oe && std::atoi(oe) == 0)) {
          const int osms = std::max(1, ctx->sms - kNnlsReserveSms);
          const ModeView pv = right_view(1);
          const std::vector<int> ptab = fast_mttkrp_unit_table(pv, t->dtype, osms);
          if (!ptab.empty()) {
            overlap_ = true;
            p0_sms_ = osms;
            p0_view_ = pv;
            p0_tab_ = DevBuf(ptab.size() * sizeof(int));
            table_upload(ctx_, p0_tab_.p, ptab.data(), ptab.size() * sizeof(int));
            p0buf_ = DevBuf(size_t(pv.I) * rank * sizeof(double));
            need = std::max(need, fast_mttkrp_partial_len(pv, t->dtype, osms));
          }
        }
      }
      if (h < N - 1) {
        ttmr_view_ = right_view(h);
        ttmr_tab_ = DevBuf(rtab.size() * sizeof(int));
        table_upload(ctx_, ttmr_tab_.p, rtab.data(), rtab.size() * sizeof(int));
        yrbuf_ = DevBuf(size_t(ttmr_view_.I) * rank * sizeof(double));
        need = std::max(need, fast_mttkrp_partial_len(ttmr_view_, t->dtype, ctx->sms));
      }
      int tiles = 1;
      for (int m = 0; m < N; ++m) {
        if (!tree_mode(m)) continue;
        const TreeView yv = tree_view(m);
        tree_chunks_[m] = tree_chunks(yv, ctx->sms);
        tiles = std::max(tiles, tree_tiles(yv));
        need = std::max(need, size_t(tree_chunks_[m]) * size_t(yv.I) * rank);
      }
      tree_tiles_max_ = tiles;
    }
  }
  partial_ = DevBuf(need * sizeof(double));
  if (tree_) {
    tree_arrivals_ = DevBuf(size_t(tree_tiles_max_) * sizeof(unsigned));
    table_zero(ctx_, tree_arrivals_.p, size_t(tree_tiles_max_) * sizeof(unsigned));
  }
  counter_ = DevBuf(2 * sizeof(unsigned));
  table_zero(ctx_, counter_.p, 2 * sizeof(unsigned));
  if (!(flags & NTF_RUN_GENERIC))
    for (int m = 0; m < t->order; ++m) {
      const std::vector<int> tab = fast_mttkrp_unit_table(view(m), t->dtype, ctx->sms);
      if (tab.empty()) continue;
      unit_tab_[m] = DevBuf(tab.size() * sizeof(int));
      table_upload(ctx_, unit_tab_[m].p, tab.data(), tab.size() * sizeof(int));
    }
  if (ctx->comm.active()) {
    const int world = ctx->comm.world;
    std::vector<long long> meta(static_cast<size_t>(2 * world));
    for (int p = 0; p < world; ++p) {
      long long b, e;
      slab_range(t->shape[0], p, world, &b, &e);
      meta[size_t(p)] = b;
      meta[size_t(world + p)] = e - b;
      maxrows_ = std::max(maxrows_, e - b);
    }
    gather_ = DevBuf(size_t(maxrows_) * world * rank * sizeof(double));
    slab_meta_ = DevBuf(meta.size() * sizeof(long long));
    table_upload(ctx_, slab_meta_.p, meta.data(), meta.size() * sizeof(long long));
  }
}

TreeView MttkrpEngine::tree_view(int mode) const {
  const ModeView v = view(mode);
  if (overlap_ && mode == order_ - 1) {  // P_0: (i1, i2) rows, contract i1 with A_1
    TreeView y{};
    y.order = 2;
    y.mode = 1;
    y.rank = rank_;
    y.dims[0] = v.dims[1];
    y.dims[1] = v.dims[2];
    y.L = v.dims[1];
    y.I = v.dims[2];
    y.R = 1;
    y.row0 = 0;
    y.foff = 1;
    return y;
  }
  // blocks < split_: Y_L over modes 0..split_-1; blocks >= split_: Y_R over
  // modes split_..N-1 (factor offset split_, no slab offset)
  const bool left = mode < split_;
  const int lo = left ? 0 : split_, hi = left ? split_ : t_->order;
  TreeView y{};
  y.order = hi - lo;
  y.mode = mode - lo;
  y.rank = rank_;
  for (int j = 0; j < y.order; ++j) y.dims[j] = v.dims[lo + j];
  y.L = 1;
  y.R = 1;
  for (int j = 0; j < y.mode; ++j) y.L *= y.dims[j];
  y.I = y.dims[y.mode];
  for (int j = y.mode + 1; j < y.order; ++j) y.R *= y.dims[j];
  y.row0 = left ? t_->row0 : 0;
  y.foff = lo;
  return y;
}

std::string MttkrpEngine::describe(int mode) const {
  if (tucker_) return "tucker (project, core " + core_eng_->describe(mode) + ", expand)";
  if (tree_mode(mode))
    return std::string("tree split=") + std::to_string(split_) + " chunks=" + std::to_string(tree_chunks_[mode]) +
           (mode == 0 ? " after Y_L " + fast_mttkrp_describe(ttm_view_, t_->dtype, ctx_->sms) : std::string()) +
           (mode == split_ ? " after Y_R " + fast_mttkrp_describe(ttmr_view_, t_->dtype, ctx_->sms) : std::string());
  const ModeView v = view(mode);
  if (!(flags_ & NTF_RUN_GENERIC) && fast_mttkrp_supported(v, t_->dtype)) return fast_mttkrp_describe(v, t_->dtype, ctx_->sms);
  return "generic segs=" + std::to_string(segs_[mode]);
}

int MttkrpEngine::kernels_per_call(int mode) const {
  if (tucker_) return 2 + core_eng_->kernels_per_call(mode);
  if (overlap_) {  // Y_L pass + contraction | contraction + the overlapped P_0 pass | contraction
    if (mode == 0) return 1 + std::min(2, fast_mttkrp_kernels(ttm_view_, t_->dtype));
    if (mode == 1) return 1 + std::min(2, fast_mttkrp_kernels(p0_view_, t_->dtype));
    return 1;
  }
  // the fast kernel reduces its split-K slabs itself (the engine passes an
  // arrival counter) unless NTF_FAST_SEPARATE_REDUCE asks for the old kernel
  const int fast_kernels = std::getenv("NTF_FAST_SEPARATE_REDUCE") ? 2 : 1;
  if (tree_mode(mode))
    return 1 + (mode == 0 ? std::min(fast_kernels, fast_mttkrp_kernels(ttm_view_, t_->dtype)) : 0) +
           (mode == split_ ? std::min(fast_kernels, fast_mttkrp_kernels(ttmr_view_, t_->dtype)) : 0);
  const ModeView v = view(mode);
  if (!(flags_ & NTF_RUN_GENERIC) && fast_mttkrp_supported(v, t_->dtype))
    return std::min(fast_kernels, fast_mttkrp_kernels(v, t_->dtype));
  return 2;
}

void MttkrpEngine::run(int mode, const DevFactors* dF, double* out, cudaStream_t s, cudaEvent_t ev0,
                       cudaEvent_t ev1) {
  if (tucker_) {
    if (ev0) NTF_CUDA(cudaEventRecord(ev0, s));
    launch_tucker_project(td_, dF, mode, order_, rank_, s);
    core_eng_->run(mode, core_dF_.as<DevFactors>(), mc_.as<double>(), s);
    launch_tucker_expand(td_, mode, rank_, mc_.as<double>(), out, s);
    if (ev1) NTF_CUDA(cudaEventRecord(ev1, s));
    return;
  }
  const ModeView v = view(mode);
  const Comm& comm = ctx_->comm;
  const bool gather = comm.active() && mode == 0;
  double* dst = gather ? gather_.as<double>() + size_t(comm.rank) * maxrows_ * rank_ : out;
  if (t_->rows_only && mode == 0) {  // a row slab on one GPU: its rows of the full I_1 x r output
    NTF_CUDA(cudaMemsetAsync(out, 0, size_t(t_->shape[0]) * rank_ * sizeof(double), s));
    dst = out + size_t(t_->row0) * rank_;
  }
  const bool seq = last_mode_ == mode - 1;
  last_mode_ = mode;
  if (ev0) NTF_CUDA(cudaEventRecord(ev0, s));
  if (tree_mode(mode)) {
    // block 0 opens the outer iteration: Y_L with the previous sweep's
    // A_split.. A_{N-1}; block split_ forms Y_R with this sweep's A_0..
    // A partial is formed by the first block of its side; a block reached
    // out of sweep order (the pivot objective's lone block N-1,
    // driver_common.hpp:50-56) forms it with the current factors.
    // kernel timing (ev0/ev1): a block that forms a partial times that full
    // tensor pass alone, the other blocks time their tree contraction
    bool pass = false;
    if (overlap_ && mode == order_ - 1) {  // block 2 from P_0 (formed after block 1's NNLS)
      if (!p0_ready_) {  // reached out of sweep order: form it now
        fast_mttkrp(t_->data.p, t_->dtype, p0_view_, dF, p0_tab_.as<int>(), partial_.as<double>(),
                    p0buf_.as<double>(), p0_sms_, s, counter_.as<unsigned>());
        pass = true;
      }
      p0_ready_ = false;
      if (ev1 && pass) NTF_CUDA(cudaEventRecord(ev1, s));
      launch_tree_mttkrp(p0buf_.as<double>(), tree_view(mode), dF, partial_.as<double>(), tree_chunks_[mode],
                         tree_arrivals_.as<unsigned>(), dst, s);
      if (ev1 && !pass) NTF_CUDA(cudaEventRecord(ev1, s));
      goto exchange;
    }
    if (mode == 0 || (mode < split_ && !seq)) {
      fast_mttkrp(t_->data.p, t_->dtype, ttm_view_, dF, ttm_tab_.as<int>(), partial_.as<double>(), ybuf_.as<double>(),
                  ctx_->sms, s, counter_.as<unsigned>());
      pass = true;
      p0_ready_ = false;  // a new sweep starts: P_0 of the previous one is stale
    }
    if (mode == split_ || (mode > split_ && !seq)) {
      fast_mttkrp(t_->data.p, t_->dtype, ttmr_view_, dF, ttmr_tab_.as<int>(), partial_.as<double>(),
                  yrbuf_.as<double>(), ctx_->sms, s, counter_.as<unsigned>());
      pass = true;
    }
    if (ev1 && pass) NTF_CUDA(cudaEventRecord(ev1, s));
    launch_tree_mttkrp(mode < split_ ? ybuf_.as<double>() : yrbuf_.as<double>(), tree_view(mode), dF,
                       partial_.as<double>(), tree_chunks_[mode], tree_arrivals_.as<unsigned>(), dst, s);
    if (ev1 && !pass) NTF_CUDA(cudaEventRecord(ev1, s));
  } else if (unit_tab_[mode].p) {  // a fast plan exists (tables are built only then)
    fast_mttkrp(t_->data.p, t_->dtype, v, dF, unit_tab_[mode].as<int>(), partial_.as<double>(), dst, ctx_->sms, s,
                counter_.as<unsigned>());
    if (ev1) NTF_CUDA(cudaEventRecord(ev1, s));
  } else {
    launch_mttkrp_generic(t_->data.p, t_->dtype, v, dF, partial_.as<double>(), segs_[mode], s);
    if (ev1) NTF_CUDA(cudaEventRecord(ev1, s));
    launch_reduce_partials(partial_.as<double>(), segs_[mode], v.I * rank_, dst, s);
  }
exchange:
  if (!comm.active()) return;
  if (gather) {
    comm.allgather(gather_.as<double>(), size_t(maxrows_) * rank_, s);
    const long long* meta = slab_meta_.as<long long>();
    launch_compact_rows(gather_.as<double>(), maxrows_, meta, meta + comm.world, comm.world, rank_, out, s);
  } else {
    comm.allreduce_sum(out, size_t(v.I) * rank_, s);
  }
}

void MttkrpEngine::after_block(int mode, const DevFactors* dF, cudaStream_t s, bool pdl, cudaEvent_t ev0,
                               cudaEvent_t ev1) {
  if (!overlap_ || mode != 1) return;
  if (ev0) NTF_CUDA(cudaEventRecord(ev0, s));
  fast_mttkrp(t_->data.p, t_->dtype, p0_view_, dF, p0_tab_.as<int>(), partial_.as<double>(), p0buf_.as<double>(),
              p0_sms_, s, counter_.as<unsigned>(), pdl);
  if (ev1) NTF_CUDA(cudaEventRecord(ev1, s));
  p0_ready_ = true;
}

// ---- Session -------------------------------------------------------------------
namespace {
constexpr int kNnlsScratch = 3072 + 64 * kMaxRank * kMaxRank;
}

Session::Session(ntf_ctx* ctx, const ntf_tensor* t, int algo, const double* init, int rank,
                 const ntf_ao_config& cfg, const ntf_her_params* params)
    : ctx_(ctx), t_(t), algo_(algo), rank_(rank), order_(t->order), cfg_(cfg) {
  if (t->rows_only)
    throw InvalidArgument("a row-slab tensor of a 1-GPU context serves MTTKRP calls only, not solver runs");
  static const bool timing = std::getenv("NTF_TIMING") != nullptr;
  const auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
  NvtxRange nvtx("ntf:session");
  NTF_CUDA(cudaSetDevice(ctx->device));
  NTF_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  for (int i = 0; i < order_; ++i) {
    rows_[i] = int(t->shape[i]);
    total_factor_len_ += (long long)rows_[i] * rank;
  }
  const auto t1 = now();
  eng_ = std::make_unique<MttkrpEngine>(ctx, t, rank, cfg.flags);
  const auto t2 = now();

  fac_ = DevBuf(size_t(2 * total_factor_len_) * sizeof(double));
  if (t->dtype == NTF_DTYPE_F32) fac32_ = DevBuf(size_t(2 * total_factor_len_) * sizeof(float));
  grams_ = DevBuf(size_t(2 * order_) * rank * rank * sizeof(double));
  int maxrows = 0;
  for (int i = 0; i < order_; ++i) maxrows = std::max(maxrows, rows_[i]);
  C_ = DevBuf(size_t(maxrows) * rank * sizeof(double));
  state_ = DevBuf(sizeof(RunState));
  trace_cap_ = cfg.max_outer_iters > 0 ? cfg.max_outer_iters : (1 << 20);
  trace_ = DevBuf(size_t(trace_cap_) * sizeof(TraceEntry));
  scratch_ = DevBuf(size_t(kNnlsScratch) * sizeof(double));
  if (cfg.solver != NTF_SOLVER_AHALS) {
    solve_buf_ = DevBuf(size_t(maxrows) * rank * sizeof(double));
    solve_work_ = DevBuf(2 * size_t(maxrows) * rank * sizeof(double));
  }
  dF_ = DevBuf(sizeof(DevFactors));
  {  // factors beyond one cluster (or NTF_NNLS_TALL=1): workspace of the grid-kernel block update
    size_t need_tall = 0;
    for (int i = 0; i < order_; ++i)
      if (nnls_needs_tall(rows_[i], rank)) need_tall = std::max(need_tall, nnls_tall_workspace(rows_[i], rank));
    if (need_tall) tall_work_ = DevBuf(need_tall * sizeof(double));
  }

  std::memset(&hF_, 0, sizeof hF_);
  hF_.order = order_;
  hF_.rank = rank;
  long long off = 0;
  for (int i = 0; i < order_; ++i) {
    const long long n = (long long)rows_[i] * rank;
    for (int b = 0; b < 2; ++b) {
      hF_.x[i][b] = fac_.as<double>() + 2 * off + b * n;
      if (fac32_.p) hF_.x32[i][b] = fac32_.as<float>() + 2 * off + b * n;
      hF_.gram[i][b] = grams_.as<double>() + (size_t(2 * i + b)) * rank * rank;
    }
    hF_.sel[i] = 0;
    hF_.rows[i] = rows_[i];
    // (kernel-parameter uploads below 1 MB: the copy engine may be busy with the tensor)
    if (size_t(n) * sizeof(double) <= (1u << 20)) {
      dev_upload(hF_.x[i][0], init + off, size_t(n) * sizeof(double), stream_);
      NTF_CUDA(cudaMemcpyAsync(hF_.x[i][1], hF_.x[i][0], size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
    } else {
      NTF_CUDA(cudaMemcpyAsync(hF_.x[i][0], init + off, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, stream_));
      NTF_CUDA(cudaMemcpyAsync(hF_.x[i][1], init + off, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, stream_));
    }
    off += n;
  }
  dev_upload(dF_.p, &hF_, sizeof hF_, stream_);

  RunState st{};
  st.beta = params ? params->beta0 : 0.0;
  st.beta_bar = 1.0;
  st.nsq = 0.0;  // copied from the tensor's device value below
  if (params) {
    st.beta0 = params->beta0;
    st.gamma = params->gamma;
    st.gamma_bar = params->gamma_bar;
    st.eta = params->eta;
  }
  st.max_time_s = cfg.max_time_s;
  st.max_iters = cfg.max_outer_iters > 0 ? cfg.max_outer_iters : trace_cap_;
  st.inner_max_iters = cfg.inner_stop.max_iters;
  st.tol = cfg.inner_stop.rel_change_tol;
  st.algo = algo;
  collective_time_ = ctx->comm.active() && cfg.max_time_s > 0.0;
  st.collective_time = collective_time_ ? 1 : 0;
  dev_upload(state_.p, &st, sizeof st, stream_);

  // GramCache::create + pivot objective f0 (driver_common.hpp:50-56), then
  // start the run clock (her.cpp:58 / ao.cpp:28). No host synchronisation:
  // everything above (small uploads from pageable memory, run on an idle
  // stream) and the Gram setup precede the wait for the tensor, so after an
  // asynchronous upload (ntf_tensor_upload_async) this constructor, the first
  // iteration's launches and the graph capture all overlap the host-to-device
  // copy of the tensor; f0's MTTKRP starts when the copy and the ||T||^2
  // reduction have finished (t->ready).
  DevFactors* dF = dF_.as<DevFactors>();
  RunState* dst = state_.as<RunState>();
  init_scratch_ = DevBuf(init_factors_scratch(hF_) * sizeof(double));
  launch_init_factors(dF, hF_, init_scratch_.as<double>(), init_scratch_.bytes / sizeof(double), stream_);
  const ntf_tensor* deps[2] = {t, t->core.get()};
  for (const ntf_tensor* dep : deps)
    if (dep && dep->ready) NTF_CUDA(cudaStreamWaitEvent(stream_, dep->ready, 0));
  NTF_CUDA(cudaMemcpyAsync(&dst->nsq, t->nsq_dev.p, sizeof(double), cudaMemcpyDeviceToDevice, stream_));
  eng_->run(order_ - 1, dF, C_.as<double>(), stream_);
  launch_objective(dF, order_, rank, order_ - 1, rows_[order_ - 1], C_.as<double>(), &dst->nsq, &dst->f0,
                   stream_);
  NTF_CUDA(cudaMemcpyAsync(&dst->f_prev, &dst->f0, sizeof(double), cudaMemcpyDeviceToDevice, stream_));
  launch_stamp_start(dst, stream_);
  if (timing) {
    const auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[ntf timing] session: stream %.2f ms, engine %.2f ms, buffers+init+f0 %.2f ms\n",
            ms(t0, t1), ms(t1, t2), ms(t2, now()));
  }
}

Session::~Session() {
  if (exec_) cudaGraphExecDestroy(exec_);
  if (graph_) cudaGraphDestroy(graph_);
  for (auto e : ev_) cudaEventDestroy(e);
  if (stream_) {
    cudaStreamSynchronize(stream_);
    cudaStreamDestroy(stream_);
  }
}

void Session::enqueue_iteration(bool timed) {
  DevFactors* dF = dF_.as<DevFactors>();
  RunState* st = state_.as<RunState>();
  for (int i = 0; i < order_; ++i) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
      NTF_CUDA(cudaEventCreate(&e0));
      NTF_CUDA(cudaEventCreate(&e1));
      ev_.push_back(e0);
      ev_.push_back(e1);
      ev_mode_.push_back(i);
    }
    {
      NvtxRange nvtx("ntf:mttkrp", i);
      eng_->run(i, dF, C_.as<double>(), stream_, e0, e1);
    }
    NvtxRange nvtx_nnls("ntf:nnls", i);
    NnlsLaunch a{};
    a.mode = i;
    a.order = order_;
    a.rows = rows_[i];
    a.rank = rank_;
    a.role = algo_;
    a.last = (i == order_ - 1) ? 1 : 0;
    a.C = C_.as<double>();
    a.F = dF;
    a.st = st;
    a.trace = trace_.as<TraceEntry>();
    a.scratch = scratch_.as<double>();
    a.bufs = hF_;
    a.has_bufs = 1;
    a.max_iters = cfg_.inner_stop.max_iters;  // the host's copy (launch count of the tall path's sweeps)
    a.tall = tall_work_.p ? tall_work_.as<double>() : nullptr;
    if (cfg_.solver != NTF_SOLVER_AHALS) {  // solve_nnls (nnls.cpp:213-222), then the fused epilogue
      NnlsLaunch b = a;
      b.solver = cfg_.solver;
      b.w_out = solve_buf_.as<double>();
      b.work = solve_work_.as<double>();
      b.error = &st->error;
      launch_nnls_solver(b, stream_);
      a.zero_sweeps = 1;
      a.w0 = solve_buf_.as<double>();
    }
    launch_nnls(a, stream_);
    if (eng_->overlap() && i == 1) {
      // the overlapped pass: launched right after block 1's NNLS as its
      // programmatic dependent (timing runs serialise it to time it alone;
      // its events replace block 1's contraction slot)
      cudaEvent_t p0 = nullptr, p1 = nullptr;
      if (timed) {
        NTF_CUDA(cudaEventCreate(&p0));
        NTF_CUDA(cudaEventCreate(&p1));
        ev_.push_back(p0);
        ev_.push_back(p1);
        ev_mode_.push_back(i);
        // drop block 1's contraction timing (its slot now holds the pass)
        ev_mode_[ev_mode_.size() - 2] = -1;
      }
      eng_->after_block(i, dF, stream_, !timed, p0, p1);
    }
  }
  if (collective_time_) {  // every rank applies the same (max) elapsed time
    ctx_->comm.allreduce_max(&st->elapsed_s, 1, stream_);
    launch_apply_time_budget(st, stream_);
  }
}

void Session::build_graph() {
  if (exec_ || graph_failed_) return;
  NvtxRange nvtx("ntf:graph");
  cudaStreamCaptureStatus cs;
  NTF_CUDA(cudaStreamIsCapturing(stream_, &cs));
  if (cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    graph_failed_ = true;
    return;
  }
  bool ok = true;
  try {
    enqueue_iteration(false);
  } catch (...) {
    ok = false;
  }
  cudaGraph_t g = nullptr;
  if (cudaStreamEndCapture(stream_, &g) != cudaSuccess || !ok) {
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    graph_failed_ = true;
    return;
  }
  if (cudaGraphInstantiate(&exec_, g, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    exec_ = nullptr;
    graph_failed_ = true;
    return;
  }
  graph_ = g;
}

void Session::step(int iters) {
  for (int k = 0; k < iters; ++k) {
    if (timing_) {
      enqueue_iteration(true);
    } else if (cfg_.flags & NTF_RUN_NO_GRAPH) {
      enqueue_iteration(false);
    } else {
      if (host_iters_ == 0 && !exec_) {
        enqueue_iteration(false);  // first iteration direct: sets kernel attributes
      } else {
        build_graph();
        if (exec_)
          NTF_CUDA(cudaGraphLaunch(exec_, stream_));
        else
          enqueue_iteration(false);
      }
    }
    ++host_iters_;
  }
}

void Session::sync() { NTF_CUDA(cudaStreamSynchronize(stream_)); }

int Session::iterations() {
  int k = 0;
  NTF_CUDA(cudaMemcpyAsync(&k, &state_.as<RunState>()->k, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  sync();
  return k;
}

bool Session::done() {
  NTF_CUDA(cudaMemcpyAsync(&done_host_, &state_.as<RunState>()->done, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  sync();
  return done_host_ != 0;
}

void Session::factors(double* out) {
  DevFactors h;
  NTF_CUDA(cudaMemcpyAsync(&h, dF_.p, sizeof h, cudaMemcpyDeviceToHost, stream_));
  sync();
  long long off = 0;
  for (int i = 0; i < order_; ++i) {
    const long long n = (long long)rows_[i] * rank_;
    NTF_CUDA(cudaMemcpyAsync(out + off, h.x[i][h.sel[i]], size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    off += n;
  }
  sync();
}

void Session::trace(double* f0, ntf_trace_record* out, int cap, int* n) {
  RunState st;
  NTF_CUDA(cudaMemcpyAsync(&st, state_.p, sizeof st, cudaMemcpyDeviceToHost, stream_));
  sync();
  if (f0) *f0 = st.f0;
  *n = st.k;
  const int m = std::min(st.k, cap);
  if (m <= 0) return;
  std::vector<TraceEntry> tr(static_cast<size_t>(m));
  NTF_CUDA(cudaMemcpyAsync(tr.data(), trace_.p, size_t(m) * sizeof(TraceEntry), cudaMemcpyDeviceToHost, stream_));
  sync();
  for (int i = 0; i < m; ++i) {
    ntf_trace_record r{};
    r.iter = i + 1;
    r.time_s = tr[size_t(i)].time_s;
    r.f = tr[size_t(i)].f;
    r.inner_sweeps = tr[size_t(i)].sweeps;
    if (algo_ == 0) {
      r.has_restarted = 1;
      r.restarted = tr[size_t(i)].restarted;
      r.has_beta = 1;
      r.beta = tr[size_t(i)].beta;
    }
    out[i] = r;
  }
}

bool Session::last_record(ntf_trace_record* out) {
  RunState st;
  NTF_CUDA(cudaMemcpyAsync(&st, state_.p, sizeof st, cudaMemcpyDeviceToHost, stream_));
  sync();
  if (st.k <= 0 || st.k > trace_cap_) return false;
  TraceEntry e;
  NTF_CUDA(cudaMemcpyAsync(&e, trace_.as<TraceEntry>() + (st.k - 1), sizeof e, cudaMemcpyDeviceToHost, stream_));
  sync();
  ntf_trace_record r{};
  r.iter = st.k;
  r.time_s = e.time_s;
  r.f = e.f;
  r.inner_sweeps = e.sweeps;
  if (algo_ == 0) {
    r.has_restarted = 1;
    r.restarted = e.restarted;
    r.has_beta = 1;
    r.beta = e.beta;
  }
  *out = r;
  return true;
}

void Session::snapshot(double* factors_out, ntf_trace_record* last, int* k, bool* done) {
  const size_t fac_bytes = factors_out ? size_t(2 * total_factor_len_) * sizeof(double) : 0;
  const size_t off_state = (sizeof(DevFactors) + 63) / 64 * 64;
  const size_t off_rec = off_state + (sizeof(RunState) + 63) / 64 * 64;
  const size_t off_fac = off_rec + 64;
  unsigned char* h = static_cast<unsigned char*>(ctx_->staging(off_fac + fac_bytes));
  // the newest record is entry host_iters_ - 1 unless the run stopped earlier (then a second, rare, copy)
  const int guess = std::min(host_iters_, trace_cap_) - 1;
  NTF_CUDA(cudaMemcpyAsync(h, dF_.p, sizeof(DevFactors), cudaMemcpyDeviceToHost, stream_));
  NTF_CUDA(cudaMemcpyAsync(h + off_state, state_.p, sizeof(RunState), cudaMemcpyDeviceToHost, stream_));
  if (guess >= 0)
    NTF_CUDA(cudaMemcpyAsync(h + off_rec, trace_.as<TraceEntry>() + guess, sizeof(TraceEntry), cudaMemcpyDeviceToHost, stream_));
  if (fac_bytes) NTF_CUDA(cudaMemcpyAsync(h + off_fac, fac_.p, fac_bytes, cudaMemcpyDeviceToHost, stream_));
  sync();
  DevFactors hf;
  RunState st;
  std::memcpy(&hf, h, sizeof hf);
  std::memcpy(&st, h + off_state, sizeof st);
  *k = st.k;
  *done = st.done != 0;
  if (factors_out) {
    const double* fac = reinterpret_cast<const double*>(h + off_fac);
    long long off = 0;
    for (int i = 0; i < order_; ++i) {
      const long long nn = (long long)rows_[i] * rank_;
      std::memcpy(factors_out + off, fac + 2 * off + (hf.sel[i] ? nn : 0), size_t(nn) * sizeof(double));
      off += nn;
    }
  }
  if (last && st.k >= 1 && st.k <= trace_cap_) {
    TraceEntry e;
    if (st.k - 1 == guess) {
      std::memcpy(&e, h + off_rec, sizeof e);
    } else {
      NTF_CUDA(cudaMemcpyAsync(&e, trace_.as<TraceEntry>() + (st.k - 1), sizeof e, cudaMemcpyDeviceToHost, stream_));
      sync();
    }
    ntf_trace_record r{};
    r.iter = st.k;
    r.time_s = e.time_s;
    r.f = e.f;
    r.inner_sweeps = e.sweeps;
    if (algo_ == 0) {
      r.has_restarted = 1;
      r.restarted = e.restarted;
      r.has_beta = 1;
      r.beta = e.beta;
    }
    *last = r;
  }
}

void Session::finish(double* out_factors, double* f0, ntf_trace_record* out, int cap, int* n) {
  const int m0 = std::max(0, std::min(cap, trace_cap_));
  if (m0 > 4096) {  // a long trace: its length first, then only the records that exist
    check_error();
    factors(out_factors);
    trace(f0, out, cap, n);
    return;
  }
  const size_t fac_bytes = size_t(2 * total_factor_len_) * sizeof(double);
  const size_t tr_bytes = size_t(m0) * sizeof(TraceEntry);
  const size_t off_state = (sizeof(DevFactors) + 63) / 64 * 64;
  const size_t off_trace = off_state + (sizeof(RunState) + 63) / 64 * 64;
  const size_t off_fac = off_trace + (tr_bytes + 63) / 64 * 64;
  unsigned char* h = static_cast<unsigned char*>(ctx_->staging(off_fac + fac_bytes));
  NTF_CUDA(cudaMemcpyAsync(h, dF_.p, sizeof(DevFactors), cudaMemcpyDeviceToHost, stream_));
  NTF_CUDA(cudaMemcpyAsync(h + off_state, state_.p, sizeof(RunState), cudaMemcpyDeviceToHost, stream_));
  if (tr_bytes) NTF_CUDA(cudaMemcpyAsync(h + off_trace, trace_.p, tr_bytes, cudaMemcpyDeviceToHost, stream_));
  NTF_CUDA(cudaMemcpyAsync(h + off_fac, fac_.p, fac_bytes, cudaMemcpyDeviceToHost, stream_));
  sync();
  DevFactors hf;
  RunState st;
  std::memcpy(&hf, h, sizeof hf);
  std::memcpy(&st, h + off_state, sizeof st);
  if (st.error) throw std::runtime_error(solver_error_message(st.error));
  const double* fac = reinterpret_cast<const double*>(h + off_fac);
  long long off = 0;
  for (int i = 0; i < order_; ++i) {  // x[i][b] = fac_ + 2 off + b n (the constructor's layout)
    const long long nn = (long long)rows_[i] * rank_;
    std::memcpy(out_factors + off, fac + 2 * off + (hf.sel[i] ? nn : 0), size_t(nn) * sizeof(double));
    off += nn;
  }
  if (f0) *f0 = st.f0;
  *n = st.k;
  const TraceEntry* tr = reinterpret_cast<const TraceEntry*>(h + off_trace);
  for (int i = 0; i < std::min(st.k, m0); ++i) {
    ntf_trace_record r{};
    r.iter = i + 1;
    r.time_s = tr[i].time_s;
    r.f = tr[i].f;
    r.inner_sweeps = tr[i].sweeps;
    if (algo_ == 0) {
      r.has_restarted = 1;
      r.restarted = tr[i].restarted;
      r.has_beta = 1;
      r.beta = tr[i].beta;
    }
    out[i] = r;
  }
}

void Session::check_error() {
  int e = 0;
  NTF_CUDA(cudaMemcpyAsync(&e, &state_.as<RunState>()->error, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  sync();
  if (e) throw std::runtime_error(solver_error_message(e));
}

void Session::set_kernel_timing(bool on) { timing_ = on; }

void Session::kernel_times(double* ms_per_mode, int* launches, int* total_kernels) {
  sync();
  for (size_t k = 0; k < ev_mode_.size(); ++k) {
    if (ev_mode_[k] < 0) continue;
    float ms = 0.f;
    NTF_CUDA(cudaEventElapsedTime(&ms, ev_[2 * k], ev_[2 * k + 1]));
    kernel_ms_[ev_mode_[k]] += ms;
    kernel_n_[ev_mode_[k]] += 1;
  }
  for (auto e : ev_) cudaEventDestroy(e);
  ev_.clear();
  ev_mode_.clear();
  int total = 0;
  for (int i = 0; i < order_; ++i) {
    if (ms_per_mode) ms_per_mode[i] = kernel_ms_[i];
    if (launches) launches[i] = kernel_n_[i];
    total += eng_->kernels_per_call(i) + 1;  // MTTKRP kernels + fused NNLS
  }
  if (total_kernels) *total_kernels = total;
}

}  // namespace ntfb

ntf_tensor::~ntf_tensor() {
  if (ready) cudaEventDestroy(ready);
}

void* ntf_ctx::staging(size_t bytes) const {
  if (bytes > pinned_bytes) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    pinned_bytes = 0;
    const size_t want = std::max<size_t>(bytes, 1 << 20);
    NTF_CUDA(cudaHostAlloc(&pinned, want, cudaHostAllocDefault));
    pinned_bytes = want;
  }
  return pinned;
}

ntf_ctx::~ntf_ctx() {
  if (pinned) cudaFreeHost(pinned);
  if (setup) cudaStreamDestroy(setup);
  if (stream) cudaStreamDestroy(stream);
}
