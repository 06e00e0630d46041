// ntf_b200.hpp — header-only C++ mirror of the reference solver API over the
// C ABI in ntf_b200.h. Names and semantics follow /root/reference/proj:
//   ntfb::AoConfig, ntfb::HerParams, ntfb::InnerStop     (ao.hpp, her.hpp, nnls.hpp)
//   ntfb::KruskalModel, ntfb::RunTrace, ntfb::TraceRecord (kruskal.hpp, trace.hpp)
//   ntfb::ObjectiveProvider / ntfb::GpuDenseProvider      (provider.hpp)
//   ntfb::her_run / ntfb::ao_run / generate / random_init (her.hpp, ao.hpp, datagen.hpp)
// Errors are rethrown as the reference's exception classes
// (std::invalid_argument, std::logic_error, std::runtime_error).
//
// Matrices are row-major here (r contiguous per row); the reference's Eigen
// col-major factors convert with a transpose copy.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <optional>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ntf_b200.h"

namespace ntfb {

inline void check(int rc) {
  if (rc == NTF_OK) return;
  char buf[1024];
  ntf_last_error(buf, sizeof buf);
  if (rc == NTF_ERR_INVALID_ARGUMENT) throw std::invalid_argument(buf);
  if (rc == NTF_ERR_LOGIC) throw std::logic_error(buf);
  throw std::runtime_error(buf);
}

// Row-major dense matrix (rows x cols).
struct Matrix {
  int rows = 0, cols = 0;
  std::vector<double> v;
  Matrix() = default;
  Matrix(int r, int c, double fill = 0.0) : rows(r), cols(c), v(size_t(r) * c, fill) {}
  double& operator()(int i, int j) { return v[size_t(i) * cols + j]; }
  double operator()(int i, int j) const { return v[size_t(i) * cols + j]; }
};

struct KruskalModel {
  std::vector<Matrix> factors;
  int order() const { return int(factors.size()); }
  int rank() const { return factors.empty() ? 0 : factors[0].cols; }
  std::vector<int> shape() const {
    std::vector<int> s;
    for (auto& f : factors) s.push_back(f.rows);
    return s;
  }
  const Matrix& factor(int mode) const { return factors[size_t(mode)]; }
  Matrix& factor(int mode) { return factors[size_t(mode)]; }
  std::vector<double> flat() const {
    std::vector<double> out;
    for (auto& f : factors) out.insert(out.end(), f.v.begin(), f.v.end());
    return out;
  }
  static KruskalModel from_flat(const double* p, const std::vector<int>& shape, int rank) {
    KruskalModel m;
    for (int d : shape) {
      Matrix a(d, rank);
      std::copy(p, p + size_t(d) * rank, a.v.begin());
      p += size_t(d) * rank;
      m.factors.push_back(std::move(a));
    }
    return m;
  }
};

enum class NnlsSolver { ahals = NTF_SOLVER_AHALS, admm, nesterov, pgd, active_set };
struct InnerStop {
  int max_iters = 50;
  double rel_change_tol = 1e-2;
};
struct AoConfig {
  NnlsSolver solver = NnlsSolver::ahals;
  InnerStop inner_stop;
  int max_outer_iters = 0;
  double max_time_s = 0.0;
  bool record_factor_error = false;
  const KruskalModel* ground_truth = nullptr;
  unsigned flags = 0;  // NTF_RUN_* (0: dimension tree, graph replay -- the production path)
  void validate() const {
    const ntf_ao_config c = c_struct(nullptr);
    check(ntf_ao_config_validate(&c));
  }
  ntf_ao_config c_struct(const std::vector<double>* truth) const {
    ntf_ao_config c;
    ntf_ao_config_default(&c);
    c.solver = int(solver);
    c.inner_stop = ntf_inner_stop{inner_stop.max_iters, inner_stop.rel_change_tol};
    c.max_outer_iters = max_outer_iters;
    c.max_time_s = max_time_s;
    c.record_factor_error = record_factor_error ? 1 : 0;
    static const double kDummy = 0.0;
    c.ground_truth = truth ? truth->data() : (record_factor_error && ground_truth ? &kDummy : nullptr);
    c.flags = flags;
    return c;
  }
};
struct HerParams {
  double beta0 = 0.5, gamma = 1.05, gamma_bar = 1.01, eta = 1.5;
  void validate() const {
    ntf_her_params p{beta0, gamma, gamma_bar, eta};
    check(ntf_her_params_validate(&p));
  }
};

struct TraceRecord {
  int iter = 0;
  double time_s = 0.0, f = 0.0;
  std::optional<double> e;
  std::optional<bool> restarted;
  std::optional<double> beta;
};
struct RunTrace {
  double f0 = 0.0;
  std::vector<TraceRecord> records;
  int restart_count() const {
    int n = 0;
    for (auto& r : records) n += (r.restarted && *r.restarted) ? 1 : 0;
    return n;
  }
  double final_f() const {
    if (records.empty()) throw std::logic_error("empty trace");
    return records.back().f;
  }
};

struct HerIterationInfo {
  int iter = 0;
  double f_hat = 0.0;
  bool restarted = false;
  double beta_used = 0.0;
  const KruskalModel* factors = nullptr;
  const KruskalModel* hat_factors = nullptr;
};
using HerObserver = std::function<void(const HerIterationInfo&)>;

// One GPU (or one rank of an NCCL world).
class Context {
 public:
  explicit Context(int device = 0) { check(ntf_ctx_create(device, &h_)); }
  Context(int device, int rank, int world, const unsigned char id[128]) {
    check(ntf_ctx_create_dist(device, rank, world, id, &h_));
  }
  ~Context() { ntf_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ntf_ctx* get() const { return h_; }

 private:
  ntf_ctx* h_ = nullptr;
};

// ObjectiveProvider (provider.hpp:14-20).
class ObjectiveProvider {
 public:
  virtual ~ObjectiveProvider() = default;
  virtual std::vector<int> shape() const = 0;
  virtual double norm_sq() const = 0;
  virtual Matrix mttkrp(const KruskalModel& m, int mode) const = 0;
};

// A provider whose data lives on the GPU (dense tensor or Tucker format):
// the drivers below run the whole iteration on the device for any of them.
class GpuProvider : public ObjectiveProvider {
 public:
  ~GpuProvider() override { ntf_tensor_destroy(t_); }
  GpuProvider(const GpuProvider&) = delete;
  GpuProvider& operator=(const GpuProvider&) = delete;

  std::vector<int> shape() const override { return shape_; }
  double norm_sq() const override {
    double v = 0.0;
    check(ntf_tensor_norm_sq(t_, &v));
    return v;
  }
  Matrix mttkrp(const KruskalModel& m, int mode) const override {
    if (m.shape() != shape_) throw std::invalid_argument("mttkrp: model/tensor shape mismatch");
    Matrix out(shape_[size_t(mode)], m.rank());
    const auto flat = m.flat();
    check(ntf_mttkrp(ctx_->get(), t_, flat.data(), m.rank(), mode, out.v.data()));
    return out;
  }
  ntf_ctx* ctx() const { return ctx_->get(); }
  const ntf_tensor* tensor() const { return t_; }

 protected:
  GpuProvider(Context& ctx, std::vector<int> shape) : ctx_(&ctx), shape_(std::move(shape)) {}
  Context* ctx_;
  std::vector<int> shape_;
  ntf_tensor* t_ = nullptr;
};

// DenseProvider (provider.hpp:22-34) with the tensor resident on the GPU.
class GpuDenseProvider final : public GpuProvider {
 public:
  // `data`: this rank's mode-1 slab (row-major, last index fastest) of a
  // tensor of full shape `shape`; FP64 or FP32.
  template <typename T>
  GpuDenseProvider(Context& ctx, const T* data, const std::vector<int>& shape) : GpuProvider(ctx, shape) {
    static_assert(std::is_same<T, double>::value || std::is_same<T, float>::value, "FP64 or FP32 tensors");
    std::vector<int64_t> s(shape.begin(), shape.end());
    check(ntf_tensor_upload(ctx.get(), data, std::is_same<T, float>::value ? NTF_DTYPE_F32 : NTF_DTYPE_F64,
                            int(shape.size()), s.data(), &t_));
  }
};

// TuckerFormat (tucker.hpp:14-35): core (row-major, dims = basis column
// counts) and one basis per mode with orthonormal columns.
struct TuckerFormat {
  std::vector<int> core_shape;
  std::vector<double> core;
  std::vector<Matrix> bases;  // I_p x r_p, row-major
  std::vector<int> full_shape() const {
    std::vector<int> s;
    for (const auto& b : bases) s.push_back(int(b.rows));
    return s;
  }
  // TuckerFormat::save / load (tucker.cpp:106-165): the NTFK container
  void save(const std::string& path) const {
    std::vector<int64_t> f, r;
    for (const auto& b : bases) f.push_back(b.rows);
    for (int d : core_shape) r.push_back(d);
    const auto flat = flat_bases();
    check(ntf_ntfk_write(path.c_str(), core.data(), flat.data(), int(bases.size()), f.data(), r.data()));
  }
  static TuckerFormat load(const std::string& path) {
    int order = 0;
    int64_t f[NTF_MAX_ORDER], r[NTF_MAX_ORDER];
    check(ntf_ntfk_info(path.c_str(), &order, f, r));
    TuckerFormat t;
    int64_t nc = 1, nb = 0;
    for (int l = 0; l < order; ++l) {
      t.core_shape.push_back(int(r[l]));
      nc *= r[l];
      nb += f[l] * r[l];
    }
    t.core.resize(size_t(nc));
    std::vector<double> flat(static_cast<size_t>(nb));
    check(ntf_ntfk_read(path.c_str(), t.core.data(), flat.data()));
    size_t off = 0;
    for (int l = 0; l < order; ++l) {
      Matrix b(f[l], r[l]);
      std::copy(flat.begin() + std::ptrdiff_t(off), flat.begin() + std::ptrdiff_t(off + b.v.size()), b.v.begin());
      off += b.v.size();
      t.bases.push_back(std::move(b));
    }
    return t;
  }
  std::vector<double> flat_bases() const {
    std::vector<double> flat;
    for (const auto& b : bases) flat.insert(flat.end(), b.v.begin(), b.v.end());
    return flat;
  }
};

// TuckerProvider (tucker.hpp:60-73): the MTTKRP runs in the compressed space
// on the GPU; norm_sq() is ||core||^2. Validates like TuckerFormat::validate.
class TuckerProvider final : public GpuProvider {
 public:
  TuckerProvider(Context& ctx, const TuckerFormat& fmt) : GpuProvider(ctx, fmt.full_shape()) {
    std::vector<int64_t> f(shape_.begin(), shape_.end()), r(fmt.core_shape.begin(), fmt.core_shape.end());
    const auto flat = fmt.flat_bases();
    check(ntf_tucker_upload(ctx.get(), fmt.core.data(), int(fmt.bases.size()), r.data(), flat.data(), f.data(), &t_));
  }
};

namespace detail {
inline RunTrace to_trace(double f0, const std::vector<ntf_trace_record>& recs, int n) {
  RunTrace t;
  t.f0 = f0;
  for (int i = 0; i < n && i < int(recs.size()); ++i) {
    const auto& r = recs[size_t(i)];
    TraceRecord o;
    o.iter = r.iter;
    o.time_s = r.time_s;
    o.f = r.f;
    if (r.has_e) o.e = r.e;
    if (r.has_restarted) o.restarted = r.restarted != 0;
    if (r.has_beta) o.beta = r.beta;
    t.records.push_back(o);
  }
  return t;
}
inline const GpuProvider& gpu(const ObjectiveProvider& p) {
  auto* g = dynamic_cast<const GpuProvider*>(&p);
  if (!g) throw std::runtime_error("her_run/ao_run need a GPU-resident provider (GpuDenseProvider, TuckerProvider)");
  return *g;
}
}  // namespace detail

// her_run (her.hpp:63-66).
inline std::pair<KruskalModel, RunTrace> her_run(const ObjectiveProvider& data, const KruskalModel& init,
                                                 const AoConfig& cfg, const HerParams& params,
                                                 const HerObserver& observer = {}) {
  const auto& g = detail::gpu(data);
  std::vector<double> truth;
  if (cfg.record_factor_error && cfg.ground_truth) truth = cfg.ground_truth->flat();
  const ntf_ao_config c = cfg.c_struct(truth.empty() ? nullptr : &truth);
  const ntf_her_params p{params.beta0, params.gamma, params.gamma_bar, params.eta};
  const auto flat = init.flat();
  std::vector<double> out(flat.size());
  const int cap = cfg.max_outer_iters > 0 ? cfg.max_outer_iters : (1 << 20);
  std::vector<ntf_trace_record> recs(static_cast<size_t>(cap));
  double f0 = 0.0;
  int n = 0;
  struct Tramp {
    const HerObserver* obs;
    std::vector<int> shape;
    int rank;
    static void call(const ntf_her_iteration_info* i, void* u) {
      auto* t = static_cast<Tramp*>(u);
      const KruskalModel acc = KruskalModel::from_flat(i->factors, t->shape, t->rank);
      const KruskalModel hat = KruskalModel::from_flat(i->hat_factors, t->shape, t->rank);
      HerIterationInfo info{i->iter, i->f_hat, i->restarted != 0, i->beta_used, &acc, &hat};
      (*t->obs)(info);
    }
  } tramp{&observer, g.shape(), init.rank()};
  check(ntf_her_run(g.ctx(), g.tensor(), flat.data(), init.rank(), &c, &p, observer ? &Tramp::call : nullptr,
                    &tramp, out.data(), &f0, recs.data(), cap, &n));
  return {KruskalModel::from_flat(out.data(), g.shape(), init.rank()), detail::to_trace(f0, recs, n)};
}

// ao_run (ao.hpp:30-31).
inline std::pair<KruskalModel, RunTrace> ao_run(const ObjectiveProvider& data, const KruskalModel& init,
                                                const AoConfig& cfg) {
  const auto& g = detail::gpu(data);
  std::vector<double> truth;
  if (cfg.record_factor_error && cfg.ground_truth) truth = cfg.ground_truth->flat();
  const ntf_ao_config c = cfg.c_struct(truth.empty() ? nullptr : &truth);
  const auto flat = init.flat();
  std::vector<double> out(flat.size());
  const int cap = cfg.max_outer_iters > 0 ? cfg.max_outer_iters : (1 << 20);
  std::vector<ntf_trace_record> recs(static_cast<size_t>(cap));
  double f0 = 0.0;
  int n = 0;
  check(ntf_ao_run(g.ctx(), g.tensor(), flat.data(), init.rank(), &c, out.data(), &f0, recs.data(), cap, &n));
  return {KruskalModel::from_flat(out.data(), g.shape(), init.rank()), detail::to_trace(f0, recs, n)};
}

// Synthetic data (datagen.hpp:14-44).
struct SyntheticSpec {
  std::vector<int> shape;
  int rank = 1;
  double noise_sigma = 0.0;
  bool ill_conditioned = false;
  std::uint64_t seed = 0;
};
inline std::uint64_t stream_seed(std::uint64_t base, std::uint64_t stream) { return ntf_stream_seed(base, stream); }
inline KruskalModel random_init(const std::vector<int>& shape, int rank, std::uint64_t seed) {
  size_t n = 0;
  for (int d : shape) n += size_t(d) * rank;
  std::vector<double> out(n);
  check(ntf_random_init(shape.data(), int(shape.size()), rank, seed, out.data()));
  return KruskalModel::from_flat(out.data(), shape, rank);
}
// Returns the row-major FP64 tensor and the truth factors.
inline std::pair<std::vector<double>, KruskalModel> generate(const SyntheticSpec& spec) {
  size_t total = 1, n = 0;
  for (int d : spec.shape) {
    total *= size_t(d);
    n += size_t(d) * spec.rank;
  }
  std::vector<double> t(total), truth(n ? n : 1);
  check(ntf_generate(spec.shape.data(), int(spec.shape.size()), spec.rank, spec.noise_sigma,
                     spec.ill_conditioned ? 1 : 0, 0, spec.seed, NTF_DTYPE_F64, t.data(), truth.data()));
  return {std::move(t), KruskalModel::from_flat(truth.data(), spec.shape, spec.rank)};
}

}  // namespace ntfb
