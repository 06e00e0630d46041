// TEST INFRASTRUCTURE ONLY -- extern "C" surface over the REAL reference
// (the unmodified sources under /root/reference/proj/src, compiled against
// the Eigen stand-in in shim/; see Makefile). It exports the same symbol
// names and signatures as oracle/oracle_capi.cpp, so oracle/pyref.py drives
// the reference through the wrappers of oracle/pyoracle.py and the tests put
// the two side by side (tests/test_ref_build.py). Every function here only
// marshals arrays and calls the reference's own public API:
//   ntf::generate / random_init / stream_seed        (datagen.hpp)
//   ntf::mttkrp / gram / hadamard_of_grams / cheap_objective / spectral_norm
//   ntf::reconstruct                                  (kernels.hpp)
//   ntf::hals_pass / ahals_solve / solve_nnls         (nnls.hpp)
//   ntf::extrapolate_block / update_betas / her_run   (her.hpp)
//   ntf::ao_run                                       (ao.hpp)
//   ntf::factor_error / hungarian                     (metrics.hpp)
//   ntf::ref::mttkrp / objective                      (reference.hpp)
//   ntf::compressed_mttkrp                            (tucker.hpp)
// Factor matrices cross this boundary row-major, modes concatenated.
#include <omp.h>

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "ntf/ao.hpp"
#include "ntf/datagen.hpp"
#include "ntf/her.hpp"
#include "ntf/kernels.hpp"
#include "ntf/metrics.hpp"
#include "ntf/nnls.hpp"
#include "ntf/reference.hpp"
#include "ntf/tucker.hpp"

namespace {

thread_local std::string g_err;

std::vector<int> to_shape(const int* shape, int order) { return std::vector<int>(shape, shape + order); }

Eigen::MatrixXd to_mat(const double* p, int rows, int cols) {
  Eigen::MatrixXd a(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) a(i, j) = p[size_t(i) * cols + j];
  return a;
}

void from_mat(const Eigen::MatrixXd& a, double* p) {
  for (Eigen::Index i = 0; i < a.rows(); ++i)
    for (Eigen::Index j = 0; j < a.cols(); ++j) p[size_t(i) * a.cols() + j] = a(i, j);
}

ntf::KruskalModel unpack(const double* flat, const int* shape, int order, int rank) {
  ntf::KruskalModel m;
  size_t off = 0;
  for (int i = 0; i < order; ++i) {
    m.factors.push_back(to_mat(flat + off, shape[i], rank));
    off += size_t(shape[i]) * rank;
  }
  return m;
}

void pack(const ntf::KruskalModel& m, double* flat) {
  size_t off = 0;
  for (const auto& a : m.factors) {
    from_mat(a, flat + off);
    off += size_t(a.rows()) * a.cols();
  }
}

// The reference stores doubles only; an FP32 data set is widened (exactly).
ntf::DenseTensor to_tensor(const void* data, int dtype, const std::vector<int>& shape) {
  ntf::DenseTensor t(shape);
  if (dtype == 1) {
    const float* s = static_cast<const float*>(data);
    for (std::int64_t i = 0; i < t.size(); ++i) t[i] = double(s[i]);
  } else {
    std::memcpy(t.data(), data, sizeof(double) * size_t(t.size()));
  }
  return t;
}

template <typename F>
int guard(F f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

struct Rec {  // the record layout of oracle_capi.cpp / pyoracle.TraceRec
  int iter, has_e, has_restart, restarted, has_beta, pad;
  double time_s, f, e, beta;
};

ntf::NnlsSolver solver_of(int s) {
  switch (s) {
    case 0: return ntf::NnlsSolver::ahals;
    case 1: return ntf::NnlsSolver::admm;
    case 2: return ntf::NnlsSolver::nesterov;
    case 3: return ntf::NnlsSolver::pgd;
    case 4: return ntf::NnlsSolver::active_set;
  }
  throw std::logic_error("unknown solver");
}

}  // namespace

extern "C" {

const char* ora_last_error() { return g_err.c_str(); }
int ora_is_reference_build() { return 1; }

unsigned long long ora_stream_seed(unsigned long long base, unsigned long long stream) {
  return ntf::stream_seed(base, stream);
}

unsigned long long ora_mt19937_64_draw(unsigned long long seed, unsigned long long skip) {
  std::mt19937_64 g(seed);
  g.discard(skip);
  return g();
}

void ora_uniform_normal(unsigned long long seed, int n, double* uni, double* nrm) {
  std::mt19937_64 g(seed);
  for (int i = 0; i < n; ++i) uni[i] = ntf::draw_uniform01(g);
  for (int i = 0; i < n; ++i) nrm[i] = ntf::draw_normal(g);
}

int ora_generate(const int* shape, int order, int rank, double sigma, int ill, int collinear,
                 unsigned long long seed, double* tensor_out, double* truth_out) {
  return guard([&] {
    if (collinear) throw std::logic_error("the collinear rule is SURVEY 8(d)'s, not a reference generator option");
    ntf::SyntheticSpec spec;
    spec.shape = to_shape(shape, order);
    spec.rank = rank;
    spec.noise_sigma = sigma;
    spec.ill_conditioned = ill != 0;
    spec.seed = seed;
    auto [t, truth] = ntf::generate(spec);
    std::memcpy(tensor_out, t.data(), sizeof(double) * size_t(t.size()));
    pack(truth, truth_out);
  });
}

int ora_random_init(const int* shape, int order, int rank, unsigned long long seed, double* out) {
  return guard([&] { pack(ntf::random_init(to_shape(shape, order), rank, seed), out); });
}

int ora_mttkrp(const void* tensor, int dtype, const int* shape, int order, const double* factors, int rank,
               int mode, double* out) {
  return guard([&] {
    const auto sh = to_shape(shape, order);
    from_mat(ntf::mttkrp(to_tensor(tensor, dtype, sh), unpack(factors, shape, order, rank), mode), out);
  });
}

int ora_ref_mttkrp(const double* tensor, const int* shape, int order, const double* factors, int rank, int mode,
                   double* out) {
  return guard([&] {
    const auto sh = to_shape(shape, order);
    from_mat(ntf::ref::mttkrp(to_tensor(tensor, 0, sh), unpack(factors, shape, order, rank), mode), out);
  });
}

int ora_ref_objective(const double* tensor, const int* shape, int order, const double* factors, int rank,
                      double* out) {
  return guard([&] {
    const auto sh = to_shape(shape, order);
    *out = ntf::ref::objective(to_tensor(tensor, 0, sh), unpack(factors, shape, order, rank));
  });
}

int ora_reconstruct(const int* shape, int order, const double* factors, int rank, double* out) {
  return guard([&] {
    const ntf::DenseTensor t = ntf::reconstruct(unpack(factors, shape, order, rank));
    std::memcpy(out, t.data(), sizeof(double) * size_t(t.size()));
  });
}

double ora_norm_sq(const void* tensor, int dtype, long long n) {
  return to_tensor(tensor, dtype, std::vector<int>{int(n)}).norm_sq();
}

void ora_gram(const double* a, int rows, int r, double* out) { from_mat(ntf::gram(to_mat(a, rows, r)), out); }

void ora_hadamard_of_grams(const double* grams, int count, int r, int skip, double* out) {
  std::vector<Eigen::MatrixXd> gs;
  for (int i = 0; i < count; ++i) gs.push_back(to_mat(grams + size_t(i) * r * r, r, r));
  from_mat(ntf::hadamard_of_grams(gs, skip), out);
}

double ora_cheap_objective(double nsq, const double* a, const double* g, const double* c, int rows, int r) {
  return ntf::cheap_objective(nsq, to_mat(a, rows, r), to_mat(g, r, r), to_mat(c, rows, r));
}

void ora_hals_pass(const double* g, const double* c, const double* w, int rows, int r, double* out) {
  ntf::NnlsProblem p;
  p.gram = to_mat(g, r, r);
  p.target = to_mat(c, rows, r);
  from_mat(ntf::hals_pass(p, to_mat(w, rows, r)), out);
}

// The reference's ahals_solve does not report its sweep count: the count
// returned here replays run_sweeps' loop (nnls.cpp:28-47) over the
// reference's own hals_pass, and the result comes from ahals_solve itself.
int ora_ahals_solve(const double* g, const double* c, const double* w0, int rows, int r, int max_iters, double tol,
                    double* out) {
  ntf::NnlsProblem p;
  p.gram = to_mat(g, r, r);
  p.target = to_mat(c, rows, r);
  p.init = to_mat(w0, rows, r);
  const ntf::InnerStop stop{max_iters, tol};
  from_mat(ntf::ahals_solve(p, stop), out);
  int sweeps = 0;
  Eigen::MatrixXd w = p.init;
  double first = -1.0;
  for (int s = 0; s < max_iters; ++s) {
    const Eigen::MatrixXd next = ntf::hals_pass(p, w);
    const double change = (next - w).norm();
    w = next;
    ++sweeps;
    if (s == 0) first = change;
    if (change <= tol * first) break;
  }
  return sweeps;
}

void ora_extrapolate(const double* a_new, const double* a_old, int rows, int r, double beta, double* out) {
  from_mat(ntf::extrapolate_block(to_mat(a_new, rows, r), to_mat(a_old, rows, r), beta), out);
}

void ora_update_betas(double* state, int restarted, double beta0, double gamma, double gamma_bar, double eta) {
  ntf::HerState s;
  s.beta = state[0];
  s.beta_bar = state[1];
  ntf::HerParams hp;
  hp.beta0 = beta0;
  hp.gamma = gamma;
  hp.gamma_bar = gamma_bar;
  hp.eta = eta;
  ntf::update_betas(s, restarted != 0, hp);
  state[0] = s.beta;
  state[1] = s.beta_bar;
}

int ora_validate_her_params(double beta0, double gamma, double gamma_bar, double eta) {
  return guard([&] {
    ntf::HerParams hp;
    hp.beta0 = beta0;
    hp.gamma = gamma;
    hp.gamma_bar = gamma_bar;
    hp.eta = eta;
    hp.validate();
  });
}

double ora_factor_error(const double* est, const double* truth, const int* shape, int order, int rank) {
  return ntf::factor_error(unpack(est, shape, order, rank), unpack(truth, shape, order, rank));
}

int ora_hungarian(const double* cost, int n, int* mapping, double* total) {
  return guard([&] {
    const ntf::PermutationAssignment a = ntf::hungarian(to_mat(cost, n, n));
    for (int i = 0; i < n; ++i) mapping[i] = a.mapping[size_t(i)];
    *total = a.cost;
  });
}

typedef void (*ora_observer_cb)(void* user, int k, double f_hat, int restarted, double beta_used,
                                const double* accepted, const double* hat);

// algo: 0 = her_run, 1 = ao_run (through DenseProvider, as the reference's
// tensor overloads do). truth may be null (no e_k).
int ora_run(int algo, int solver, const void* tensor, int dtype, const int* shape, int order, const double* init,
            int rank, int inner_max_iters, double inner_tol, int max_outer_iters, double max_time_s,
            const double* truth, double beta0, double gamma, double gamma_bar, double eta, double* out_factors,
            double* f0, void* records, int cap, int* n_records, ora_observer_cb cb, void* user) {
  return guard([&] {
    const auto sh = to_shape(shape, order);
    const ntf::DenseTensor t = to_tensor(tensor, dtype, sh);
    const ntf::KruskalModel m0 = unpack(init, shape, order, rank);
    ntf::KruskalModel tm;
    ntf::AoConfig cfg;
    cfg.solver = solver_of(solver);
    cfg.inner_stop = ntf::InnerStop{inner_max_iters, inner_tol};
    cfg.max_outer_iters = max_outer_iters;
    cfg.max_time_s = max_time_s;
    if (truth) {
      tm = unpack(truth, shape, order, rank);
      cfg.record_factor_error = true;
      cfg.ground_truth = &tm;
    }
    ntf::HerParams hp;
    hp.beta0 = beta0;
    hp.gamma = gamma;
    hp.gamma_bar = gamma_bar;
    hp.eta = eta;
    size_t total = 0;
    for (int i = 0; i < order; ++i) total += size_t(shape[i]) * rank;
    std::vector<double> acc(total), hat(total);
    ntf::HerObserver obs;
    if (cb)
      obs = [&](const ntf::HerIterationInfo& info) {
        pack(*info.factors, acc.data());
        pack(*info.hat_factors, hat.data());
        cb(user, info.iter, info.f_hat, info.restarted ? 1 : 0, info.beta_used, acc.data(), hat.data());
      };
    auto result = algo == 0 ? ntf::her_run(t, m0, cfg, hp, obs) : ntf::ao_run(t, m0, cfg);
    pack(result.first, out_factors);
    const ntf::RunTrace& trace = result.second;
    *f0 = trace.f0;
    *n_records = int(trace.records.size());
    Rec* recs = static_cast<Rec*>(records);
    for (int i = 0; i < *n_records && i < cap; ++i) {
      const ntf::TraceRecord& r = trace.records[size_t(i)];
      recs[i] = Rec{r.iter,           r.e.has_value() ? 1 : 0, r.restarted.has_value() ? 1 : 0, r.restarted.value_or(false) ? 1 : 0,
                    r.beta.has_value() ? 1 : 0, 0, r.time_s, r.f, r.e.value_or(0.0), r.beta.value_or(0.0)};
    }
  });
}

int ora_set_threads(int n) {
  const int prev = omp_get_max_threads();
  if (n > 0) omp_set_num_threads(n);
  return prev;
}

void ora_set_sum_order(int) {}  // an oracle-only experiment switch; the reference has one order

int ora_compressed_mttkrp(const double* core, const int* core_shape, const double* bases, const int* full_shape,
                          int order, const double* factors, int rank, int mode, double* out) {
  return guard([&] {
    ntf::TuckerFormat fmt;
    fmt.core = to_tensor(core, 0, to_shape(core_shape, order));
    size_t off = 0;
    for (int l = 0; l < order; ++l) {
      fmt.bases.push_back(to_mat(bases + off, full_shape[l], core_shape[l]));
      off += size_t(full_shape[l]) * core_shape[l];
    }
    from_mat(ntf::compressed_mttkrp(fmt, unpack(factors, full_shape, order, rank), mode), out);
  });
}

int ora_solve_nnls(int solver, const double* g, const double* c, const double* w0, int rows, int r, int max_iters,
                   double tol, double* out) {
  return guard([&] {
    ntf::NnlsProblem p;
    p.gram = to_mat(g, r, r);
    p.target = to_mat(c, rows, r);
    p.init = to_mat(w0, rows, r);
    from_mat(ntf::solve_nnls(solver_of(solver), p, ntf::InnerStop{max_iters, tol}), out);
  });
}

double ora_spectral_norm(const double* g, int r) { return ntf::spectral_norm(to_mat(g, r, r)); }

}  // extern "C"
