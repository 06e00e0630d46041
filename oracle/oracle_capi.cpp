// TEST INFRASTRUCTURE ONLY — extern "C" surface of the CPU oracle, loaded by
// tests/ (ctypes) and by bench.py's cpu_baseline / --impl reference legs.
// Factor matrices cross this boundary row-major, modes concatenated.
#include <omp.h>

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "ntf_oracle.hpp"

namespace {

thread_local std::string g_err;

std::vector<int> to_shape(const int* shape, int order) { return std::vector<int>(shape, shape + order); }

ora::Model unpack(const double* flat, const int* shape, int order, int rank) {
  ora::Model m;
  size_t off = 0;
  for (int i = 0; i < order; ++i) {
    ora::Mat a(shape[i], rank);
    std::memcpy(a.v.data(), flat + off, sizeof(double) * a.v.size());
    off += a.v.size();
    m.push_back(std::move(a));
  }
  return m;
}

void pack(const ora::Model& m, double* flat) {
  size_t off = 0;
  for (auto& a : m) {
    std::memcpy(flat + off, a.v.data(), sizeof(double) * a.v.size());
    off += a.v.size();
  }
}

ora::Mat to_mat(const double* p, int rows, int cols) {
  ora::Mat a(rows, cols);
  std::memcpy(a.v.data(), p, sizeof(double) * a.v.size());
  return a;
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

struct Rec {  // mirrors ora_trace_record below
  int iter, has_e, has_restart, restarted, has_beta, pad;
  double time_s, f, e, beta;
};

void export_trace(const ora::RunTrace& t, double* f0, Rec* recs, int cap, int* n) {
  *f0 = t.f0;
  *n = int(t.records.size());
  for (int i = 0; i < *n && i < cap; ++i) {
    const auto& r = t.records[size_t(i)];
    recs[i] = Rec{r.iter, r.has_e, r.has_restart, r.restarted, r.has_beta, 0, r.time_s, r.f, r.e, r.beta};
  }
}

}  // namespace

extern "C" {

const char* ora_last_error() { return g_err.c_str(); }

unsigned long long ora_stream_seed(unsigned long long base, unsigned long long stream) {
  return ora::stream_seed(base, stream);
}

// The (skip+1)-th output of std::mt19937_64(seed).
unsigned long long ora_mt19937_64_draw(unsigned long long seed, unsigned long long skip) {
  std::mt19937_64 g(seed);
  g.discard(skip);
  return g();
}

void ora_uniform_normal(unsigned long long seed, int n, double* uni, double* nrm) {
  std::mt19937_64 g(seed);
  for (int i = 0; i < n; ++i) uni[i] = ora::draw_uniform01(g);
  for (int i = 0; i < n; ++i) nrm[i] = ora::draw_normal(g);
}

int ora_generate(const int* shape, int order, int rank, double sigma, int ill, int collinear,
                 unsigned long long seed, double* tensor_out, double* truth_out) {
  return guard([&] {
    std::vector<double> t;
    ora::Model truth;
    ora::generate(to_shape(shape, order), rank, sigma, ill != 0, collinear != 0, seed, t, truth);
    std::memcpy(tensor_out, t.data(), sizeof(double) * t.size());
    pack(truth, truth_out);
  });
}

int ora_random_init(const int* shape, int order, int rank, unsigned long long seed, double* out) {
  return guard([&] { pack(ora::random_init(to_shape(shape, order), rank, seed), out); });
}

int ora_mttkrp(const void* tensor, int dtype, const int* shape, int order, const double* factors,
               int rank, int mode, double* out) {
  return guard([&] {
    const auto sh = to_shape(shape, order);
    const auto m = unpack(factors, shape, order, rank);
    const ora::Mat c = dtype == 1 ? ora::mttkrp(static_cast<const float*>(tensor), sh, m, mode)
                                  : ora::mttkrp(static_cast<const double*>(tensor), sh, m, mode);
    std::memcpy(out, c.v.data(), sizeof(double) * c.v.size());
  });
}

int ora_ref_mttkrp(const double* tensor, const int* shape, int order, const double* factors, int rank,
                   int mode, double* out) {
  return guard([&] {
    const auto m = unpack(factors, shape, order, rank);
    const ora::Mat c = ora::ref_mttkrp(tensor, to_shape(shape, order), m, mode);
    std::memcpy(out, c.v.data(), sizeof(double) * c.v.size());
  });
}

int ora_ref_objective(const double* tensor, const int* shape, int order, const double* factors, int rank,
                      double* out) {
  return guard([&] {
    *out = ora::ref_objective(tensor, to_shape(shape, order), unpack(factors, shape, order, rank));
  });
}

int ora_reconstruct(const int* shape, int order, const double* factors, int rank, double* out) {
  return guard([&] {
    std::vector<double> t;
    ora::reconstruct(unpack(factors, shape, order, rank), t);
    std::memcpy(out, t.data(), sizeof(double) * t.size());
  });
}

double ora_norm_sq(const void* tensor, int dtype, long long n) {
  return dtype == 1 ? ora::norm_sq(static_cast<const float*>(tensor), n)
                    : ora::norm_sq(static_cast<const double*>(tensor), n);
}

void ora_gram(const double* a, int rows, int r, double* out) {
  const ora::Mat g = ora::gram(to_mat(a, rows, r));
  std::memcpy(out, g.v.data(), sizeof(double) * g.v.size());
}

// grams: `count` r x r matrices back to back.
void ora_hadamard_of_grams(const double* grams, int count, int r, int skip, double* out) {
  std::vector<ora::Mat> gs;
  for (int i = 0; i < count; ++i) gs.push_back(to_mat(grams + size_t(i) * r * r, r, r));
  const ora::Mat h = ora::hadamard_of_grams(gs, skip);
  std::memcpy(out, h.v.data(), sizeof(double) * h.v.size());
}

double ora_cheap_objective(double nsq, const double* a, const double* g, const double* c, int rows, int r) {
  return ora::cheap_objective(nsq, to_mat(a, rows, r), to_mat(g, r, r), to_mat(c, rows, r));
}

void ora_hals_pass(const double* g, const double* c, const double* w, int rows, int r, double* out) {
  const ora::Mat o = ora::hals_pass(to_mat(g, r, r), to_mat(c, rows, r), to_mat(w, rows, r));
  std::memcpy(out, o.v.data(), sizeof(double) * o.v.size());
}

int ora_ahals_solve(const double* g, const double* c, const double* w0, int rows, int r, int max_iters,
                    double tol, double* out) {
  int sweeps = 0;
  const ora::Mat o = ora::ahals_solve(to_mat(g, r, r), to_mat(c, rows, r), to_mat(w0, rows, r),
                                      ora::InnerStop{max_iters, tol}, &sweeps);
  std::memcpy(out, o.v.data(), sizeof(double) * o.v.size());
  return sweeps;
}

void ora_extrapolate(const double* a_new, const double* a_old, int rows, int r, double beta, double* out) {
  const ora::Mat o = ora::extrapolate_block(to_mat(a_new, rows, r), to_mat(a_old, rows, r), beta);
  std::memcpy(out, o.v.data(), sizeof(double) * o.v.size());
}

// state = {beta, beta_bar}
void ora_update_betas(double* state, int restarted, double beta0, double gamma, double gamma_bar, double eta) {
  ora::HerState s;
  s.beta = state[0];
  s.beta_bar = state[1];
  ora::update_betas(s, restarted != 0, ora::HerParams{beta0, gamma, gamma_bar, eta});
  state[0] = s.beta;
  state[1] = s.beta_bar;
}

int ora_validate_her_params(double beta0, double gamma, double gamma_bar, double eta) {
  return guard([&] { ora::validate_her_params(ora::HerParams{beta0, gamma, gamma_bar, eta}); });
}

double ora_factor_error(const double* est, const double* truth, const int* shape, int order, int rank) {
  return ora::factor_error(unpack(est, shape, order, rank), unpack(truth, shape, order, rank));
}

int ora_hungarian(const double* cost, int n, int* mapping, double* total) {
  return guard([&] {
    const auto m = ora::hungarian(to_mat(cost, n, n), total);
    for (int i = 0; i < n; ++i) mapping[i] = m[size_t(i)];
  });
}

typedef void (*ora_observer_cb)(void* user, int k, double f_hat, int restarted, double beta_used,
                                const double* accepted, const double* hat);

namespace {
struct ObsCtx {
  ora_observer_cb cb;
  void* user;
  std::vector<double> acc, hat;
};
void obs_tramp(void* u, int k, double f, int rs, double b, const ora::Model& acc, const ora::Model& hat) {
  auto* o = static_cast<ObsCtx*>(u);
  pack(acc, o->acc.data());
  pack(hat, o->hat.data());
  o->cb(o->user, k, f, rs, b, o->acc.data(), o->hat.data());
}
}  // namespace

// algo: 0 = HER, 1 = AO. truth may be null (no e_k).
int ora_run(int algo, int solver, const void* tensor, int dtype, const int* shape, int order, const double* init,
            int rank, int inner_max_iters, double inner_tol, int max_outer_iters, double max_time_s,
            const double* truth, double beta0, double gamma, double gamma_bar, double eta,
            double* out_factors, double* f0, void* records, int cap, int* n_records,
            ora_observer_cb cb, void* user) {
  return guard([&] {
    const auto sh = to_shape(shape, order);
    const auto m0 = unpack(init, shape, order, rank);
    ora::Model tm;
    ora::AoConfig cfg;
    cfg.inner = ora::InnerStop{inner_max_iters, inner_tol};
    cfg.solver = solver;
    cfg.max_outer_iters = max_outer_iters;
    cfg.max_time_s = max_time_s;
    if (truth) {
      tm = unpack(truth, shape, order, rank);
      cfg.ground_truth = &tm;
    }
    ora::RunTrace trace;
    ora::Model out;
    size_t total = 0;
    for (int i = 0; i < order; ++i) total += size_t(shape[i]) * rank;
    ObsCtx octx{cb, user, std::vector<double>(total), std::vector<double>(total)};
    ora::HerObserverFn obs;
    if (cb) {
      obs.fn = obs_tramp;
      obs.user = &octx;
    }
    const ora::HerParams hp{beta0, gamma, gamma_bar, eta};
    if (dtype == 1) {
      const float* t = static_cast<const float*>(tensor);
      out = algo == 0 ? ora::her_run(t, sh, m0, cfg, hp, trace, obs) : ora::ao_run(t, sh, m0, cfg, trace);
    } else {
      const double* t = static_cast<const double*>(tensor);
      out = algo == 0 ? ora::her_run(t, sh, m0, cfg, hp, trace, obs) : ora::ao_run(t, sh, m0, cfg, trace);
    }
    pack(out, out_factors);
    export_trace(trace, f0, static_cast<Rec*>(records), cap, n_records);
  });
}

}  // extern "C"

// OpenMP thread count of the oracle's parallel loops (bench.py's 1-thread and
// all-core CPU baselines); returns the previous maximum.
extern "C" int ora_set_threads(int n) {
  const int prev = omp_get_max_threads();
  if (n > 0) omp_set_num_threads(n);
  return prev;
}

// MTTKRP summation order (0 = the reference's, 1 = descending): conditioning
// experiments only (tools/r02/oracle_sensitivity.py).
extern "C" void ora_set_sum_order(int order) { ora::g_sum_order = order; }

// compressed_mttkrp (tucker.cpp:62-77): core row-major (core_shape), bases
// concatenated row-major (full_shape[l] x core_shape[l]), factors as usual.
extern "C" int ora_compressed_mttkrp(const double* core, const int* core_shape, const double* bases,
                                     const int* full_shape, int order, const double* factors, int rank, int mode,
                                     double* out) {
  try {
    std::vector<ora::Mat> bs;
    size_t off = 0;
    for (int l = 0; l < order; ++l) {
      ora::Mat b(full_shape[l], core_shape[l]);
      std::memcpy(b.v.data(), bases + off, b.v.size() * sizeof(double));
      off += b.v.size();
      bs.push_back(std::move(b));
    }
    const ora::Model m = unpack(factors, full_shape, order, rank);
    const ora::Mat c = ora::compressed_mttkrp(core, std::vector<int>(core_shape, core_shape + order), bs, m, mode);
    std::memcpy(out, c.v.data(), c.v.size() * sizeof(double));
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// solve_nnls (nnls.cpp:213-222) with any solver: g r x r, c / w0 / out rows x r.
extern "C" int ora_solve_nnls(int solver, const double* g, const double* c, const double* w0, int rows, int r,
                              int max_iters, double tol, double* out) {
  return guard([&] {
    ora::Mat gm(r, r), cm(rows, r), wm(rows, r);
    std::memcpy(gm.v.data(), g, gm.v.size() * sizeof(double));
    std::memcpy(cm.v.data(), c, cm.v.size() * sizeof(double));
    std::memcpy(wm.v.data(), w0, wm.v.size() * sizeof(double));
    const ora::Mat w = ora::solve_nnls(solver, gm, cm, wm, ora::InnerStop{max_iters, tol});
    std::memcpy(out, w.v.data(), w.v.size() * sizeof(double));
  });
}

extern "C" double ora_spectral_norm(const double* g, int r) {
  ora::Mat gm(r, r);
  std::memcpy(gm.v.data(), g, gm.v.size() * sizeof(double));
  return ora::spectral_norm(gm);
}
