// =============================================================================
// TEST INFRASTRUCTURE ONLY — CPU oracle for the HER-AHALS hot path.
//
// This is a plain C++17 + OpenMP restatement of the reference's dense NTF
// inner loop (arXiv 2001.04321 toolkit under /root/reference/proj). It exists
// so that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs can CHECK the CUDA path and time a CPU baseline. The
// product library (paper_2001_04321_b200/libntf_b200.so) never links, loads or
// calls anything in oracle/.
//
// Parity pinning: the reference's CMake build needs Eigen3, doctest, CLI11 and
// nlohmann-json (absent from the image), but its hot-path sources compile,
// unmodified and from where they lie, against the small Eigen stand-in of
// oracle/ref_build/ into oracle/_ref/libntf_ref.so, and the reference's own
// unit suites pass over that build. This oracle is pinned to that build
// function by function and trace by trace (tests/test_ref_build.py: datagen
// bit for bit, MTTKRP, HALS / every inner solver, whole her_run / ao_run traces
// with identical restart decisions and final factors), to the reference-
// produced runs at the BASELINE configs (tests/golden/refrun_c*.npz), and to
// every known-answer and property test the reference's own suites hold for
// the path (std::mt19937_64 10000th draw, rank-one MTTKRP identity,
// Hadamard-of-Grams == KR^T KR, cheap objective == residual, HALS scalar
// formula, update_betas arithmetic, beta->0 reduction to AO, restart
// bookkeeping, determinism; tests/test_oracle.py). Arithmetic the reference
// delegates to Eigen (GEMV inside hals_pass, Gram GEMM, Frobenius norms,
// redux sums) is restated in plain ascending order -- as the stand-in does --
// so agreement with a real Eigen build is "to rounding", not bitwise.
//
// Storage conventions (shared with the product's C ABI):
//   * tensors: row-major, last index fastest (tensor.hpp:11-13);
//   * factor matrices: row-major I_n x r, modes concatenated in mode order.
// =============================================================================
#pragma once

#include <cstdint>
#include <random>
#include <string>
#include <vector>

namespace ora {

// Row-major dense matrix of doubles.
struct Mat {
  int64_t rows = 0, cols = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(int64_t r, int64_t c, double fill = 0.0) : rows(r), cols(c), v(size_t(r * c), fill) {}
  double& operator()(int64_t i, int64_t j) { return v[size_t(i * cols + j)]; }
  double operator()(int64_t i, int64_t j) const { return v[size_t(i * cols + j)]; }
};

using Model = std::vector<Mat>;  // one I_i x r factor per mode

// ---- datagen (datagen.cpp:13-80, datagen.hpp:31-33) ------------------------
uint64_t splitmix64_next(uint64_t& state);
uint64_t stream_seed(uint64_t base, uint64_t stream);
double draw_uniform01(std::mt19937_64& gen);
double draw_normal(std::mt19937_64& gen);
Mat uniform_matrix(int rows, int cols, std::mt19937_64& gen);
Model random_init(const std::vector<int>& shape, int rank, uint64_t seed);
// generate(): truth factors + tensor (double). `collinear` is the build's
// BASELINE config-4 rule (not in the reference).
void generate(const std::vector<int>& shape, int rank, double sigma, bool ill_conditioned,
              bool collinear, uint64_t seed, std::vector<double>& tensor, Model& truth);

// ---- kernels (kernels.cpp) -------------------------------------------------
struct Split { int64_t left = 1, mid = 1, right = 1; };
Split split_around(const std::vector<int>& shape, int mode);
Mat khatri_rao(const std::vector<const Mat*>& ms);
template <typename T>
Mat mttkrp(const T* data, const std::vector<int>& shape, const Model& m, int mode);
extern int g_sum_order;  // 0 = reference order; 1 = descending (conditioning experiments)
Mat gram(const Mat& a);
Mat hadamard_of_grams(const std::vector<Mat>& grams, int skip);
double cheap_objective(double norm_sq, const Mat& a, const Mat& g, const Mat& c);
template <typename T>
double norm_sq(const T* data, int64_t n);
void reconstruct(const Model& m, std::vector<double>& out);

// ---- naive enumeration oracles (reference.cpp:20-105) ----------------------
Mat ref_mttkrp(const double* data, const std::vector<int>& shape, const Model& m, int mode);
double ref_objective(const double* data, const std::vector<int>& shape, const Model& m);

// ---- NNLS (nnls.cpp:15-49) -------------------------------------------------
struct InnerStop { int max_iters = 50; double rel_change_tol = 1e-2; };
Mat hals_pass(const Mat& g, const Mat& c, Mat w);
Mat ahals_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop, int* sweeps_out);

// ---- drivers (ao.cpp, her.cpp, driver_common.hpp) --------------------------
// NnlsSolver (nnls.hpp:53) and the solvers of nnls.cpp:51-211.
enum Solver { kAhals = 0, kAdmm = 1, kNesterov = 2, kPgd = 3, kActiveSet = 4 };
double spectral_norm(const Mat& m);
double nnls_objective(const Mat& g, const Mat& c, const Mat& w);
Mat pgd_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop);
Mat nesterov_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop);
Mat admm_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop);
Mat active_set_solve(const Mat& g, const Mat& c);
Mat solve_nnls(int solver, const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop);

struct AoConfig {
  int solver = kAhals;
  InnerStop inner;
  int max_outer_iters = 0;
  double max_time_s = 0.0;
  const Model* ground_truth = nullptr;  // record e_k when set
};
struct HerParams { double beta0 = 0.5, gamma = 1.05, gamma_bar = 1.01, eta = 1.5; };
struct HerState { double beta = 0.0, beta_bar = 1.0, f_hat_prev = 0.0; };
struct TraceRecord {
  int iter = 0;
  double time_s = 0.0, f = 0.0, e = 0.0, beta = 0.0;
  bool has_e = false, has_restart = false, restarted = false, has_beta = false;
};
struct RunTrace { double f0 = 0.0; std::vector<TraceRecord> records; };

void validate_her_params(const HerParams& p);
void validate_ao_config(const AoConfig& c);
Mat extrapolate_block(const Mat& a_new, const Mat& a_old, double beta);
void update_betas(HerState& s, bool restarted, const HerParams& p);

// Per-iteration observer: (k, f_hat, restarted, beta_used, accepted, hat).
struct HerObserverFn {
  void (*fn)(void* user, int k, double f_hat, int restarted, double beta_used, const Model& acc,
             const Model& hat) = nullptr;
  void* user = nullptr;
};

template <typename T>
Model her_run(const T* data, const std::vector<int>& shape, const Model& init, const AoConfig& cfg,
              const HerParams& params, RunTrace& trace, HerObserverFn obs = {});
template <typename T>
Model ao_run(const T* data, const std::vector<int>& shape, const Model& init, const AoConfig& cfg,
             RunTrace& trace);

// ---- metrics (metrics.cpp:10-111) ------------------------------------------
// ---- TuckerProvider (tucker.hpp:60-73, tucker.cpp:62-77) -------------------
// U_mode * MTTKRP(core, {U_l^T A_l}_l, mode); bases[l] is I_l x r_l.
Mat compressed_mttkrp(const double* core, const std::vector<int>& core_shape, const std::vector<Mat>& bases,
                      const Model& m, int mode);

Mat normalize_columns(const Mat& a);
std::vector<int> hungarian(const Mat& cost, double* cost_out);
double factor_error(const Model& est, const Model& truth);

}  // namespace ora
