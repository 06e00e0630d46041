// TEST INFRASTRUCTURE ONLY — see ntf_oracle.hpp for scope and pinning.
// Every function cites the reference file:line (under /root/reference/proj)
// whose arithmetic it restates.
#include "ntf_oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace ora {

// ---------------------------------------------------------------- datagen --

// SplitMix64 step (src/datagen.cpp:13-19).
uint64_t splitmix64_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Sub-stream k of a base seed = the (k+1)-th SplitMix64 output
// (src/datagen.cpp:30-35).
uint64_t stream_seed(uint64_t base, uint64_t stream) {
  uint64_t s = base, out = 0;
  for (uint64_t k = 0; k <= stream; ++k) out = splitmix64_next(s);
  return out;
}

// Top 53 bits into [0,1) (include/ntf/datagen.hpp:31-33).
double draw_uniform01(std::mt19937_64& gen) { return double(gen() >> 11) * 0x1.0p-53; }

// Box-Muller, cosine branch, u1 == 0 replaced by 2^-53 (src/datagen.cpp:41-46).
double draw_normal(std::mt19937_64& gen) {
  double u1 = draw_uniform01(gen);
  if (u1 == 0.0) u1 = 0x1.0p-53;
  const double u2 = draw_uniform01(gen);
  const double two_pi = 6.283185307179586476925286766559;  // 2 * std::numbers::pi
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
}

// Row-major fill order (src/datagen.cpp:21-26).
Mat uniform_matrix(int rows, int cols, std::mt19937_64& gen) {
  Mat m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m(i, j) = draw_uniform01(gen);
  return m;
}

// src/datagen.cpp:72-80: stream i of `seed` for mode i.
Model random_init(const std::vector<int>& shape, int rank, uint64_t seed) {
  if (rank < 1) throw std::invalid_argument("rank must be >= 1");
  Model m;
  for (size_t i = 0; i < shape.size(); ++i) {
    std::mt19937_64 gen(stream_seed(seed, i));
    m.push_back(uniform_matrix(shape[i], rank, gen));
  }
  return m;
}

// src/datagen.cpp:48-70. The collinear variant is the build's definition for
// BASELINE config 4 (no reference counterpart): column j of mode i is
// 0.5 * s_i + 0.5 * U_i[:, j], with U_i from stream i (as in the reference)
// and the shared vector s_i from stream N + 1 + i.
void generate(const std::vector<int>& shape, int rank, double sigma, bool ill_conditioned,
              bool collinear, uint64_t seed, std::vector<double>& tensor, Model& truth) {
  if (rank < 1) throw std::invalid_argument("rank must be >= 1");
  if (sigma < 0.0) throw std::invalid_argument("noise level must be >= 0");
  if (ill_conditioned && rank < 2) throw std::invalid_argument("ill-conditioned instances need rank >= 2");
  const int n = int(shape.size());
  truth.clear();
  for (int i = 0; i < n; ++i) {
    std::mt19937_64 gen(stream_seed(seed, uint64_t(i)));
    Mat a = uniform_matrix(shape[size_t(i)], rank, gen);
    if (ill_conditioned)
      for (int64_t r = 0; r < a.rows; ++r) a(r, 0) = 0.99 * a(r, 1) + 0.01 * a(r, 0);
    if (collinear) {
      std::mt19937_64 sg(stream_seed(seed, uint64_t(n + 1 + i)));
      std::vector<double> s(size_t(a.rows));
      for (auto& x : s) x = draw_uniform01(sg);
      for (int64_t r = 0; r < a.rows; ++r)
        for (int64_t j = 0; j < a.cols; ++j) a(r, j) = 0.5 * s[size_t(r)] + 0.5 * a(r, j);
    }
    truth.push_back(std::move(a));
  }
  reconstruct(truth, tensor);
  if (sigma > 0.0) {
    std::mt19937_64 gen(stream_seed(seed, uint64_t(n)));
    for (auto& t : tensor) t = std::max(0.0, t + sigma * draw_normal(gen));
  }
}

// ---------------------------------------------------------------- kernels --

// (left, mid, right) around `mode` (src/kernels.cpp:18-27).
Split split_around(const std::vector<int>& shape, int mode) {
  if (mode < 0 || mode >= int(shape.size())) throw std::invalid_argument("mode out of range");
  Split s;
  for (int l = 0; l < mode; ++l) s.left *= shape[size_t(l)];
  s.mid = shape[size_t(mode)];
  for (int l = mode + 1; l < int(shape.size()); ++l) s.right *= shape[size_t(l)];
  return s;
}

// Row-wise Khatri-Rao: the LAST listed matrix's row runs fastest, and the row
// product accumulates from the last listed matrix to the first, starting from
// ones (src/kernels.cpp:90-113).
Mat khatri_rao(const std::vector<const Mat*>& ms) {
  if (ms.empty()) throw std::invalid_argument("khatri_rao of an empty list");
  const int64_t r = ms[0]->cols;
  int64_t rows = 1;
  for (auto* m : ms) {
    if (m->cols != r) throw std::invalid_argument("khatri_rao column counts disagree");
    rows *= m->rows;
  }
  Mat out(rows, r);
  const int k = int(ms.size());
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < rows; ++row) {
    int64_t rest = row;
    double* o = &out.v[size_t(row * r)];
    for (int64_t c = 0; c < r; ++c) o[c] = 1.0;
    for (int l = k - 1; l >= 0; --l) {
      const Mat& m = *ms[size_t(l)];
      const int64_t j = rest % m.rows;
      rest /= m.rows;
      for (int64_t c = 0; c < r; ++c) o[c] *= m(j, c);
    }
  }
  return out;
}

static void check_model(const std::vector<int>& shape, const Model& m) {
  if (m.size() != shape.size()) throw std::invalid_argument("mttkrp: model/tensor shape mismatch");
  for (size_t i = 0; i < shape.size(); ++i)
    if (m[i].rows != shape[i] || m[i].cols != m[0].cols)
      throw std::invalid_argument("mttkrp: model/tensor shape mismatch");
}

// Dense MTTKRP in the reference's loop order (src/kernels.cpp:161-191):
// per output row `mid`, for each `left`: inner = sum_right T * wr[right,:]
// (ascending right), then acc += wl[left,:] .* inner.
// Summation-order variant (conditioning experiments only, tools/r02/
// oracle_sensitivity.py): 1 walks `left` and `right` in descending order -- the
// same algorithm, rounded differently; 2 rounds the Khatri-Rao rows to float
// (what FP32 factor mirrors do to an FP32 tensor's MTTKRP). 0 (default) is the
// reference's order.
int g_sum_order = 0;

template <typename T>
Mat mttkrp(const T* data, const std::vector<int>& shape, const Model& m, int mode) {
  check_model(shape, m);
  const Split s = split_around(shape, mode);
  const int n = int(shape.size());
  const int64_t r = m[0].cols;
  std::vector<const Mat*> lows, highs;
  for (int l = 0; l < mode; ++l) lows.push_back(&m[size_t(l)]);
  for (int l = mode + 1; l < n; ++l) highs.push_back(&m[size_t(l)]);
  Mat wl = lows.empty() ? Mat(1, r, 1.0) : khatri_rao(lows);
  Mat wr = highs.empty() ? Mat(1, r, 1.0) : khatri_rao(highs);
  if (g_sum_order == 2) {  // FP32-mirror emulation: Khatri-Rao rows rounded to float (conditioning experiments)
    for (double& x : wl.v) x = double(float(x));
    for (double& x : wr.v) x = double(float(x));
  }
  Mat out(s.mid, r);
#pragma omp parallel for schedule(static)
  for (int64_t mid = 0; mid < s.mid; ++mid) {
    std::vector<double> acc(static_cast<size_t>(r), 0.0), inner(static_cast<size_t>(r));
    for (int64_t li = 0; li < s.left; ++li) {
      const int64_t left = g_sum_order == 1 ? s.left - 1 - li : li;
      const T* src = data + (left * s.mid + mid) * s.right;
      std::fill(inner.begin(), inner.end(), 0.0);
      for (int64_t ri = 0; ri < s.right; ++ri) {
        const int64_t right = g_sum_order == 1 ? s.right - 1 - ri : ri;
        const double t = double(src[right]);
        const double* w = &wr.v[size_t(right * r)];
        for (int64_t c = 0; c < r; ++c) inner[size_t(c)] += t * w[c];
      }
      const double* wlr = &wl.v[size_t(left * r)];
      for (int64_t c = 0; c < r; ++c) acc[size_t(c)] += wlr[c] * inner[size_t(c)];
    }
    for (int64_t c = 0; c < r; ++c) out(mid, c) = acc[size_t(c)];
  }
  return out;
}
template Mat mttkrp<double>(const double*, const std::vector<int>&, const Model&, int);
template Mat mttkrp<float>(const float*, const std::vector<int>&, const Model&, int);

// A^T A (include/ntf/kernels.hpp:38), summed over rows in ascending order.
Mat gram(const Mat& a) {
  Mat g(a.cols, a.cols);
  for (int64_t p = 0; p < a.cols; ++p)
    for (int64_t q = 0; q < a.cols; ++q) {
      double s = 0.0;
      for (int64_t i = 0; i < a.rows; ++i) s += a(i, p) * a(i, q);
      g(p, q) = s;
    }
  return g;
}

// Ones, times every Gram except `skip`, ascending (src/kernels.cpp:193-200).
Mat hadamard_of_grams(const std::vector<Mat>& grams, int skip) {
  if (grams.empty()) throw std::invalid_argument("no grams");
  const int64_t r = grams[0].rows;
  Mat out(r, r, 1.0);
  for (int l = 0; l < int(grams.size()); ++l)
    if (l != skip)
      for (size_t e = 0; e < out.v.size(); ++e) out.v[e] *= grams[size_t(l)].v[e];
  return out;
}

// 0.5||T||^2 - <A,C> + 0.5<A^T A, G> (src/kernels.cpp:298-303).
double cheap_objective(double nsq, const Mat& a, const Mat& g, const Mat& c) {
  double cross = 0.0;
  for (size_t e = 0; e < a.v.size(); ++e) cross += a.v[e] * c.v[e];
  const Mat ga = gram(a);
  double quad = 0.0;
  for (size_t e = 0; e < ga.v.size(); ++e) quad += ga.v[e] * g.v[e];
  return 0.5 * nsq - cross + 0.5 * quad;
}

// Flat-order serial sum of squares (src/tensor.cpp:43-47).
template <typename T>
double norm_sq(const T* data, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += double(data[i]) * double(data[i]);
  return s;
}
template double norm_sq<double>(const double*, int64_t);
template double norm_sq<float>(const float*, int64_t);

// Flat layout == (prod of leading dims) x I_N: entry = sum_p wl[row,p]*A_N[col,p]
// (src/kernels.cpp:202-215); the sum runs over p in ascending order.
void reconstruct(const Model& m, std::vector<double>& out) {
  const int n = int(m.size());
  const int64_t r = m[0].cols;
  std::vector<const Mat*> lows;
  for (int l = 0; l + 1 < n; ++l) lows.push_back(&m[size_t(l)]);
  const Mat wl = lows.empty() ? Mat(1, r, 1.0) : khatri_rao(lows);
  const Mat& last = m[size_t(n - 1)];
  out.assign(size_t(wl.rows * last.rows), 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < wl.rows; ++row)
    for (int64_t col = 0; col < last.rows; ++col) {
      double s = 0.0;
      for (int64_t p = 0; p < r; ++p) s += wl(row, p) * last(col, p);
      out[size_t(row * last.rows + col)] = s;
    }
}

// ------------------------------------------------ naive enumeration oracles --

// unfold(T, mode) * KR(factors excluding mode, listed N-1..0)
// (src/reference.cpp:44-67, 89-95), evaluated element by element.
Mat ref_mttkrp(const double* data, const std::vector<int>& shape, const Model& m, int mode) {
  check_model(shape, m);
  const int n = int(shape.size());
  const int64_t r = m[0].cols;
  Mat out(shape[size_t(mode)], r);
  std::vector<int> idx(size_t(n), 0);
  int64_t total = 1;
  for (int d : shape) total *= d;
  for (int64_t flat = 0; flat < total; ++flat) {
    for (int64_t c = 0; c < r; ++c) {
      double w = 1.0;
      for (int l = n - 1; l >= 0; --l)
        if (l != mode) w *= m[size_t(l)](idx[size_t(l)], c);
      out(idx[size_t(mode)], c) += data[flat] * w;
    }
    for (int l = n - 1; l >= 0; --l) {
      if (++idx[size_t(l)] < shape[size_t(l)]) break;
      idx[size_t(l)] = 0;
    }
  }
  return out;
}

// 0.5 * ||T - [[A]]||^2 by explicit reconstruction (src/reference.cpp:97-105).
double ref_objective(const double* data, const std::vector<int>& shape, const Model& m) {
  const int n = int(shape.size());
  const int64_t r = m[0].cols;
  std::vector<int> idx(size_t(n), 0);
  int64_t total = 1;
  for (int d : shape) total *= d;
  double s = 0.0;
  for (int64_t flat = 0; flat < total; ++flat) {
    double v = 0.0;
    for (int64_t p = 0; p < r; ++p) {
      double prod = 1.0;
      for (int l = 0; l < n; ++l) prod *= m[size_t(l)](idx[size_t(l)], p);
      v += prod;
    }
    const double d = data[flat] - v;
    s += d * d;
    for (int l = n - 1; l >= 0; --l) {
      if (++idx[size_t(l)] < shape[size_t(l)]) break;
      idx[size_t(l)] = 0;
    }
  }
  return 0.5 * s;
}

// ------------------------------------------------------------------- NNLS --

// One Gauss-Seidel pass over the columns (src/nnls.cpp:15-26): columns whose
// Gram diagonal is <= 1e-12 * max diag are skipped; otherwise
// W[:,j] = max(0, (C[:,j] - W G[:,j] + G_jj W[:,j]) / G_jj).
Mat hals_pass(const Mat& g, const Mat& c, Mat w) {
  const int64_t r = g.rows;
  double dmax = -std::numeric_limits<double>::infinity();
  for (int64_t j = 0; j < r; ++j) dmax = std::max(dmax, g(j, j));
  const double floor_ = 1e-12 * dmax;
  for (int64_t j = 0; j < r; ++j) {
    const double gjj = g(j, j);
    if (gjj <= floor_) continue;
    for (int64_t i = 0; i < w.rows; ++i) {
      double prod = 0.0;
      for (int64_t l = 0; l < r; ++l) prod += w(i, l) * g(l, j);
      const double numer = (c(i, j) - prod) + gjj * w(i, j);
      w(i, j) = std::max(numer / gjj, 0.0);
    }
  }
  return w;
}

// Sweep loop with the global Frobenius stop rule (src/nnls.cpp:31-49):
// stop after max_iters sweeps or when ||W_{s+1}-W_s|| <= tol * ||W_1-W_0||.
Mat ahals_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop, int* sweeps_out) {
  Mat w = w0;
  double first = -1.0;
  int s = 0;
  for (; s < stop.max_iters; ++s) {
    Mat next = hals_pass(g, c, w);
    double sq = 0.0;
    for (size_t e = 0; e < w.v.size(); ++e) {
      const double d = next.v[e] - w.v[e];
      sq += d * d;
    }
    const double change = std::sqrt(sq);
    w = std::move(next);
    if (s == 0) first = change;
    if (change <= stop.rel_change_tol * first) { ++s; break; }
  }
  if (sweeps_out) *sweeps_out = s;
  return w;
}

// ------------------------------------------------ the other inner solvers --
// Restated from nnls.cpp:51-211 (and spectral_norm, kernels.cpp:262-280),
// plain ascending loops instead of Eigen: agreement "to rounding".

namespace {

Mat matmul(const Mat& a, const Mat& b) {  // a (n x k) * b (k x m)
  Mat out(a.rows, b.cols);
  for (int64_t i = 0; i < a.rows; ++i)
    for (int64_t j = 0; j < b.cols; ++j) {
      double acc = 0.0;
      for (int64_t k = 0; k < a.cols; ++k) acc += a(i, k) * b(k, j);
      out(i, j) = acc;
    }
  return out;
}

double fro_diff(const Mat& a, const Mat& b) {
  double sq = 0.0;
  for (size_t e = 0; e < a.v.size(); ++e) sq += (a.v[e] - b.v[e]) * (a.v[e] - b.v[e]);
  return std::sqrt(sq);
}

// Cholesky L L^T = a (lower, row-major); false unless positive definite
// (Eigen::LLT's info() != Success).
bool cholesky(const Mat& a, Mat* l) {
  const int64_t n = a.rows;
  *l = Mat(n, n);
  for (int64_t j = 0; j < n; ++j) {
    double d = a(j, j);
    for (int64_t k = 0; k < j; ++k) d -= (*l)(j, k) * (*l)(j, k);
    if (!(d > 0.0)) return false;
    (*l)(j, j) = std::sqrt(d);
    for (int64_t i = j + 1; i < n; ++i) {
      double v = a(i, j);
      for (int64_t k = 0; k < j; ++k) v -= (*l)(i, k) * (*l)(j, k);
      (*l)(i, j) = v / (*l)(j, j);
    }
  }
  return true;
}

// x = (L L^T)^{-1} b for one vector
std::vector<double> chol_solve(const Mat& l, std::vector<double> b) {
  const int64_t n = l.rows;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = 0; k < i; ++k) b[size_t(i)] -= l(i, k) * b[size_t(k)];
    b[size_t(i)] /= l(i, i);
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    for (int64_t k = i + 1; k < n; ++k) b[size_t(i)] -= l(k, i) * b[size_t(k)];
    b[size_t(i)] /= l(i, i);
  }
  return b;
}

// Largest |eigenvalue| of a symmetric matrix by cyclic Jacobi rotations:
// the fallback of spectral_norm (Eigen::SelfAdjointEigenSolver there).
double jacobi_max_abs_eig(Mat a) {
  const int64_t n = a.rows;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int64_t p = 0; p < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) off += a(p, q) * a(p, q);
    if (off <= 1e-300) break;
    for (int64_t p = 0; p < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        if (a(p, q) == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int64_t k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
      }
  }
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) m = std::max(m, std::abs(a(i, i)));
  return m;
}

}  // namespace

// kernels.cpp:262-280: power iteration from the normalised ones vector.
double spectral_norm(const Mat& m) {
  const int64_t r = m.rows;
  if (r == 0) return 0.0;
  if (r == 1) return std::abs(m(0, 0));
  std::vector<double> v(static_cast<size_t>(r), 1.0 / std::sqrt(double(r))), w(static_cast<size_t>(r));
  double lambda = 0.0;
  for (int it = 0; it < 1000; ++it) {
    double nrm = 0.0;
    for (int64_t i = 0; i < r; ++i) {
      double acc = 0.0;
      for (int64_t k = 0; k < r; ++k) acc += m(i, k) * v[size_t(k)];
      w[size_t(i)] = acc;
      nrm += acc * acc;
    }
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) return 0.0;
    for (int64_t i = 0; i < r; ++i) v[size_t(i)] = w[size_t(i)] / nrm;
    double next = 0.0;
    for (int64_t i = 0; i < r; ++i) {
      double acc = 0.0;
      for (int64_t k = 0; k < r; ++k) acc += m(i, k) * v[size_t(k)];
      next += v[size_t(i)] * acc;
    }
    if (std::abs(next - lambda) <= 1e-10 * std::max(1.0, std::abs(next))) return next;
    lambda = next;
  }
  return jacobi_max_abs_eig(m);
}

// nnls.cpp:11-13: 0.5 <W^T W, G> - <W, C>.
double nnls_objective(const Mat& g, const Mat& c, const Mat& w) {
  const Mat ww = gram(w);
  double q = 0.0, l = 0.0;
  for (size_t e = 0; e < ww.v.size(); ++e) q += ww.v[e] * g.v[e];
  for (size_t e = 0; e < w.v.size(); ++e) l += w.v[e] * c.v[e];
  return 0.5 * q - l;
}

// nnls.cpp:51-57 (run_sweeps, nnls.cpp:31-44: stop on the first change).
Mat pgd_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop) {
  const double lip = spectral_norm(g);
  if (lip <= 0.0) throw std::runtime_error("pgd_solve: zero Gram matrix");
  Mat w = w0;
  double first = -1.0;
  for (int s = 0; s < stop.max_iters; ++s) {
    const Mat wg = matmul(w, g);
    Mat next(w.rows, w.cols);
    for (size_t e = 0; e < w.v.size(); ++e) next.v[e] = std::max(0.0, w.v[e] - (wg.v[e] - c.v[e]) / lip);
    const double change = fro_diff(next, w);
    w = std::move(next);
    if (s == 0) first = change;
    if (change <= stop.rel_change_tol * first) break;
  }
  return w;
}

// nnls.cpp:59-87.
Mat nesterov_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop) {
  const double lip = spectral_norm(g);
  if (lip <= 0.0) throw std::runtime_error("nesterov_solve: zero Gram matrix");
  Mat w = w0, y = w0, best = w0;
  double best_obj = nnls_objective(g, c, w);
  double t = 1.0, first = -1.0;
  for (int s = 0; s < stop.max_iters; ++s) {
    const Mat yg = matmul(y, g);
    Mat next(w.rows, w.cols);
    for (size_t e = 0; e < w.v.size(); ++e) next.v[e] = std::max(0.0, y.v[e] - (yg.v[e] - c.v[e]) / lip);
    const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    for (size_t e = 0; e < w.v.size(); ++e) y.v[e] = next.v[e] + ((t - 1.0) / t_next) * (next.v[e] - w.v[e]);
    const double change = fro_diff(next, w);
    w = std::move(next);
    t = t_next;
    const double obj = nnls_objective(g, c, w);
    if (obj < best_obj) {
      best_obj = obj;
      best = w;
    }
    if (s == 0) first = change;
    if (change <= stop.rel_change_tol * first) break;
  }
  return best;
}

// nnls.cpp:89-121.
Mat admm_solve(const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop) {
  const int64_t r = g.rows;
  double tr = 0.0;
  for (int64_t j = 0; j < r; ++j) tr += g(j, j);
  const double rho = tr / double(r);
  if (rho <= 0.0) throw std::runtime_error("admm_solve: zero Gram matrix");
  Mat shifted = g;
  for (int64_t j = 0; j < r; ++j) shifted(j, j) += rho;
  Mat l;
  if (!cholesky(shifted, &l)) throw std::runtime_error("admm_solve: factorization failed");
  Mat z = w0, u(w0.rows, w0.cols), best = w0;
  double best_obj = nnls_objective(g, c, z);
  double first = -1.0;
  for (int s = 0; s < stop.max_iters; ++s) {
    Mat w(z.rows, z.cols), zn(z.rows, z.cols);
    for (int64_t i = 0; i < z.rows; ++i) {  // W (G + rho I) = C + rho (Z - U), row by row
      std::vector<double> rhs(static_cast<size_t>(r));
      for (int64_t j = 0; j < r; ++j) rhs[size_t(j)] = c(i, j) + rho * (z(i, j) - u(i, j));
      const std::vector<double> x = chol_solve(l, rhs);
      for (int64_t j = 0; j < r; ++j) w(i, j) = x[size_t(j)];
    }
    for (size_t e = 0; e < z.v.size(); ++e) {
      zn.v[e] = std::max(0.0, w.v[e] + u.v[e]);
      u.v[e] += w.v[e] - zn.v[e];
    }
    const double change = fro_diff(zn, z);
    z = std::move(zn);
    const double obj = nnls_objective(g, c, z);
    if (obj < best_obj) {
      best_obj = obj;
      best = z;
    }
    if (s == 0) first = change;
    if (change <= stop.rel_change_tol * first) break;
  }
  return best;
}

namespace {

// nnls.cpp:125-191: Lawson-Hanson on the normal equations for one row.
bool solve_row_active_set(const Mat& g, const std::vector<double>& c, std::vector<double>& x) {
  const int64_t r = g.rows;
  double cmax = 0.0, gmax = -std::numeric_limits<double>::infinity();
  for (int64_t j = 0; j < r; ++j) {
    cmax = std::max(cmax, std::abs(c[size_t(j)]));
    gmax = std::max(gmax, g(j, j));
  }
  const double enter_tol = 1e-11 * std::max({1.0, cmax, gmax});
  x.assign(size_t(r), 0.0);
  std::vector<int64_t> passive;
  std::vector<bool> in_passive(size_t(r), false);
  const int max_additions = 3 * int(r);
  for (int additions = 0;; ++additions) {
    int64_t enter = -1;
    double best = enter_tol;
    for (int64_t j = 0; j < r; ++j) {
      double gx = 0.0;
      for (int64_t k = 0; k < r; ++k) gx += g(j, k) * x[size_t(k)];
      const double dual = c[size_t(j)] - gx;
      if (!in_passive[size_t(j)] && dual > best) {
        best = dual;
        enter = j;
      }
    }
    if (enter < 0) return true;
    if (additions >= max_additions) return false;
    passive.push_back(enter);
    in_passive[size_t(enter)] = true;
    for (;;) {
      const int64_t np = int64_t(passive.size());
      Mat gp(np, np);
      std::vector<double> cp(static_cast<size_t>(np));
      for (int64_t a = 0; a < np; ++a) {
        cp[size_t(a)] = c[size_t(passive[size_t(a)])];
        for (int64_t b = 0; b < np; ++b) gp(a, b) = g(passive[size_t(a)], passive[size_t(b)]);
      }
      Mat l;
      cholesky(gp, &l);  // Eigen's llt().solve on a positive-definite principal submatrix
      const std::vector<double> zp = chol_solve(l, cp);
      bool all_pos = true;
      for (double v : zp) all_pos = all_pos && v > 0.0;
      if (all_pos) {
        std::fill(x.begin(), x.end(), 0.0);
        for (int64_t a = 0; a < np; ++a) x[size_t(passive[size_t(a)])] = zp[size_t(a)];
        break;
      }
      double alpha = 1.0;
      for (int64_t a = 0; a < np; ++a)
        if (zp[size_t(a)] <= 0.0) {
          const double xa = x[size_t(passive[size_t(a)])];
          alpha = std::min(alpha, xa / (xa - zp[size_t(a)]));
        }
      for (int64_t a = 0; a < np; ++a) {
        const int64_t j = passive[size_t(a)];
        x[size_t(j)] += alpha * (zp[size_t(a)] - x[size_t(j)]);
      }
      for (size_t a = passive.size(); a-- > 0;) {
        const int64_t j = passive[a];
        if (x[size_t(j)] <= 0.0 || (zp[a] <= 0.0 && x[size_t(j)] < 1e-14)) {
          x[size_t(j)] = 0.0;
          in_passive[size_t(j)] = false;
          passive.erase(passive.begin() + std::ptrdiff_t(a));
        }
      }
    }
  }
}

}  // namespace

// nnls.cpp:195-211.
Mat active_set_solve(const Mat& g, const Mat& c) {
  Mat l;
  if (!cholesky(g, &l)) throw std::runtime_error("active_set_solve: Gram matrix is not positive definite");
  Mat w(c.rows, g.cols);
  bool ok = true;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < c.rows; ++i) {
    std::vector<double> row(static_cast<size_t>(c.cols)), x;
    for (int64_t j = 0; j < c.cols; ++j) row[size_t(j)] = c(i, j);
    if (solve_row_active_set(g, row, x)) {
      for (int64_t j = 0; j < c.cols; ++j) w(i, j) = x[size_t(j)];
    } else {
#pragma omp atomic write
      ok = false;
    }
  }
  if (!ok) throw std::runtime_error("active_set_solve: pass budget exceeded");
  return w;
}

// nnls.cpp:213-222.
Mat solve_nnls(int solver, const Mat& g, const Mat& c, const Mat& w0, const InnerStop& stop) {
  switch (solver) {
    case kAhals: return ahals_solve(g, c, w0, stop, nullptr);
    case kAdmm: return admm_solve(g, c, w0, stop);
    case kNesterov: return nesterov_solve(g, c, w0, stop);
    case kPgd: return pgd_solve(g, c, w0, stop);
    case kActiveSet: return active_set_solve(g, c);
  }
  throw std::logic_error("unknown solver");
}

// ---------------------------------------------------------------- drivers --

// src/her.cpp:10-14.
void validate_her_params(const HerParams& p) {
  if (!(p.beta0 > 0.0 && p.beta0 < 1.0)) throw std::invalid_argument("beta0 must lie in (0,1)");
  if (!(1.0 < p.gamma_bar && p.gamma_bar <= p.gamma && p.gamma <= p.eta))
    throw std::invalid_argument("parameters must satisfy 1 < gamma_bar <= gamma <= eta");
}

// src/ao.cpp:10-15 (the record_e / ground-truth pairing is carried by the
// pointer here).
void validate_ao_config(const AoConfig& c) {
  if (c.max_outer_iters <= 0 && c.max_time_s <= 0.0)
    throw std::invalid_argument("set an iteration or time budget");
}

// max(0, A_new + beta (A_new - A_old)) (src/her.cpp:16-19).
Mat extrapolate_block(const Mat& a_new, const Mat& a_old, double beta) {
  Mat out = a_new;
  for (size_t e = 0; e < out.v.size(); ++e)
    out.v[e] = std::max(a_new.v[e] + beta * (a_new.v[e] - a_old.v[e]), 0.0);
  return out;
}

// src/her.cpp:21-30.
void update_betas(HerState& s, bool restarted, const HerParams& p) {
  if (restarted) {
    s.beta_bar = s.beta;
    s.beta /= p.eta;
  } else {
    s.beta = std::min(s.beta_bar, s.beta * p.gamma);
    s.beta_bar = std::min(1.0, s.beta_bar * p.gamma_bar);
  }
}

namespace {

// driver_common.hpp:14-25.
void check_inputs(const std::vector<int>& shape, const Model& init, const AoConfig& cfg) {
  validate_ao_config(cfg);
  if (init.empty()) throw std::invalid_argument("model must have at least one factor");
  for (auto& a : init)
    if (a.cols != init[0].cols) throw std::invalid_argument("factor column counts disagree");
  if (init.size() != shape.size()) throw std::invalid_argument("initial model does not match the tensor shape");
  for (size_t i = 0; i < shape.size(); ++i)
    if (init[i].rows != shape[i]) throw std::invalid_argument("initial model does not match the tensor shape");
  for (auto& a : init)
    for (double x : a.v)
      if (x < 0.0) throw std::invalid_argument("initial model must be entrywise nonnegative");
  if (cfg.ground_truth && (cfg.ground_truth->size() != init.size() ||
                           (*cfg.ground_truth)[0].cols != init[0].cols))
    throw std::invalid_argument("ground truth does not match the initial model");
}

struct Clock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double elapsed() const {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};

// driver_common.hpp:38-42.
bool budget_exhausted(const AoConfig& cfg, int k, double t) {
  if (cfg.max_outer_iters > 0 && k >= cfg.max_outer_iters) return true;
  if (cfg.max_time_s > 0.0 && t >= cfg.max_time_s) return true;
  return false;
}

// driver_common.hpp:50-56: one MTTKRP at the last mode.
template <typename T>
double pivot_objective(const T* data, const std::vector<int>& shape, const Model& m,
                       const std::vector<Mat>& grams, double nsq) {
  const int pivot = int(m.size()) - 1;
  const Mat c = mttkrp(data, shape, m, pivot);
  return cheap_objective(nsq, m[size_t(pivot)], hadamard_of_grams(grams, pivot), c);
}

}  // namespace

// Algorithm 2, step order of src/her.cpp:40-110.
template <typename T>
Model her_run(const T* data, const std::vector<int>& shape, const Model& init, const AoConfig& cfg,
              const HerParams& params, RunTrace& trace, HerObserverFn obs) {
  check_inputs(shape, init, cfg);
  validate_her_params(params);
  const int n = int(init.size());
  int64_t total = 1;
  for (int d : shape) total *= d;
  const double nsq = norm_sq(data, total);

  Model accepted = init, hat = init, solved = init;
  HerState st;
  st.beta = params.beta0;
  std::vector<Mat> hat_grams;
  for (auto& a : hat) hat_grams.push_back(gram(a));

  trace = RunTrace{};
  trace.f0 = pivot_objective(data, shape, accepted, hat_grams, nsq);
  st.f_hat_prev = trace.f0;

  Clock clock;
  for (int k = 1;; ++k) {
    const double beta_used = st.beta;
    Mat last_c;
    for (int i = 0; i < n; ++i) {
      const Mat g = hadamard_of_grams(hat_grams, i);
      Mat c = mttkrp(data, shape, hat, i);
      solved[size_t(i)] = solve_nnls(cfg.solver, g, c, accepted[size_t(i)], cfg.inner);
      hat[size_t(i)] = extrapolate_block(solved[size_t(i)], accepted[size_t(i)], beta_used);
      hat_grams[size_t(i)] = gram(hat[size_t(i)]);
      if (i == n - 1) last_c = std::move(c);
    }
    // f_hat (src/her.cpp:32-38): mixed point, no extra MTTKRP.
    const double fk = cheap_objective(nsq, solved[size_t(n - 1)],
                                      hadamard_of_grams(hat_grams, n - 1), last_c);
    const bool restarted = fk > st.f_hat_prev;
    if (restarted) {
      hat = solved;
      for (int i = 0; i < n; ++i) hat_grams[size_t(i)] = gram(hat[size_t(i)]);
      accepted = solved;
    } else {
      accepted = hat;
    }
    st.f_hat_prev = fk;
    update_betas(st, restarted, params);

    TraceRecord rec;
    rec.iter = k;
    rec.time_s = clock.elapsed();
    rec.f = fk;
    if (cfg.ground_truth) {
      rec.e = factor_error(accepted, *cfg.ground_truth);
      rec.has_e = true;
    }
    rec.has_restart = true;
    rec.restarted = restarted;
    rec.has_beta = true;
    rec.beta = beta_used;
    trace.records.push_back(rec);
    if (obs.fn) obs.fn(obs.user, k, fk, restarted ? 1 : 0, beta_used, accepted, hat);
    if (budget_exhausted(cfg, k, rec.time_s)) break;
  }
  return accepted;
}
template Model her_run<double>(const double*, const std::vector<int>&, const Model&, const AoConfig&,
                               const HerParams&, RunTrace&, HerObserverFn);
template Model her_run<float>(const float*, const std::vector<int>&, const Model&, const AoConfig&,
                              const HerParams&, RunTrace&, HerObserverFn);

// Algorithm 1, step order of src/ao.cpp:17-52.
template <typename T>
Model ao_run(const T* data, const std::vector<int>& shape, const Model& init, const AoConfig& cfg,
             RunTrace& trace) {
  check_inputs(shape, init, cfg);
  const int n = int(init.size());
  int64_t total = 1;
  for (int d : shape) total *= d;
  const double nsq = norm_sq(data, total);
  Model model = init;
  std::vector<Mat> grams;
  for (auto& a : model) grams.push_back(gram(a));
  trace = RunTrace{};
  trace.f0 = pivot_objective(data, shape, model, grams, nsq);
  Clock clock;
  for (int k = 1;; ++k) {
    double f = 0.0;
    for (int i = 0; i < n; ++i) {
      const Mat g = hadamard_of_grams(grams, i);
      const Mat c = mttkrp(data, shape, model, i);
      Mat w = solve_nnls(cfg.solver, g, c, model[size_t(i)], cfg.inner);
      if (i == n - 1) f = cheap_objective(nsq, w, g, c);
      model[size_t(i)] = std::move(w);
      grams[size_t(i)] = gram(model[size_t(i)]);
    }
    TraceRecord rec;
    rec.iter = k;
    rec.time_s = clock.elapsed();
    rec.f = f;
    if (cfg.ground_truth) {
      rec.e = factor_error(model, *cfg.ground_truth);
      rec.has_e = true;
    }
    trace.records.push_back(rec);
    if (budget_exhausted(cfg, k, rec.time_s)) break;
  }
  return model;
}
template Model ao_run<double>(const double*, const std::vector<int>&, const Model&, const AoConfig&, RunTrace&);
template Model ao_run<float>(const float*, const std::vector<int>&, const Model&, const AoConfig&, RunTrace&);

// ---------------------------------------------------------------- metrics --

// Unit-norm columns; zero columns pass through (src/metrics.cpp:10-17).
Mat normalize_columns(const Mat& a) {
  Mat out = a;
  for (int64_t j = 0; j < a.cols; ++j) {
    double sq = 0.0;
    for (int64_t i = 0; i < a.rows; ++i) sq += a(i, j) * a(i, j);
    const double nrm = std::sqrt(sq);
    if (nrm > 0.0)
      for (int64_t i = 0; i < a.rows; ++i) out(i, j) /= nrm;
  }
  return out;
}

// Minimum-cost assignment by shortest augmenting paths with potentials
// (src/metrics.cpp:19-77). Returns mapping[row] = column.
std::vector<int> hungarian(const Mat& cost, double* cost_out) {
  if (cost.rows != cost.cols) throw std::invalid_argument("cost matrix must be square");
  const int n = int(cost.rows);
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> u(size_t(n) + 1, 0.0), v(size_t(n) + 1, 0.0);
  std::vector<int> owner(size_t(n) + 1, 0), via(size_t(n) + 1, 0);
  for (int row = 1; row <= n; ++row) {
    owner[0] = row;
    int col0 = 0;
    std::vector<double> slack(size_t(n) + 1, inf);
    std::vector<char> done(size_t(n) + 1, 0);
    while (true) {
      done[size_t(col0)] = 1;
      const int r0 = owner[size_t(col0)];
      double delta = inf;
      int col1 = 0;
      for (int c = 1; c <= n; ++c) {
        if (done[size_t(c)]) continue;
        const double red = cost(r0 - 1, c - 1) - u[size_t(r0)] - v[size_t(c)];
        if (red < slack[size_t(c)]) {
          slack[size_t(c)] = red;
          via[size_t(c)] = col0;
        }
        if (slack[size_t(c)] < delta) {
          delta = slack[size_t(c)];
          col1 = c;
        }
      }
      for (int c = 0; c <= n; ++c) {
        if (done[size_t(c)]) {
          u[size_t(owner[size_t(c)])] += delta;
          v[size_t(c)] -= delta;
        } else {
          slack[size_t(c)] -= delta;
        }
      }
      col0 = col1;
      if (owner[size_t(col0)] == 0) break;
    }
    while (col0 != 0) {
      const int prev = via[size_t(col0)];
      owner[size_t(col0)] = owner[size_t(prev)];
      col0 = prev;
    }
  }
  std::vector<int> mapping(size_t(n), -1);
  for (int c = 1; c <= n; ++c)
    if (owner[size_t(c)] > 0) mapping[size_t(owner[size_t(c)] - 1)] = c - 1;
  if (cost_out) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += cost(i, mapping[size_t(i)]);
    *cost_out = s;
  }
  return mapping;
}

// Joint-permutation factor error (src/metrics.cpp:79-111).
double factor_error(const Model& est, const Model& truth) {
  if (est.size() != truth.size() || est.empty() || est[0].cols != truth[0].cols)
    throw std::invalid_argument("factor_error: model shapes disagree");
  for (size_t i = 0; i < est.size(); ++i)
    if (est[i].rows != truth[i].rows) throw std::invalid_argument("factor_error: model shapes disagree");
  const int n = int(est.size());
  const int64_t r = est[0].cols;
  std::vector<Mat> ne, nt;
  for (int i = 0; i < n; ++i) {
    ne.push_back(normalize_columns(est[size_t(i)]));
    nt.push_back(normalize_columns(truth[size_t(i)]));
  }
  Mat cost(r, r);
  for (int i = 0; i < n; ++i)
    for (int64_t p = 0; p < r; ++p)
      for (int64_t q = 0; q < r; ++q) {
        double sq = 0.0;
        for (int64_t row = 0; row < ne[size_t(i)].rows; ++row) {
          const double d = ne[size_t(i)](row, p) - nt[size_t(i)](row, q);
          sq += d * d;
        }
        cost(p, q) += sq;
      }
  const std::vector<int> pi = hungarian(cost, nullptr);
  double err = 0.0;
  for (int i = 0; i < n; ++i) {
    double num = 0.0, den = 0.0;
    for (int64_t row = 0; row < ne[size_t(i)].rows; ++row)
      for (int64_t p = 0; p < r; ++p) {
        // permuted column pi[p] holds normalized estimate column p
        const double d = nt[size_t(i)](row, pi[size_t(p)]) - ne[size_t(i)](row, p);
        num += d * d;
      }
    for (double x : nt[size_t(i)].v) den += x * x;
    err += std::sqrt(num) / std::sqrt(den);
  }
  return err / n;
}

// compressed_mttkrp (tucker.cpp:62-77): project every other factor into the
// compressed space (P_l = U_l^T A_l), contract the core with their
// Khatri-Rao product -- the reference's unfold(core, mode) * khatri_rao(P)
// with its ordering convention is the MTTKRP of the core with the P_l
// (kernels.cpp:161-191; the reference pins compressed == dense MTTKRP in
// test_tucker.cpp:71-99) -- then U_mode times it.
Mat compressed_mttkrp(const double* core, const std::vector<int>& core_shape, const std::vector<Mat>& bases,
                      const Model& m, int mode) {
  const int n = int(m.size());
  if (int(bases.size()) != n || int(core_shape.size()) != n)
    throw std::invalid_argument("compressed_mttkrp: order mismatch");
  const int64_t r = m[0].cols;
  Model proj;
  for (int l = 0; l < n; ++l) {
    const Mat& u = bases[size_t(l)];
    Mat pl(u.cols, r);
    if (l != mode)
      for (int64_t a = 0; a < u.cols; ++a)
        for (int64_t c = 0; c < r; ++c) {
          double acc = 0.0;
          for (int64_t i = 0; i < u.rows; ++i) acc += u(i, a) * m[size_t(l)](i, c);
          pl(a, c) = acc;
        }
    proj.push_back(pl);
  }
  const Mat mc = mttkrp(core, core_shape, proj, mode);
  const Mat& um = bases[size_t(mode)];
  Mat out(um.rows, r);
  for (int64_t i = 0; i < um.rows; ++i)
    for (int64_t c = 0; c < r; ++c) {
      double acc = 0.0;
      for (int64_t a = 0; a < um.cols; ++a) acc += um(i, a) * mc(a, c);
      out(i, c) = acc;
    }
  return out;
}

}  // namespace ora
