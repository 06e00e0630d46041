// Host-side synthetic instances and the factor-error metric.
//
// Instance generation must be bit-exact with the reference generator
// (src/datagen.cpp:13-80): SplitMix64 sub-stream seeds feeding
// std::mt19937_64 (whose output sequence the C++ standard fixes), top-53-bit
// uniforms, cosine-branch Box-Muller, row-major factor fills, noise drawn in
// flat order from sub-stream N. It is inherently sequential in the noise
// stream, so it stays on the host; the reconstruction part is parallel.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#include "ntf_internal.h"
#include "runtime.h"

namespace ntfb {

namespace {

inline uint64_t splitmix_step(uint64_t& st) {
  st += 0x9E3779B97F4A7C15ull;
  uint64_t z = st;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline double unit_draw(std::mt19937_64& g) { return double(g() >> 11) * 0x1.0p-53; }

inline double gauss_draw(std::mt19937_64& g) {
  double u1 = unit_draw(g);
  if (u1 == 0.0) u1 = 0x1.0p-53;
  const double u2 = unit_draw(g);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

std::vector<int> check_shape(const int* shape, int order, int rank) {
  if (order < 1 || order > kMaxOrder) throw InvalidArgument("tensor order must lie in 1..8");
  if (rank < 1) throw InvalidArgument("rank must be >= 1");
  std::vector<int> s(shape, shape + order);
  for (int d : s)
    if (d < 1) throw InvalidArgument("tensor dimensions must be positive");
  return s;
}

// Row-major uniform fill (datagen.cpp:21-26) into `out` (rows x r).
void fill_uniform(double* out, int rows, int r, std::mt19937_64& g) {
  for (long long e = 0; e < (long long)rows * r; ++e) out[e] = unit_draw(g);
}

}  // namespace

uint64_t stream_seed(uint64_t base, uint64_t stream) {
  uint64_t st = base, out = 0;
  for (uint64_t k = 0; k <= stream; ++k) out = splitmix_step(st);
  return out;
}

void random_init(const int* shape, int order, int rank, uint64_t seed, double* out) {
  const auto s = check_shape(shape, order, rank);
  long long off = 0;
  for (int i = 0; i < order; ++i) {
    std::mt19937_64 g(stream_seed(seed, uint64_t(i)));
    fill_uniform(out + off, s[size_t(i)], rank, g);
    off += (long long)s[size_t(i)] * rank;
  }
}

// generate(): truth factors, T = reconstruct(truth) with the entry summed
// over p ascending (kernels.cpp:202-215), then max(0, T + sigma N(0,1)) in
// flat order from sub-stream N. The build-defined collinear rule (BASELINE
// config 4): A_i[:,j] = 0.5 s_i + 0.5 U_i[:,j], s_i from sub-stream N+1+i.
template <typename T>
static void generate_impl(const std::vector<int>& s, int rank, double sigma, bool ill, bool collinear,
                          uint64_t seed, T* tensor, double* truth) {
  const int n = int(s.size());
  std::vector<const double*> A(static_cast<size_t>(n));
  long long off = 0;
  for (int i = 0; i < n; ++i) {
    double* a = truth + off;
    const int rows = s[size_t(i)];
    std::mt19937_64 g(stream_seed(seed, uint64_t(i)));
    fill_uniform(a, rows, rank, g);
    if (ill)
      for (int row = 0; row < rows; ++row)
        a[(long long)row * rank] = 0.99 * a[(long long)row * rank + 1] + 0.01 * a[(long long)row * rank];
    if (collinear) {
      std::mt19937_64 sg(stream_seed(seed, uint64_t(n + 1 + i)));
      std::vector<double> shared(static_cast<size_t>(rows));
      for (auto& x : shared) x = unit_draw(sg);
      for (int row = 0; row < rows; ++row)
        for (int j = 0; j < rank; ++j)
          a[(long long)row * rank + j] = 0.5 * shared[size_t(row)] + 0.5 * a[(long long)row * rank + j];
    }
    A[size_t(i)] = a;
    off += (long long)rows * rank;
  }
  // Leading-mode Khatri-Rao rows, product from the last listed factor down
  // to the first (kernels.cpp:104-109), computed per row on the fly.
  long long lead = 1;
  for (int i = 0; i + 1 < n; ++i) lead *= s[size_t(i)];
  const int last = s[size_t(n - 1)];
  const double* An = A[size_t(n - 1)];
  std::mt19937_64 noise(stream_seed(seed, uint64_t(n)));
  const long long chunk = 4096;
  std::vector<double> buf;
  for (long long r0 = 0; r0 < lead; r0 += chunk) {
    const long long r1 = std::min(lead, r0 + chunk);
    buf.assign(size_t((r1 - r0) * last), 0.0);
#pragma omp parallel for schedule(static)
    for (long long row = r0; row < r1; ++row) {
      double kr[kMaxRank * 4];
      std::vector<double> krv;
      double* w = kr;
      if (rank > kMaxRank * 4) {
        krv.resize(size_t(rank));
        w = krv.data();
      }
      for (int p = 0; p < rank; ++p) w[p] = 1.0;
      long long rest = row;
      for (int l = n - 2; l >= 0; --l) {
        const long long j = rest % s[size_t(l)];
        rest /= s[size_t(l)];
        for (int p = 0; p < rank; ++p) w[p] *= A[size_t(l)][j * rank + p];
      }
      for (int col = 0; col < last; ++col) {
        double v = 0.0;
        for (int p = 0; p < rank; ++p) v += w[p] * An[(long long)col * rank + p];
        buf[size_t((row - r0) * last + col)] = v;
      }
    }
    for (long long e = 0; e < (r1 - r0) * last; ++e) {
      double v = buf[size_t(e)];
      if (sigma > 0.0) v = std::max(0.0, v + sigma * gauss_draw(noise));
      tensor[r0 * last + e] = T(v);
    }
  }
}

void generate(const int* shape, int order, int rank, double sigma, int ill, int collinear, uint64_t seed,
              int dtype, void* tensor, double* truth) {
  const auto s = check_shape(shape, order, rank);
  if (sigma < 0.0) throw InvalidArgument("noise level must be >= 0");
  if (ill && rank < 2) throw InvalidArgument("ill-conditioned instances need rank >= 2");
  if (dtype == NTF_DTYPE_F32)
    generate_impl(s, rank, sigma, ill != 0, collinear != 0, seed, static_cast<float*>(tensor), truth);
  else if (dtype == NTF_DTYPE_F64)
    generate_impl(s, rank, sigma, ill != 0, collinear != 0, seed, static_cast<double*>(tensor), truth);
  else
    throw InvalidArgument("unknown dtype");
}

// ---- factor error (metrics.cpp:10-111) --------------------------------------

namespace {

// Column-normalised copy (zero columns unchanged).
std::vector<double> unit_columns(const double* a, int rows, int r) {
  std::vector<double> out(a, a + (long long)rows * r);
  for (int j = 0; j < r; ++j) {
    double sq = 0.0;
    for (int i = 0; i < rows; ++i) sq += out[size_t(i) * r + j] * out[size_t(i) * r + j];
    const double nrm = std::sqrt(sq);
    if (nrm > 0.0)
      for (int i = 0; i < rows; ++i) out[size_t(i) * r + j] /= nrm;
  }
  return out;
}

// Min-cost perfect assignment (Jonker-Volgenant style augmenting paths with
// dual potentials); returns assign[row] = column.
std::vector<int> min_cost_assignment(const std::vector<double>& cost, int n) {
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> pr(size_t(n) + 1, 0.0), pc(size_t(n) + 1, 0.0);
  std::vector<int> col_owner(size_t(n) + 1, 0), back(size_t(n) + 1, 0);
  for (int row = 1; row <= n; ++row) {
    col_owner[0] = row;
    int cur = 0;
    std::vector<double> best(size_t(n) + 1, inf);
    std::vector<char> seen(size_t(n) + 1, 0);
    do {
      seen[size_t(cur)] = 1;
      const int rr = col_owner[size_t(cur)];
      double step = inf;
      int nxt = 0;
      for (int c = 1; c <= n; ++c) {
        if (seen[size_t(c)]) continue;
        const double red = cost[size_t(rr - 1) * n + (c - 1)] - pr[size_t(rr)] - pc[size_t(c)];
        if (red < best[size_t(c)]) {
          best[size_t(c)] = red;
          back[size_t(c)] = cur;
        }
        if (best[size_t(c)] < step) {
          step = best[size_t(c)];
          nxt = c;
        }
      }
      for (int c = 0; c <= n; ++c) {
        if (seen[size_t(c)]) {
          pr[size_t(col_owner[size_t(c)])] += step;
          pc[size_t(c)] -= step;
        } else {
          best[size_t(c)] -= step;
        }
      }
      cur = nxt;
    } while (col_owner[size_t(cur)] != 0);
    do {
      const int prev = back[size_t(cur)];
      col_owner[size_t(cur)] = col_owner[size_t(prev)];
      cur = prev;
    } while (cur != 0);
  }
  std::vector<int> assign(size_t(n), -1);
  for (int c = 1; c <= n; ++c)
    if (col_owner[size_t(c)] > 0) assign[size_t(col_owner[size_t(c)] - 1)] = c - 1;
  return assign;
}

}  // namespace

double factor_error(const double* est, const double* truth, const int* shape, int order, int rank) {
  const auto s = check_shape(shape, order, rank);
  std::vector<std::vector<double>> ne, nt;
  long long off = 0;
  for (int i = 0; i < order; ++i) {
    ne.push_back(unit_columns(est + off, s[size_t(i)], rank));
    nt.push_back(unit_columns(truth + off, s[size_t(i)], rank));
    off += (long long)s[size_t(i)] * rank;
  }
  std::vector<double> cost(size_t(rank) * rank, 0.0);
  for (int i = 0; i < order; ++i)
    for (int p = 0; p < rank; ++p)
      for (int q = 0; q < rank; ++q) {
        double sq = 0.0;
        for (int row = 0; row < s[size_t(i)]; ++row) {
          const double d = ne[size_t(i)][size_t(row) * rank + p] - nt[size_t(i)][size_t(row) * rank + q];
          sq += d * d;
        }
        cost[size_t(p) * rank + q] += sq;
      }
  const auto pi = min_cost_assignment(cost, rank);
  double err = 0.0;
  for (int i = 0; i < order; ++i) {
    double num = 0.0, den = 0.0;
    for (int row = 0; row < s[size_t(i)]; ++row)
      for (int p = 0; p < rank; ++p) {
        const double d = nt[size_t(i)][size_t(row) * rank + pi[size_t(p)]] - ne[size_t(i)][size_t(row) * rank + p];
        num += d * d;
      }
    for (double x : nt[size_t(i)]) den += x * x;
    err += std::sqrt(num) / std::sqrt(den);
  }
  return err / order;
}

}  // namespace ntfb
