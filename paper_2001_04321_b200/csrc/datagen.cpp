// Host-side synthetic instances and the factor-error metric.
//
// Instance generation must be bit-exact with the reference generator
// (src/datagen.cpp:13-80): SplitMix64 sub-stream seeds feeding
// std::mt19937_64 (whose output sequence the C++ standard fixes), top-53-bit
// uniforms, cosine-branch Box-Muller, row-major factor fills, noise drawn in
// flat order from sub-stream N. It is inherently sequential in the noise
// stream, so it stays on the host; the reconstruction part is parallel.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <thread>
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
                          uint64_t seed, T* tensor, double* truth, long long slab_b, long long slab_e) {
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
  // The tensor entries of the mode-1 slab [slab_b, slab_e): flat range
  // [f0, f1). Entry e = T_rec[e] (Khatri-Rao row of the leading modes, product
  // from the last listed factor down to the first, kernels.cpp:104-109, dotted
  // with A_last's row in ascending p), then max(0, . + sigma N(0,1)) with
  // the Box-Muller pair drawn from noise draws 2e, 2e+1 of sub-stream N
  // (exactly two draws per entry, no rejection). The noise stream is serial,
  // so one producer thread walks it (discard) and snapshots the engine at
  // every chunk start while OpenMP workers reconstruct and add the noise of
  // whole chunks from their snapshot: same draws, same arithmetic, any
  // thread count.
  long long stride0 = 1;
  for (int i = 1; i < n; ++i) stride0 *= s[size_t(i)];
  const int last = s[size_t(n - 1)];
  const long long f0 = slab_b * stride0, f1 = slab_e * stride0;
  const long long count = f1 - f0;
  if (count <= 0) return;
  // A_last transposed (p-major): the chunk loop runs over columns innermost,
  // which keeps each entry's ascending-p sum while vectorising across entries
  std::vector<double> AnT(size_t(rank) * size_t(last));
  for (int col = 0; col < last; ++col)
    for (int p = 0; p < rank; ++p) AnT[size_t(p) * last + col] = A[size_t(n - 1)][(long long)col * rank + p];
  const long long chunk = 1LL << 20;
  const long long nchunks = (count + chunk - 1) / chunk;
  const bool noisy = sigma > 0.0;
  std::vector<std::mt19937_64> snaps;
  std::atomic<long long> ready{0};
  std::thread producer;
  if (noisy) {
    snaps.resize(size_t(nchunks));
    producer = std::thread([&] {
      std::mt19937_64 g(stream_seed(seed, uint64_t(n)));
      g.discard(2ull * uint64_t(f0));
      for (long long c = 0; c < nchunks; ++c) {
        snaps[size_t(c)] = g;
        ready.store(c + 1, std::memory_order_release);
        if (c + 1 < nchunks) g.discard(2ull * uint64_t(chunk));
      }
    });
  }
#pragma omp parallel
  {
    std::vector<double> buf(static_cast<size_t>(chunk)), w(static_cast<size_t>(rank));
#pragma omp for schedule(dynamic, 1)
    for (long long c = 0; c < nchunks; ++c) {
      const long long a = f0 + c * chunk, z = std::min(f1, a + chunk);
      for (long long e = a; e < z;) {
        const long long row = e / last;  // leading-mode row
        const int c0 = int(e - row * last);
        const int c1 = int(std::min<long long>(last, c0 + (z - e)));
        for (int p = 0; p < rank; ++p) w[size_t(p)] = 1.0;
        long long rest = row;
        for (int l = n - 2; l >= 0; --l) {
          const long long j = rest % s[size_t(l)];
          rest /= s[size_t(l)];
          for (int p = 0; p < rank; ++p) w[size_t(p)] *= A[size_t(l)][j * rank + p];
        }
        double* out = buf.data() + (e - a) - c0;
        for (int col = c0; col < c1; ++col) out[col] = 0.0;
        for (int p = 0; p < rank; ++p) {
          const double wp = w[size_t(p)];
          const double* an = AnT.data() + size_t(p) * last;
          for (int col = c0; col < c1; ++col) out[col] += wp * an[col];
        }
        e += c1 - c0;
      }
      T* dst = tensor + (a - f0);
      if (noisy) {
        while (ready.load(std::memory_order_acquire) <= c) std::this_thread::yield();
        std::mt19937_64 g = snaps[size_t(c)];
        for (long long e = 0; e < z - a; ++e) dst[e] = T(std::max(0.0, buf[size_t(e)] + sigma * gauss_draw(g)));
      } else {
        for (long long e = 0; e < z - a; ++e) dst[e] = T(buf[size_t(e)]);
      }
    }
  }
  if (producer.joinable()) producer.join();
}

void generate(const int* shape, int order, int rank, double sigma, int ill, int collinear, uint64_t seed,
              int dtype, void* tensor, double* truth, long long slab_b, long long slab_e) {
  const auto s = check_shape(shape, order, rank);
  if (sigma < 0.0) throw InvalidArgument("noise level must be >= 0");
  if (ill && rank < 2) throw InvalidArgument("ill-conditioned instances need rank >= 2");
  if (slab_b < 0 && slab_e < 0) {
    slab_b = 0;
    slab_e = s[0];
  }
  if (slab_b < 0 || slab_e < slab_b || slab_e > s[0]) throw InvalidArgument("slab outside the first mode");
  if (dtype == NTF_DTYPE_F32)
    generate_impl(s, rank, sigma, ill != 0, collinear != 0, seed, static_cast<float*>(tensor), truth, slab_b, slab_e);
  else if (dtype == NTF_DTYPE_F64)
    generate_impl(s, rank, sigma, ill != 0, collinear != 0, seed, static_cast<double*>(tensor), truth, slab_b,
                  slab_e);
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
