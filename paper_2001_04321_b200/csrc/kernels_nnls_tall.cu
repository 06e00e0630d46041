// Fused block update for factors too tall for one thread-block cluster
// (I_n > 4096, or beyond the fused kernels' per-rank row limits) or ranks
// above the fused kernels' 64 (up to 128).
//
// The fused kernels (kernels_nnls.cu) keep a whole factor on one 16-CTA
// cluster; the reference has no height limit (nnls.cpp:15-49 loops over all
// rows), so taller factors take this path instead of being refused. Same
// algorithm, split into plain grid kernels with the factor's rows in global
// memory (L2-resident between sweeps):
//
//   setup    G = Hadamard of the other modes' Grams (kernels.cpp:193-200),
//            the skipped columns (G_jj <= 1e-12 max diag, nnls.cpp:16-19),
//            the run scalars
//   init     W := accepted A_i (or the given warm start)
//   sweep x max_iters   one Gauss-Seidel pass over every row (nnls.cpp:20-27,
//            one thread per row), ||W_{s+1} - W_s||_F^2 as per-block partials
//            summed in block order by the last block to finish, which applies
//            the stop rule (nnls.cpp:31-45); later launches are no-ops once a
//            stop is decided -- a fixed launch count, so the sequence
//            captures into the iteration's CUDA graph
//   epilogue HER: S_i := W, X_i := max(0, W + beta (W - A_i)) (her.cpp:66-70);
//            AO: X_i := W; <W, C> partials of the last mode
//   grams    of the written buffers (kernels.cpp:294-296)
//   finish   last mode: F-hat / f (her.cpp:32-38, ao.cpp:37), the restart
//            decision and beta update (her.cpp:73-85, :21-30), the trace record
//
// Every reduction runs in a fixed order: bit-reproducible. One launch of the
// sweep kernel costs a few microseconds, so a block update takes ~0.3 ms at
// 50 sweeps -- a correct fallback, not the fast path.
#include <algorithm>
#include <cstdlib>

#include "ntf_internal.h"

namespace ntfb {
namespace {

constexpr int kTallThreads = 256;
constexpr int kGramRowsPerBlock = 1024;

struct TallCtl {
  int stopped, sweeps, skip, max_iters;  // skip: the run's budget is exhausted (whole update is a no-op)
  unsigned long long okbits[2];          // columns updated (G_jj above the floor), r <= 128
  double tol, first, beta;
  unsigned counter;
};

// workspace layout (doubles)
struct TallWs {
  double* G;       // r x r
  TallCtl* ctl;    // 16 doubles reserved
  double* W;       // rows x r
  double* part;    // nb partials of the sweep / nb of <W,C> / Gram partials
};

__host__ __device__ inline TallWs tall_ws(double* base, int rows, int r) {
  TallWs w;
  w.G = base;
  w.ctl = reinterpret_cast<TallCtl*>(base + size_t(r) * r);
  w.W = base + size_t(r) * r + 16;
  w.part = w.W + size_t(rows) * r;
  return w;
}

__device__ __forceinline__ unsigned long long tall_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool tall_stop_rule(double ch2, double thr) {  // sqrt(ch2) <= thr (nnls.cpp:38)
  if (!(thr >= 0.0)) return sqrt(ch2) <= thr;
  const double t2 = thr * thr;
  if (ch2 < t2 * (1.0 - 1e-12)) return true;
  if (ch2 > t2 * (1.0 + 1e-12)) return false;
  return sqrt(ch2) <= thr;
}

// Deterministic block sum (every thread returns the same value).
__device__ double tall_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

__device__ __forceinline__ const double* buf_x(const NnlsLaunch& a, int mode, int b) {
  return a.has_bufs ? a.bufs.x[mode][b] : a.F->x[mode][b];
}

__global__ void tall_setup_kernel(NnlsLaunch a, double* ws) {
  const int r = a.rank, mode = a.mode;
  TallWs w = tall_ws(ws, a.rows, r);
  __shared__ double dmax_s;
  __shared__ int skip_s;
  if (threadIdx.x == 0) skip_s = (a.F && a.st->done) ? 1 : 0;
  __syncthreads();
  if (skip_s) {
    if (threadIdx.x == 0) w.ctl->skip = 1;
    return;
  }
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    double g = 1.0;
    if (a.role == 2) {
      g = a.gram_in[e];
    } else {
      for (int j = 0; j < a.order; ++j)
        if (j != mode) {
          const double* src = a.has_bufs ? a.bufs.gram[j][a.F->sel[j]] : a.F->gram[j][a.F->sel[j]];
          g *= src[e];
        }
    }
    w.G[e] = g;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double dmax = -INFINITY;
    for (int j = 0; j < r; ++j) dmax = fmax(dmax, w.G[j * r + j]);
    dmax_s = dmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double floor_ = 1e-12 * dmax_s;  // nnls.cpp:16-19
    unsigned long long ok[2] = {0, 0};
    for (int j = 0; j < r; ++j)
      if (w.G[j * r + j] > floor_) ok[j >> 6] |= 1ull << (j & 63);
    TallCtl c{};
    c.okbits[0] = ok[0];
    c.okbits[1] = ok[1];
    c.skip = 0;
    if (a.F) {
      c.max_iters = a.zero_sweeps ? 0 : a.st->inner_max_iters;
      c.tol = a.st->tol;
      c.beta = a.role == 0 ? a.st->beta : 0.0;
    } else {
      c.max_iters = a.zero_sweeps ? 0 : a.max_iters;
      c.tol = a.tol;
      c.beta = 0.0;
    }
    c.stopped = c.max_iters <= 0 ? 1 : 0;
    c.sweeps = 0;
    c.first = 0.0;
    c.counter = 0u;
    *w.ctl = c;
  }
}

__global__ void tall_init_kernel(NnlsLaunch a, double* ws) {
  const int r = a.rank;
  TallWs w = tall_ws(ws, a.rows, r);
  if (w.ctl->skip) return;
  const double* src = (a.role == 2 || a.zero_sweeps) ? a.w0 : buf_x(a, a.mode, a.F->sel[a.mode]);
  const long long n = (long long)a.rows * r;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    w.W[e] = src[e];
}

// One Gauss-Seidel pass over every row (hals_pass, nnls.cpp:15-27).
__global__ void __launch_bounds__(kTallThreads) tall_sweep_kernel(NnlsLaunch a, double* ws, int s) {
  extern __shared__ double Gs[];  // r x r
  __shared__ double red[kTallThreads / 32];
  __shared__ int last_s;
  const int r = a.rank;
  TallWs w = tall_ws(ws, a.rows, r);
  TallCtl* ctl = w.ctl;
  if (ctl->skip || ctl->stopped || s >= ctl->max_iters) return;  // uniform over the grid (set by earlier launches)
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) Gs[e] = w.G[e];
  __syncthreads();
  const unsigned long long ok[2] = {ctl->okbits[0], ctl->okbits[1]};
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (row < a.rows) {
    double x[kMaxTallRank];
    double* wr = w.W + (long long)row * r;
    const double* cr = a.C + (long long)row * r;
    for (int l = 0; l < r; ++l) x[l] = wr[l];
    for (int j = 0; j < r; ++j) {
      if (!((ok[j >> 6] >> (j & 63)) & 1)) continue;
      const double gjj = Gs[j * r + j];
      double acc = 0.0;  // W_{i,:} G_{:,j} with the latest entries
      for (int l = 0; l < r; ++l) acc = fma(x[l], Gs[l * r + j], acc);
      const double numer = cr[j] - acc + gjj * x[j];
      double nw = numer / gjj;
      nw = nw < 0.0 ? 0.0 : nw;
      const double dd = nw - x[j];
      d2 = fma(dd, dd, d2);
      x[j] = nw;
    }
    for (int l = 0; l < r; ++l) wr[l] = x[l];
  }
  const double bsum = tall_block_sum(d2, red);
  if (threadIdx.x == 0) {
    w.part[blockIdx.x] = bsum;
    __threadfence();
    last_s = atomicAdd(&ctl->counter, 1u) == gridDim.x - 1 ? 1 : 0;
  }
  __syncthreads();
  if (!last_s || threadIdx.x != 0) return;
  __threadfence();
  double ch2 = 0.0;  // ||W_{s+1} - W_s||_F^2, blocks in order
  for (unsigned b = 0; b < gridDim.x; ++b) ch2 += __ldcg(w.part + b);
  if (s == 0) ctl->first = sqrt(ch2);
  ctl->sweeps = s + 1;
  if (s + 1 >= ctl->max_iters || tall_stop_rule(ch2, ctl->tol * ctl->first)) ctl->stopped = 1;
  ctl->counter = 0u;
}

// Writes the block; <W, C> partials for the last mode.
__global__ void __launch_bounds__(kTallThreads) tall_epilogue_kernel(NnlsLaunch a, double* ws) {
  __shared__ double red[kTallThreads / 32];
  const int r = a.rank, mode = a.mode;
  TallWs w = tall_ws(ws, a.rows, r);
  if (w.ctl->skip) return;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  double cross = 0.0;
  if (a.role == 2) {
    if (row < a.rows)
      for (int l = 0; l < r; ++l) a.w_out[(long long)row * r + l] = w.W[(long long)row * r + l];
    if (row == 0 && a.sweeps_out) *a.sweeps_out = w.ctl->sweeps;
    return;
  }
  const int sel = a.F->sel[mode];
  const DevFactors& B = a.has_bufs ? a.bufs : *a.F;
  double* X = B.x[mode][sel];
  double* S = B.x[mode][sel ^ 1];
  float* X32 = B.x32[mode][sel];
  float* S32 = B.x32[mode][sel ^ 1];
  const double beta = w.ctl->beta;
  if (row < a.rows) {
    for (int l = 0; l < r; ++l) {
      const long long o = (long long)row * r + l;
      const double v = w.W[o];
      cross = fma(v, a.C[o], cross);
      double h = v;
      if (a.role == 0) {
        const double old = X[o];
        const double t = __dadd_rn(v, __dmul_rn(beta, __dsub_rn(v, old)));  // her.cpp:16-19
        h = t < 0.0 ? 0.0 : t;
        S[o] = v;
        if (S32) S32[o] = float(v);
      }
      X[o] = h;
      if (X32) X32[o] = float(h);
    }
  }
  if (a.last) {
    const double bsum = tall_block_sum(cross, red);
    if (threadIdx.x == 0) w.part[blockIdx.x] = bsum;
  }
}

// Gram partials of `rows` x r rows of buf: block b covers kGramRowsPerBlock rows.
__global__ void __launch_bounds__(kTallThreads) tall_gram_partial_kernel(NnlsLaunch a, double* ws, int which,
                                                                         double* part) {
  const int r = a.rank, mode = a.mode;
  TallWs w = tall_ws(ws, a.rows, r);
  if (w.ctl->skip) return;
  const int sel = a.F->sel[mode];
  const double* buf = buf_x(a, mode, which ? sel ^ 1 : sel);
  const int r0 = blockIdx.x * kGramRowsPerBlock;
  const int r1 = min(a.rows, r0 + kGramRowsPerBlock);
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int p = e / r, q = e % r;
    if (p > q) continue;
    double s0 = 0.0, s1 = 0.0;
    int i = r0;
    for (; i + 1 < r1; i += 2) {
      s0 = fma(buf[(long long)i * r + p], buf[(long long)i * r + q], s0);
      s1 = fma(buf[(long long)(i + 1) * r + p], buf[(long long)(i + 1) * r + q], s1);
    }
    if (i < r1) s0 = fma(buf[(long long)i * r + p], buf[(long long)i * r + q], s0);
    part[(size_t)blockIdx.x * r * r + e] = s0 + s1;
  }
}

__global__ void tall_gram_finish_kernel(NnlsLaunch a, double* ws, int which, const double* part, int nblk) {
  const int r = a.rank, mode = a.mode;
  TallWs w = tall_ws(ws, a.rows, r);
  if (w.ctl->skip) return;
  const int sel = a.F->sel[mode];
  double* g = a.has_bufs ? a.bufs.gram[mode][which ? sel ^ 1 : sel] : a.F->gram[mode][which ? sel ^ 1 : sel];
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int p = e / r, q = e % r;
    if (p > q) continue;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(size_t)b * r * r + e];
    g[p * r + q] = s;
    g[q * r + p] = s;
  }
}

// last_sweeps; last mode: the objective, the restart decision, the trace record
__global__ void tall_finish_kernel(NnlsLaunch a, double* ws, int nb_cross) {
  __shared__ double red[kTallThreads / 32];
  const int r = a.rank, mode = a.mode;
  TallWs w = tall_ws(ws, a.rows, r);
  if (w.ctl->skip) return;
  RunState* st = a.st;
  DevFactors* F = a.F;
  const int s = w.ctl->sweeps;
  if (!a.last) {
    if (threadIdx.x == 0) st->last_sweeps[mode] = s;
    return;
  }
  const int sel = F->sel[mode];
  // <W^T W, G>: the Gram of the solved block (HER: the S buffer, AO: X)
  const double* gw = a.has_bufs ? a.bufs.gram[mode][a.role == 0 ? sel ^ 1 : sel] : F->gram[mode][a.role == 0 ? sel ^ 1 : sel];
  double q = 0.0;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) q = fma(gw[e], w.G[e], q);
  const double quad = tall_block_sum(q, red);
  if (threadIdx.x != 0) return;
  double cross = 0.0;
  for (int b = 0; b < nb_cross; ++b) cross += w.part[b];
  const double f = 0.5 * st->nsq - cross + 0.5 * quad;
  int sweeps_before = 0;
  for (int j = 0; j < a.order; ++j)
    if (j != mode) sweeps_before += st->last_sweeps[j];
  st->last_sweeps[mode] = s;
  const int kk = st->k + 1;
  const double time_s = double(tall_timer() - st->t_start_ns) * 1e-9;
  TraceEntry rec;
  rec.f = f;
  rec.time_s = time_s;
  rec.sweeps = sweeps_before + s;
  const double beta = w.ctl->beta;
  if (a.role == 0) {
    const bool restarted = f > st->f_prev;  // strict (her.cpp:75)
    if (restarted)
      for (int j = 0; j < a.order; ++j) F->sel[j] ^= 1;  // X := S for every mode
    st->f_prev = f;                                      // even on rejection (:84)
    rec.beta = beta;
    rec.restarted = restarted ? 1 : 0;
    if (restarted) {  // update_betas (her.cpp:21-30)
      st->beta_bar = beta;
      st->beta = __ddiv_rn(beta, st->eta);
    } else {
      const double bb = st->beta_bar;
      st->beta = fmin(bb, __dmul_rn(beta, st->gamma));
      st->beta_bar = fmin(1.0, __dmul_rn(bb, st->gamma_bar));
    }
  } else {
    rec.beta = 0.0;
    rec.restarted = 0;
  }
  a.trace[kk - 1] = rec;
  st->f_last = f;
  st->k = kk;
  st->elapsed_s = time_s;
  if ((st->max_iters > 0 && kk >= st->max_iters) ||
      (!st->collective_time && st->max_time_s > 0.0 && time_s >= st->max_time_s))
    st->done = 1;
}

}  // namespace

size_t nnls_tall_workspace(int rows, int rank) {
  const size_t nb = size_t((rows + kTallThreads - 1) / kTallThreads);
  const size_t ng = size_t((rows + kGramRowsPerBlock - 1) / kGramRowsPerBlock);
  return size_t(rank) * rank + 16 + size_t(rows) * rank + (nb + 7) / 8 * 8 + ng * rank * rank + 64;
}

// max_iters_host: the inner sweep budget as the host knows it (the launch count of the sweep kernel)
void launch_nnls_tall(const NnlsLaunch& a, cudaStream_t s, int max_iters_host) {
  if (!a.tall) throw LogicError("tall NNLS path without a workspace");
  if (a.rank > kMaxTallRank) throw Unsupported("rank outside the NNLS kernels' range (1..128)");
  double* ws = a.tall;
  const int nb = (a.rows + kTallThreads - 1) / kTallThreads;
  const int ng = (a.rows + kGramRowsPerBlock - 1) / kGramRowsPerBlock;
  TallWs w = tall_ws(ws, a.rows, a.rank);
  tall_setup_kernel<<<1, 256, 0, s>>>(a, ws);
  tall_init_kernel<<<std::min(nb, 1024), kTallThreads, 0, s>>>(a, ws);
  const size_t smem = size_t(a.rank) * a.rank * sizeof(double);
  if (smem > 48 * 1024)
    NTF_CUDA(cudaFuncSetAttribute(tall_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  for (int it = 0; it < max_iters_host; ++it) tall_sweep_kernel<<<nb, kTallThreads, smem, s>>>(a, ws, it);
  tall_epilogue_kernel<<<nb, kTallThreads, 0, s>>>(a, ws);
  if (a.role != 2) {
    double* gp = w.part + ((nb + 7) / 8) * 8;  // Gram partials behind the <W,C> partials
    const int nmat = a.role == 0 ? 2 : 1;
    for (int m = 0; m < nmat; ++m) {
      tall_gram_partial_kernel<<<ng, kTallThreads, 0, s>>>(a, ws, m, gp);
      tall_gram_finish_kernel<<<1, 256, 0, s>>>(a, ws, m, gp, ng);
    }
    tall_finish_kernel<<<1, kTallThreads, 0, s>>>(a, ws, nb);
  }
  NTF_CUDA(cudaGetLastError());
}

}  // namespace ntfb
