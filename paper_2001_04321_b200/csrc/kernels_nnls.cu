// Fused block update for one mode of an outer iteration:
//
//   G   = hadamard of the other modes' X-role Grams       (kernels.cpp:193-200)
//   W   = AHALS(G, C, W0 = accepted A_i), <= max_iters      (nnls.cpp:15-49)
//         Gauss-Seidel column sweeps with the global stop rule
//         ||W_{s+1} - W_s||_F <= tol * ||W_1 - W_0||_F
//   HER: S_i := W, X_i := max(0, W + beta (W - A_i))        (her.cpp:66-70)
//   AO : X_i := W                                            (ao.cpp:35-39)
//   Grams of the written buffers                             (kernels.cpp:294-296)
//   last mode: F-hat / f = 0.5||T||^2 - <W,C> + 0.5<W^T W, G> (her.cpp:32-38,
//         ao.cpp:37) and, for HER, the restart decision and beta update
//         (her.cpp:73-85, :21-30) plus the trace record — all on the device,
//         so an outer iteration needs no host synchronisation.
//
// One thread owns one row of W (rows are independent inside a pass,
// nnls.cpp:22); the row lives in registers for all sweeps. The rows are
// spread over a thread-block cluster of up to 16 CTAs (one SM each) so the
// rows*r^2 FMAs of a sweep and the column recurrence of each row run in
// parallel; the per-sweep stop rule, the Grams and <W,C> are reduced through
// distributed shared memory in a fixed CTA order (bit-reproducible) with one
// cluster barrier per reduction.
#include <cooperative_groups.h>

#include <cstdlib>

#include "ntf_internal.h"

namespace cg = cooperative_groups;

namespace ntfb {
namespace {

constexpr int kMaxCluster = 16;

// diagnostics: CTA 0's sweep-loop cycles, of which in the cluster reduction,
// sweeps, calls (read with ntfb::nnls_prof_read)
__device__ unsigned long long g_nnls_prof[4];

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Deterministic block sum; every thread receives the same value.
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (blockDim.x == 32) return v;
  __syncthreads();  // red may still be read from a previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) s += red[w];
  return s;
}

// Sum over the cluster, same bits in every thread of every CTA: each CTA
// publishes its block sum in its own shared slot pub[parity]; after the
// cluster barrier every thread adds the slots in CTA-rank order. Callers
// alternate `parity` so a slot is never rewritten before every CTA has read
// it (the rewrite happens after the next barrier).
__device__ double cluster_sum(double v, double* red, double* pub, int parity, cg::cluster_group& cl) {
  const double b = block_sum(v, red);
  const unsigned n = cl.num_blocks();
  if (n == 1) return b;
  // push: lane k of warp 0 stores this CTA's sum into slot [parity][me] of
  // CTA k (remote shared stores are fire-and-forget); the cluster barrier's
  // release/acquire makes them visible, then every CTA reads locally
  const unsigned me = cl.block_rank();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < n) *cl.map_shared_rank(&pub[parity * kMaxCluster + me], unsigned(lane)) = b;
  cl.sync();
  double s = 0.0;
  for (unsigned k = 0; k < n; ++k) s += pub[parity * kMaxCluster + k];
  return s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Sum over the cluster without a cluster barrier, in two halves so a sweep
// can run between them: cluster_post sends this CTA's block sum to slot [me]
// of every CTA with st.async, which completes transaction bytes on the
// receiver's mbarrier `bar` (expecting n*8 bytes plus its own arrival);
// cluster_fin waits for the n slots (`phase` = parity of this use of `bar`)
// and adds them in CTA-rank order. The same bits reach every CTA. A slot
// buffer is reused two reductions later: a CTA can only post there after
// every CTA has posted the reduction in between, i.e. after reading it.
__device__ double cluster_post(double v, double* red, double* slots, uint64_t* bar, cg::cluster_group& cl) {
  const double b = block_sum(v, red);
  const unsigned n = cl.num_blocks();
  if (n == 1) return b;
  const unsigned me = cl.block_rank();
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(n * 8u)
                 : "memory");
  if (threadIdx.x < n) {
    uint32_t raddr, rbar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(&slots[me])), "r"(threadIdx.x));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(bar)), "r"(threadIdx.x));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(b)), "r"(rbar)
                 : "memory");
  }
  return b;
}

__device__ double cluster_fin(double b, const double* slots, uint64_t* bar, uint32_t phase, cg::cluster_group& cl) {
  const unsigned n = cl.num_blocks();
  if (n == 1) return b;
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
  // (st.async data is visible once its complete_tx is observed; no
  // cluster-scope acquire, which would invalidate L1)
  double s = 0.0;
  for (unsigned k = 0; k < n; ++k) s += slots[k];
  __syncwarp();  // every lane has read the slots before any lane posts again
  return s;
}

// sqrt(ch2) <= thr (nnls.cpp:38) without the square root on the sweep
// loop's critical path unless ch2 is within rounding of thr^2.
__device__ __forceinline__ bool stop_rule(double ch2, double thr) {
  if (!(thr >= 0.0)) return sqrt(ch2) <= thr;
  const double t2 = thr * thr;
  if (ch2 < t2 * (1.0 - 1e-12)) return true;
  if (ch2 > t2 * (1.0 + 1e-12)) return false;
  return sqrt(ch2) <= thr;
}

// Eigen's cwiseMax(0.0): (a < 0) ? 0 : a.
__device__ __forceinline__ double clip0(double a) { return a < 0.0 ? 0.0 : a; }

// Gram of the rows staged in `stage` ([blockDim][RP+1]) of every CTA of the
// cluster, written to `dst` (r x r): per-CTA partials in shared memory, then
// CTA k sums entries e == k (mod n) over the CTAs in rank order.
template <int RP>
__device__ void cluster_gram(const double* stage, int nrows, double* part, int r, double* dst,
                             cg::cluster_group& cl) {
  constexpr int LD = RP + 1;
  const int nt = blockDim.x;
  for (int e = threadIdx.x; e < r * r; e += nt) {
    const int p = e / r, q = e % r;
    if (p > q) continue;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int i = 0; i < nrows; i += 4) {
      s0 += stage[(i + 0) * LD + p] * stage[(i + 0) * LD + q];
      s1 += stage[(i + 1) * LD + p] * stage[(i + 1) * LD + q];
      s2 += stage[(i + 2) * LD + p] * stage[(i + 2) * LD + q];
      s3 += stage[(i + 3) * LD + p] * stage[(i + 3) * LD + q];
    }
    part[e] = (s0 + s1) + (s2 + s3);
  }
  const unsigned n = cl.num_blocks();
  cl.sync();  // partials visible cluster-wide (n == 1: a plain CTA barrier)
  const unsigned me = cl.block_rank();
  for (int e = threadIdx.x * int(n) + int(me); e < r * r; e += nt * int(n)) {
    const int p = e / r, q = e % r;
    if (p > q) continue;
    double s = 0.0;
    double vals[kMaxCluster];  // all remote loads in flight before the ordered sum
#pragma unroll
    for (int k = 0; k < kMaxCluster; ++k) vals[k] = k < int(n) ? cl.map_shared_rank(part, unsigned(k))[e] : 0.0;
#pragma unroll
    for (int k = 0; k < kMaxCluster; ++k)
      if (k < int(n)) s += vals[k];
    dst[p * r + q] = s;
    dst[q * r + p] = s;
  }
  cl.sync();  // partials are reused by the next Gram; dst visible cluster-wide
}

template <int RP, int RPT, int TPB>
__global__ void __launch_bounds__(TPB) nnls_kernel(NnlsLaunch a) {
  constexpr int LD = RP + 1;
  extern __shared__ double smem[];
  double* Gs = smem;                 // RP*RP
  double* red = Gs + RP * RP;        // 32
  double* pub = red + 32;            // 2 x kMaxCluster: pushed block sums (by parity)
  double* part = pub + 2 * kMaxCluster;  // RP*RP: Gram partial of this CTA
  double* Ginv = part + RP * RP;     // RP: 1 / G_jj (0 for skipped columns)
  double* Hs = Ginv + RP;            // RP: G_{j-1,j} / G_jj (0 for skipped columns)
  double* stage = Hs + RP;           // (blockDim*RPT) * LD: staged rows (Grams)
  double* Cs = stage + size_t(blockDim.x) * RPT * LD;  // (blockDim*RPT) * LD: rows of C
  double* aslots = Cs + size_t(blockDim.x) * RPT * LD;  // 2 x kMaxCluster: st.async sums
  uint64_t* abar = reinterpret_cast<uint64_t*>(aslots + 2 * kMaxCluster);  // 2 mbarriers
  cg::cluster_group cl = cg::this_cluster();

  RunState* st = a.st;
  if (st && st->done) return;  // budget exhausted: the whole iteration is a no-op (uniform)

  const int r = a.rank, mode = a.mode;
  const int nloc = int(blockDim.x) * RPT;                              // row slots per CTA
  const int rpc = (a.rows + int(gridDim.x) - 1) / int(gridDim.x);    // rows per CTA
  // thread t owns local rows t, t + blockDim, ... (coalesced loads/stores)
  int row[RPT];
  bool valid[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int lr = int(threadIdx.x) + i * int(blockDim.x);
    row[i] = int(blockIdx.x) * rpc + lr;
    valid[i] = lr < rpc && row[i] < a.rows;
  }
  DevFactors* F = a.F;
  const int sel = F ? F->sel[mode] : 0;
  double* X = F ? F->x[mode][sel] : nullptr;
  const double beta = (a.role == 0) ? st->beta : 0.0;
  const int max_iters = (a.role == 2) ? a.max_iters : st->inner_max_iters;
  const double tol = (a.role == 2) ? a.tol : st->tol;
  const double* w0 = (a.role == 2) ? a.w0 : X;
  const double* C = a.C;

  // ---- G: Hadamard of the other modes' Grams (ones, ascending modes).
  for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) {
    const int p = e / RP, q = e % RP;
    double g = 0.0;
    if (p < r && q < r) {
      if (a.role == 2) {
        g = a.gram_in[p * r + q];
      } else {
        g = 1.0;
        for (int j = 0; j < a.order; ++j)
          if (j != mode) g *= F->gram[j][F->sel[j]][p * r + q];
      }
    }
    Gs[e] = g;
  }
  // rows of C in shared memory (read once per column per sweep, off the chain)
  for (int e = threadIdx.x; e < nloc * RP; e += blockDim.x) {
    const int lr = e / RP, l = e % RP;
    const int gr = int(blockIdx.x) * rpc + lr;
    Cs[lr * LD + l] = (lr < rpc && gr < a.rows && l < r) ? C[(long long)gr * r + l] : 0.0;
  }
  __syncthreads();
  double dmax = -INFINITY;
  for (int j = 0; j < r; ++j) dmax = fmax(dmax, Gs[j * RP + j]);
  const double diag_floor = 1e-12 * dmax;  // nnls.cpp:16-19
  // columns with G_jj <= floor are skipped: ginv = h = 0 leaves them as they are
  unsigned long long okmask = 0;
  for (int j = 0; j < r; ++j)
    if (Gs[j * RP + j] > diag_floor) okmask |= 1ull << j;
  for (int j = threadIdx.x; j < RP; j += blockDim.x) {
    const bool ok = (okmask >> j) & 1;
    const double gi = ok ? 1.0 / Gs[j * RP + j] : 0.0;
    Ginv[j] = gi;
    Hs[j] = (ok && j > 0) ? Gs[(j - 1) * RP + j] * gi : 0.0;
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&abar[b])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();  // every CTA's mbarriers exist before any st.async targets them; Ginv/Hs visible

  double W[RPT][RP];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int l = 0; l < RP; ++l) W[i][l] = (valid[i] && l < r) ? w0[(long long)row[i] * r + l] : 0.0;

  // ---- AHALS sweeps.
  // Column j of a pass needs prod_j = (W G)[row, j] with columns < j already
  // updated in this pass (nnls.cpp:22). It is assembled as
  //   P[j] = sum_{l >= j} W_old[l] G[l][j]      (all j at once, ILP)
  //        + sum_{l < j}  W_new[l] G[l][j]      (added as columns finish),
  // so column j needs no dot product once column j-1 is known.
  // The division by G_jj is a multiply by its reciprocal (<= 1 ulp apart).
  // RPT rows per thread share every G read and interleave their chains.
  double first = -1.0;
  int s = 0;
  long long prof_red = 0;  // diagnostics: cycles in the per-sweep cluster reduction
  const long long prof_t0 = clock64();
  constexpr bool kIncremental = RP <= 32;  // P[] costs RPT*RP more registers
  auto sweep = [&]() -> double {
    double P[RPT][kIncremental ? RP : 1];
    if constexpr (kIncremental) {
      // row l of G is contiguous: 16-byte broadcast reads; P[j] still sums
      // l = j, j+1, ... in ascending order
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int j = 0; j < RP; ++j) P[i][j] = 0.0;
#pragma unroll
      for (int l = 0; l < RP; ++l) {
#pragma unroll
        for (int j = 0; j <= l; j += 2) {
          const double2 g = *reinterpret_cast<const double2*>(&Gs[l * RP + j]);
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            P[i][j] = fma(W[i][l], g.x, P[i][j]);
            if (j + 1 <= l) P[i][j + 1] = fma(W[i][l], g.y, P[i][j + 1]);
          }
        }
      }
    }
    double d2 = 0.0;
    if constexpr (kIncremental) {
      // Branch-free: padded (j >= r) and skipped columns have ginv = h = 0 and
      // come out unchanged. With P[j] holding every term of (W G)[row, j] but
      // column j-1's,
      //   numer_j / G_jj = (C_j - P[j]) / G_jj + W_j - h_j * Wnew_{j-1},
      // whose first part is ready a column early: the serial chain from
      // column j-1 to j is one FMA and the clip.
      double prev[RPT];
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const double ginv = Ginv[j], h = Hs[j];
        const bool ok = (okmask >> j) & 1ull;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const double c = Cs[(int(threadIdx.x) + i * int(blockDim.x)) * LD + j];
          const double t = fma(c - P[i][j], ginv, W[i][j]);
          const double v = j == 0 ? t : fma(-h, prev[i], t);
          const double nw = (ok && v < 0.0) ? 0.0 : v;  // cwiseMax(0.0)
          const double d = nw - W[i][j];
          d2 = fma(d, d, d2);
          W[i][j] = nw;
          prev[i] = nw;
        }
        // columns q >= j + 2 (column j + 1 takes this one through h)
#pragma unroll
        for (int q = (j + 2) & ~1; q < RP; q += 2) {
          const double2 g = *reinterpret_cast<const double2*>(&Gs[j * RP + q]);
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            if (q >= j + 2) P[i][q] = fma(W[i][j], g.x, P[i][q]);
            P[i][q + 1] = fma(W[i][j], g.y, P[i][q + 1]);
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        if (j < r) {
          const double gjj = Gs[j * RP + j];
          const double ginv = Ginv[j];
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
            for (int l = 0; l < RP; l += 4) {
              p0 = fma(W[i][l + 0], Gs[(l + 0) * RP + j], p0);
              p1 = fma(W[i][l + 1], Gs[(l + 1) * RP + j], p1);
              p2 = fma(W[i][l + 2], Gs[(l + 2) * RP + j], p2);
              p3 = fma(W[i][l + 3], Gs[(l + 3) * RP + j], p3);
            }
            const double prod = (p0 + p1) + (p2 + p3);
            if (gjj > diag_floor) {
              const double c = Cs[(int(threadIdx.x) + i * int(blockDim.x)) * LD + j];
              const double numer = __dadd_rn(__dsub_rn(c, prod), __dmul_rn(gjj, W[i][j]));
              const double nw = clip0(__dmul_rn(numer, ginv));
              const double d = nw - W[i][j];
              d2 = fma(d, d, d2);
              W[i][j] = nw;
            }
          }
        }
      }
    }
    return d2;
  };
  // Sweep s + 1 runs speculatively while the cluster reduction of sweep s's
  // change is in flight; if sweep s meets the stop rule its result is
  // restored from Wsave (nnls.cpp:33-39: the stop test follows the sweep).
  constexpr bool kSpeculate = kIncremental;
  auto post = [&](double d2, int k) {
    return cluster_post(d2, red, aslots + (k & 1) * kMaxCluster, &abar[k & 1], cl);
  };
  auto fin = [&](double b, int k) {
    return cluster_fin(b, aslots + (k & 1) * kMaxCluster, &abar[k & 1], uint32_t(k >> 1) & 1u, cl);
  };
  if (max_iters > 0) {
    double b = post(sweep(), 0);
    for (;;) {
      const bool spec = kSpeculate && s + 1 < max_iters;
      double Wsave[RPT][RP];
      double d2n = 0.0;
      if (spec) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
#pragma unroll
          for (int l = 0; l < RP; ++l) Wsave[i][l] = W[i][l];
        d2n = sweep();
      }
      const long long tr0 = clock64();
      const double ch2 = fin(b, s);  // ||W_{s+1} - W_s||_F^2
      prof_red += clock64() - tr0;
      if (s == 0) first = sqrt(ch2);
      ++s;
      if (stop_rule(ch2, tol * first)) {
        if (spec) {
#pragma unroll
          for (int i = 0; i < RPT; ++i)
#pragma unroll
            for (int l = 0; l < RP; ++l) W[i][l] = Wsave[i][l];
        }
        break;
      }
      if (s >= max_iters) break;
      if (!spec) d2n = sweep();
      b = post(d2n, s);
    }
  }

  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_nnls_prof[0] += clock64() - prof_t0;
    g_nnls_prof[1] += prof_red;
    g_nnls_prof[2] += s;
    g_nnls_prof[3] += 1;
  }
  if (a.role == 2) {
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (valid[i]) {
#pragma unroll
        for (int l = 0; l < RP; ++l)
          if (l < r) a.w_out[(long long)row[i] * r + l] = W[i][l];
      }
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s;
    return;
  }

  // ---- Gram(W): needed by F-hat / f and, on a restart, as the new Gram.
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int l = 0; l < RP; ++l)
      stage[(int(threadIdx.x) + i * int(blockDim.x)) * LD + l] = (valid[i] && l < r) ? W[i][l] : 0.0;
  __syncthreads();
  double* gW = (a.role == 0) ? F->gram[mode][sel ^ 1] : F->gram[mode][sel];
  cluster_gram<RP>(stage, nloc, part, r, gW, cl);

  // ---- write the block (HER: solved + extrapolated twin; AO: in place);
  // the twin is staged for its Gram as it is produced.
  double* S = F->x[mode][sel ^ 1];
  float* X32 = F->x32[mode][sel];
  float* S32 = F->x32[mode][sel ^ 1];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
#pragma unroll
    for (int l = 0; l < RP; ++l) {
      double h = 0.0;
      if (valid[i] && l < r) {
        const long long o = (long long)row[i] * r + l;
        if (a.role == 0) {
          const double old = X[o];
          h = clip0(__dadd_rn(W[i][l], __dmul_rn(beta, __dsub_rn(W[i][l], old))));
          S[o] = W[i][l];
          if (S32) S32[o] = float(W[i][l]);
        } else {
          h = W[i][l];
        }
        X[o] = h;
        if (X32) X32[o] = float(h);
      }
      if (a.role == 0) stage[(int(threadIdx.x) + i * int(blockDim.x)) * LD + l] = h;
    }
  }
  if (a.role == 0) {
    __syncthreads();
    cluster_gram<RP>(stage, nloc, part, r, F->gram[mode][sel], cl);
  }
  if (!a.last) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->last_sweeps[mode] = s;
    return;
  }

  // ---- objective at the (mixed) point: <W, C> and <W^T W, G>.
  double cross = 0.0;
#pragma unroll
  for (int i = 0; i < RPT; ++i)
    if (valid[i]) {
#pragma unroll
      for (int l = 0; l < RP; ++l)
        if (l < r) cross += W[i][l] * Cs[(int(threadIdx.x) + i * int(blockDim.x)) * LD + l];
    }
  cross = cluster_sum(cross, red, pub, (s + 1) & 1, cl);
  if (blockIdx.x != 0 || threadIdx.x != 0) return;

  double quad = 0.0;
  for (int p = 0; p < r; ++p)
    for (int q = 0; q < r; ++q) quad += gW[p * r + q] * Gs[p * RP + q];
  const double f = 0.5 * st->nsq - cross + 0.5 * quad;

  st->last_sweeps[mode] = s;
  const int k = st->k + 1;
  const double time_s = double(globaltimer() - st->t_start_ns) * 1e-9;
  TraceEntry rec;
  rec.f = f;
  rec.time_s = time_s;
  rec.sweeps = 0;
  for (int j = 0; j < a.order; ++j) rec.sweeps += st->last_sweeps[j];
  if (a.role == 0) {
    const bool restarted = f > st->f_prev;  // strict (her.cpp:75)
    if (restarted)
      for (int j = 0; j < a.order; ++j) F->sel[j] ^= 1;  // X := S for every mode
    st->f_prev = f;                                      // even on rejection (:84)
    rec.beta = st->beta;                                 // beta_used
    rec.restarted = restarted ? 1 : 0;
    if (restarted) {  // update_betas (her.cpp:21-30)
      st->beta_bar = st->beta;
      st->beta = __ddiv_rn(st->beta, st->eta);
    } else {
      st->beta = fmin(st->beta_bar, __dmul_rn(st->beta, st->gamma));
      st->beta_bar = fmin(1.0, __dmul_rn(st->beta_bar, st->gamma_bar));
    }
  } else {
    rec.beta = 0.0;
    rec.restarted = 0;
  }
  a.trace[k - 1] = rec;
  st->f_last = f;
  st->k = k;
  if ((st->max_iters > 0 && k >= st->max_iters) || (st->max_time_s > 0.0 && time_s >= st->max_time_s))
    st->done = 1;
}

// Cluster size: one warp of RPT-row threads per CTA when the factor allows,
// at most 16 CTAs (non-portable cluster size, B200 allows it).
int cluster_size(int rows, int rows_per_warp) {
  return std::max(1, std::min((rows + rows_per_warp - 1) / rows_per_warp, kMaxCluster));
}

template <int RP, int RPT, int TPB>
void launch_rpt(const NnlsLaunch& a, cudaStream_t s) {
  const int cl = cluster_size(a.rows, 32 * RPT);
  const int rpc = (a.rows + cl - 1) / cl;
  const int threads = ((rpc + RPT - 1) / RPT + 31) / 32 * 32;
  if (threads > TPB) throw Unsupported("factor too tall for the fused NNLS kernel");
  const size_t nloc = size_t(threads) * RPT;
  const size_t smem =
      sizeof(double) * (2 * RP * RP + 32 + 2 * kMaxCluster + 2 * RP + 2 * nloc * (RP + 1) + 2 * kMaxCluster + 2);
  auto fn = nnls_kernel<RP, RPT, TPB>;
  NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  if (cl > 8) NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  NnlsLaunch args = a;
  void* params[] = {&args};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  NTF_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(fn), params));
}

// One row per thread (the sweep is latency-bound per warp).
template <int RP, int TPB>
void launch_rp(const NnlsLaunch& a, cudaStream_t s) {
  launch_rpt<RP, 1, TPB>(a, s);
}

}  // namespace

void nnls_prof_read(unsigned long long out[4], bool reset) {
  NTF_CUDA(cudaMemcpyFromSymbol(out, g_nnls_prof, sizeof(unsigned long long) * 4));
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    NTF_CUDA(cudaMemcpyToSymbol(g_nnls_prof, z, sizeof z));
  }
}

void launch_nnls(const NnlsLaunch& a, cudaStream_t s) {
  const int r = a.rank;
  if (r < 1 || r > kMaxRank) throw Unsupported("rank outside the fused NNLS kernel's range (1..64)");
  if (a.rows > kMaxCluster * 256) throw Unsupported("factor taller than 4096 rows");
  if (r <= 4) return launch_rp<4, 256>(a, s);
  if (r <= 8) return launch_rp<8, 256>(a, s);
  if (r <= 12) return launch_rp<12, 256>(a, s);
  if (r <= 16) return launch_rp<16, 256>(a, s);
  if (r <= 20) return launch_rp<20, 256>(a, s);
  if (r <= 24) return launch_rp<24, 256>(a, s);
  if (r <= 32) return launch_rp<32, 256>(a, s);
  if (r <= 48) return launch_rp<48, 256>(a, s);
  return launch_rp<64, 256>(a, s);
}

}  // namespace ntfb
