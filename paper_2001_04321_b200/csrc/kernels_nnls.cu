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
constexpr int kMaxWarps = 8;  // per CTA (256 threads)

// diagnostics: CTA 0's sweep-loop cycles, of which in the cluster reduction,
// sweeps, calls (read with ntfb::nnls_prof_read)
__device__ unsigned long long g_nnls_prof[8];  // + [4] cycles in passes, [5] passes, [6] triangle cycles
// per-pass probes (compile with -DNTF_NNLS_PROFILE=1): clock reads cost ~30 cycles each
#ifndef NTF_NNLS_PROFILE
#define NTF_NNLS_PROFILE 0
#endif
#ifndef NTF_NNLS_SYNCWARP
#define NTF_NNLS_SYNCWARP 1
#endif
__device__ __forceinline__ long long pclock() { return NTF_NNLS_PROFILE ? clock64() : 0; }
// globaltimer of post / fin completion of pass 4, per (CTA, warp), last call (profile builds)
__device__ unsigned long long g_nnls_skew[3][128];

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

// Sum over the cluster without any barrier, in two halves so a sweep can
// run between them. cluster_post: every warp reduces its lanes (butterfly,
// same bits in every lane) and sends the value to slot [cta * nwarps + warp]
// of every CTA with st.async, which completes transaction bytes on the
// receiver's mbarrier `bar` (expecting n * nwarps * 8 bytes plus one arrival,
// by thread 0). cluster_fin waits for the slots (`phase` = parity of this use
// of `bar`) and adds them in a fixed order. The same bits reach every thread.
// A slot buffer is reused two reductions later: a warp can only post there
// after every warp has posted the reduction in between, i.e. after reading.
__device__ void cluster_post(double v, double* slots, uint64_t* bar, cg::cluster_group& cl) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const unsigned n = cl.num_blocks(), me = cl.block_rank();
  const unsigned nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(n * nw * 8u)
                 : "memory");
  if (lane < n) {
    uint32_t raddr, rbar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(&slots[me * nw + warp])), "r"(lane));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(bar)), "r"(lane));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
  }
}

__device__ double cluster_fin(const double* slots, uint64_t* bar, uint32_t phase, cg::cluster_group& cl) {
  const unsigned total = cl.num_blocks() * (blockDim.x >> 5);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
  // (st.async data is visible once its complete_tx is observed; no
  // cluster-scope acquire, which would invalidate L1)
  // lane l adds slots l, l + 32, ... (loads in flight together), then a
  // butterfly: identical operations in every warp, so identical bits
  const unsigned lane = threadIdx.x & 31;
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < kMaxCluster * kMaxWarps / 32; ++i) {
    const unsigned e = lane + 32u * i;
    const double x = e < total ? slots[e] : 0.0;
    v = i == 0 ? x : v + x;
  }
  __syncwarp();  // every lane has read the slots before any lane posts again
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
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

// Lanes per row Q (see the sweep below).
template <int RP, int Q>
struct SweepShape {
  static constexpr bool kIncremental = RP <= 32;  // per-column partial sums in registers
  static constexpr int PQ = RP / Q;               // columns per lane
  static constexpr int PQP = (PQ + 1) & ~1;        // padded: 16-byte aligned per-lane runs
  static constexpr int RS = Q * PQP;               // row stride of the lane-permuted matrices
  static_assert(RP % Q == 0 && (Q == 1 || kIncremental), "lane split needs the incremental sweep");
};

template <int RP, int Q, int TPB>
__global__ void __launch_bounds__(TPB, 1) nnls_kernel(NnlsLaunch a) {
  using Shape = SweepShape<RP, Q>;
  constexpr int LD = RP + 1;
  constexpr int PQ = Shape::PQ, PQP = Shape::PQP, RS = Shape::RS;
  constexpr bool kIncremental = Shape::kIncremental;
  extern __shared__ double smem[];
  const int nloc = int(blockDim.x) / Q;  // row slots per CTA
  double* Gs = smem;                     // RP*RP
  double* red = Gs + RP * RP;            // 32
  double* pub = red + 32;                // 2 x kMaxCluster: pushed block sums (by parity)
  double* part = pub + 2 * kMaxCluster;  // RP*RP: Gram partial of this CTA
  double* Ginv = part + RP * RP;         // RP: 1 / G_jj (0 for skipped columns)
  // column constants (hd_j, lo_j) = (G[j-1][j] / G_jj, clip bound 0), (0, -inf) when skipped
  double* HL = Ginv + RP;                // 2*RP
  // lane-permuted [l][k][m] (column q = m Q + k, lane k's run contiguous):
  double* HmP = HL + 2 * RP;             // RP*RS: G[l][q] / G_qq for l + 2 <= q (pushes), else 0
  double* GtP = HmP + (kIncremental ? RP * RS : 0);  // RP*RS: G[l][q] / G_qq for l > q, -1 at l == q if skipped
  double* stage = GtP + (kIncremental ? RP * RS : 0);  // nloc * LD: staged rows (Grams)
  double* Cs = stage + size_t(nloc) * LD;  // nloc * LD: rows of C
  double* aslots = Cs + size_t(nloc) * LD;  // 2 x kMaxCluster*kMaxWarps: st.async sums
  uint64_t* abar = reinterpret_cast<uint64_t*>(aslots + 2 * kMaxCluster * kMaxWarps);  // 2 mbarriers
  cg::cluster_group cl = cg::this_cluster();

  RunState* st = a.st;
  if (st && st->done) return;  // budget exhausted: the whole iteration is a no-op (uniform)

  const int r = a.rank, mode = a.mode;
  const int rpc = (a.rows + int(gridDim.x) - 1) / int(gridDim.x);  // rows per CTA
  // Q consecutive lanes own one row: lane k of the group keeps the sweep
  // products of columns k, k + Q, ...; W is replicated in the group.
  const int lr = int(threadIdx.x) / Q, k = int(threadIdx.x) % Q;
  const int row = int(blockIdx.x) * rpc + lr;
  const bool valid = lr < rpc && row < a.rows;
  const bool lead = valid && k == 0;  // writes the row
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
  // rows of C in shared memory
  for (int e = threadIdx.x; e < nloc * RP; e += blockDim.x) {
    const int i = e / RP, l = e % RP;
    const int gr = int(blockIdx.x) * rpc + i;
    Cs[i * LD + l] = (i < rpc && gr < a.rows && l < r) ? C[(long long)gr * r + l] : 0.0;
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
    HL[2 * j] = j > 0 ? Gs[(j - 1) * RP + j] * gi : 0.0;
    HL[2 * j + 1] = ok ? 0.0 : -INFINITY;
  }
  for (int e = threadIdx.x; kIncremental && e < RP * RS; e += blockDim.x) {
    const int l = e / RS, kk = (e % RS) / PQP, m = e % PQP, q = m * Q + kk;
    double h = 0.0, g = 0.0;
    if (m < PQ) {
      const bool ok = (okmask >> q) & 1;
      const double gi = ok ? 1.0 / Gs[q * RP + q] : 0.0;
      h = l + 2 <= q ? Gs[l * RP + q] * gi : 0.0;
      g = l > q ? Gs[l * RP + q] * gi : (l == q && !ok ? -1.0 : 0.0);
    }
    HmP[e] = h;
    GtP[e] = g;
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&abar[b])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();  // every CTA's mbarriers exist before any st.async targets them; Ginv/Hm/Gm visible

  double W[RP], WB[RP];  // the sweeps alternate W -> WB -> W ...
#pragma unroll
  for (int l = 0; l < RP; ++l) W[l] = (valid && l < r) ? w0[(long long)row * r + l] : 0.0;
  double cs[kIncremental ? PQ : 1];  // C / G_qq of this lane's columns q = m Q + k
#pragma unroll
  for (int m = 0; m < (kIncremental ? PQ : 1); ++m) cs[m] = Cs[lr * LD + m * Q + k] * Ginv[m * Q + k];
  const int gbase = (int(threadIdx.x) & 31) & ~(Q - 1);  // first lane of the group

  // ---- AHALS sweeps (nnls.cpp:15-49).
  // Column j of a pass is (Gauss-Seidel, nnls.cpp:22)
  //   numer_j / G_jj = t_j - sum_{l < j} G[l][j] / G_jj W_new[l],
  //   t_j = C_j / G_jj - sum_{l > j} G[l][j] / G_jj W_old[l]
  // (the reference's "minus W G_j plus G_jj W_j", the l = j terms cancelled).
  // Lane k of a row's group owns the pending sums u of columns k, k + Q, ...:
  // it forms their t (the triangle) at the start of the pass and pushes every
  // new W[l] into them, except into column l + 1. Column j's owner hands u_j
  // to the group two columns early (shuffle); every lane adds the last term
  // -hd_j W_new[j-1] itself and clips, so the serial chain per column is one
  // FMA and the clip, and the shuffle has a column of slack. Division by G_jj
  // is a multiply by its reciprocal (<= 1 ulp apart). Padded (j >= r) and
  // skipped columns have t_j = W_j (GtP diagonal -1), no terms, no clip.
  // __syncwarp() between columns keeps ptxas from sinking work into long
  // per-column chains (in-order issue would serialise them); every operand
  // of column j + 1 is loaded during column j. A pass reads Wi, writes Wo.
  double first = -1.0;
  int s = 0;
  long long prof_red = 0;  // diagnostics: cycles in the per-sweep cluster reduction
  const long long prof_t0 = clock64();
  long long prof_pass = 0, prof_tri = 0, prof_np = 0;
  auto sweep = [&](const double(&Wi)[RP], double(&Wo)[RP]) -> double {
    const long long ps0 = pclock();
    double d2 = 0.0;
    if constexpr (kIncremental) {
      const double* gt = GtP + k * PQP;
      const double* hm = HmP + k * PQP;
      double u[PQP], ub[PQP];  // two accumulators per slot (even / odd l): half the chain
#pragma unroll
      for (int m = 0; m < PQP; ++m) u[m] = ub[m] = 0.0;
#pragma unroll
      for (int l = 0; l < RP; ++l) {
        const int mmax = (l / Q < PQ - 1) ? l / Q : PQ - 1;  // slots with a column <= l
        double* acc = (l & 1) ? ub : u;
#pragma unroll
        for (int m = 0; m <= mmax; m += 2) {
          const double2 g = *reinterpret_cast<const double2*>(gt + l * RS + m);
          acc[m] = fma(Wi[l], g.x, acc[m]);
          if (m + 1 <= mmax) acc[m + 1] = fma(Wi[l], g.y, acc[m + 1]);
        }
      }
#pragma unroll
      for (int m = 0; m < PQ; ++m) u[m] = cs[m] - (u[m] + ub[m]);
      prof_tri += pclock() - ps0;
      auto bcast = [&](int j) {  // u_j from its owner
        if constexpr (Q > 1)
          return __shfl_sync(0xffffffffu, u[j / Q], gbase | (j % Q));
        else
          return u[j];
      };
      // operands of the pushes of column j (hm row j, slots m >= (j + 2) / Q)
      // and of its chain step (hd_j, lo_j), loaded two columns ahead (shared
      // loads take ~50 cycles; ptxas issues them no earlier than written)
      double hp[3][PQP];
      double2 hl[3];
      auto load_ops = [&](int j) {
        const int m0 = ((j + 2) / Q) & ~1;
#pragma unroll
        for (int m = m0; m < PQ; m += 2) {
          const double2 h = *reinterpret_cast<const double2*>(hm + j * RS + m);
          hp[j % 3][m] = h.x;
          hp[j % 3][m + 1] = h.y;
        }
        hl[j % 3] = *reinterpret_cast<const double2*>(HL + 2 * j);
      };
      double pend[RP];  // u_j as handed over (all terms but column j-1's)
      pend[0] = bcast(0);
      if (RP > 1) pend[1] = bcast(1);
      load_ops(0);
      if (RP > 1) load_ops(1);
      double d2b = 0.0;
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        if (j + 2 < RP) load_ops(j + 2);
        const double v = j == 0 ? pend[0] : fma(-hl[j % 3].x, Wo[j - 1], pend[j]);
        const double nw = v < hl[j % 3].y ? 0.0 : v;  // cwiseMax(0.0)
        const double dd = nw - Wi[j];
        if (j & 1)
          d2b = fma(dd, dd, d2b);
        else
          d2 = fma(dd, dd, d2);
        Wo[j] = nw;
#pragma unroll
        for (int m = (j + 2) / Q; m < PQ; ++m) u[m] = fma(-nw, hp[j % 3][m], u[m]);
        if (j + 2 < RP) pend[j + 2] = bcast(j + 2);
        if (NTF_NNLS_SYNCWARP) __syncwarp();
      }
      d2 += d2b;
    } else {
#pragma unroll
      for (int j = 0; j < RP; ++j) Wo[j] = Wi[j];
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        if (j < r) {
          const double gjj = Gs[j * RP + j];
          const double ginv = Ginv[j];
          double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
          for (int l = 0; l < RP; l += 4) {
            p0 = fma(Wo[l + 0], Gs[(l + 0) * RP + j], p0);
            p1 = fma(Wo[l + 1], Gs[(l + 1) * RP + j], p1);
            p2 = fma(Wo[l + 2], Gs[(l + 2) * RP + j], p2);
            p3 = fma(Wo[l + 3], Gs[(l + 3) * RP + j], p3);
          }
          const double prod = (p0 + p1) + (p2 + p3);
          if (gjj > diag_floor) {
            const double c = Cs[lr * LD + j];
            const double numer = __dadd_rn(__dsub_rn(c, prod), __dmul_rn(gjj, Wo[j]));
            const double nw = clip0(__dmul_rn(numer, ginv));
            const double dd = nw - Wo[j];
            d2 = fma(dd, dd, d2);
            Wo[j] = nw;
          }
        }
      }
    }
    prof_pass += pclock() - ps0;
    ++prof_np;
    return k == 0 ? d2 : 0.0;  // each row counted once
  };

  // Sweep s + 1 runs speculatively while the cluster reduction of sweep s's
  // change is in flight; if sweep s meets the stop rule, its result (the
  // other buffer) is kept (nnls.cpp:33-39: the stop test follows the sweep).
  constexpr bool kSpeculate = kIncremental;
  auto post = [&](double d2, int j) {
    if (NTF_NNLS_PROFILE && j == 4 && (threadIdx.x & 31) == 0)
      g_nnls_skew[0][cl.block_rank() * (blockDim.x >> 5) + (threadIdx.x >> 5)] = globaltimer();
    cluster_post(d2, aslots + (j & 1) * kMaxCluster * kMaxWarps, &abar[j & 1], cl);
  };
  auto fin = [&](int j) {
    return cluster_fin(aslots + (j & 1) * kMaxCluster * kMaxWarps, &abar[j & 1], uint32_t(j >> 1) & 1u, cl);
  };
  bool inB = false;  // result in WB
  if (max_iters > 0) {
    post(sweep(W, WB), 0);
    bool done = false;
    // current result in Wc (posted); the next pass goes to Wn
    auto step = [&](double(&Wc)[RP], double(&Wn)[RP]) {
      const bool spec = kSpeculate && s + 1 < max_iters;
      double d2n = 0.0;
      if (spec) d2n = sweep(Wc, Wn);
      const long long tr0 = pclock();
      if (NTF_NNLS_PROFILE && s == 4 && (threadIdx.x & 31) == 0)
        g_nnls_skew[2][cl.block_rank() * (blockDim.x >> 5) + (threadIdx.x >> 5)] = globaltimer();
      const double ch2 = fin(s);  // ||W_{s+1} - W_s||_F^2
      prof_red += pclock() - tr0;
      if (NTF_NNLS_PROFILE && s == 4 && (threadIdx.x & 31) == 0)
        g_nnls_skew[1][cl.block_rank() * (blockDim.x >> 5) + (threadIdx.x >> 5)] = globaltimer();
      if (s == 0) first = sqrt(ch2);
      ++s;
      if (s >= max_iters || stop_rule(ch2, tol * first)) {
        done = true;
        return;
      }
      if constexpr (!kSpeculate) d2n = sweep(Wc, Wn);
      post(d2n, s);
    };
    for (;;) {
      step(WB, W);
      if (done) {
        inB = true;
        break;
      }
      step(W, WB);
      if (done) break;
    }
  }
  if (inB) {
#pragma unroll
    for (int l = 0; l < RP; ++l) W[l] = WB[l];
  }

  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g_nnls_prof[0] += clock64() - prof_t0;
    g_nnls_prof[1] += prof_red;
    g_nnls_prof[2] += s;
    g_nnls_prof[3] += 1;
    g_nnls_prof[4] += prof_pass;
    g_nnls_prof[5] += prof_np;
    g_nnls_prof[6] += prof_tri;
  }
  if (a.role == 2) {
    if (lead) {
#pragma unroll
      for (int l = 0; l < RP; ++l)
        if (l < r) a.w_out[(long long)row * r + l] = W[l];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s;
    return;
  }

  // ---- Gram(W): needed by F-hat / f and, on a restart, as the new Gram.
  if (k == 0) {
#pragma unroll
    for (int l = 0; l < RP; ++l) stage[lr * LD + l] = (valid && l < r) ? W[l] : 0.0;
  }
  __syncthreads();
  double* gW = (a.role == 0) ? F->gram[mode][sel ^ 1] : F->gram[mode][sel];
  cluster_gram<RP>(stage, nloc, part, r, gW, cl);

  // ---- write the block (HER: solved + extrapolated twin; AO: in place);
  // the twin is staged for its Gram as it is produced.
  double* S = F->x[mode][sel ^ 1];
  float* X32 = F->x32[mode][sel];
  float* S32 = F->x32[mode][sel ^ 1];
  if (k == 0) {
#pragma unroll
    for (int l = 0; l < RP; ++l) {
      double h = 0.0;
      if (valid && l < r) {
        const long long o = (long long)row * r + l;
        if (a.role == 0) {
          const double old = X[o];
          h = clip0(__dadd_rn(W[l], __dmul_rn(beta, __dsub_rn(W[l], old))));  // her.cpp:16-19
          S[o] = W[l];
          if (S32) S32[o] = float(W[l]);
        } else {
          h = W[l];
        }
        X[o] = h;
        if (X32) X32[o] = float(h);
      }
      if (a.role == 0) stage[lr * LD + l] = h;
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
  if (lead) {
#pragma unroll
    for (int l = 0; l < RP; ++l)
      if (l < r) cross += W[l] * Cs[lr * LD + l];
  }
  cross = cluster_sum(cross, red, pub, (s + 1) & 1, cl);
  if (blockIdx.x != 0 || threadIdx.x != 0) return;

  double quad = 0.0;
  for (int p = 0; p < r; ++p)
    for (int q = 0; q < r; ++q) quad += gW[p * r + q] * Gs[p * RP + q];
  const double f = 0.5 * st->nsq - cross + 0.5 * quad;

  st->last_sweeps[mode] = s;
  const int kk = st->k + 1;
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
  a.trace[kk - 1] = rec;
  st->f_last = f;
  st->k = kk;
  if ((st->max_iters > 0 && kk >= st->max_iters) || (st->max_time_s > 0.0 && time_s >= st->max_time_s))
    st->done = 1;
}

// Launch shape: Q lanes per row, about four warps per CTA (one per SM
// sub-partition), at most 16 CTAs (non-portable cluster size, allowed on
// B200); taller factors put more warps in each CTA.
template <int RP, int Q, int TPB>
bool launch_q(const NnlsLaunch& a, cudaStream_t s) {
  const long long lanes = (long long)a.rows * Q;
  const int cl = int(std::max(1LL, std::min<long long>((lanes + 127) / 128, kMaxCluster)));
  const int rpc = (a.rows + cl - 1) / cl;
  const int threads = (rpc * Q + 31) / 32 * 32;
  if (threads > TPB) return false;
  const size_t nloc = size_t(threads) / Q;
  using Shape = SweepShape<RP, Q>;
  const size_t smem = sizeof(double) * (2 * RP * RP + (Shape::kIncremental ? 2 * RP * Shape::RS : 0) + 32 +
                                        2 * kMaxCluster + 3 * RP + 2 * nloc * (RP + 1) + 2 * kMaxCluster * kMaxWarps + 2);
  auto fn = nnls_kernel<RP, Q, TPB>;
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
  return true;
}

// Preferred lane split by padded rank, falling back to one lane per row for
// factors too tall for it. NTF_NNLS_Q=1 forces one lane per row.
template <int RP, int TPB>
void launch_rp(const NnlsLaunch& a, cudaStream_t s) {
  static const int qenv = [] {
    const char* e = std::getenv("NTF_NNLS_Q");
    return e ? std::atoi(e) : 0;
  }();
  // measured (tools/tune.py, r01): one lane per row is as fast or faster up
  // to r = 16 (the triangle is short); from r = 20 four lanes per row win
  if constexpr (RP >= 20 && RP <= 32) {
    if (qenv != 1 && launch_q<RP, 4, TPB>(a, s)) return;
  }
  if (!launch_q<RP, 1, TPB>(a, s)) throw Unsupported("factor too tall for the fused NNLS kernel");
}

}  // namespace

void nnls_prof_read(unsigned long long out[8 + 384], bool reset) {
  NTF_CUDA(cudaMemcpyFromSymbol(out, g_nnls_prof, sizeof(unsigned long long) * 8));
  NTF_CUDA(cudaMemcpyFromSymbol(out + 8, g_nnls_skew, sizeof(unsigned long long) * 384));
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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
