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
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // see nnls_stream_kernel
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
  const int max_iters = (a.role == 2) ? a.max_iters : (a.zero_sweeps ? 0 : st->inner_max_iters);
  const double tol = (a.role == 2) ? a.tol : st->tol;
  const double* w0 = (a.role == 2 || a.zero_sweeps) ? a.w0 : X;
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
  st->elapsed_s = time_s;
  if ((st->max_iters > 0 && kk >= st->max_iters) ||
      (!st->collective_time && st->max_time_s > 0.0 && time_s >= st->max_time_s))
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


// ===========================================================================
// Stream AHALS (r <= 32): the column updates of all sweeps form one stream
// t = s * RP + j. Every evaluation of column j pushes the new W[j] into the
// pending sums of all other columns, so the "triangle" of a Gauss-Seidel
// pass (the sum over W_old[l > j]) is never formed at the pass start:
//
//   P_q  = C_q / G_qq - sum_{l != q} (G_lq / G_qq) W_latest[l]
//   W[q] = max(0, P_q)            (nnls.cpp:22, the l = q terms cancelled)
//
// and after the evaluation P_q restarts from C_q / G_qq. Q lanes own one row;
// lane k keeps the sums of columns q = m Q + k. The owner hands P_c to the
// group (shuffle) L columns before c is due; the L-1 newest terms are added
// by every lane itself, the last one (W[c-1]) as the only FMA on the serial
// chain, followed by the clip. Padded and skipped (G_jj <= floor) columns
// have no incoming terms and restart from their own value, so they stay
// unchanged. The stop rule (nnls.cpp:31-45, ||W_{s+1}-W_s||_F against the
// first change, cluster-wide) is decided by one reducer warp per CTA from
// per-row partials while the row warps run up to D sweeps ahead; each sweep's
// result is kept in a D-deep shared-memory stash, so the rows just stop and
// take the stashed result of the deciding sweep.
// ===========================================================================

constexpr int kStreamTPB = 160;  // up to four row warps + the reducer warp: <= 2 warps per SM sub-partition, 255 registers
constexpr int kStreamDC = 16;    // cluster exchange ring (slots per CTA): 2 D, see the reducer
constexpr int kStreamRowLanes = 64;  // target row lanes per CTA (r01h sweep: 16-CTA clusters at C2, 3113 -> 3151 iters/s)

template <int RP, int Q, int L>
struct StreamShape {
  static constexpr int PQ = RP / Q;         // owned columns per lane
  static constexpr int PQ2 = (PQ + 1) / 2;  // as double2
  static constexpr int WN2 = L / 2;         // window coefficients h_{j,j+1..j+L-1} as double2 (L-1 used)
  static constexpr int D = 8;               // sweeps in flight (stash depth)
  static_assert(RP % Q == 0 && L >= 2 && L < RP && (Q == 1 || L >= 3), "stream shape");
  static_assert((32 / Q) % 4 == 0 || Q == 16, "row slots per warp: a multiple of four (Gram partials)");
};

// Non-blocking: has the phase with this parity completed? (warp-uniform via lane 0)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// max(0, v) for okm == -1 (Eigen's cwiseMax, up to the sign of zero), v for
// okm == 0 (skipped column): sign-bit masking, two integer ops on the chain.
__device__ __forceinline__ double clip_mask(double v, int okm) {
#ifndef NTF_NNLS_FCLIP
  // arithmetic shift of the sign, then one 3-input LOP3 per word
  // (x & ~(sign & okm), immLut 0x70): two dependent steps on the chain
  const int hi = __double2hiint(v), lo = __double2loint(v);
  int h2, l2;
  asm("{\n\t.reg .b32 m;\n\tshr.s32 m, %2, 31;\n\tlop3.b32 %0, %2, m, %4, 0x70;\n\t"
      "lop3.b32 %1, %3, m, %4, 0x70;\n\t}"
      : "=r"(h2), "=r"(l2)
      : "r"(hi), "r"(lo), "r"(okm));
  return __hiloint2double(h2, l2);
#else
  return (okm != 0 && v < 0.0) ? 0.0 : v;
#endif
}

template <int RP, int Q, int L>
__global__ void __launch_bounds__(kStreamTPB, 1) nnls_stream_kernel(NnlsLaunch a) {
  using SS = StreamShape<RP, Q, L>;
  constexpr int PQ = SS::PQ, PQ2 = SS::PQ2, WN2 = SS::WN2, D = SS::D;
  constexpr int LDC = RP + 1;
  constexpr int LDW = RP + 2;  // row stride of the stash / twin buffers (16-byte rows)
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cl = cg::this_cluster();

  RunState* st = a.st;
  const int r = a.rank, mode = a.mode;
  DevFactors* F = a.F;
  // one round of global loads: the role bits, the budget flag and the
  // driver scalars (the buffer pointers come with the launch: a.bufs)
  int selv[kMaxOrder] = {};
  const double* gp0[kMaxOrder] = {};
  const double* gp1[kMaxOrder] = {};
  double* xp0 = nullptr;
  double* xp1 = nullptr;
  int sel = 0, done = 0;
  double beta = 0.0, tol = a.tol;
  int max_iters = a.max_iters;
  if (F) {
    done = st->done;
    beta = (a.role == 0) ? st->beta : 0.0;
    max_iters = a.zero_sweeps ? 0 : st->inner_max_iters;
    tol = st->tol;
#pragma unroll
    for (int j = 0; j < kMaxOrder; ++j)
      if (j < a.order) {
        selv[j] = F->sel[j];
        gp0[j] = a.has_bufs ? a.bufs.gram[j][0] : F->gram[j][0];
        gp1[j] = a.has_bufs ? a.bufs.gram[j][1] : F->gram[j][1];
      }
    xp0 = a.has_bufs ? a.bufs.x[mode][0] : F->x[mode][0];
    xp1 = a.has_bufs ? a.bufs.x[mode][1] : F->x[mode][1];
#pragma unroll
    for (int j = 0; j < kMaxOrder; ++j)
      if (j == mode) sel = selv[j];
  }
  // a programmatic dependent (the overlapped tensor pass) may start now, on
  // the SMs this cluster leaves free: it reads nothing this kernel writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (done) return;  // budget exhausted: the whole iteration is a no-op (uniform)
  const long long t_begin = clock64();
  // the last mode's decision scalars, loaded now by the deciding thread so
  // that no global round trip sits between the final barrier and the record
  struct Dec {
    double nsq, f_prev, beta_bar, eta, gamma, gamma_bar, max_time_s;
    unsigned long long t_start_ns;
    int k, max_iters, collective_time, sweeps_before;
  } dec{};
  const bool decider = F && a.last && blockIdx.x == 0 && threadIdx.x == 0;
  if (decider) {
    dec.nsq = st->nsq;
    dec.f_prev = st->f_prev;
    dec.beta_bar = st->beta_bar;
    dec.eta = st->eta;
    dec.gamma = st->gamma;
    dec.gamma_bar = st->gamma_bar;
    dec.max_time_s = st->max_time_s;
    dec.t_start_ns = st->t_start_ns;
    dec.k = st->k;
    dec.max_iters = st->max_iters;
    dec.collective_time = st->collective_time;
    for (int j = 0; j < a.order; ++j)
      if (j != mode) dec.sweeps_before += st->last_sweeps[j];
  }

  const int nrw = int(blockDim.x >> 5) - 1;  // row warps; warp nrw reduces
  const int nloc = nrw * 32 / Q;              // row slots per CTA
  const int rpc = (a.rows + int(gridDim.x) - 1) / int(gridDim.x);
  const unsigned ncta = cl.num_blocks(), me = cl.block_rank();

  double2* pushc = reinterpret_cast<double2*>(smem);  // [RP][PQ2][Q]: h_{j,q}, q = m Q + k (pushed terms)
  double2* wins = pushc + RP * PQ2 * Q;               // [RP][WN2]: h_{j,j+d}, d = 1..L-1 (window terms)
  double* Gs = reinterpret_cast<double*>(wins + RP * WN2);  // RP*RP
  double* Ginv = Gs + RP * RP;                             // RP
  double* stash = Ginv + RP;                               // [D][nloc][LDW]: W after each sweep
  double* Cs = stash + D * nloc * LDW;                     // [nloc][LDC]: rows of C
  double* stage = Cs + nloc * LDC;                         // [nloc][LDW]: extrapolated twin
  double* part = stage + nloc * LDW;                       // 2*RP*RP + 2: Gram partials, <W,C>, quad
  double* d2part = part + 2 * RP * RP + 2;                 // [D][nloc]: per-row ||dW||^2
  double* cslot = d2part + D * nloc;                       // [kStreamDC][kMaxCluster]
  double* red = cslot + kStreamDC * kMaxCluster;           // 32
  uint64_t* rowbar = reinterpret_cast<uint64_t*>(red + 32);  // D
  uint64_t* cbar = rowbar + D;                                // kStreamDC
  unsigned long long* ctl = reinterpret_cast<unsigned long long*>(cbar + kStreamDC);  // (stop << 32) | decided

  double* X = sel ? xp1 : xp0;
  const double* w0 = (a.role == 2 || a.zero_sweeps) ? a.w0 : X;
  const double* C = a.C;

  // rows of C: the first batch of loads is issued before the G loads (both
  // round trips overlap); its stores follow the G loop
  auto load_c = [&](int e0, double(&cv)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * int(blockDim.x);
      const int i = e / RP, l = e % RP;
      const int gr = int(blockIdx.x) * rpc + i;
      cv[u] = (e < nloc * RP && i < rpc && gr < a.rows && l < r) ? C[(long long)gr * r + l] : 0.0;
    }
  };
  auto store_c = [&](int e0, const double(&cv)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * int(blockDim.x);
      if (e < nloc * RP) Cs[(e / RP) * LDC + e % RP] = cv[u];
    }
  };
  const long long t_q0 = clock64();
  // ---- G: Hadamard of the other modes' Grams (kernels.cpp:193-200).
  // (global loads of four entries per thread in flight together)
  for (int e0 = threadIdx.x; e0 < RP * RP; e0 += 4 * blockDim.x) {
    // every factor value first (independent read-only loads, all in flight),
    // then the products in ascending mode order
    double v[4][kMaxOrder];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * int(blockDim.x);
      const int p = e / RP, q = e % RP;
      const bool in = e < RP * RP && p < r && q < r;
#pragma unroll
      for (int j = 0; j < kMaxOrder; ++j) {
        const bool use = in && (a.role == 2 ? j == 0 : (j < a.order && j != mode));
        const double* src = a.role == 2 ? a.gram_in : (selv[j] ? gp1[j] : gp0[j]);
        v[u][j] = use ? __ldg(src + p * r + q) : 1.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * int(blockDim.x);
      const int p = e / RP, q = e % RP;
      double g = 1.0;
#pragma unroll
      for (int j = 0; j < kMaxOrder; ++j) g *= v[u][j];
      if (e < RP * RP) Gs[e] = (p < r && q < r) ? g : 0.0;
    }
  }
  const long long t_q1 = clock64();
  const long long t_q2 = clock64();
  if (threadIdx.x == 0) {
    for (int b = 0; b < D; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&rowbar[b])) : "memory");
    for (int b = 0; b < kStreamDC; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[b])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *ctl = 0ull;
  }
  __syncthreads();
  const long long t_p1 = clock64();
  // max diagonal and the updated columns: every warp reads the diagonal once
  // (lane j < r), a shuffle max and a ballot (r <= 32 here)
  const int ln = int(threadIdx.x & 31);
  const double gjj = ln < r ? Gs[ln * RP + ln] : -INFINITY;
  double dmax = gjj;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const double diag_floor = 1e-12 * dmax;  // nnls.cpp:16-19
  const unsigned okbits = __ballot_sync(0xffffffffu, ln < r && gjj > diag_floor);  // updated (and clipped) columns
  for (int j = threadIdx.x; j < RP; j += blockDim.x) Ginv[j] = ((okbits >> j) & 1) ? 1.0 / Gs[j * RP + j] : 0.0;
  __syncthreads();
  {
    double* pc = reinterpret_cast<double*>(pushc);
    for (int e = threadIdx.x; e < RP * PQ2 * Q * 2; e += blockDim.x) {
      const int j = e / (PQ2 * Q * 2), rem = e % (PQ2 * Q * 2);
      const int m2 = rem / (Q * 2), k = (rem / 2) % Q, half = rem & 1;
      const int m = 2 * m2 + half, q = m * Q + k;
      double h = 0.0;
      if (m < PQ && q < r && j < r && q != j && ((q - j + RP) % RP) >= L && ((okbits >> q) & 1))
        h = Gs[j * RP + q] * Ginv[q];
      pc[e] = h;
    }
    double* wn = reinterpret_cast<double*>(wins);
    for (int e = threadIdx.x; e < RP * WN2 * 2; e += blockDim.x) {
      const int j = e / (WN2 * 2), d = e % (WN2 * 2) + 1, c = (j + d) % RP;
      double h = 0.0;
      if (d <= L - 1 && j < r && c < r && ((okbits >> c) & 1)) h = Gs[j * RP + c] * Ginv[c];
      wn[e] = h;
    }
  }
  // Everything above depends only on earlier blocks (Grams, roles) and runs
  // while the kernel producing C (the block's MTTKRP contraction, of which
  // this kernel is a programmatic dependent) finishes: wait for it now,
  // then the C rows (and, with another inner solver, its result rows w0).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int e0 = int(threadIdx.x); e0 < nloc * RP; e0 += 4 * int(blockDim.x)) {
    double cv[4];
    load_c(e0, cv);
    store_c(e0, cv);
  }
  const long long t_p2 = clock64();
  cl.sync();  // tables, C rows and every CTA's mbarriers exist before any st.async targets them
  const long long t_loop = clock64();

  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  int red_np = 0, red_nd = -1;  // reducer: sweeps posted / the deciding sweep (for the drain)
  if (warp < nrw) {
    // ------------------------------------------------------------ row warps
    const int slot = (warp * 32 + lane) / Q, k = lane % Q, gbase = lane & ~(Q - 1);
    const int row = int(blockIdx.x) * rpc + slot;
    const bool valid = slot < rpc && row < a.rows;
    double Wl[RP];  // latest value of every column of the row (all lanes of the group)
#pragma unroll
    for (int l = 0; l < RP; ++l) Wl[l] = (valid && l < r) ? w0[(long long)row * r + l] : 0.0;
    const double* pcd = reinterpret_cast<const double*>(pushc);
    // restart values and pending sums of the owned columns (as if the
    // previous sweep had pushed W0[l > q]; W0[l < q] arrive in sweep 0)
    double rv[PQ], P[PQ];
#pragma unroll
    for (int m = 0; m < PQ; ++m) {
      const int q = m * Q + k;
      double v = 0.0;
      if (q < r) v = ((okbits >> q) & 1) ? Cs[slot * LDC + q] * Ginv[q] : (valid ? w0[(long long)row * r + q] : 0.0);
      rv[m] = v;
      double pm = v;
#pragma unroll
      for (int j = 0; j < RP; ++j)
        if (j > q) pm = fma(-Wl[j], pcd[((j * PQ2 + m / 2) * Q + k) * 2 + (m & 1)], pm);
      P[m] = pm;
    }
    auto bcast = [&](double v, int c) -> double {
      if constexpr (Q > 1)
        return __shfl_sync(0xffffffffu, v, gbase | (c % Q));
      else
        return v;
    };
    auto win = [&](int j, int d) -> double {  // h_{j, j+d}
      return reinterpret_cast<const double*>(wins)[j * WN2 * 2 + d - 1];
    };
    double acc[RP];  // per column: its handed-over sum plus the window terms so far
#pragma unroll
    for (int c = 0; c < L; ++c) {
      acc[c] = bcast(P[c / Q], c);
#pragma unroll
      for (int d = L - 1; d >= 2; --d)
        if (d > c) acc[c] = fma(-win((c - d + RP) % RP, d), Wl[(c - d + RP) % RP], acc[c]);
    }
    if constexpr (L >= Q) {
      // groups whose restart step (m Q + Q - 1 - L) precedes sweep 0 have
      // just handed over their initial sums: they restart now
#pragma unroll
      for (int m = 0; m < PQ; ++m)
        if (m * Q + Q - 1 - L < 0) P[m] = rv[m];
    }
    // coefficient registers of the next two steps (rows j of pushc / wins)
    double2 pcr[RP][PQ2], wr[RP][WN2];
    auto load_row = [&](int j) {
#pragma unroll
      for (int m2 = 0; m2 < PQ2; ++m2) pcr[j][m2] = pushc[(j * PQ2 + m2) * Q + k];
#pragma unroll
      for (int w = 0; w < WN2; ++w) wr[j][w] = wins[j * WN2 + w];
    };
    // coefficient rows are loaded PF steps ahead (a ring of PF + 1 rows in registers)
    constexpr int PF = 2;
    load_row(RP - 1);
    load_row(0);
    if constexpr (PF == 2) load_row(1);
    auto wcoef = [&](int j, int d) -> double {  // h_{j,j+d} from the registers
      const double2 x = wr[j][(d - 1) / 2];
      return ((d - 1) & 1) ? x.y : x.x;
    };
    auto pcoef = [&](int j, int m) -> double {
      const double2 x = pcr[j][m / 2];
      return (m & 1) ? x.y : x.x;
    };

    // sweep s's result is stashed during sweep s + 1 (each column just before
    // it is overwritten) or on leaving the loop; the per-row change goes to
    // the reducer with st.async (completes bytes on rowbar, no fence)
    const uint32_t d2addr = smem_u32(d2part + slot);
    int s = 0;
    long long passes = 0, pass_cyc = 0;
    unsigned long long c = ld_volatile_u64(ctl);
    long long gate_cyc = 0, gate_n = 0;
    const long long rows_t0 = pclock();
    // one sweep of the row (false: a stop was decided before it started);
    // two per loop trip, so the rotating registers of Wl come back to their
    // loop-entry allocation without a block of moves
    auto one_pass = [&]() -> bool {
      if (c >> 32) return false;
      if (s >= max_iters || (s >= D && int(c & 0xffffffffu) < s - D + 1)) {
        const long long tg = pclock();
        ++gate_n;
        do {
          __nanosleep(20);
          c = ld_volatile_u64(ctl);
        } while (!(c >> 32) && (s >= max_iters || int(c & 0xffffffffu) < s - D + 1));
        gate_cyc += pclock() - tg;
        if (c >> 32) return false;
      }
      double d2 = 0.0;
      double* stp = stash + (((s + D - 1) % D) * nloc + slot) * LDW;  // row of sweep s - 1
      const long long tp0 = pclock();
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const int jm1 = (j + RP - 1) % RP;
        const double v = fma(-wcoef(jm1, 1), Wl[jm1], acc[j]);
        const double nw = clip_mask(v, -int((okbits >> j) & 1u));
        if (k == 0) stp[j] = Wl[j];
        const double dd = nw - Wl[j];
        d2 = fma(dd, dd, d2);
        Wl[j] = nw;
#pragma unroll
        for (int d = 2; d < L; ++d) acc[(j + d) % RP] = fma(-wcoef(j, d), nw, acc[(j + d) % RP]);
#pragma unroll
        for (int m = 0; m < PQ; ++m) P[m] = fma(-nw, pcoef(j, m), P[m]);
        acc[(j + L) % RP] = bcast(P[((j + L) % RP) / Q], (j + L) % RP);
        if constexpr (L >= Q) {
          // every sum of the column group m is idle from its hand-over (L
          // steps before it is due) until after its evaluation, so the
          // whole group restarts at once, unconditionally, right after the
          // last of the group's hand-overs (step m Q + Q - 1 - L)
#pragma unroll
          for (int m = 0; m < PQ; ++m)
            if (((m * Q + Q - 1 - L) % RP + RP) % RP == j) P[m] = rv[m];
        } else {
          if (k == j % Q) P[j / Q] = rv[j / Q];
        }
        load_row((j + PF) % RP);
        if (j == RP / 2) c = ld_volatile_u64(ctl);  // decisions so far, checked after the pass
      }
      pass_cyc += pclock() - tp0;
      if (k == 0) {
        const int b = s % D;
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                         d2addr + uint32_t(b * nloc * 8)),
                     "l"(__double_as_longlong(d2)), "r"(smem_u32(&rowbar[b]))
                     : "memory");
      }
      ++s;
      ++passes;
      return true;
    };
    for (;;) {
      if (!one_pass()) break;
      if (!one_pass()) break;
    }
    if (k == 0) {  // the last sweep's result (or W0 when no sweep ran)
      double* stp = stash + (((s + D - 1) % D) * nloc + slot) * LDW;
#pragma unroll
      for (int l = 0; l < RP; ++l) stp[l] = Wl[l];
    }
    if (NTF_NNLS_PROFILE && blockIdx.x == 0 && threadIdx.x == 0) {
      g_nnls_prof[5] += passes;
      g_nnls_prof[6] += pass_cyc;
      g_nnls_prof[7] += gate_cyc;
      g_nnls_skew[2][80] += gate_n;
      g_nnls_skew[2][81] += pclock() - rows_t0;
    }
  } else {
    // -------------------------------------------------------- reducer warp
    // Two decoupled stages over the sweeps, in order: post (this CTA's rows
    // are done with sweep np: sum their partials, send the sum to every CTA)
    // and decide (every CTA's sum of sweep nd has arrived: add them in rank
    // order -- the same bits in every CTA -- and apply the stop rule). Posts
    // run ahead of decisions, so the cluster latency overlaps the sweeps.
    double first = 0.0;
    if (max_iters <= 0) {
      if (lane == 0) asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(smem_u32(ctl)), "l"(1ull << 32) : "memory");
    } else {
      int np = 0, nd = 0;
      if (lane == 0)
        for (int b = 0; b < D; ++b)
          asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                           smem_u32(&rowbar[b])),
                       "r"(unsigned(nloc) * 8u)
                       : "memory");
      for (;;) {
        bool idle = true;
        if (np < max_iters && mbar_test(&rowbar[np % D], uint32_t(np / D) & 1u)) {
          const int b = np % D;
          double x = 0.0;
          for (int i = lane; i < nloc; i += 32) x += d2part[b * nloc + i];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          const int cb = np % kStreamDC;
          if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&cbar[cb])),
                         "r"(ncta * 8u)
                         : "memory");
          if (unsigned(lane) < ncta) {
            uint32_t raddr, rbar;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(raddr)
                         : "r"(smem_u32(&cslot[cb * kMaxCluster + me])), "r"(lane));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&cbar[cb])), "r"(lane));
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                         "l"(__double_as_longlong(x)), "r"(rbar)
                         : "memory");
          }
          if (lane == 0)  // re-arm this barrier for sweep np + D
            asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&rowbar[b])),
                         "r"(unsigned(nloc) * 8u)
                         : "memory");
          ++np;
          idle = false;
        }
        if (nd < np && mbar_test(&cbar[nd % kStreamDC], uint32_t(nd / kStreamDC) & 1u)) {
          const int cb = nd % kStreamDC;
          double ch2 = 0.0;  // ||W_{s+1} - W_s||_F^2, CTAs in rank order: same bits everywhere
          for (unsigned c = 0; c < ncta; ++c) ch2 += cslot[cb * kMaxCluster + c];
          if (nd == 0) first = sqrt(ch2);
          const bool stop = (nd + 1 >= max_iters) || stop_rule(ch2, tol * first);
          if (lane == 0) {
            const unsigned long long w = (stop ? (1ull << 32) : 0ull) | unsigned(nd + 1);
            asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(smem_u32(ctl)), "l"(w) : "memory");
          }
          if (stop) {
            red_nd = nd;
            break;
          }
          ++nd;
          idle = false;
        }
        if (idle) __nanosleep(64);
      }
      red_np = np;
    }
  }
  // Before the last cluster barrier every st.async aimed at this CTA must
  // have landed (no CTA may leave while traffic can still target its shared
  // memory). Rows run at most D - 1 sweeps past the decisions, so reducers
  // posted sweeps <= red_nd + D - 1 at most, each CTA its own count. The
  // reducer posts zeros for the sweeps it has not posted up to that bound
  // (arming its own ring slot each time), so every slot phase up to it gets
  // exactly one post from every CTA, then waits for those phases. (The rows'
  // st.async into their own CTA's ring come from threads of this CTA, which
  // are all behind the final barrier.)
  auto drain = [&]() {
    if (warp != nrw || max_iters <= 0 || red_nd < 0) return;
    const int last = min(red_nd + D - 1, max_iters - 1);
    for (int x = red_np; x <= last; ++x) {
      const int cb = x % kStreamDC;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&cbar[cb])),
                     "r"(ncta * 8u)
                     : "memory");
      if (unsigned(lane) < ncta) {
        uint32_t raddr, rbar;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(raddr)
                     : "r"(smem_u32(&cslot[cb * kMaxCluster + me])), "r"(lane));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&cbar[cb])), "r"(lane));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                     "l"(0ll), "r"(rbar)
                     : "memory");
      }
    }
    for (int x = red_nd + 1; x <= last; ++x)
      while (!mbar_test(&cbar[x % kStreamDC], uint32_t(x / kStreamDC) & 1u)) __nanosleep(32);
  };
  __syncthreads();
  const long long t_loop_end = clock64();
  const int s = int(*ctl & 0xffffffffu);  // sweeps run (nnls.cpp:31-45)
  const int fs = (s + D - 1) % D;         // stash slot of the result

  if (a.role == 2) {
    for (int e = threadIdx.x; e < nloc * RP; e += blockDim.x) {
      const int i = e / RP, l = e % RP;
      const int row = int(blockIdx.x) * rpc + i;
      if (i < rpc && row < a.rows && l < r) a.w_out[(long long)row * r + l] = stash[(fs * nloc + i) * LDW + l];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s;
    drain();
    cl.sync();  // no CTA leaves while cluster traffic may target it
    return;
  }

  // ---- write the block (HER: solved + extrapolated twin; AO: in place).
  const double* Wf = stash + fs * nloc * LDW;  // [nloc][LDW]
  double* S = sel ? xp0 : xp1;
  const DevFactors& B = a.has_bufs ? a.bufs : *F;
  float* X32 = B.x32[mode][sel];
  float* S32 = B.x32[mode][sel ^ 1];
  for (int e0 = threadIdx.x; e0 < nloc * RP; e0 += 4 * blockDim.x) {
    double old[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // the accepted block's values, loads in flight together
      const int e = e0 + u * int(blockDim.x);
      const int i = e / RP, l = e % RP;
      const int row = int(blockIdx.x) * rpc + i;
      old[u] = (a.role == 0 && e < nloc * RP && i < rpc && row < a.rows && l < r) ? X[(long long)row * r + l] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * int(blockDim.x);
      if (e >= nloc * RP) break;
      const int i = e / RP, l = e % RP;
      const int row = int(blockIdx.x) * rpc + i;
      const double w = Wf[i * LDW + l];
      double h = 0.0;
      if (i < rpc && row < a.rows && l < r) {
        const long long o = (long long)row * r + l;
        if (a.role == 0) {
          h = clip0(__dadd_rn(w, __dmul_rn(beta, __dsub_rn(w, old[u]))));  // her.cpp:16-19
          S[o] = w;
          if (S32) S32[o] = float(w);
        } else {
          h = w;
        }
        X[o] = h;
        if (X32) X32[o] = float(h);
      }
      if (a.role == 0) stage[i * LDW + l] = h;
    }
  }
  __syncthreads();
  const long long t_e1 = clock64();
  // ---- Gram partials of this CTA's rows (W, and the twin for HER): one
  // 2 x 2 block of entries per task, two accumulators per entry (even / odd
  // rows), columns of the [RP][nloc] buffers read as double2
  {
    constexpr int NB = RP / 2;
    constexpr int NBLK = NB * (NB + 1) / 2;  // blocks on or above the diagonal
    const int nmat = (a.role == 0) ? 2 : 1;
    for (int t = threadIdx.x; t < nmat * NBLK; t += blockDim.x) {
      const int mat = t / NBLK;
      int bi = t % NBLK, pb = 0;
      while (bi >= NB - pb) {
        bi -= NB - pb;
        ++pb;
      }
      const int p = 2 * pb, q = 2 * (pb + bi);
      if (p >= r) continue;
      const double* base = mat ? stage : Wf;
      double e00 = 0.0, e01 = 0.0, e10 = 0.0, e11 = 0.0, o00 = 0.0, o01 = 0.0, o10 = 0.0, o11 = 0.0;
      for (int i = 0; i < nloc; i += 2) {
        const double2 a0 = *reinterpret_cast<const double2*>(base + i * LDW + p);
        const double2 b0 = *reinterpret_cast<const double2*>(base + i * LDW + q);
        const double2 a1 = *reinterpret_cast<const double2*>(base + (i + 1) * LDW + p);
        const double2 b1 = *reinterpret_cast<const double2*>(base + (i + 1) * LDW + q);
        e00 = fma(a0.x, b0.x, e00);
        e01 = fma(a0.x, b0.y, e01);
        e10 = fma(a0.y, b0.x, e10);
        e11 = fma(a0.y, b0.y, e11);
        o00 = fma(a1.x, b1.x, o00);
        o01 = fma(a1.x, b1.y, o01);
        o10 = fma(a1.y, b1.x, o10);
        o11 = fma(a1.y, b1.y, o11);
      }
      double* dst = part + mat * RP * RP;
      dst[p * RP + q] = e00 + o00;
      if (q + 1 < RP) dst[p * RP + q + 1] = e01 + o01;
      if (p + 1 <= q) dst[(p + 1) * RP + q] = e10 + o10;
      if (q + 1 < RP) dst[(p + 1) * RP + q + 1] = e11 + o11;
    }
  }
  if (a.last) {
    // <W, C> and <W^T W, G> of this CTA (the cheap objective's data terms)
    __syncthreads();
    double cr = 0.0, qd = 0.0;
    for (int e = threadIdx.x; e < nloc * RP; e += blockDim.x) {
      const int i = e / RP, l = e % RP;
      if (l < r) cr += Wf[i * LDW + l] * Cs[i * LDC + l];
    }
    for (int e = threadIdx.x; e < RP * RP; e += blockDim.x) {
      const int p = e / RP, q = e % RP;
      if (p < r && q < r) qd += part[p <= q ? p * RP + q : q * RP + p] * Gs[e];
    }
    cr = block_sum(cr, red);
    qd = block_sum(qd, red);
    if (threadIdx.x == 0) {
      part[2 * RP * RP] = cr;
      part[2 * RP * RP + 1] = qd;
    }
  }
  const long long t_e2 = clock64();
  cl.sync();  // partials visible cluster-wide
  const long long t_e3 = clock64();
  double* gW = (a.role == 0) ? B.gram[mode][sel ^ 1] : B.gram[mode][sel];
  double* gH = B.gram[mode][sel];
  const int nmat = (a.role == 0) ? 2 : 1;
  for (int e = int(threadIdx.x) * int(ncta) + int(me); e < nmat * RP * RP; e += int(blockDim.x) * int(ncta)) {
    const int mat = e / (RP * RP), pq = e % (RP * RP);
    const int p = pq / RP, q = pq % RP;
    if (p > q || q >= r) continue;
    double vals[kMaxCluster];
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c) vals[c] = c < int(ncta) ? cl.map_shared_rank(part, unsigned(c))[e] : 0.0;
    double v = 0.0;
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c)
      if (c < int(ncta)) v += vals[c];
    double* dst = mat ? gH : gW;
    dst[p * r + q] = v;
    dst[q * r + p] = v;
  }
  // <W,C> and <W^T W, G> of the cluster, by CTA 0's last thread while the
  // others reduce the Grams (remote loads of both in flight together); the
  // decider reads them after the final cluster barrier
  if (a.last && blockIdx.x == 0 && threadIdx.x == blockDim.x - 1) {
    double cv[kMaxCluster], qv[kMaxCluster];  // all remote loads in flight before the ordered sums
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c) {
      const double* pc = cl.map_shared_rank(part, unsigned(c < int(ncta) ? c : 0));
      cv[c] = c < int(ncta) ? pc[2 * RP * RP] : 0.0;
      qv[c] = c < int(ncta) ? pc[2 * RP * RP + 1] : 0.0;
    }
    double cross = 0.0, quad = 0.0;
#pragma unroll
    for (int c = 0; c < kMaxCluster; ++c)
      if (c < int(ncta)) {
        cross += cv[c];
        quad += qv[c];
      }
    red[30] = cross;
    red[31] = quad;
  }
  const long long t_e4 = clock64();
  drain();
  cl.sync();  // remote reads and every cluster post done before any CTA exits
  if (NTF_NNLS_PROFILE && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t_end = clock64();
    unsigned long long* ph = &g_nnls_skew[2][64];  // phase cycles (diagnostics, -DNTF_NNLS_PROFILE=1)
    ph[0] += t_p1 - t_begin;
    ph[1] += t_p2 - t_p1;
    ph[2] += t_loop - t_p2;
    ph[3] += t_e1 - t_loop_end;
    ph[4] += t_e2 - t_e1;
    ph[5] += t_e3 - t_e2;
    ph[6] += t_e4 - t_e3;
    ph[7] += t_end - t_e4;
    ph[8] += t_q0 - t_begin;
    ph[9] += t_q1 - t_q0;
    ph[10] += t_q2 - t_q1;
    g_nnls_prof[0] += t_loop_end - t_loop;
    g_nnls_prof[1] += t_loop - t_begin;
    g_nnls_prof[2] += s;
    g_nnls_prof[3] += 1;
    g_nnls_prof[4] += t_end - t_loop_end;
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  if (!a.last) {
    st->last_sweeps[mode] = s;
    return;
  }
  const double cross = red[30], quad = red[31];
  const double f = 0.5 * dec.nsq - cross + 0.5 * quad;
  st->last_sweeps[mode] = s;
  const int kk = dec.k + 1;
  const double time_s = double(globaltimer() - dec.t_start_ns) * 1e-9;
  TraceEntry rec;
  rec.f = f;
  rec.time_s = time_s;
  rec.sweeps = dec.sweeps_before + s;
  if (a.role == 0) {
    const bool restarted = f > dec.f_prev;  // strict (her.cpp:75)
    if (restarted)
      for (int j = 0; j < a.order; ++j) F->sel[j] = selv[j] ^ 1;  // X := S for every mode
    st->f_prev = f;                                                // even on rejection (:84)
    rec.beta = beta;                                               // beta_used
    rec.restarted = restarted ? 1 : 0;
    if (restarted) {  // update_betas (her.cpp:21-30)
      st->beta_bar = beta;
      st->beta = __ddiv_rn(beta, dec.eta);
    } else {
      st->beta = fmin(dec.beta_bar, __dmul_rn(beta, dec.gamma));
      st->beta_bar = fmin(1.0, __dmul_rn(dec.beta_bar, dec.gamma_bar));
    }
  } else {
    rec.beta = 0.0;
    rec.restarted = 0;
  }
  a.trace[kk - 1] = rec;
  st->f_last = f;
  st->k = kk;
  st->elapsed_s = time_s;
  if ((dec.max_iters > 0 && kk >= dec.max_iters) ||
      (!dec.collective_time && dec.max_time_s > 0.0 && time_s >= dec.max_time_s))
    st->done = 1;
}

template <int RP, int Q, int L>
bool launch_stream_q(const NnlsLaunch& a, cudaStream_t s) {
  using SS = StreamShape<RP, Q, L>;
  const long long lanes = (long long)a.rows * Q;
  static const int row_lanes = [] {  // tuning: NTF_NNLS_ROW_LANES overrides the target row lanes per CTA
    const char* e = std::getenv("NTF_NNLS_ROW_LANES");
    return e ? std::max(32, std::atoi(e)) : kStreamRowLanes;
  }();
  const int cl = int(std::max(1LL, std::min<long long>((lanes + row_lanes - 1) / row_lanes, kMaxCluster)));
  const int rpc = (a.rows + cl - 1) / cl;
  const int roww = (rpc * Q + 31) / 32;
  const int threads = (roww + 1) * 32;
  if (threads > kStreamTPB) return false;
  const size_t nloc = size_t(roww) * 32 / Q;
  const size_t smem = sizeof(double2) * (RP * SS::PQ2 * Q + RP * SS::WN2) +
                      sizeof(double) * (RP * RP + RP + SS::D * nloc * (RP + 2) + nloc * (RP + 1) + nloc * (RP + 2) +
                                        2 * RP * RP + 2 + SS::D * nloc + kStreamDC * kMaxCluster + 32) +
                      sizeof(uint64_t) * (SS::D + kStreamDC + 1);
  auto fn = nnls_stream_kernel<RP, Q, L>;
  NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  if (cl > 8) NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  NnlsLaunch args = a;
  void* params[] = {&args};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // drivers: a programmatic dependent of the block's MTTKRP kernel (the
  // prologue overlaps it; griddepcontrol.wait before the C rows)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = (a.role != 2 && !std::getenv("NTF_NNLS_NO_PDL")) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  NTF_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(fn), params));
  return true;
}

// Lane split by padded rank: about four owned columns per lane, narrower
// groups for factors too tall for the cluster.
template <int RP, int Q0>
bool launch_stream_rp(const NnlsLaunch& a, cudaStream_t s) {
  if constexpr (Q0 > 1) {
    if (launch_stream_q<RP, Q0, 4>(a, s)) return true;
    return launch_stream_rp<RP, Q0 / 2>(a, s);
  } else {
    return launch_stream_q<RP, 1, 2>(a, s);
  }
}

bool launch_stream(const NnlsLaunch& a, cudaStream_t s) {
  static const bool off = [] {
    const char* e = std::getenv("NTF_NNLS_OLD");
    return e && std::atoi(e) != 0;
  }();
  if (off) return false;
  const int r = a.rank;
  if (r <= 4) return launch_stream_rp<4, 1>(a, s);
  if (r <= 8) return launch_stream_rp<8, 2>(a, s);
  if (r <= 10) return launch_stream_rp<10, 2>(a, s);
  if (r <= 12) return launch_stream_rp<12, 4>(a, s);
  if (r <= 16) return launch_stream_rp<16, 4>(a, s);
  if (r <= 20) {
    // window length (terms every lane adds itself) of the r = 20 plan: 3 (r02ak sweep at C2:
    // L = 3 4372, 4 4336, 5 4333, 6 4263 iters/s); NTF_NNLS_L overrides
    static const int lwin = [] {
      const char* e = std::getenv("NTF_NNLS_L");
      return e ? std::atoi(e) : 3;
    }();
    if (lwin == 3 && launch_stream_q<20, 4, 3>(a, s)) return true;
    if (lwin == 5 && launch_stream_q<20, 4, 5>(a, s)) return true;
    if (lwin == 6 && launch_stream_q<20, 4, 6>(a, s)) return true;
    return launch_stream_rp<20, 4>(a, s);
  }
  if (r <= 24) return launch_stream_rp<24, 8>(a, s);
  if (r <= 32) return launch_stream_rp<32, 8>(a, s);
  return false;
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

// One cluster holds at most 4096 rows (one lane per row, 16 CTAs x 256); the spilling plans of
// r > 32 at most 2048. NTF_NNLS_TALL=1 sends every update through the tall path (tests).
bool nnls_needs_tall(int rows, int rank) {
  static const bool force = [] {
    const char* e = std::getenv("NTF_NNLS_TALL");
    return e && std::atoi(e) != 0;
  }();
  return force || rows > kMaxNnlsRows || (rank > 32 && rows > 2048) || rank > kMaxRank;
}

void launch_nnls(const NnlsLaunch& a, cudaStream_t s) {
  const int r = a.rank;
  if (r < 1 || r > kMaxTallRank) throw Unsupported("rank outside the NNLS kernels' range (1..128)");
  if (nnls_needs_tall(a.rows, r)) {
    if (!a.tall) throw Unsupported("factor taller than one cluster holds and no tall-path workspace");
    return launch_nnls_tall(a, s, a.zero_sweeps ? 0 : a.max_iters);
  }
  if (launch_stream(a, s)) return;
  if (a.rows > kMaxNnlsRows) throw Unsupported("factor taller than 4096 rows");
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
