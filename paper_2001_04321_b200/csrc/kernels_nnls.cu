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
// nnls.cpp:22); the row lives in registers for all sweeps. A single CTA
// serves up to kTpb rows; taller factors use a cooperative grid whose CTAs
// meet at grid.sync() for the global stop rule and the Gram reductions.
#include <cooperative_groups.h>

#include "ntf_internal.h"

namespace cg = cooperative_groups;

namespace ntfb {
namespace {

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Deterministic block sum; every thread receives the same value.
template <int TPB>
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // red may still be read from a previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int w = 0; w < TPB / 32; ++w)
    if (w < nw) s += red[w];
  return s;
}

// Sum of a per-CTA value over the whole (cooperative) grid, same bits in
// every thread. `slots` is double-buffered by the caller's parity.
template <int TPB>
__device__ double grid_sum(double v, double* red, double* slots, cg::grid_group& grid) {
  const double b = block_sum<TPB>(v, red);
  if (gridDim.x == 1) return b;
  if (threadIdx.x == 0) slots[blockIdx.x] = b;
  grid.sync();
  double s = 0.0;
  for (unsigned i = 0; i < gridDim.x; ++i) s += slots[i];
  return s;
}

// Eigen's cwiseMax(0.0): (a < 0) ? 0 : a.
__device__ __forceinline__ double clip0(double a) { return a < 0.0 ? 0.0 : a; }

// Gram of the rows staged in `stage` ([TPB][RP+1]) for this CTA, written to
// `dst` (r x r). With several CTAs, per-CTA partials go to `slots` and CTA 0
// sums them in CTA order after a grid barrier.
template <int RP, int TPB>
__device__ void cta_gram(const double* stage, int r, double* dst, double* slots, cg::grid_group& grid) {
  constexpr int LD = RP + 1;
  const bool multi = gridDim.x > 1;
  const int nt = blockDim.x;
  for (int e = threadIdx.x; e < r * r; e += nt) {
    const int p = e / r, q = e % r;
    if (p > q) continue;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int i = 0; i < nt; i += 4) {
      s0 += stage[(i + 0) * LD + p] * stage[(i + 0) * LD + q];
      s1 += stage[(i + 1) * LD + p] * stage[(i + 1) * LD + q];
      s2 += stage[(i + 2) * LD + p] * stage[(i + 2) * LD + q];
      s3 += stage[(i + 3) * LD + p] * stage[(i + 3) * LD + q];
    }
    const double s = (s0 + s1) + (s2 + s3);
    if (multi) {
      slots[blockIdx.x * (RP * RP) + p * r + q] = s;
    } else {
      dst[p * r + q] = s;
      dst[q * r + p] = s;
    }
  }
  if (!multi) return;
  grid.sync();
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < r * r; e += nt) {
      const int p = e / r, q = e % r;
      if (p > q) continue;
      double s = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) s += slots[b * (RP * RP) + p * r + q];
      dst[p * r + q] = s;
      dst[q * r + p] = s;
    }
  }
  grid.sync();  // slots are reused by the next Gram
}

template <int RP, int TPB>
__global__ void __launch_bounds__(TPB) nnls_kernel(NnlsLaunch a) {
  constexpr int LD = RP + 1;
  extern __shared__ double smem[];
  double* Gs = smem;             // RP*RP
  double* red = Gs + RP * RP;    // 32
  double* stage = red + 32;      // TPB*LD
  cg::grid_group grid = cg::this_grid();

  RunState* st = a.st;
  if (st && st->done) return;  // budget exhausted: the whole iteration is a no-op

  const int r = a.rank, mode = a.mode;
  const int row = blockIdx.x * TPB + threadIdx.x;
  const bool valid = row < a.rows;
  DevFactors* F = a.F;
  const int sel = F ? F->sel[mode] : 0;
  double* X = F ? F->x[mode][sel] : nullptr;
  const double beta = (a.role == 0) ? st->beta : 0.0;
  const int max_iters = (a.role == 2) ? a.max_iters : st->inner_max_iters;
  const double tol = (a.role == 2) ? a.tol : st->tol;
  // scratch layout: [0,2048) sweep sums (double-buffered by sweep parity),
  // [2048,3072) the <W,C> sums, [3072, ...) per-CTA Gram partials.
  double* slots_sweep = a.scratch;
  double* slots_cross = a.scratch + 2048;
  double* slots_gram = a.scratch + 3072;

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
  __syncthreads();

  double dmax = -INFINITY;
  for (int j = 0; j < r; ++j) dmax = fmax(dmax, Gs[j * RP + j]);
  const double diag_floor = 1e-12 * dmax;

  const double* w0 = (a.role == 2) ? a.w0 : X;
  const double* C = a.C;
  double W[RP];
#pragma unroll
  for (int l = 0; l < RP; ++l) W[l] = (valid && l < r) ? w0[(long long)row * r + l] : 0.0;

  // ---- AHALS sweeps.
  // Column j of a pass needs prod_j = (W G)[row, j] with columns < j already
  // updated in this pass (nnls.cpp:22). It is assembled as
  //   P[j] = sum_{l >= j} W_old[l] G[l][j]      (all j at once, ILP)
  //        + sum_{l < j}  W_new[l] G[l][j]      (added as columns finish),
  // so the serial chain from column j-1 to j is one FMA, not a dot product.
  // The division by G_jj is a multiply by its reciprocal (<= 1 ulp apart).
  double* Ginv = stage;  // RP reciprocals (stage is free until the Grams)
  for (int j = threadIdx.x; j < RP; j += blockDim.x) Ginv[j] = (j < r && Gs[j * RP + j] > 0.0) ? 1.0 / Gs[j * RP + j] : 0.0;
  __syncthreads();
  double first = -1.0;
  int s = 0;
  constexpr bool kIncremental = RP <= 24;  // P[] costs RP more registers
  for (; s < max_iters; ++s) {
    double P[kIncremental ? RP : 1];
    if constexpr (kIncremental) {
      // row l of G is contiguous: 16-byte broadcast reads, P[j] still sums
      // l = j, j+1, ... in ascending order
#pragma unroll
      for (int j = 0; j < RP; ++j) P[j] = 0.0;
#pragma unroll
      for (int l = 0; l < RP; ++l) {
#pragma unroll
        for (int j = 0; j <= l; j += 2) {
          const double2 g = *reinterpret_cast<const double2*>(&Gs[l * RP + j]);
          P[j] = fma(W[l], g.x, P[j]);
          if (j + 1 <= l) P[j + 1] = fma(W[l], g.y, P[j + 1]);
        }
      }
    }
    double d2 = 0.0;
#pragma unroll
    for (int j = 0; j < RP; ++j) {
      if (j < r) {
        const double gjj = Gs[j * RP + j];
        double prod;
        if constexpr (kIncremental) {
          prod = P[j];
        } else {
          double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
          for (int l = 0; l < RP; l += 4) {
            p0 = fma(W[l + 0], Gs[(l + 0) * RP + j], p0);
            p1 = fma(W[l + 1], Gs[(l + 1) * RP + j], p1);
            p2 = fma(W[l + 2], Gs[(l + 2) * RP + j], p2);
            p3 = fma(W[l + 3], Gs[(l + 3) * RP + j], p3);
          }
          prod = (p0 + p1) + (p2 + p3);
        }
        if (gjj > diag_floor) {
          const double c = valid ? __ldg(&C[(long long)row * r + j]) : 0.0;
          const double numer = __dadd_rn(__dsub_rn(c, prod), __dmul_rn(gjj, W[j]));
          const double nw = clip0(__dmul_rn(numer, Ginv[j]));
          const double d = nw - W[j];
          d2 = fma(d, d, d2);
          W[j] = nw;
        }
        if constexpr (kIncremental) {
#pragma unroll
          for (int q = (j + 1) & ~1; q < RP; q += 2) {
            const double2 g = *reinterpret_cast<const double2*>(&Gs[j * RP + q]);
            if (q > j) P[q] = fma(W[j], g.x, P[q]);
            P[q + 1] = fma(W[j], g.y, P[q + 1]);
          }
        }
      }
    }
    const double change = sqrt(grid_sum<TPB>(valid ? d2 : 0.0, red, slots_sweep + (s & 1) * 1024, grid));
    if (s == 0) first = change;
    if (change <= tol * first) {
      ++s;
      break;
    }
  }

  if (a.role == 2) {
    if (valid) {
#pragma unroll
      for (int l = 0; l < RP; ++l)
        if (l < r) a.w_out[(long long)row * r + l] = W[l];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = s;
    return;
  }

  // ---- Gram(W): needed by F-hat / f and, on a restart, as the new Gram.
#pragma unroll
  for (int l = 0; l < RP; ++l) stage[threadIdx.x * LD + l] = (valid && l < r) ? W[l] : 0.0;
  __syncthreads();
  double* gW = (a.role == 0) ? F->gram[mode][sel ^ 1] : F->gram[mode][sel];
  cta_gram<RP, TPB>(stage, r, gW, slots_gram, grid);
  __syncthreads();

  // ---- write the block (HER: solved + extrapolated twin; AO: in place);
  // the twin is staged for its Gram as it is produced.
  double* S = F->x[mode][sel ^ 1];
  float* X32 = F->x32[mode][sel];
  float* S32 = F->x32[mode][sel ^ 1];
#pragma unroll
  for (int l = 0; l < RP; ++l) {
    double h = 0.0;
    if (valid && l < r) {
      const long long o = (long long)row * r + l;
      if (a.role == 0) {
        const double old = X[o];
        h = clip0(__dadd_rn(W[l], __dmul_rn(beta, __dsub_rn(W[l], old))));
        S[o] = W[l];
        if (S32) S32[o] = float(W[l]);
      } else {
        h = W[l];
      }
      X[o] = h;
      if (X32) X32[o] = float(h);
    }
    if (a.role == 0) stage[threadIdx.x * LD + l] = h;
  }
  if (a.role == 0) {
    __syncthreads();
    cta_gram<RP, TPB>(stage, r, F->gram[mode][sel], slots_gram, grid);
    __syncthreads();
  }
  if (!a.last) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->last_sweeps[mode] = s;
    return;
  }

  // ---- objective at the (mixed) point: <W, C> and <W^T W, G>.
  double cross = 0.0;
  if (valid) {
#pragma unroll
    for (int l = 0; l < RP; ++l)
      if (l < r) cross += W[l] * C[(long long)row * r + l];
  }
  cross = grid_sum<TPB>(cross, red, slots_cross, grid);
  if (gridDim.x > 1) grid.sync();  // gram written by CTA 0 is visible to all
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

template <int RP, int TPB>
void launch_rp(const NnlsLaunch& a, cudaStream_t s) {
  const int grid = (a.rows + TPB - 1) / TPB;
  if (grid > 1024) throw Unsupported("factor too tall for the fused NNLS kernel");
  const size_t smem = sizeof(double) * (RP * RP + 32 + size_t(TPB) * (RP + 1));
  auto fn = nnls_kernel<RP, TPB>;
  NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  NnlsLaunch args = a;
  void* params[] = {&args};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  // a single CTA runs exactly the warps its rows need
  cfg.blockDim = dim3(grid == 1 ? unsigned((a.rows + 31) / 32 * 32) : unsigned(TPB));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = grid > 1 ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  NTF_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(fn), params));
}

}  // namespace

void launch_nnls(const NnlsLaunch& a, cudaStream_t s) {
  const int r = a.rank;
  if (r < 1 || r > kMaxRank) throw Unsupported("rank outside the fused NNLS kernel's range (1..64)");
  if (r <= 4) return launch_rp<4, 512>(a, s);
  if (r <= 8) return launch_rp<8, 512>(a, s);
  if (r <= 12) return launch_rp<12, 384>(a, s);
  if (r <= 16) return launch_rp<16, 384>(a, s);
  if (r <= 20) return launch_rp<20, 384>(a, s);
  if (r <= 24) return launch_rp<24, 256>(a, s);
  if (r <= 32) return launch_rp<32, 256>(a, s);
  if (r <= 48) return launch_rp<48, 128>(a, s);
  return launch_rp<64, 128>(a, s);
}

}  // namespace ntfb
