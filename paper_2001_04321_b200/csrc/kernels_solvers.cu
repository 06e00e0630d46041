// The reference's other inner NNLS solvers (nnls.cpp:51-211) on the GPU:
// projected gradient (PGD), Nesterov's accelerated gradient, ADMM and the
// row-wise Lawson-Hanson active set, behind the same solve_nnls dispatch
// (nnls.cpp:213-222). One thread-block cluster (up to 16 CTAs, one thread
// per row of W) runs every sweep of a solve: the rows are independent inside
// a sweep, and the stop rule's ||W_{s+1} - W_s||_F and the NNLS objective
// (nnls.cpp:11-13, for the "best iterate" of Nesterov / ADMM) are reduced
// over the cluster in a fixed order -- the same bits in every CTA, so the
// decisions are uniform and the result is reproducible. Row state lives in
// a global work area (each thread reads and writes only its own rows).
//
// These solvers are selectable alternatives to AHALS (which runs in the fused
// kernel of kernels_nnls.cu); inside the drivers their result is handed to
// that kernel with zero sweeps for the extrapolation, Grams and decision.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "ntf_internal.h"

namespace cg = cooperative_groups;

namespace ntfb {

namespace {

constexpr int kSolverCluster = 16;
constexpr int kSolverTPB = 256;

enum SolverError : int {
  kErrNone = 0,
  kErrPgdZero = 1,
  kErrNesterovZero = 2,
  kErrAdmmZero = 3,
  kErrAdmmFactor = 4,
  kErrActiveSetPd = 5,
  kErrActiveSetBudget = 6,
};

__device__ double solver_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// Cluster sum, same bits in every thread of every CTA (CTA-rank order);
// `parity` alternates so a slot is rewritten only after every CTA read it.
__device__ double solver_cluster_sum(double v, double* red, double* pub, int parity, cg::cluster_group& cl) {
  const double b = solver_block_sum(v, red);
  const unsigned n = cl.num_blocks();
  if (n == 1) return b;
  const unsigned me = cl.block_rank();
  if (threadIdx.x < n) *cl.map_shared_rank(&pub[parity * kSolverCluster + me], threadIdx.x) = b;
  cl.sync();
  double s = 0.0;
  for (unsigned k = 0; k < n; ++k) s += pub[parity * kSolverCluster + k];
  return s;
}

// Cholesky L L^T = a (n x n, leading dimension ld, lower triangle into l);
// false unless positive definite (Eigen::LLT info() != Success).
__device__ bool chol(const double* a, int n, int ld, double* l) {
  for (int j = 0; j < n; ++j) {
    double d = a[j * ld + j];
    for (int k = 0; k < j; ++k) d -= l[j * ld + k] * l[j * ld + k];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d);
    l[j * ld + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double v = a[i * ld + j];
      for (int k = 0; k < j; ++k) v -= l[i * ld + k] * l[j * ld + k];
      l[i * ld + j] = v / ljj;
    }
  }
  return true;
}

// b := (L L^T)^{-1} b
__device__ void chol_solve(const double* l, int n, int ld, double* b) {
  for (int i = 0; i < n; ++i) {
    double v = b[i];
    for (int k = 0; k < i; ++k) v -= l[i * ld + k] * b[k];
    b[i] = v / l[i * ld + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double v = b[i];
    for (int k = i + 1; k < n; ++k) v -= l[k * ld + i] * b[k];
    b[i] = v / l[i * ld + i];
  }
}

// spectral_norm (kernels.cpp:262-280): power iteration from the normalised
// ones vector by one warp (lane l owns rows l, l + 32, ...); the full
// symmetric eigen-solve fallback is cyclic Jacobi by lane 0. v / w: 2 r
// doubles of scratch.
__device__ double spectral_norm_warp(const double* g, int r, int ld, double* v, double* w, double* jac) {
  const int lane = threadIdx.x & 31;
  if (r == 1) return fabs(g[0]);
  for (int i = lane; i < r; i += 32) v[i] = 1.0 / sqrt(double(r));
  __syncwarp();
  double lambda = 0.0;
  for (int it = 0; it < 1000; ++it) {
    double part = 0.0;
    for (int i = lane; i < r; i += 32) {
      double acc = 0.0;
      for (int k = 0; k < r; ++k) acc += g[i * ld + k] * v[k];
      w[i] = acc;
      part += acc * acc;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const double nrm = sqrt(part);
    if (nrm == 0.0) return 0.0;
    __syncwarp();
    for (int i = lane; i < r; i += 32) v[i] = w[i] / nrm;
    __syncwarp();
    double nx = 0.0;
    for (int i = lane; i < r; i += 32) {
      double acc = 0.0;
      for (int k = 0; k < r; ++k) acc += g[i * ld + k] * v[k];
      nx += v[i] * acc;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nx += __shfl_xor_sync(0xffffffffu, nx, o);
    if (fabs(nx - lambda) <= 1e-10 * fmax(1.0, fabs(nx))) return nx;
    lambda = nx;
    __syncwarp();
  }
  double m = 0.0;
  if (lane == 0) {  // cyclic Jacobi on a copy
    for (int i = 0; i < r; ++i)
      for (int k = 0; k < r; ++k) jac[i * ld + k] = g[i * ld + k];
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0;
      for (int p = 0; p < r; ++p)
        for (int q = p + 1; q < r; ++q) off += jac[p * ld + q] * jac[p * ld + q];
      if (off <= 1e-300) break;
      for (int p = 0; p < r; ++p)
        for (int q = p + 1; q < r; ++q) {
          const double apq = jac[p * ld + q];
          if (apq == 0.0) continue;
          const double theta = (jac[q * ld + q] - jac[p * ld + p]) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
          for (int k = 0; k < r; ++k) {
            const double akp = jac[k * ld + p], akq = jac[k * ld + q];
            jac[k * ld + p] = c * akp - s * akq;
            jac[k * ld + q] = s * akp + c * akq;
          }
          for (int k = 0; k < r; ++k) {
            const double apk = jac[p * ld + k], aqk = jac[q * ld + k];
            jac[p * ld + k] = c * apk - s * aqk;
            jac[q * ld + k] = s * apk + c * aqk;
          }
        }
    }
    for (int i = 0; i < r; ++i) m = fmax(m, fabs(jac[i * ld + i]));
  }
  return __shfl_sync(0xffffffffu, m, 0);
}

// Lawson-Hanson for one row (nnls.cpp:125-191): min_{x>=0} 0.5 x^T G x - c^T x.
// gp / lp: RP x RP local scratch. False when the addition budget runs out.
template <int RP>
__device__ bool active_set_row(const double* g, int r, const double* c, double* x) {
  double gp[RP * RP], lp[RP * RP], cp[RP];
  int passive[RP];
  bool in_p[RP];
  double cmax = 0.0, gmax = -INFINITY;
  for (int j = 0; j < r; ++j) {
    cmax = fmax(cmax, fabs(c[j]));
    gmax = fmax(gmax, g[j * RP + j]);
    x[j] = 0.0;
    in_p[j] = false;
  }
  const double enter_tol = 1e-11 * fmax(1.0, fmax(cmax, gmax));
  int np = 0;
  const int max_additions = 3 * r;
  for (int additions = 0;; ++additions) {
    int enter = -1;
    double best = enter_tol;
    for (int j = 0; j < r; ++j) {
      double gx = 0.0;
      for (int k = 0; k < r; ++k) gx += g[j * RP + k] * x[k];
      const double dual = c[j] - gx;
      if (!in_p[j] && dual > best) {
        best = dual;
        enter = j;
      }
    }
    if (enter < 0) return true;
    if (additions >= max_additions) return false;
    passive[np++] = enter;
    in_p[enter] = true;
    for (;;) {
      for (int a2 = 0; a2 < np; ++a2) {
        cp[a2] = c[passive[a2]];
        for (int b2 = 0; b2 < np; ++b2) gp[a2 * RP + b2] = g[passive[a2] * RP + passive[b2]];
      }
      chol(gp, np, RP, lp);
      chol_solve(lp, np, RP, cp);  // cp := zp
      bool all_pos = true;
      for (int a2 = 0; a2 < np; ++a2) all_pos = all_pos && cp[a2] > 0.0;
      if (all_pos) {
        for (int j = 0; j < r; ++j) x[j] = 0.0;
        for (int a2 = 0; a2 < np; ++a2) x[passive[a2]] = cp[a2];
        break;
      }
      double alpha = 1.0;
      for (int a2 = 0; a2 < np; ++a2)
        if (cp[a2] <= 0.0) {
          const double xa = x[passive[a2]];
          alpha = fmin(alpha, xa / (xa - cp[a2]));
        }
      for (int a2 = 0; a2 < np; ++a2) {
        const int j = passive[a2];
        x[j] += alpha * (cp[a2] - x[j]);
      }
      for (int a2 = np; a2-- > 0;) {
        const int j = passive[a2];
        if (x[j] <= 0.0 || (cp[a2] <= 0.0 && x[j] < 1e-14)) {
          x[j] = 0.0;
          in_p[j] = false;
          for (int b2 = a2; b2 + 1 < np; ++b2) {
            passive[b2] = passive[b2 + 1];
            cp[b2] = cp[b2 + 1];
          }
          --np;
        }
      }
    }
  }
}

template <int RP>
__global__ void __launch_bounds__(kSolverTPB, 1) nnls_solver_kernel(NnlsLaunch a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double dyn[];  // Gs[RP * RP], Ls[RP * RP]: G and its Cholesky factor (ADMM) / Jacobi scratch
  double* Gs = dyn;
  double* Ls = dyn + RP * RP;
  __shared__ double vec[2 * RP];
  __shared__ double red[32];
  __shared__ double pub[2 * kSolverCluster];
  __shared__ double scal[2];
  __shared__ int serr;

  const int r = a.rank, mode = a.mode;
  RunState* st = a.st;
  DevFactors* F = a.F;
  if (F && st->done) return;  // budget exhausted: the iteration is a no-op (uniform)
  const int solver = a.solver;
  const int max_iters = (a.role == 2) ? a.max_iters : st->inner_max_iters;
  const double tol = (a.role == 2) ? a.tol : st->tol;
  const double* X = F ? F->x[mode][F->sel[mode]] : nullptr;
  const double* w0 = (a.role == 2) ? a.w0 : X;

  // G = Hadamard of the other modes' X-role Grams (kernels.cpp:193-200:
  // ones, times every Gram except `mode`, ascending), or the given Gram
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
  if (threadIdx.x == 0) serr = kErrNone;
  __syncthreads();
  // solver constants (computed redundantly by every CTA: same bits)
  if (threadIdx.x < 32) {
    if (solver == NTF_SOLVER_PGD || solver == NTF_SOLVER_NESTEROV) {
      const double lip = spectral_norm_warp(Gs, r, RP, vec, vec + RP, Ls);
      if (threadIdx.x == 0) {
        scal[0] = lip;
        if (lip <= 0.0) serr = solver == NTF_SOLVER_PGD ? kErrPgdZero : kErrNesterovZero;
      }
    } else if (solver == NTF_SOLVER_ADMM && threadIdx.x == 0) {
      double tr = 0.0;
      for (int j = 0; j < r; ++j) tr += Gs[j * RP + j];
      const double rho = tr / double(r);
      scal[0] = rho;
      if (rho <= 0.0) {
        serr = kErrAdmmZero;
      } else {
        for (int j = 0; j < r; ++j) Gs[j * RP + j] += rho;  // G + rho I for the factorisation
        if (!chol(Gs, r, RP, Ls)) serr = kErrAdmmFactor;
        for (int j = 0; j < r; ++j) Gs[j * RP + j] -= rho;
      }
    } else if (solver == NTF_SOLVER_ACTIVE_SET && threadIdx.x == 0) {
      if (!chol(Gs, r, RP, Ls)) serr = kErrActiveSetPd;
    }
  }
  __syncthreads();

  const int rpc = (a.rows + int(gridDim.x) - 1) / int(gridDim.x);
  const int row = int(blockIdx.x) * rpc + int(threadIdx.x);
  const bool valid = int(threadIdx.x) < rpc && row < a.rows;
  double* out = a.w_out;
  const long long n_all = (long long)a.rows * r;
  double* B = a.work + n_all;  // best iterate (the first n_all doubles: spare per-row state)
  double w[RP], c[RP];
  for (int j = 0; j < RP; ++j) {
    w[j] = (valid && j < r) ? w0[(long long)row * r + j] : 0.0;
    c[j] = (valid && j < r) ? a.C[(long long)row * r + j] : 0.0;
  }
  if (serr != kErrNone) {  // the reference throws; keep the warm start and report
    if (valid)
      for (int j = 0; j < r; ++j) out[(long long)row * r + j] = w[j];
    if (threadIdx.x == 0 && blockIdx.x == 0 && a.error) atomicCAS(a.error, 0, serr);
    cl.sync();
    return;
  }
  auto row_obj = [&](const double (&x)[RP]) {  // 0.5 x G x^T - x c^T of this row (nnls.cpp:11-13)
    double q = 0.0, l = 0.0;
    for (int j = 0; j < r; ++j) {
      double gx = 0.0;
      for (int k = 0; k < r; ++k) gx += Gs[j * RP + k] * x[k];
      q += x[j] * gx;
      l += x[j] * c[j];
    }
    return valid ? 0.5 * q - l : 0.0;
  };
  int parity = 0;
  int sweeps = 0;
  if (solver == NTF_SOLVER_ACTIVE_SET) {
    double x[RP];
    bool ok = true;
    if (valid) ok = active_set_row<RP>(Gs, r, c, x);
    if (!ok) atomicCAS(&serr, 0, kErrActiveSetBudget);
    if (valid)
      for (int j = 0; j < r; ++j) out[(long long)row * r + j] = ok ? x[j] : w[j];
  } else {
    const double k1 = scal[0];  // lip (PGD, Nesterov) or rho (ADMM)
    double y[RP];  // Nesterov: y; ADMM: u
    for (int j = 0; j < RP; ++j) y[j] = solver == NTF_SOLVER_NESTEROV ? w[j] : 0.0;
    const bool track_best = solver != NTF_SOLVER_PGD;
    double best_obj = 0.0;
    if (track_best) {
      best_obj = solver_cluster_sum(row_obj(w), red, pub, parity, cl);
      parity ^= 1;
      if (valid)
        for (int j = 0; j < r; ++j) B[(long long)row * r + j] = w[j];
    }
    double t = 1.0, first = -1.0;
    for (int s = 0; s < max_iters; ++s) {
      double next[RP];
      double d2 = 0.0;
      if (solver == NTF_SOLVER_ADMM) {
        // W (G + rho I) = C + rho (Z - U); Z' = max(0, W + U); U += W - Z'
        double rhs[RP];
        for (int j = 0; j < r; ++j) rhs[j] = c[j] + k1 * (w[j] - y[j]);
        chol_solve(Ls, r, RP, rhs);
        for (int j = 0; j < r; ++j) {
          next[j] = fmax(0.0, rhs[j] + y[j]);
          y[j] += rhs[j] - next[j];
        }
      } else {
        // PGD: W - (W G - C) / L from W; Nesterov: the same step from Y
        const double* src = solver == NTF_SOLVER_PGD ? w : y;
        for (int j = 0; j < r; ++j) {
          double g = 0.0;
          for (int k = 0; k < r; ++k) g += src[k] * Gs[k * RP + j];
          next[j] = fmax(0.0, src[j] - (g - c[j]) / k1);
        }
        if (solver == NTF_SOLVER_NESTEROV) {
          const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
          for (int j = 0; j < r; ++j) y[j] = next[j] + ((t - 1.0) / t_next) * (next[j] - w[j]);
          t = t_next;
        }
      }
      for (int j = 0; j < r; ++j) {
        const double d = valid ? next[j] - w[j] : 0.0;
        d2 += d * d;
        w[j] = next[j];
      }
      const double change = sqrt(solver_cluster_sum(d2, red, pub, parity, cl));
      parity ^= 1;
      ++sweeps;
      if (track_best) {
        const double obj = solver_cluster_sum(row_obj(w), red, pub, parity, cl);
        parity ^= 1;
        if (obj < best_obj) {
          best_obj = obj;
          if (valid)
            for (int j = 0; j < r; ++j) B[(long long)row * r + j] = w[j];
        }
      }
      if (s == 0) first = change;
      if (change <= tol * first) break;
    }
    if (valid)
      for (int j = 0; j < r; ++j) out[(long long)row * r + j] = track_best ? B[(long long)row * r + j] : w[j];
  }
  __syncthreads();
  if (threadIdx.x == 0 && serr != kErrNone && a.error) atomicCAS(a.error, 0, serr);
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.sweeps_out) *a.sweeps_out = sweeps;
  cl.sync();  // remote slot writes done before any CTA exits
}

template <int RP>
void launch_rp_solver(const NnlsLaunch& a, cudaStream_t s) {
  const int cl = std::max(1, std::min(kSolverCluster, (a.rows + kSolverTPB - 1) / kSolverTPB));
  const int rpc = (a.rows + cl - 1) / cl;
  const int threads = std::max(32, (rpc + 31) / 32 * 32);
  auto fn = nnls_solver_kernel<RP>;
  const size_t smem = 2 * size_t(RP) * RP * sizeof(double);
  NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  if (cl > 8) NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  NnlsLaunch args = a;
  void* params[] = {&args};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(cl));
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(cl);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  NTF_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(fn), params));
}

}  // namespace

void launch_nnls_solver(const NnlsLaunch& a, cudaStream_t s) {
  if (a.rows > kSolverCluster * kSolverTPB) throw Unsupported("factor taller than 4096 rows");
  if (a.solver == NTF_SOLVER_ACTIVE_SET && a.rank > 32)
    throw Unsupported("the GPU active-set solver serves ranks up to 32");
  if (a.rank <= 8) return launch_rp_solver<8>(a, s);
  if (a.rank <= 16) return launch_rp_solver<16>(a, s);
  if (a.rank <= 32) return launch_rp_solver<32>(a, s);
  if (a.rank <= 64) return launch_rp_solver<64>(a, s);
  throw Unsupported("rank outside the solver kernel's range (1..64)");
}

const char* solver_error_message(int code) {
  switch (code) {
    case kErrPgdZero: return "pgd_solve: zero Gram matrix";
    case kErrNesterovZero: return "nesterov_solve: zero Gram matrix";
    case kErrAdmmZero: return "admm_solve: zero Gram matrix";
    case kErrAdmmFactor: return "admm_solve: factorization failed";
    case kErrActiveSetPd: return "active_set_solve: Gram matrix is not positive definite";
    case kErrActiveSetBudget: return "active_set_solve: pass budget exceeded";
    default: return "inner solver failure";
  }
}

}  // namespace ntfb
