// Dimension-tree MTTKRP reuse.
//
// Inside one HER / AO outer iteration, block n contracts the tensor with
// the current sweep's blocks j < n and the previous sweep's (or restart
// values) j > n (her.cpp:64-65). With a split point h the two partial
// contractions
//     Y_L[i_0..i_{h-1}][c] = sum_{i_h..i_{N-1}} T[i] * prod_{j>=h} A_j[i_j][c]
//     Y_R[i_h..i_{N-1}][c] = sum_{i_0..i_{h-1}} T[i] * prod_{j<h}  A_j[i_j][c]
// are each one streaming pass of the fast MTTKRP kernel (Y_L: ROW view with
// the rows before h merged; Y_R: COL view with the columns from h merged),
// formed when block 0 (Y_L, previous sweep's A_h..) and block h (Y_R, this
// sweep's A_0..A_{h-1}) come up; blocks on each side then only need
//     M_n[i][c] = sum_{l, rho} Y[l][i][rho][c] * wl[l][c] * wr[rho][c]
// with wl / wr the Khatri-Rao rows of the other blocks of that side
// (kernels.cpp:90-113). Full tensor passes per iteration drop from N to 2.
// h = N-1 (3-way) leaves Y_R = block N-1's MTTKRP itself and Y_L = 14.4 MB
// at BASELINE config 2 (L2-resident); h = 2 at 4-way makes both partials
// 1.28 MB at config 3 instead of one 128 MB Y. Results differ from the
// direct MTTKRP only by summation order.
//
// tree_mttkrp_kernel: CTA (chunk, tile) owns a contiguous range of the
// flattened reduction index q = l * R' + rho and a tile of (i, c) output
// pairs (one pair per thread, consecutive pairs on consecutive lanes); it
// forms the chunk's Khatri-Rao rows in shared memory and streams Y with
// kTreeQB loads in flight per thread (the first batch before the factor
// round trips). The chunks of a tile form one thread-block cluster (<= 8)
// and sum their partials in chunk order over distributed shared memory.
// Fallback when a chunk's Khatri-Rao rows exceed shared memory: more
// chunks, partials in global slots, and the last CTA of a tile to arrive
// (self-resetting arrival counter) sums them in chunk order. No atomics on
// data either way: bit-reproducible.
#include <cooperative_groups.h>

#include <cstdlib>

#include "ntf_internal.h"

namespace ntfb {
namespace {

namespace cg = cooperative_groups;

constexpr int kTreeThreads = 256;
constexpr int kTreeTile = kTreeThreads;  // output pairs per CTA tile
constexpr int kTreeQB = 16;              // q steps per load batch

// CLUSTER: the chunks of a tile are one thread-block cluster (grid.x = the
// cluster size); the chunk partials are summed in chunk order over
// distributed shared memory, no global slots, fences or arrival counters.
template <bool CLUSTER>
__global__ void __launch_bounds__(kTreeThreads) tree_mttkrp_kernel(const double* __restrict__ Y, TreeView v,
                                                                   const DevFactors* __restrict__ F,
                                                                   double* __restrict__ partial, int qpc,
                                                                   unsigned* __restrict__ arrivals,
                                                                   double* __restrict__ out) {
  extern __shared__ double wsh[];  // [qpc][r]
  __shared__ const double* fac[kMaxOrder];
  __shared__ unsigned last;
  const int r = v.rank;
  // every index below fits 32 bits (checked by the launcher)
  const int Q = int(v.L * v.R);
  const int q0 = int(blockIdx.x) * qpc;
  const int q1 = q0 + qpc < Q ? q0 + qpc : Q;
  const int I = int(v.I), R = int(v.R);
  const int pairs = I * r;
  const int p = int(blockIdx.y) * kTreeTile + int(threadIdx.x);
  const bool ok = p < pairs;
  const int i = ok ? p / r : 0;
  const int col = ok ? p - i * r : 0;
  const double* yp = Y + (long long)i * R * r + col;
  const long long istride = (long long)I * R * r;  // one step of l
  // (l, rho) of q advance by counting, no division in the loop
  int l = q0 / R, rho = q0 - (q0 / R) * R;
  // Y does not depend on the factors: the first batch of loads is issued
  // before the factor-pointer and Khatri-Rao round trips, and every later
  // batch while the previous one is consumed (two register buffers)
  double y[kTreeQB];
  auto load_batch = [&](double* dst, int n) {
#pragma unroll
    for (int b = 0; b < kTreeQB; ++b)
      if (b < n) {
        dst[b] = __ldg(yp + l * istride + (long long)rho * r);
        if (++rho == R) {
          rho = 0;
          ++l;
        }
      }
  };
  if (ok) load_batch(y, min(kTreeQB, q1 - q0));

  // factor pointers of the current roles: one round trip (sel and both
  // candidate pointers in flight together), then shared by the CTA
  if (threadIdx.x < unsigned(v.order)) {
    const int j = threadIdx.x + v.foff;
    const int sel = F->sel[j];
    const double* x0 = F->x[j][0];
    const double* x1 = F->x[j][1];
    fac[threadIdx.x] = sel ? x1 : x0;
  }
  __syncthreads();

  // Khatri-Rao rows of the chunk: rho digits over the blocks after n (last
  // fastest), l digits over the blocks before n (block 0 carries the slab
  // offset on a multi-GPU context).
  for (int e = threadIdx.x; e < (q1 - q0) * r; e += blockDim.x) {
    const int q = q0 + e / r;
    const int c = e % r;
    int lq = q / R, rq = q - (q / R) * R;
    double w = 1.0;
    for (int j = v.order - 1; j > v.mode; --j) {
      const int d = rq % v.dims[j];
      rq /= v.dims[j];
      w *= fac[j][(long long)d * r + c];
    }
    for (int j = v.mode - 1; j >= 0; --j) {
      const int d = lq % v.dims[j];
      lq /= v.dims[j];
      w *= fac[j][((long long)d + (j == 0 && v.foff == 0 ? v.row0 : 0)) * r + c];
    }
    wsh[e] = w;
  }
  __syncthreads();

  double acc = 0.0;
  if (ok) {
    for (int q = q0; q < q1;) {
      const int n = min(kTreeQB, q1 - q);
      double ynext[kTreeQB];
      load_batch(ynext, min(kTreeQB, q1 - q - n));
#pragma unroll
      for (int b = 0; b < kTreeQB; ++b)
        if (b < n) acc = fma(y[b], wsh[(q + b - q0) * r + col], acc);  // q order
#pragma unroll
      for (int b = 0; b < kTreeQB; ++b) y[b] = ynext[b];
      q += n;
    }
    if (!CLUSTER) partial[(long long)blockIdx.x * pairs + p] = acc;
  }
  if constexpr (CLUSTER) {
    __shared__ double cpart[kTreeThreads];
    cg::cluster_group cl = cg::this_cluster();
    cpart[threadIdx.x] = acc;
    cl.sync();
    // CTA k of the cluster sums pairs [k*per, (k+1)*per) of the tile over
    // the cluster's CTAs in rank (= chunk) order
    const int ncl = int(cl.num_blocks()), me = int(cl.block_rank());
    const int per = kTreeThreads / ncl;
    if (int(threadIdx.x) < per) {
      const int e = me * per + int(threadIdx.x);
      double s = 0.0;
      for (int c = 0; c < ncl; ++c) s += cl.map_shared_rank(cpart, c)[e];
      const int pe = int(blockIdx.y) * kTreeTile + e;
      if (pe < pairs) out[pe] = s;
    }
    cl.sync();  // no CTA leaves while another still reads its partials
    return;
  }

  // last arrival of the tile sums the chunk slots in chunk order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&arrivals[blockIdx.y], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (ok) {
    const int nch = int(gridDim.x);
    double s = 0.0;
    int k = 0;
    for (; k + kTreeQB <= nch; k += kTreeQB) {
      double x[kTreeQB];
#pragma unroll
      for (int b = 0; b < kTreeQB; ++b) x[b] = __ldcg(partial + (long long)(k + b) * pairs + p);
#pragma unroll
      for (int b = 0; b < kTreeQB; ++b) s += x[b];
    }
    for (; k < nch; ++k) s += __ldcg(partial + (long long)k * pairs + p);
    out[p] = s;
  }
  if (threadIdx.x == 0) arrivals[blockIdx.y] = 0;
}

// Two-mode partials (every tree view of 3- and 4-way tensors): one CTA per
// output row i, M[i][c] = sum_q Y(i, q)[c] * A(q)[c] over the other mode q
// (rows of Y are contiguous for the inner mode, strided by I r for the
// outer one). Thread (g, c) of the CTA (G = blockDim / r groups) adds
// q = g, g + G, ... with all its loads in flight (4 partial sums), then the
// groups fold in group order through shared memory: a fixed order,
// bit-reproducible; one round trip per CTA instead of the chunked
// general kernel's chains (C2: 11.8 -> ~3 us per contraction).
template <int R_MAX>
__global__ void __launch_bounds__(256) tree2_kernel(const double* __restrict__ Y, TreeView v,
                                                    const DevFactors* __restrict__ F, double* __restrict__ out) {
  __shared__ double fold[256];
  // the block's NNLS (a programmatic dependent) may launch and run its
  // prologue now; it waits for this grid before reading the result
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int r = v.rank;
  const int i = int(blockIdx.x);
  const int G = int(blockDim.x) / r;
  const int g = int(threadIdx.x) / r, c = int(threadIdx.x) - g * r;
  const bool inner = v.mode == 0;  // reduce the view's dim 1 (contiguous) or dim 0 (strided)
  const int Q = inner ? v.dims[1] : v.dims[0];
  const int fq = (inner ? 1 : 0) + v.foff;  // factor of the reduced dim
  const long long qoff = (!inner && v.foff == 0) ? v.row0 : 0;  // slab offset of mode 1's rows
  const double* A = F->x[fq][F->sel[fq]];
  constexpr int U = 8;  // terms per trip: 2 U independent loads in flight per thread
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  if (g < G) {
    const double* yrow = inner ? Y + (long long)i * Q * r + c : Y + (long long)i * r + c;
    const long long ystep = inner ? r : (long long)v.dims[1] * r;
    for (int q = g; q < Q; q += U * G) {
      double y[U], a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int qq = q + u * G;
        y[u] = qq < Q ? __ldg(yrow + qq * ystep) : 0.0;
        a[u] = qq < Q ? __ldg(A + (qq + qoff) * r + c) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) s[u & 3] = fma(y[u], a[u], s[u & 3]);
    }
  }
  fold[threadIdx.x] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (int(threadIdx.x) < r) {
    double t = 0.0;
    for (int k = 0; k < G; ++k) t += fold[k * r + threadIdx.x];
    out[(long long)i * r + threadIdx.x] = t;
  }
}

}  // namespace

int tree_tiles(const TreeView& v) { return int((v.I * v.rank + kTreeTile - 1) / kTreeTile); }

int tree_chunks(const TreeView& v, int sms) {
  const long long tiles = tree_tiles(v);
  const long long Q = v.L * v.R;
  // at most two CTAs per SM over the whole grid (two are resident at 92
  // registers x 256 threads): one wave, no tail (r01e at C2: 24 tiles x 13
  // chunks = 312 CTAs ran a 16-CTA second wave, 17 us per launch)
  long long chunks = std::max(1LL, (2LL * sms) / tiles);
  // a chunk's Khatri-Rao rows live in shared memory (<= 192 KB)
  const long long min_chunks = (Q * v.rank * (long long)sizeof(double) + 192 * 1024 - 1) / (192 * 1024);
  chunks = std::max(1LL, std::min(std::max(chunks, min_chunks), Q));
  return int(chunks);
}

void launch_tree_mttkrp(const double* Y, const TreeView& v, const DevFactors* dF, double* partial, int chunks,
                        unsigned* arrivals, double* out, cudaStream_t s) {
  const long long pairs = v.I * v.rank;
  const long long Q = v.L * v.R;
  if (Q >= (1LL << 31) || pairs >= (1LL << 31)) throw Unsupported("dimension tree: view too large for 32-bit indexing");
  if (v.order == 2 && v.rank <= 256 && v.I < (1LL << 31) && !std::getenv("NTF_TREE_GENERAL")) {
    tree2_kernel<0><<<unsigned(v.I), 256, 0, s>>>(Y, v, dF, out);
    NTF_CUDA(cudaGetLastError());
    return;
  }
  const int tiles = tree_tiles(v);
  // cluster path: up to 8 chunks per tile, one wave of at most two CTAs per
  // SM (NTF_TREE_ATOMIC=1: always the global-slot path)
  {
    int ncl = 8;
    const int sms = device_sm_count();
    while (ncl > 1 && (ncl > Q || (long long)tiles * ncl > 2LL * sms)) ncl /= 2;
    const long long qpc = (Q + ncl - 1) / ncl;
    const size_t smem = size_t(qpc) * v.rank * sizeof(double);
    // measured (r01g): clusters win when a chunk is at most two load
    // batches (C3 split tree: 12.0 -> 10.5 us per block) and lose to more,
    // shorter chunks otherwise (C2: 38-step chunks 16.0 vs 14.6 us)
    if (smem <= 192 * 1024 && qpc <= 2 * kTreeQB && !std::getenv("NTF_TREE_ATOMIC")) {
      auto fn = tree_mttkrp_kernel<true>;
      if (smem > 48 * 1024) NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(unsigned(ncl), unsigned(tiles));
      cfg.blockDim = dim3(kTreeThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = unsigned(ncl);
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      NTF_CUDA(cudaLaunchKernelEx(&cfg, fn, Y, v, dF, partial, int(qpc), arrivals, out));
      return;
    }
  }
  const long long qpc = (Q + chunks - 1) / chunks;
  const int nchunk = int((Q + qpc - 1) / qpc);
  const size_t smem = size_t(qpc) * v.rank * sizeof(double);
  if (smem > 200 * 1024) throw Unsupported("dimension tree: chunk too large");
  if (smem > 48 * 1024)
    NTF_CUDA(cudaFuncSetAttribute(tree_mttkrp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(nchunk), unsigned(tiles));
  cfg.blockDim = dim3(kTreeThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  NTF_CUDA(cudaLaunchKernelEx(&cfg, tree_mttkrp_kernel<false>, Y, v, dF, partial, int(qpc), arrivals, out));
}

}  // namespace ntfb
