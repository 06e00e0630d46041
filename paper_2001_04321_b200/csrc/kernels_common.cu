#include <cstring>
#include <algorithm>
// Generic MTTKRP, deterministic reductions, Grams and the cheap objective.
//
// Determinism contract (README.md:155-157 of the reference): every value is
// produced by a fixed accumulation order that depends only on the shapes and
// the launch configuration, never on scheduling — no floating-point atomics.
#include <cstdio>

#include "ntf_internal.h"

namespace ntfb {

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
           file, line, what);
  throw CudaError(buf);
}

int device_sm_count() {
  int dev = 0, n = 0;
  NTF_CUDA(cudaGetDevice(&dev));
  NTF_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

namespace {

constexpr int kGenThreads = 256;
constexpr int kGenCols = 8;

// Fixed-shape tree reduction of kGenThreads values per column.
__device__ __forceinline__ void block_tree_sum(double (&acc)[kGenCols], double* sm) {
  const int t = threadIdx.x;
#pragma unroll
  for (int c = 0; c < kGenCols; ++c) sm[c * kGenThreads + t] = acc[c];
  __syncthreads();
  for (int half = kGenThreads / 2; half > 0; half >>= 1) {
    if (t < half) {
#pragma unroll
      for (int c = 0; c < kGenCols; ++c) sm[c * kGenThreads + t] += sm[c * kGenThreads + t + half];
    }
    __syncthreads();
  }
}

// One block per (output row, segment of the (left,right) plane, 8-column
// group). Each element contributes T * prod_{l != mode} A_l[i_l, c]
// (kernels.cpp:161-191, without materialising the Khatri-Rao rows).
template <typename T>
__global__ void __launch_bounds__(kGenThreads)
    mttkrp_generic_kernel(const T* __restrict__ t, ModeView v, const DevFactors* __restrict__ F,
                          double* __restrict__ partial, long long seg_len) {
  __shared__ double sm[kGenCols * kGenThreads];
  const long long mid = blockIdx.x;
  const long long seg = blockIdx.y;
  const int c0 = blockIdx.z * kGenCols;
  const int r = v.rank;
  const long long plane = v.L * v.R;
  const long long e0 = seg * seg_len;
  const long long e1 = min(plane, e0 + seg_len);
  const double* A[kMaxOrder];
  for (int l = 0; l < v.order; ++l) A[l] = F->x[l][F->sel[l]];

  double acc[kGenCols];
#pragma unroll
  for (int c = 0; c < kGenCols; ++c) acc[c] = 0.0;
  for (long long e = e0 + threadIdx.x; e < e1; e += kGenThreads) {
    const long long left = e / v.R;
    const long long right = e - left * v.R;
    const double tv = double(t[(left * v.I + mid) * v.R + right]);
    int idx[kMaxOrder];
    long long rem = right;
    for (int l = v.order - 1; l > v.mode; --l) {
      idx[l] = int(rem % v.dims[l]);
      rem /= v.dims[l];
    }
    rem = left;
    for (int l = v.mode - 1; l >= 0; --l) {
      idx[l] = int(rem % v.dims[l]);
      rem /= v.dims[l];
    }
    if (v.mode != 0) idx[0] += int(v.row0);  // slab rows index the full A_1
#pragma unroll
    for (int c = 0; c < kGenCols; ++c) {
      if (c0 + c < r) {
        double w = tv;
        for (int l = 0; l < v.order; ++l)
          if (l != v.mode) w *= A[l][(long long)idx[l] * r + c0 + c];
        acc[c] += w;
      }
    }
  }
  block_tree_sum(acc, sm);
  if (threadIdx.x < kGenCols && c0 + threadIdx.x < r)
    partial[(seg * v.I + mid) * r + c0 + threadIdx.x] = sm[threadIdx.x * kGenThreads];
}

// out[i] = sum_k partial[k][i]. A block covers 64 outputs with 4 slot
// groups (k mod 4) of 64 threads; each thread keeps 4 interleaved sums so
// 4 independent loads are in flight, and the groups are folded in a fixed
// order: the result depends only on `segs`, never on scheduling.
constexpr int kRedOut = 64;
__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* __restrict__ partial, int segs,
                                                              long long n, double* __restrict__ out) {
  __shared__ double sm[4][kRedOut];
  const int e = threadIdx.x % kRedOut, g = threadIdx.x / kRedOut;
  const long long i = blockIdx.x * (long long)kRedOut + e;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (i < n) {
    int k = g;
    for (; k + 12 < segs; k += 16) {
      a0 += __ldg(&partial[(long long)k * n + i]);
      a1 += __ldg(&partial[(long long)(k + 4) * n + i]);
      a2 += __ldg(&partial[(long long)(k + 8) * n + i]);
      a3 += __ldg(&partial[(long long)(k + 12) * n + i]);
    }
    for (; k < segs; k += 4) a0 += __ldg(&partial[(long long)k * n + i]);
  }
  sm[g][e] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (g == 0 && i < n) out[i] = (sm[0][e] + sm[1][e]) + (sm[2][e] + sm[3][e]);
}

constexpr int kNormBlocks = 592;  // fixed, so the sum order is device-independent

template <typename T>
__global__ void __launch_bounds__(256) norm_sq_kernel(const T* __restrict__ t, long long n,
                                                      double* __restrict__ scratch) {
  __shared__ double sm[256];
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * kNormBlocks) {
    const double x = double(t[i]);
    s += x * x;
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int half = 128; half > 0; half >>= 1) {
    if (threadIdx.x < half) sm[threadIdx.x] += sm[threadIdx.x + half];
    __syncthreads();
  }
  if (threadIdx.x == 0) scratch[blockIdx.x] = sm[0];
}

__global__ void sum_scratch_kernel(const double* __restrict__ scratch, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += scratch[i];
    *out = s;
  }
}

// Gram of one row-major rows x r matrix, ascending-row order per entry.
// Fixed-order block sum of one value per thread (blockDim a power of two).
__device__ double block_sum(double v, double* __restrict__ red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int half = int(blockDim.x) / 2; half > 0; half >>= 1) {
    if (int(threadIdx.x) < half) red[threadIdx.x] += red[threadIdx.x + half];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

constexpr int kSetupThreads = 1024;
constexpr int kGramThreads = 256;
constexpr int kGramRows = 32;  // rows per partial-Gram CTA

// Partial Grams of the X-role buffers: CTA (mode, chunk) sums its rows'
// outer products (thread e: entries e, e + 256, ...; rows in ascending
// order), one slot per chunk; gram_finish adds the slots in chunk order.
__global__ void __launch_bounds__(kGramThreads) gram_partial_kernel(const DevFactors* __restrict__ F,
                                                                    double* __restrict__ part, int chunks) {
  const int mode = blockIdx.x, chunk = blockIdx.y;
  const int rows = F->rows[mode], r = F->rank;
  const int rpc = (rows + chunks - 1) / chunks;
  const int i0 = chunk * rpc, i1 = min(rows, i0 + rpc);
  const double* a = F->x[mode][F->sel[mode]];
  double* dst = part + ((size_t)mode * chunks + chunk) * r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int p = e / r, q = e % r;
    double s0 = 0.0, s1 = 0.0;
    int i = i0;
    for (; i + 1 < i1; i += 2) {
      s0 += a[(long long)i * r + p] * a[(long long)i * r + q];
      s1 += a[(long long)(i + 1) * r + p] * a[(long long)(i + 1) * r + q];
    }
    if (i < i1) s0 += a[(long long)i * r + p] * a[(long long)i * r + q];
    dst[e] = s0 + s1;
  }
}

__global__ void __launch_bounds__(kGramThreads) gram_finish_kernel(DevFactors* F, const double* __restrict__ part,
                                                                   int chunks) {
  const int mode = blockIdx.x, r = F->rank;
  double* g = F->gram[mode][F->sel[mode]];
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    double t = 0.0;
    for (int c = 0; c < chunks; ++c) t += part[((size_t)mode * chunks + c) * r * r + e];
    g[e] = t;
  }
}

// FP32 mirrors of both buffers of every mode (grid-stride, blockIdx.y = mode)
__global__ void mirror_kernel(DevFactors* F) {
  const int mode = blockIdx.y;
  const long long n = (long long)F->rows[mode] * F->rank;
  for (int bb = 0; bb < 2; ++bb) {
    float* m = F->x32[mode][bb];
    const double* x = F->x[mode][bb];
    if (m && x)
      for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
        m[e] = float(x[e]);
  }
}

// cheap_objective at `pivot` (kernels.cpp:298-303 with the pivot of :305-311);
// every Gram (the pivot's included) is current: launch_init_factors ran on
// the same factors
__global__ void __launch_bounds__(kSetupThreads) objective_kernel(const DevFactors* __restrict__ F, int order,
                                                                  int r, int pivot, int rows,
                                                                  const double* __restrict__ C,
                                                                  const double* __restrict__ nsq,
                                                                  double* __restrict__ out) {
  __shared__ double red[kSetupThreads];
  const double* a = F->x[pivot][F->sel[pivot]];
  double cross = 0.0;
  for (long long e = threadIdx.x; e < (long long)rows * r; e += blockDim.x) cross += a[e] * C[e];
  cross = block_sum(cross, red);
  const double* gp[kMaxOrder];
  for (int j = 0; j < order; ++j) gp[j] = F->gram[j][F->sel[j]];
  double quad = 0.0;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    double g = 1.0;
    for (int j = 0; j < order; ++j)
      if (j != pivot) g *= gp[j][e];
    quad += gp[pivot][e] * g;
  }
  quad = block_sum(quad, red);
  if (threadIdx.x == 0) *out = 0.5 * (*nsq) - cross + 0.5 * quad;
}

__global__ void stamp_start_kernel(RunState* st) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  st->t_start_ns = t;
}

__global__ void apply_time_budget_kernel(RunState* st) {
  if (st->max_time_s > 0.0 && st->elapsed_s >= st->max_time_s) st->done = 1;
}

__global__ void compact_rows_kernel(const double* __restrict__ gathered, long long maxrows,
                                    const long long* __restrict__ begins, const long long* __restrict__ counts,
                                    int world, int r, double* __restrict__ out) {
  for (int p = 0; p < world; ++p) {
    const long long n = counts[p] * r;
    const double* src = gathered + (long long)p * maxrows * r;
    double* dst = out + begins[p] * r;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
      dst[e] = src[e];
  }
}

}  // namespace

void launch_mttkrp_generic(const void* t, int dtype, const ModeView& v, const DevFactors* dF, double* partial,
                           int segs, cudaStream_t s) {
  const long long plane = v.L * v.R;
  const long long seg_len = (plane + segs - 1) / segs;
  dim3 grid(unsigned(v.I), unsigned(segs), unsigned((v.rank + kGenCols - 1) / kGenCols));
  if (dtype == NTF_DTYPE_F32)
    mttkrp_generic_kernel<float><<<grid, kGenThreads, 0, s>>>(static_cast<const float*>(t), v, dF, partial, seg_len);
  else
    mttkrp_generic_kernel<double><<<grid, kGenThreads, 0, s>>>(static_cast<const double*>(t), v, dF, partial,
                                                               seg_len);
  NTF_CUDA(cudaGetLastError());
}

void launch_reduce_partials(const double* partial, int segs, long long n, double* out, cudaStream_t s) {
  const long long blocks = (n + kRedOut - 1) / kRedOut;
  reduce_partials_kernel<<<unsigned(blocks), 256, 0, s>>>(partial, segs, n, out);
  NTF_CUDA(cudaGetLastError());
}

void launch_norm_sq(const void* t, int dtype, long long n, double* scratch, int scratch_len, double* out,
                    cudaStream_t s) {
  if (scratch_len < kNormBlocks) throw LogicError("norm_sq scratch too small");
  if (dtype == NTF_DTYPE_F32)
    norm_sq_kernel<float><<<kNormBlocks, 256, 0, s>>>(static_cast<const float*>(t), n, scratch);
  else
    norm_sq_kernel<double><<<kNormBlocks, 256, 0, s>>>(static_cast<const double*>(t), n, scratch);
  sum_scratch_kernel<<<1, 32, 0, s>>>(scratch, kNormBlocks, out);
  NTF_CUDA(cudaGetLastError());
}

size_t init_factors_scratch(const DevFactors& hF) {
  int rows = 1;
  for (int i = 0; i < hF.order; ++i) rows = std::max(rows, hF.rows[i]);
  const int chunks = std::max(1, std::min(64, (rows + kGramRows - 1) / kGramRows));
  return size_t(hF.order) * chunks * hF.rank * hF.rank;
}

void launch_init_factors(DevFactors* dF, const DevFactors& hF, double* scratch, size_t scratch_len, cudaStream_t s) {
  int rows = 1;
  for (int i = 0; i < hF.order; ++i) rows = std::max(rows, hF.rows[i]);
  int chunks = std::max(1, std::min(64, (rows + kGramRows - 1) / kGramRows));
  const size_t per = size_t(hF.order) * hF.rank * hF.rank;
  chunks = int(std::max<size_t>(1, std::min<size_t>(size_t(chunks), scratch_len / per)));
  if (scratch_len < per) throw LogicError("init_factors scratch too small");
  gram_partial_kernel<<<dim3(unsigned(hF.order), unsigned(chunks)), kGramThreads, 0, s>>>(dF, scratch, chunks);
  gram_finish_kernel<<<unsigned(hF.order), kGramThreads, 0, s>>>(dF, scratch, chunks);
  bool mirrors = false;
  for (int i = 0; i < hF.order; ++i) mirrors = mirrors || hF.x32[i][0] || hF.x32[i][1];
  if (mirrors) mirror_kernel<<<dim3(64u, unsigned(hF.order)), 256, 0, s>>>(dF);
  NTF_CUDA(cudaGetLastError());
}

void launch_objective(const DevFactors* dF, int order, int rank, int pivot, int rows, const double* C,
                      const double* nsq_dev, double* out, cudaStream_t s) {
  objective_kernel<<<1, kSetupThreads, 0, s>>>(dF, order, rank, pivot, rows, C, nsq_dev, out);
  NTF_CUDA(cudaGetLastError());
}

void launch_stamp_start(RunState* st, cudaStream_t s) {
  stamp_start_kernel<<<1, 1, 0, s>>>(st);
  NTF_CUDA(cudaGetLastError());
}

void launch_apply_time_budget(RunState* st, cudaStream_t s) {
  apply_time_budget_kernel<<<1, 1, 0, s>>>(st);
  NTF_CUDA(cudaGetLastError());
}

void launch_compact_rows(const double* gathered, long long maxrows, const long long* begins,
                         const long long* counts, int world, int r, double* out, cudaStream_t s) {
  compact_rows_kernel<<<64, 256, 0, s>>>(gathered, maxrows, begins, counts, world, r, out);
  NTF_CUDA(cudaGetLastError());
}


// ---- small host -> device uploads as kernel parameters --------------------
// A cudaMemcpy of a small table queues behind whatever the copy engine is
// doing -- behind the 216 MB tensor upload of an asynchronous ntf_tensor_upload,
// which would stall session setup for milliseconds. Kernel parameters travel
// with the launch instead: the payload is cut into chunks that ride in the
// parameter buffer and a few threads write them out.
namespace {
constexpr int kParamChunk = 28672;  // bytes per launch (CUDA 12.1+: 32 764 bytes of kernel parameters on sm_70+)
struct ParamBlob {
  unsigned long long w[kParamChunk / 8];
};
__global__ void param_upload_kernel(unsigned long long* dst, ParamBlob blob, int n8, unsigned char* tail_dst,
                                    unsigned long long tail, int tail_n) {
  for (int i = threadIdx.x; i < n8; i += blockDim.x) dst[i] = blob.w[i];
  if (threadIdx.x < tail_n) tail_dst[threadIdx.x] = (unsigned char)(tail >> (8 * threadIdx.x));
}
}  // namespace

namespace {
__global__ void zero_kernel(unsigned* dst, size_t n4) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) dst[i] = 0u;
}
}  // namespace

void dev_zero(void* dst, size_t bytes, cudaStream_t s) {
  if (bytes % 4 || reinterpret_cast<uintptr_t>(dst) % 4) throw LogicError("dev_zero: 4-byte granularity");
  if (!bytes) return;
  const size_t n4 = bytes / 4;
  zero_kernel<<<unsigned(std::min<size_t>(64, (n4 + 255) / 256)), 256, 0, s>>>(static_cast<unsigned*>(dst), n4);
  NTF_CUDA(cudaGetLastError());
}

void dev_upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (reinterpret_cast<uintptr_t>(dst) % 8) throw LogicError("dev_upload: destination must be 8-byte aligned");
  const unsigned char* p = static_cast<const unsigned char*>(src);
  unsigned char* d = static_cast<unsigned char*>(dst);
  size_t off = 0;
  while (off < bytes) {
    const size_t n = std::min(bytes - off, size_t(kParamChunk));
    ParamBlob blob;
    const int n8 = int(n / 8), tail_n = int(n % 8);
    std::memcpy(blob.w, p + off, size_t(n8) * 8);
    unsigned long long tail = 0;
    if (tail_n) std::memcpy(&tail, p + off + size_t(n8) * 8, size_t(tail_n));
    param_upload_kernel<<<1, 128, 0, s>>>(reinterpret_cast<unsigned long long*>(d + off), blob, n8,
                                          d + off + size_t(n8) * 8, tail, tail_n);
    off += n;
  }
  NTF_CUDA(cudaGetLastError());
}

}  // namespace ntfb
