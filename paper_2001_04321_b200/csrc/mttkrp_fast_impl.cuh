// Fast dense MTTKRP for sm_100a — kernel template (included by the
// per-dtype translation units).
//
// View of the local tensor around `mode` (kernels.cpp:10-27): T[l][m][rho]
// with l over the modes before `mode`, m the output row, rho over the modes
// after it. The contraction is
//     M[m][c] = sum_{l,rho} T[l][m][rho] * wl[l][c] * wr[rho][c]
// where wl / wr are Khatri-Rao rows of the other factors (kernels.cpp:90-113)
// formed on the fly in shared memory, never materialised in HBM.
//
// Two shared-memory layouts, picked by which index is contiguous in HBM:
//   ROW (R > 1): a unit is one (l, 128-byte rho box) for all m of the CTA
//     tile; TMA brings a [m_tile][128 B] box with the 128-byte swizzle, so a
//     lane can read 16 B of one row (2 doubles / 4 floats along rho) without
//     bank conflicts while its neighbours read other rows.
//   COL (R == 1, the last mode): a unit is KL consecutive l for all m; TMA
//     brings [KL][m_tile] rows, lanes read 16 B = consecutive output rows.
//
// Warp specialisation: warp 0 is the producer (one lane issues the TMA boxes,
// all 32 lanes build the stage's Khatri-Rao rows W[k][c] = wl*wr), warps
// 1.. are consumers with register-blocked accumulators: lane = (rg, cg)
// owns A rows x B columns, W values are warp-broadcast reads, T values are
// 16-byte reads. Stages are handed over with mbarriers (full: TMA tx bytes +
// 32 producer arrivals; empty: one arrival per consumer warp).
//
// Each CTA owns a contiguous range of units of one m-tile (split-K) and
// writes its FP64 partial M to its own slot; a fixed-order reduction over the
// slots follows (no atomics: bit-reproducible, README.md:155-157).
#pragma once

#include <cuda.h>

#include "mttkrp_fast_launch.h"
#include "ntf_internal.h"

namespace ntfb {
namespace fast {

template <typename T>
struct Vec;
template <>
struct Vec<double> {
  using V = double2;
  static constexpr int N = 2;
  __device__ static double get(const V& v, int i) { return i == 0 ? v.x : v.y; }
};
template <>
struct Vec<float> {
  using V = float4;
  static constexpr int N = 4;
  __device__ static float get(const V& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

template <typename T>
__device__ __forceinline__ const T* factor_ptr(const DevFactors* F, int j);
template <>
__device__ __forceinline__ const double* factor_ptr<double>(const DevFactors* F, int j) {
  return F->x[j][F->sel[j]];
}
template <>
__device__ __forceinline__ const float* factor_ptr<float>(const DevFactors* F, int j) {
  return F->x32[j][F->sel[j]];
}

// G column groups of B columns each (padded to BP so 16-byte loads stay
// aligned); RG = 32/G row groups; A rows per lane.
template <typename T, int G, int B, int A, int LAYOUT>
__global__ void __launch_bounds__(384, 1) mttkrp_fast_kernel(const __grid_constant__ CUtensorMap tmap, Params p) {
  using VT = Vec<T>;
  using V = typename VT::V;
  constexpr int VEC = VT::N;
  constexpr int RG = 32 / G;
  constexpr int BP = (B + VEC - 1) / VEC * VEC;
  constexpr int NV = BP / VEC;
  static_assert(LAYOUT == kRow || A % VEC == 0, "COL layout reads VEC consecutive rows");

  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ModeView& v = p.v;
  const int r = v.rank;
  const int stages = p.stages;
  unsigned char* t_base = smem;
  T* w_base = reinterpret_cast<T*>(smem + size_t(stages) * p.t_stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(w_base) +
                                               size_t(stages) * p.w_stage_bytes);
  uint64_t* empty = full + stages;

  const int mt = blockIdx.x / p.ctas_per_mtile;
  const int j = blockIdx.x % p.ctas_per_mtile;
  const long long u0 = p.units * j / p.ctas_per_mtile;
  const long long u1 = p.units * (j + 1) / p.ctas_per_mtile;
  const int n_consumers = p.MW * p.KW;
  const int NP = p.NP;  // producer warps

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], n_consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  }
  {
    // padding columns of every W stage stay zero for the whole kernel
    constexpr int KB = 128 / int(sizeof(T));
    for (int e = threadIdx.x; e < stages * KB * p.wld; e += blockDim.x) {
      const int cc = e % p.wld;
      if (cc % BP >= B || (cc / BP) * B + cc % BP >= r) w_base[e] = T(0);
    }
  }
  __syncthreads();

  if (warp < NP) {
    // ------------------------------------------------------------ producer
    // Lane owns columns c = lane (+32); the k-varying modes (ROW: modes after
    // `mode`, i.e. rho; COL: all modes before it, i.e. l) advance as an
    // odometer, so a unit costs KB x (#varying modes) coalesced row loads per
    // lane, all independent, and no integer division inside the k loop.
    constexpr int KB = 128 / int(sizeof(T));
    constexpr int CPL = (G * B + 31) / 32;  // columns per lane
    const T* fac[kMaxOrder];
    int dims[kMaxOrder];
    bool vary[kMaxOrder], fixd[kMaxOrder];
#pragma unroll
    for (int q = 0; q < kMaxOrder; ++q) {
      fac[q] = q < v.order ? factor_ptr<T>(p.F, q) : nullptr;
      dims[q] = q < v.order ? v.dims[q] : 1;
      vary[q] = q < v.order && (LAYOUT == kRow ? q > v.mode : q < v.mode);
      fixd[q] = LAYOUT == kRow && q < v.mode;
    }
    const int row0 = int(v.row0);
    // Producer warp `warp` owns the units i = warp, warp + NP, ... of this
    // CTA's range; unit i lives in stage i % stages during round i / stages.
    for (long long i = warp; i < u1 - u0; i += NP) {
      const long long u = u0 + i;
      const int s = int(i % stages);
      const uint32_t round = uint32_t(i / stages);
      if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
      long long l, rho0;
      if (LAYOUT == kRow) {
        l = u / p.nbox_r;
        rho0 = (u - l * p.nbox_r) * p.kbox;
      } else {
        l = u * p.kbox;
        rho0 = 0;
      }
      unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
      if (lane == 0) {
        mbar_expect_tx(&full[s], p.tx_bytes);
        for (int mb = 0; mb < p.n_mbox; ++mb) {
          const int m0 = mt * p.m_cta + mb * p.m_box;
          if (LAYOUT == kRow)
            tma_load_3d(ts + size_t(mb) * p.m_box * 128, &tmap, &full[s], int(rho0), m0, int(l));
          else
            tma_load_3d(ts + size_t(mb) * p.m_box * p.kbox * sizeof(T), &tmap, &full[s], m0, int(l), 0);
        }
      }
      // Khatri-Rao rows of this unit: W[k][cg*BP + b] for column c = cg*B + b.
      T* ws = w_base + size_t(s) * (p.w_stage_bytes / sizeof(T));
      int dig[kMaxOrder];
      {
        // l and rho0 are < 2^31 on the fast path (checked by the planner)
        unsigned rem = unsigned((LAYOUT == kRow) ? rho0 : l);  // digits of the first k
        unsigned lrem = unsigned(l);                           // ROW: fixed digits of l
#pragma unroll
        for (int q = kMaxOrder - 1; q >= 0; --q) {
          dig[q] = 0;
          if (vary[q]) {
            dig[q] = int(rem % unsigned(dims[q]));
            rem /= unsigned(dims[q]);
          } else if (fixd[q]) {
            dig[q] = int(lrem % unsigned(dims[q]));
            lrem /= unsigned(dims[q]);
          }
        }
      }
      const long long kmax = (LAYOUT == kRow) ? v.R - rho0 : v.L - l;  // valid k < kmax
      // Only the last varying digit (mode qL) moves between consecutive k,
      // except at a wrap: W[k][c] = base[c] * A_qL[dl + k][c] with base the
      // product of every other factor row, recomputed only after a wrap.
      const int qL = (LAYOUT == kRow) ? v.order - 1 : v.order - 2;
      const T* __restrict__ fL = fac[0];
#pragma unroll
      for (int q = 1; q < kMaxOrder; ++q)
        if (q == qL) fL = fac[q];
      const int offL = (qL == 0) ? row0 : 0;
      int dimL = dims[0];
#pragma unroll
      for (int q = 1; q < kMaxOrder; ++q)
        if (q == qL) dimL = dims[q];
#pragma unroll
      for (int ci = 0; ci < CPL; ++ci) {
        const int c = lane + 32 * ci;
        if (c >= r) continue;
        int d[kMaxOrder];
#pragma unroll
        for (int q = 0; q < kMaxOrder; ++q) d[q] = dig[q];
        auto make_base = [&]() {
          T b = T(1);
#pragma unroll
          for (int q = 0; q < kMaxOrder; ++q)
            if ((fixd[q] || vary[q]) && q != qL) b *= __ldg(&fac[q][(d[q] + (q == 0 ? row0 : 0)) * r + c]);
          return b;
        };
        const T base0 = make_base();
        int dl0 = 0;
#pragma unroll
        for (int q = 0; q < kMaxOrder; ++q)
          if (q == qL) dl0 = d[q];
        T* dst = ws + (c / B) * BP + (c % B);
        const int kwrap = dimL - dl0;  // first k whose last digit wraps to 0
        if (kwrap < KB && dimL < KB) {
          // tiny last mode (several wraps per unit): plain odometer walk
          int dl = dl0;
          T base = base0;
          for (int k = 0; k < KB; ++k) {
            const T val = base * __ldg(&fL[(dl + offL) * r + c]);
            dst[k * p.wld] = (k < kmax) ? val : T(0);
            if (++dl == dimL) {
              dl = 0;
              bool carry = true;
#pragma unroll
              for (int q = kMaxOrder - 1; q >= 0; --q) {
                if (vary[q] && q < qL && carry) {
                  if (++d[q] < dims[q])
                    carry = false;
                  else
                    d[q] = 0;
                }
              }
              base = make_base();
            }
          }
          continue;
        }
        // at most one wrap: base1 (after the carry) is fetched up front and
        // every factor-row load of the unit is independent of the others
        T base1 = base0;
        if (kwrap < KB) {
          bool carry = true;
#pragma unroll
          for (int q = kMaxOrder - 1; q >= 0; --q) {
            if (vary[q] && q < qL && carry) {
              if (++d[q] < dims[q])
                carry = false;
              else
                d[q] = 0;
            }
          }
          base1 = make_base();
        }
        T row_val[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          const int row = dl0 + k - (k >= kwrap ? dimL : 0);
          row_val[k] = __ldg(&fL[(row + offL) * r + c]);
        }
#pragma unroll
        for (int k = 0; k < KB; ++k)
          dst[k * p.wld] = (k < kmax) ? (k >= kwrap ? base1 : base0) * row_val[k] : T(0);
      }
      mbar_arrive(&full[s]);
    }
  } else if (warp < NP + n_consumers) {
    // ------------------------------------------------------------ consumers
    const int cw = warp - NP;
    const int mw = cw % p.MW, kw = cw / p.MW;
    const int rg = lane % RG, cg = lane / RG;
    const int RW = RG * A;
    T acc[A][B];
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int b = 0; b < B; ++b) acc[i][b] = T(0);

    // per-lane smem offsets of its rows (constant over units)
    int off[A];
#pragma unroll
    for (int i = 0; i < A; ++i) {
      if (LAYOUT == kRow) {
        const int m = mw * RW + rg + RG * i;
        off[i] = m;  // row index; byte offset m*128, swizzle key m & 7
      } else {
        const int m = mw * RW + VEC * rg + (i % VEC) + VEC * RG * (i / VEC);
        off[i] = (m / p.m_box) * p.m_box * p.kbox + (m % p.m_box);  // element offset at k = 0
      }
    }
    int s = 0;
    uint32_t phase = 0;
    for (long long u = u0; u < u1; ++u) {
      mbar_wait(&full[s], phase);
      const unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
      const T* ws = w_base + size_t(s) * (p.w_stage_bytes / sizeof(T)) + cg * BP;
      if (LAYOUT == kRow) {
        constexpr int KCH = 128 / 16;  // 16-byte chunks per 128-byte row
        for (int pc = kw; pc < KCH; pc += p.KW) {
          T w[VEC][BP];
#pragma unroll
          for (int kk = 0; kk < VEC; ++kk)
#pragma unroll
            for (int q = 0; q < NV; ++q) {
              const V x = *reinterpret_cast<const V*>(ws + (pc * VEC + kk) * p.wld + q * VEC);
#pragma unroll
              for (int e = 0; e < VEC; ++e) w[kk][q * VEC + e] = VT::get(x, e);
            }
          V tv[A];
#pragma unroll
          for (int i = 0; i < A; ++i) {
            const int m = off[i];
            tv[i] = *reinterpret_cast<const V*>(ts + m * 128 + (((pc ^ m) & 7) << 4));
          }
          // kk outermost: an accumulator is reused only after all A*B others
          // (DFMA latency exceeds a B-long dependency distance)
#pragma unroll
          for (int kk = 0; kk < VEC; ++kk)
#pragma unroll
            for (int i = 0; i < A; ++i) {
              const T t = VT::get(tv[i], kk);
#pragma unroll
              for (int b = 0; b < B; ++b) acc[i][b] = fma(t, w[kk][b], acc[i][b]);
            }
        }
      } else {
        const T* tt = reinterpret_cast<const T*>(ts);
        for (int k = kw; k < p.kbox; k += p.KW) {
          T w[BP];
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const V x = *reinterpret_cast<const V*>(ws + k * p.wld + q * VEC);
#pragma unroll
            for (int e = 0; e < VEC; ++e) w[q * VEC + e] = VT::get(x, e);
          }
#pragma unroll
          for (int i4 = 0; i4 < A / VEC; ++i4) {
            const V tv = *reinterpret_cast<const V*>(tt + off[i4 * VEC] + k * p.m_box);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const T t = VT::get(tv, e);
#pragma unroll
              for (int b = 0; b < B; ++b) acc[i4 * VEC + e][b] = fma(t, w[b], acc[i4 * VEC + e][b]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == stages) {
        s = 0;
        phase ^= 1;
      }
    }

    // ------------------------------------------------------------ epilogue
    // k-split warps fold into kw == 0 in kw order through shared memory
    // (the stage buffers are idle once every unit has been consumed).
    T* red = reinterpret_cast<T*>(smem);
    const int ld = G * B;
    asm volatile("bar.sync 1, %0;" ::"r"(n_consumers * 32) : "memory");
    for (int src = 1; src < p.KW; ++src) {
      if (kw == src) {
#pragma unroll
        for (int i = 0; i < A; ++i) {
          const int m = (LAYOUT == kRow) ? off[i] : mw * RW + VEC * rg + (i % VEC) + VEC * RG * (i / VEC);
#pragma unroll
          for (int b = 0; b < B; ++b) red[m * ld + cg * B + b] = acc[i][b];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(n_consumers * 32) : "memory");
      if (kw == 0) {
#pragma unroll
        for (int i = 0; i < A; ++i) {
          const int m = (LAYOUT == kRow) ? off[i] : mw * RW + VEC * rg + (i % VEC) + VEC * RG * (i / VEC);
#pragma unroll
          for (int b = 0; b < B; ++b) acc[i][b] += red[m * ld + cg * B + b];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(n_consumers * 32) : "memory");
    }
    if (kw == 0) {
      double* out = p.partial + (size_t(j) * v.I) * r;
#pragma unroll
      for (int i = 0; i < A; ++i) {
        const int m = (LAYOUT == kRow) ? off[i] : mw * RW + VEC * rg + (i % VEC) + VEC * RG * (i / VEC);
        const long long row = (long long)mt * p.m_cta + m;
        if (m < p.m_cta && row < v.I) {
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const int c = cg * B + b;
            if (c < r) out[row * r + c] = double(acc[i][b]);
          }
        }
      }
    }
  }
}

}  // namespace fast
}  // namespace ntfb
