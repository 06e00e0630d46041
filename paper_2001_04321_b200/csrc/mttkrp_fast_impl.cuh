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

#ifndef NTF_FAST_PROFILE
#define NTF_FAST_PROFILE 0
#endif

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
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(tx)
               : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
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
// FP64 tensor-core step (DMMA): D[8x8] += A[8x4] B[4x8]; lane (g, t) holds
// A[g][t], B[t][g] and D[g][2t], D[g][2t+1] (g = lane / 4, t = lane % 4).
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// LAYOUT: kRow / kCol with CUDA-core FMAs; kRowMma / kColMma (FP64 only):
// the consumers run the same stages through DMMA (see the consumer loop).
template <typename T, int G, int B, int A, int LAYOUT>
__global__ void __launch_bounds__(max_threads_es(A, B, int(sizeof(T))), 1) mttkrp_fast_kernel(const __grid_constant__ CUtensorMap tmap, Params p) {
  constexpr bool MMA = LAYOUT >= kRowMma;
  constexpr int LAY = LAYOUT & 1;
  using VT = Vec<T>;
  using V = typename VT::V;
  constexpr int VEC = VT::N;
  constexpr int RG = 32 / G;
  constexpr int BP = (B + VEC - 1) / VEC * VEC;
  constexpr int NV = BP / VEC;

  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ModeView& v = p.v;
  const int r = v.rank;
  const int stages = p.stages;
  unsigned char* t_base = smem;
  T* w_base = reinterpret_cast<T*>(smem + size_t(stages) * p.t_stage_bytes);
  T* aq_base = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(w_base) + size_t(stages) * p.w_stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(aq_base) +
                                               size_t(stages) * p.aq_stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* aqb = empty + stages;  // factor rows of a unit landed (producer-only)

  const int mt = blockIdx.x / p.ctas_per_mtile;
  const int j = blockIdx.x % p.ctas_per_mtile;
  const long long u0 = p.units * j / p.ctas_per_mtile;
  const long long u1 = p.units * (j + 1) / p.ctas_per_mtile;
  const int n_consumers = p.MW * p.KW;
  const int NP = p.NP;  // producer warps
  // diagnostics only: compiled in with -DNTF_FAST_PROFILE=1
  const bool prof_on = NTF_FAST_PROFILE && p.prof != nullptr;

  if (prof_on && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    p.prof[blockIdx.x * kProfSlots + 6] = g;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], n_consumers);
      mbar_init(&aqb[s], 1);
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
    // W[k][c] = base[c] * A_qL[dl0 + k][c]: only the last varying digit
    // (mode qL) moves between consecutive k of a unit, so the unit's KB rows
    // of A_qL are consecutive in memory (two runs at a wrap). They arrive
    // with one or two cp.async.bulk copies issued D units ahead on the aq
    // barrier; `base` (every other factor row) changes rarely and is an L1
    // hit. The producer then only multiplies shared-memory rows.
    // Everything shape-dependent about a unit (TMA coordinates, first row and
    // wrap of the last varying digit, base-row indices) comes from the
    // host-built unit table, so the producer does no index arithmetic.
    constexpr int KB = 128 / int(sizeof(T));
    constexpr int CPL = (G * B + 31) / 32;  // columns per lane
    const T* fL = factor_ptr<T>(p.F, p.qL);
    const T* bfac[kMaxBase];
#pragma unroll
    for (int t = 0; t < kMaxBase; ++t) bfac[t] = t < p.nb ? factor_ptr<T>(p.F, p.bq[t]) : nullptr;
    const unsigned row_bytes = unsigned(r * sizeof(T));
    // aq stage: [KB rows of A_qL][nb base rows][nb base rows after the wrap]
    // then two ints (valid k count, first k after the wrap).
    const int aq_elems = int(p.aq_stage_bytes / sizeof(T));
    auto aq_of = [&](int s) { return aq_base + size_t(s) * aq_elems; };
    auto info_of = [&](int s) { return reinterpret_cast<int*>(aq_of(s) + (KB + 2 * kMaxBase) * r); };

    // Producer warp `warp` owns the units i = warp + NP*jj of this CTA's
    // range; unit i lives in stage i % stages during round i / stages
    // (NP | stages, so each producer cycles through its own stages).
    const long long n_units = u1 - u0;
    const long long n_mine = n_units > warp ? (n_units - warp + NP - 1) / NP : 0;
    // copies of a unit are issued D units before its W is formed (1 <= D <
    // stages/NP, so the stage wait in issue() only ever depends on W already
    // produced: no deadlock)
    const int D = (stages / NP) / 2 > 1 ? (stages / NP) / 2 : 1;
    long long pw_empty = 0, pw_aq = 0;  // diagnostics (p.prof)
    const long long pt0 = prof_on ? clock64() : 0;
    // Unit-table entries are read by lane 0 one iteration ahead.
    struct Ent {
      int e[kUnitInts];
    };
    auto fetch = [&](long long jj) {
      Ent t;
      if (lane == 0) {
        const int2* src = reinterpret_cast<const int2*>(p.utab + size_t(u0 + warp + jj * NP) * kUnitInts);
#pragma unroll
        for (int q = 0; q < kUnitInts / 2; ++q) {
          const int2 x = __ldg(src + q);
          t.e[2 * q] = x.x;
          t.e[2 * q + 1] = x.y;
        }
      }
      return t;
    };
    // stage / round of the next unit to issue and to form (NP | stages)
    int s_is = warp, s_cp = warp;
    uint32_t r_is = 0, r_cp = 0;
    auto issue = [&](const Ent& en) {
      const int s = s_is;
      if (r_is > 0) {
        const long long t0 = prof_on ? clock64() : 0;
        mbar_wait(&empty[s], (r_is - 1) & 1);
        if (prof_on) pw_empty += clock64() - t0;
      }
      if ((s_is += NP) >= stages) {
        s_is -= stages;
        ++r_is;
      }
      if (lane == 0) {
        const int* e = en.e;
        const int n_valid = e[3], n1 = e[4], kwrap = e[5];
        unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
        mbar_expect_tx(&full[s], p.tx_bytes);
        for (int mb = 0; mb < p.n_mbox; ++mb) {
          const int m0 = mt * p.m_cta + mb * p.m_box;
          if (LAY == kRow)
            tma_load_3d(ts + size_t(mb) * p.m_box * 128, &tmap, &full[s], e[0], m0, e[1]);
          else
            tma_load_3d(ts + size_t(mb) * p.m_pitch * p.kbox * sizeof(T), &tmap, &full[s], m0, e[0], 0);
        }
        T* aq = aq_of(s);
        int* info = info_of(s);
        info[0] = n_valid;
        info[1] = kwrap;
        const bool wrap = kwrap < KB;
        // this warp's generic reads of the previous use of aq[s] precede the copies
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&aqb[s], unsigned(n_valid + p.nb * (wrap ? 2 : 1)) * row_bytes);
        bulk_load(aq, fL + size_t(e[2]) * r, unsigned(n1) * row_bytes, &aqb[s]);
        if (n_valid > n1)
          bulk_load(aq + size_t(n1) * r, fL + size_t(p.rowL_wrap) * r, unsigned(n_valid - n1) * row_bytes, &aqb[s]);
#pragma unroll
        for (int t = 0; t < kMaxBase; ++t)
          if (t < p.nb) {
            bulk_load(aq + size_t(KB + t) * r, bfac[t] + size_t(e[6 + t]) * r, row_bytes, &aqb[s]);
            if (wrap)
              bulk_load(aq + size_t(KB + kMaxBase + t) * r, bfac[t] + size_t(e[6 + kMaxBase + t]) * r, row_bytes,
                        &aqb[s]);
          }
      }
    };
    // Iteration jj issues the copies of unit jj (as soon as its stage is
    // free) and forms W of unit jj - D, whose copies have had D iterations to
    // land: W runs up to `stages/NP` units ahead of the consumers.
    Ent ent = fetch(0);
    for (long long jj = 0; jj < n_mine + D; ++jj) {
      if (jj < n_mine) {
        const Ent ent_next = (jj + 1 < n_mine) ? fetch(jj + 1) : ent;
        issue(ent);
        ent = ent_next;
      }
      if (jj < D) continue;
      const int s = s_cp;
      const uint32_t round = r_cp;
      if ((s_cp += NP) >= stages) {
        s_cp -= stages;
        ++r_cp;
      }
      T* ws = w_base + size_t(s) * (p.w_stage_bytes / sizeof(T));
      const T* aq = aq_of(s);
      {
        const long long t0 = prof_on ? clock64() : 0;
        mbar_wait(&aqb[s], round & 1);
        if (prof_on) pw_aq += clock64() - t0;
      }
      const int* info = info_of(s);
      const int kmax = info[0];   // valid k < kmax
      const int kwrap = info[1];  // first k after the wrap of the last varying digit
      const bool wrap = kwrap < KB;
#pragma unroll
      for (int ci = 0; ci < CPL; ++ci) {
        const int c = lane + 32 * ci;
        if (c >= r) continue;
        T base0 = T(1), base1 = T(1);
#pragma unroll
        for (int t = 0; t < kMaxBase; ++t)
          if (t < p.nb) {
            base0 *= aq[(KB + t) * r + c];
            base1 *= aq[(KB + (wrap ? kMaxBase : 0) + t) * r + c];
          }
        T* dst = ws + (c / B) * BP + (c % B);
#pragma unroll
        for (int k = 0; k < KB; ++k)
          dst[k * p.wld] = (k < kmax) ? (k >= kwrap ? base1 : base0) * aq[k * r + c] : T(0);
      }
      mbar_arrive(&full[s]);
    }
    if (prof_on && warp == 0 && lane == 0) {
      p.prof[blockIdx.x * kProfSlots + 0] = clock64() - pt0;
      p.prof[blockIdx.x * kProfSlots + 1] = pw_empty;
      p.prof[blockIdx.x * kProfSlots + 2] = pw_aq;
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

    // Rows owned by the lane. ROW: rg + RG*i. COL: groups of VEC consecutive
    // rows (one 16-byte read), the last A % VEC rows one by one.
    constexpr int AV = (A / VEC) * VEC;
    auto lane_row = [&](int i) {
      if (LAY == kRow) return mw * RW + rg + RG * i;
      if (i < AV) return mw * RW + VEC * rg + (i % VEC) + VEC * RG * (i / VEC);
      return mw * RW + VEC * RG * (A / VEC) + rg + RG * (i - AV);
    };
    // per-lane smem offsets of its rows (constant over units)
    int off[A];
#pragma unroll
    for (int i = 0; i < A; ++i) {
      const int m = lane_row(i);
      if (LAY == kRow)
        off[i] = m;  // row index; byte offset m*128, swizzle key m & 7
      else
        off[i] = (m / p.m_box) * p.m_pitch * p.kbox + (m % p.m_box);  // element offset at k = 0
    }
    // periodic FP64 flush of the FP32 accumulators (KW == 1: each output
    // entry of the CTA belongs to exactly one lane, so no race)
    double* const slab = (p.ctas_per_mtile == 1 ? p.out : p.partial) + (size_t(j) * v.I) * r;
    bool flushed = false;
    int since_flush = 0;
    auto flush_acc = [&]() {
#pragma unroll
      for (int i = 0; i < A; ++i) {
        const int m = lane_row(i);
        const long long row = (long long)mt * p.m_cta + m;
        if (m < p.m_cta && row < v.I) {
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const int c = cg * B + b;
            if (c < r) {
              double* q = slab + row * r + c;
              *q = flushed ? *q + double(acc[i][b]) : double(acc[i][b]);
            }
          }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) acc[i][b] = T(0);
      }
      flushed = true;
    };
    int s = 0;
    uint32_t phase = 0;
    long long cw_full = 0;
    const long long ct0 = prof_on ? clock64() : 0;
    if constexpr (MMA) {
      // ---- FP64 DMMA consumer. The warp's RW rows are NMF 8-row fragments,
      // the G*B columns NNF 8-column fragments; per 4-k step a lane loads one
      // T value per row fragment and one W value per column fragment for
      // NMF*NNF DMMAs (256 FMAs each): ~1/10 of the shared-memory operand
      // traffic per FMA of the register-blocked DFMA loop, which is bound by
      // that traffic (128 B/clk/SM against 64 DFMA/clk). ROW fragments take
      // rows with swizzle keys (m & 7) = 0,2,4,6 | 1,3,5,7 on the two
      // half-warps so the 16-byte chunks of a k pair never share banks.
      constexpr int RWc = RG * A;
      constexpr int NMF = RWc / 8;
      constexpr int NNF = (G * B + 7) / 8;
      static_assert(RWc % 8 == 0, "DMMA consumer needs 8-row fragments");
      const int g8 = lane >> 2, t4 = lane & 3;
      const int frow = LAY == kRow ? (((g8 & 3) << 1) | (g8 >> 2)) : g8;
      int wcol[NNF];
#pragma unroll
      for (int jn = 0; jn < NNF; ++jn) {
        const int c = 8 * jn + g8;
        wcol[jn] = c < G * B ? (c / B) * BP + c % B : 0;  // padded columns: any finite column, discarded
      }
      int moff[NMF];
#pragma unroll
      for (int f = 0; f < NMF; ++f) {
        const int m = mw * RWc + 8 * f + frow;
        moff[f] = LAY == kRow ? m : (m / p.m_box) * p.m_pitch * p.kbox + (m % p.m_box);
      }
      double dacc[NMF][NNF][2];
#pragma unroll
      for (int f = 0; f < NMF; ++f)
#pragma unroll
        for (int jn = 0; jn < NNF; ++jn) dacc[f][jn][0] = dacc[f][jn][1] = 0.0;
      const int ksteps = p.kbox / 4;
      for (long long u = u0; u < u1; ++u) {
        mbar_wait(&full[s], phase);
        const unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
        const double* wsd = reinterpret_cast<const double*>(w_base) + size_t(s) * (p.w_stage_bytes / sizeof(double));
        for (int ks = kw; ks < ksteps; ks += p.KW) {
          const int k = 4 * ks + t4;
          double bv[NNF];
#pragma unroll
          for (int jn = 0; jn < NNF; ++jn) bv[jn] = wsd[k * p.wld + wcol[jn]];
#pragma unroll
          for (int f = 0; f < NMF; ++f) {
            double av;
            if (LAY == kRow) {
              const int m = moff[f];
              av = *reinterpret_cast<const double*>(ts + m * 128 + ((((k >> 1) ^ m) & 7) << 4) + ((k & 1) << 3));
            } else {
              av = reinterpret_cast<const double*>(ts)[moff[f] + k * p.m_pitch];
            }
#pragma unroll
            for (int jn = 0; jn < NNF; ++jn) dmma_8x8x4(dacc[f][jn], av, bv[jn]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == stages) {
          s = 0;
          phase ^= 1;
        }
      }
      // fragments -> the (rg, cg) register layout of the epilogue, through a
      // per-warp scratch in the idle stage buffers (every consumer is past
      // its last stage read after the barrier; the host checks the size)
      constexpr int LDS = NNF * 8 + 1;
      asm volatile("bar.sync 1, %0;" ::"r"(n_consumers * 32) : "memory");
      double* scr = reinterpret_cast<double*>(smem) + size_t(cw) * RWc * LDS;
#pragma unroll
      for (int f = 0; f < NMF; ++f)
#pragma unroll
        for (int jn = 0; jn < NNF; ++jn) {
          scr[(8 * f + frow) * LDS + 8 * jn + 2 * t4] = dacc[f][jn][0];
          scr[(8 * f + frow) * LDS + 8 * jn + 2 * t4 + 1] = dacc[f][jn][1];
        }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < A; ++i)
#pragma unroll
        for (int b = 0; b < B; ++b) acc[i][b] = T(scr[(lane_row(i) - mw * RWc) * LDS + cg * B + b]);
    } else
    for (long long u = u0; u < u1; ++u) {
      {
        const long long t0 = prof_on ? clock64() : 0;
        mbar_wait(&full[s], phase);
        if (prof_on) cw_full += clock64() - t0;
      }
      const unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
      const T* ws = w_base + size_t(s) * (p.w_stage_bytes / sizeof(T)) + cg * BP;
      if (LAY == kRow) {
        constexpr int KCH = 128 / 16;  // 16-byte chunks per 128-byte row
        for (int pc = kw; pc < KCH; pc += p.KW) {
          // Shared-memory bandwidth (128 B/clk/SM, every lane receiving its
          // 16 or 8 bytes even on a broadcast) is the budget: per k a lane
          // reads B W values and A T values for A*B FMAs, so A and B are
          // large. A lane's 16-byte chunk of a row holds all VEC k of the
          // chunk: one read per row, then VEC rank-1 updates.
          T w[VEC][BP];
#pragma unroll
          for (int kk = 0; kk < VEC; ++kk)
#pragma unroll
            for (int q = 0; q < NV; ++q) {
              const V x = *reinterpret_cast<const V*>(ws + (pc * VEC + kk) * p.wld + q * VEC);
#pragma unroll
              for (int e = 0; e < VEC; ++e) w[kk][q * VEC + e] = VT::get(x, e);
            }
#pragma unroll
          for (int i = 0; i < A; ++i) {
            const int m = off[i];
            const V tv = *reinterpret_cast<const V*>(ts + m * 128 + (((pc ^ m) & 7) << 4));
#pragma unroll
            for (int kk = 0; kk < VEC; ++kk) {
              const T t = VT::get(tv, kk);
#pragma unroll
              for (int b = 0; b < B; ++b) acc[i][b] = fma(t, w[kk][b], acc[i][b]);
            }
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
            const V tv = *reinterpret_cast<const V*>(tt + off[i4 * VEC] + k * p.m_pitch);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const T t = VT::get(tv, e);
#pragma unroll
              for (int b = 0; b < B; ++b) acc[i4 * VEC + e][b] = fma(t, w[b], acc[i4 * VEC + e][b]);
            }
          }
#pragma unroll
          for (int i = AV; i < A; ++i) {
            const T t = tt[off[i] + k * p.m_pitch];
#pragma unroll
            for (int b = 0; b < B; ++b) acc[i][b] = fma(t, w[b], acc[i][b]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == stages) {
        s = 0;
        phase ^= 1;
      }
      if constexpr (sizeof(T) == 4) {  // FP32 only (FP64 sums need no flush)
        if (p.flush_units > 0 && ++since_flush == p.flush_units) {
          since_flush = 0;
          flush_acc();
        }
      }
    }

    if (prof_on && cw == 0 && lane == 0) {
      p.prof[blockIdx.x * kProfSlots + 3] = clock64() - ct0;
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      p.prof[blockIdx.x * kProfSlots + 7] = g;
      p.prof[blockIdx.x * kProfSlots + 4] = cw_full;
      p.prof[blockIdx.x * kProfSlots + 5] = u1 - u0;
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
          const int m = lane_row(i);
#pragma unroll
          for (int b = 0; b < B; ++b) red[m * ld + cg * B + b] = acc[i][b];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(n_consumers * 32) : "memory");
      if (kw == 0) {
#pragma unroll
        for (int i = 0; i < A; ++i) {
          const int m = lane_row(i);
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
        const int m = lane_row(i);
        const long long row = (long long)mt * p.m_cta + m;
        if (m < p.m_cta && row < v.I) {
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const int c = cg * B + b;
            if (c < r) {
              if (sizeof(T) == 4 && flushed)
                out[row * r + c] += double(acc[i][b]);
              else
                out[row * r + c] = double(acc[i][b]);
            }
          }
        }
      }
    }
    auto gstamp = [&](int slot) {
      if (prof_on && cw == 0 && lane == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        p.prof[blockIdx.x * kProfSlots + slot] = g;
      }
    };
    gstamp(8);
    if (p.counter) {
      // ---------------------------------------------- slab reduction
      // arrive once every slab row of this CTA is written; wait for all CTAs
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(n_consumers * 32) : "memory");
      if (cw == 0 && lane == 0) {
        // sense-reversing grid barrier: counter[0] arrivals, counter[1]
        // generation; the last arrival resets the count and bumps the
        // generation (any grid size per launch)
        unsigned gen;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(p.counter + 1) : "memory");
        const unsigned old = atomicAdd(p.counter, 1u);
        if (old == gridDim.x - 1) {
          p.counter[0] = 0u;
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.counter + 1), "r"(gen + 1u) : "memory");
        } else {
          unsigned seen;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.counter + 1) : "memory");
          } while (seen == gen);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(n_consumers * 32) : "memory");
      gstamp(9);
      // Eight lanes per output element: lane t of the octet adds slabs
      // t, t + 8, ... in order with all its loads in flight, then the octet
      // folds (xor 1, 2, 4). The order depends only on the slab count, so
      // the result is bit-reproducible; every lane of the CTA takes part.
      const long long n = v.I * r;
      const long long per = (n + gridDim.x - 1) / gridDim.x;
      const long long e0 = (long long)blockIdx.x * per;
      const long long e1 = e0 + per < n ? e0 + per : n;
      const int nsl = p.ctas_per_mtile;
      const int oct = (cw * 32 + lane) >> 3, t8 = lane & 7;
      const int n_oct = n_consumers * 4;
      for (long long eb = e0; eb < e1; eb += n_oct) {
        const long long e = eb + oct;
        const bool ok = e < e1;
        // up to 24 slabs per lane loaded in one round (148 slabs: 19)
        double x[24];
#pragma unroll
        for (int u = 0; u < 24; ++u) {
          const int q = t8 + 8 * u;
          x[u] = (ok && q < nsl) ? __ldcg(p.partial + (size_t(q) * n + e)) : 0.0;
        }
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int u = 0; u < 24; u += 4) {
          s0 += x[u];
          s1 += x[u + 1];
          s2 += x[u + 2];
          s3 += x[u + 3];
        }
        for (int q = t8 + 8 * 24; q < nsl; q += 8) s0 += ok ? __ldcg(p.partial + (size_t(q) * n + e)) : 0.0;
        double sum = (s0 + s1) + (s2 + s3);
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        if (ok && t8 == 0) p.out[e] = sum;
      }
      gstamp(10);
    }
  }
}

}  // namespace fast
}  // namespace ntfb
