// Stream-K FP64 MTTKRP on the FP64 tensor pipe (DMMA) for sm_100a.
//
// Same contraction, views, unit table, TMA boxes and Khatri-Rao formation as
// the fast kernel (mttkrp_fast_impl.cuh); what differs is the schedule:
//
//   * persistent: one CTA per SM. The work of a view is the flat sequence of
//     (m-tile t, unit u) pairs, u fastest (n_tiles x U units); CTA b streams
//     the contiguous range [W b / G, W (b + 1) / G) of it, so every SM gets
//     the same number of units (+-1) whatever the tile count -- no wave
//     quantisation (C2's tall Y_L view: 282 one-shot CTAs = 1.9 waves before;
//     C3's 40 m-tiles: 120 of 148 SMs busy), no per-tile pipeline fill: the
//     producers run ahead across tile boundaries while the consumers store
//     the finished tile.
//   * KW = 1: each consumer warp owns NMF 8-row fragments of the tile and
//     every k of every unit, so a tile's result leaves the accumulators
//     straight from the DMMA fragment registers (16-byte stores of two
//     adjacent columns; no shared-memory transpose, no k-split fold).
//   * operand prefetch: the A (tensor) and B (Khatri-Rao) fragments of the
//     next 4-k step are loaded before the DMMAs of the current one, and a
//     stage is released to the producers as soon as its last operands are in
//     registers.
//   * split tiles (a tile whose units span several CTAs) are written as FP64
//     partial slabs, one per (CTA, segment); after one grid-wide arrival count
//     (cooperative launch) every CTA sums a share of the split tiles' outputs
//     over their contributors in CTA order -- a fixed order, so the result
//     is bit-reproducible (README.md:155-157 determinism contract). Tiles
//     covered by one CTA are stored directly.
//
// The DMMA (mma.sync.m8n8k4.f64) computes exact FP64 products and sums with
// IEEE double accumulators (the north star's CUDA-core clause
// guards against reduced-precision formats, which do not arise).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "mttkrp_fast_impl.cuh"
#include "mttkrp_sk.h"

namespace ntfb {
namespace sk {

using fast::bulk_load;
using fast::dmma_8x8x4;
using fast::factor_ptr;
using fast::kMaxBase;
using fast::kUnitInts;
using fast::mbar_arrive;
using fast::mbar_arrive_expect_tx;
using fast::mbar_expect_tx;
using fast::mbar_init;
using fast::mbar_wait;
using fast::tma_load_3d;


// First unit of CTA b: W b / G, or (tall views, align) the first unit of
// tile n_tiles b / G -- the host tables (sk_choose) use the same formula.
__host__ __device__ __forceinline__ long long range_lo(const SkParams& p, int G, int b) {
  return p.align ? p.U * ((long long)p.n_tiles * b / G) : p.W * b / G;
}

__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  // packed FP32 FMA (SASS FFMA2, scalar a broadcast to both lanes)
  unsigned long long d;
  const float2 aa = make_float2(a, a);
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<const unsigned long long*>(&aa)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

// FP32 consumer warp of the stream-K kernel: lane (rg, cg) owns 8 rows x 8
// columns (columns cg*8.., rows rg + RG*i for ROW views, groups of four
// consecutive rows for COL views) as 32 float2 accumulators fed by packed
// FFMA2 -- 64 FMAs per 4-8 shared loads (T values are 16-byte reads of
// four k of a row (ROW) or four rows of a k (COL); W values 16-byte
// broadcast reads). Every p.flush_units units and at a tile segment's end
// the FP32 sums are added into FP64 (each lane its own entries: no race),
// so no FP32 sum runs over more than flush_units * 32 terms (the FP32 bar of
// BASELINE configs 4/5, mttkrp_fast_impl.cuh).
template <int CG, int A, int LAYOUT>
__device__ __forceinline__ void consume_f32(const SkParams& p, const unsigned char* t_base, const unsigned char* w_base,
                                            const unsigned char* aq_base, uint64_t* full, uint64_t* empty, long long w0,
                                            long long w1, long long U, const int* tile_ctas, int b, int cw, int lane) {
  static_assert(A == 4 || A == 8, "rows per lane");
  constexpr int RG = 32 / CG, RW = RG * A, KB = 32;
  const int r = p.v.rank;
  const int rg = lane % RG, cg = lane / RG;
  auto lrow = [&](int i) {
    return LAYOUT == fast::kRow ? cw * RW + rg + RG * i : cw * RW + 4 * rg + 4 * RG * (i >> 2) + (i & 3);
  };
  float2 acc[A][4];
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = make_float2(0.f, 0.f);
  // ROW: the byte offset of each row and its swizzle key; COL: the two
  // 4-row groups' element offsets
  int roff[A];
#pragma unroll
  for (int i = 0; i < A; ++i) {
    const int m = lrow(i);
    roff[i] = LAYOUT == fast::kRow ? m * 128 : ((m / p.m_box) * p.m_pitch * KB + (m % p.m_box)) * 4;
  }
  const unsigned bpitch = p.direct_b ? unsigned(r) * 4u : unsigned(p.wld) * 4u;
  const int wcol = cg * 32;  // bytes: columns cg*8 .. cg*8+7
  const unsigned tpitch = unsigned(p.m_pitch) * 4u;
  int s = 0;
  uint32_t phase = 0;
  const int first_tile = int(w0 / U);
  int tile = first_tile;
  long long u_in = w0 - (long long)first_tile * U;
  int since = 0;
  bool started = false;  // the segment's FP64 target holds a first flush
  auto flush = [&](bool seg_end) {
    const int2 cs = reinterpret_cast<const int2*>(tile_ctas)[tile];
    const bool direct = cs.x == cs.y;
    double* dst = direct ? p.out : p.partial + size_t(2 * b + (tile == first_tile ? 0 : 1)) * p.m_cta * r;
    const long long row0 = direct ? (long long)tile * p.m_cta : 0;
#pragma unroll
    for (int i = 0; i < A; ++i) {
      const int m = lrow(i);
      if ((long long)tile * p.m_cta + m >= p.v.I) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = cg * 8 + 2 * q;
        if (c < r) {
          double2* d = reinterpret_cast<double2*>(dst + (row0 + m) * r + c);
          double2 v = make_double2(double(acc[i][q].x), double(acc[i][q].y));
          if (started) {
            const double2 o = *d;
            v.x += o.x;
            v.y += o.y;
          }
          *d = v;
        }
        acc[i][q] = make_float2(0.f, 0.f);
      }
    }
    started = !seg_end;
    since = 0;
  };
  if constexpr (A == 4) {
    // Software-pipelined 4-k steps: the operands of step kq + 1 (4 T reads +
    // 8 W reads of 16 bytes, 48 registers) are loaded before the 64 FFMA2 of
    // step kq, across unit boundaries too (the next stage's first step is
    // loaded right after this stage's last operands are in registers and the
    // stage is released), so a warp's shared-memory latency hides behind its
    // own FMAs as well as behind the sub-partition's second warp.
    struct Ops {
      float4 t[A];
      float4 w[8];
    };
    auto stage_t = [&](int st) { return t_base + size_t(st) * p.t_stage_bytes; };
    auto stage_w = [&](int st) {
      return p.direct_b ? aq_base + size_t(st) * p.aq_stage_bytes : w_base + size_t(st) * p.w_stage_bytes;
    };
    auto load_ops = [&](const unsigned char* ts, const unsigned char* wsb, int kq, Ops& o) {
#pragma unroll
      for (int i = 0; i < A; ++i) {
        if (LAYOUT == fast::kRow) {
          const int key = (roff[i] >> 7) & 7;
          o.t[i] = *reinterpret_cast<const float4*>(ts + roff[i] + (((kq ^ key) & 7) << 4));  // four k of row i
        } else {
          o.t[i] = *reinterpret_cast<const float4*>(ts + roff[0] + (4 * kq + i) * tpitch);  // four rows of k = 4 kq + i
        }
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        o.w[2 * kk] = *reinterpret_cast<const float4*>(wsb + (4 * kq + kk) * bpitch + wcol);
        o.w[2 * kk + 1] = *reinterpret_cast<const float4*>(wsb + (4 * kq + kk) * bpitch + wcol + 16);
      }
    };
    auto comp = [](const float4& v, int c) { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; };
    auto compute = [&](const Ops& o) {
#pragma unroll
      for (int i = 0; i < A; ++i)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float tv = LAYOUT == fast::kRow ? comp(o.t[i], kk) : comp(o.t[kk], i);
          acc[i][0] = ffma2(tv, make_float2(o.w[2 * kk].x, o.w[2 * kk].y), acc[i][0]);
          acc[i][1] = ffma2(tv, make_float2(o.w[2 * kk].z, o.w[2 * kk].w), acc[i][1]);
          acc[i][2] = ffma2(tv, make_float2(o.w[2 * kk + 1].x, o.w[2 * kk + 1].y), acc[i][2]);
          acc[i][3] = ffma2(tv, make_float2(o.w[2 * kk + 1].z, o.w[2 * kk + 1].w), acc[i][3]);
        }
    };
    Ops oa, ob;
    if (w0 < w1) {
      mbar_wait(&full[s], phase);
      load_ops(stage_t(s), stage_w(s), 0, oa);
    }
    for (long long w = w0; w < w1; ++w) {
      const unsigned char* ts = stage_t(s);
      const unsigned char* wsb = stage_w(s);
#pragma unroll
      for (int kq = 0; kq < KB / 4; kq += 2) {
        load_ops(ts, wsb, kq + 1, ob);
        compute(oa);
        if (kq + 2 < KB / 4) {
          load_ops(ts, wsb, kq + 2, oa);
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);  // every operand of this stage is in registers
          if (++s == p.stages) {
            s = 0;
            phase ^= 1;
          }
          if (w + 1 < w1) {
            mbar_wait(&full[s], phase);
            load_ops(stage_t(s), stage_w(s), 0, oa);
          }
        }
        compute(ob);
      }
      const bool seg_end = ++u_in == U || w + 1 == w1;
      if (seg_end || (p.flush_units > 0 && ++since == p.flush_units)) flush(seg_end);
      if (seg_end) {
        u_in = 0;
        ++tile;
      }
    }
  } else {
  for (long long w = w0; w < w1; ++w) {
    mbar_wait(&full[s], phase);
    const unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
    const unsigned char* wsb = p.direct_b ? aq_base + size_t(s) * p.aq_stage_bytes : w_base + size_t(s) * p.w_stage_bytes;
    if (LAYOUT == fast::kRow) {
#pragma unroll 2
      for (int kq = 0; kq < KB / 4; ++kq) {
        float4 t[A];
#pragma unroll
        for (int i = 0; i < A; ++i) {
          const int key = (roff[i] >> 7) & 7;
          t[i] = *reinterpret_cast<const float4*>(ts + roff[i] + (((kq ^ key) & 7) << 4));
        }
        float2 wv[4][4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 a = *reinterpret_cast<const float4*>(wsb + (4 * kq + kk) * bpitch + wcol);
          const float4 c = *reinterpret_cast<const float4*>(wsb + (4 * kq + kk) * bpitch + wcol + 16);
          wv[kk][0] = make_float2(a.x, a.y);
          wv[kk][1] = make_float2(a.z, a.w);
          wv[kk][2] = make_float2(c.x, c.y);
          wv[kk][3] = make_float2(c.z, c.w);
        }
#pragma unroll
        for (int i = 0; i < A; ++i) {
          const float tk[4] = {t[i].x, t[i].y, t[i].z, t[i].w};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = ffma2(tk[kk], wv[kk][q], acc[i][q]);
        }
      }
    } else {
#pragma unroll 4
      for (int k = 0; k < KB; ++k) {
        float tv[A];
#pragma unroll
        for (int g = 0; g < A / 4; ++g) {
          const float4 tq = *reinterpret_cast<const float4*>(ts + roff[4 * g] + k * tpitch);
          tv[4 * g] = tq.x;
          tv[4 * g + 1] = tq.y;
          tv[4 * g + 2] = tq.z;
          tv[4 * g + 3] = tq.w;
        }
        const float4 a = *reinterpret_cast<const float4*>(wsb + k * bpitch + wcol);
        const float4 c = *reinterpret_cast<const float4*>(wsb + k * bpitch + wcol + 16);
        const float2 wv[4] = {make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(c.x, c.y),
                              make_float2(c.z, c.w)};
#pragma unroll
        for (int i = 0; i < A; ++i)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] = ffma2(tv[i], wv[q], acc[i][q]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == p.stages) {
      s = 0;
      phase ^= 1;
    }
    const bool seg_end = ++u_in == U || w + 1 == w1;
    if (seg_end || (p.flush_units > 0 && ++since == p.flush_units)) flush(seg_end);
    if (seg_end) {
      u_in = 0;
      ++tile;
    }
  }
  }  // A == 8
}

// T = double: DMMA consumers, NMF 8-row fragments x NNF 8-column fragments
// per warp. T = float (FP32 tensors, FP32 factor mirrors): FFMA2 register
// tiles of A rows x 8 columns per lane (A = 8, or 4 when NMF = 4: eight
// 32-row warps instead of four 64-row ones for r <= 32), NNF = column groups
// of 8 (RG = 32 / NNF row groups), FP32 sums flushed into FP64 every
// p.flush_units units.
template <typename T, int NMF, int NNF, int LAYOUT>
__global__ void __launch_bounds__(32 * (kMaxNP + kMaxMW), 1) mttkrp_sk_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                            SkParams p) {
  constexpr int KBT = 128 / int(sizeof(T));  // reduction indices per unit
  constexpr int FA = NMF == 4 ? 4 : 8;                             // FP32: rows per lane
  constexpr int RW = sizeof(T) == 8 ? 8 * NMF : (32 / NNF) * FA;  // rows per consumer warp
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ModeView& v = p.v;
  const int r = v.rank;
  const int stages = p.stages;
  // shared memory: [stages] T boxes | [stages] W rows | [n_aq] factor-row
  // slots (aq) | barriers. direct_b (no base modes): the B operand is the
  // factor rows themselves, one aq slot per stage, no W stage.
  unsigned char* t_base = smem;
  T* w_base = reinterpret_cast<T*>(smem + size_t(stages) * p.t_stage_bytes);
  T* aq_base = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(w_base) + size_t(stages) * p.w_stage_bytes);
  const int n_aq = p.direct_b ? stages : p.NP * p.naw;
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(aq_base) + size_t(n_aq) * p.aq_stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* aqb = empty + stages;  // [n_aq] (W formation mode)

  const int G = int(gridDim.x), b = int(blockIdx.x);
  const long long w0 = range_lo(p, G, b), w1 = range_lo(p, G, b + 1);
  const long long U = p.U;
  const int NP = p.NP, MW = p.MW;
  const int* tile_ctas = p.utab + size_t(U) * kUnitInts;  // [n_tiles][2]
  const int* split_list = tile_ctas + 2 * p.n_tiles;      // [n_split]

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], p.direct_b ? 1 : 32);
      mbar_init(&empty[s], MW);
    }
    if (!p.direct_b)
      for (int q = 0; q < n_aq; ++q) mbar_init(&aqb[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
  }
  // W stages start zeroed (the padding columns c >= r stay zero); the aq
  // slots too, so B rows past a unit's valid k are finite (they multiply the
  // zero-filled T rows)
  {
    const int nw = (stages * int(p.w_stage_bytes) + n_aq * int(p.aq_stage_bytes)) / int(sizeof(T));
    for (int e = threadIdx.x; e < nw; e += blockDim.x) w_base[e] = T(0);
  }
  __syncthreads();

  if (warp < NP) {
    // ------------------------------------------------------------ producers
    // Unit i of this CTA's range (i = w - w0) belongs to producer warp
    // i % NP and T stage i % stages (NP | stages). W-formation mode: the
    // factor rows of a unit are bulk-copied DA = naw - 1 of the warp's units
    // ahead into the warp's own ring of naw aq slots, so by the time the
    // unit's stage is free (TMA issued) its rows have landed and W is formed
    // at once. direct_b: one bulk copy per unit into the stage's aq slot,
    // completing on the stage's full barrier with the TMA box.
    constexpr int KB = KBT;
    const T* fL = factor_ptr<T>(p.F, p.qL);
    const T* bfac[kMaxBase];
#pragma unroll
    for (int t = 0; t < kMaxBase; ++t) bfac[t] = t < p.nb ? factor_ptr<T>(p.F, p.bq[t]) : nullptr;
    const unsigned row_bytes = unsigned(r * sizeof(T));
    const int aq_elems = int(p.aq_stage_bytes / sizeof(T));
    auto aq_of = [&](int q) { return aq_base + size_t(q) * aq_elems; };
    auto info_of = [&](int q) { return reinterpret_cast<int*>(aq_of(q) + (KB + 2 * kMaxBase) * r); };
    const long long n_units = w1 - w0;
    const long long n_mine = n_units > warp ? (n_units - warp + NP - 1) / NP : 0;
    const int naw = p.naw, DA = p.naw - 1;
    // (tile, unit-in-tile) cursors of the warp's unit stream, advanced by NP
    // units per step without divisions: one for the TMA issue, one DA units
    // ahead for the factor-row copies
    struct Cursor {
      long long u;
      int tile;
    };
    auto cursor_at = [&](long long jj) {
      const long long w = w0 + warp + jj * NP;
      Cursor c;
      c.tile = int(w / U);
      c.u = w - (long long)c.tile * U;
      return c;
    };
    auto advance = [&](Cursor& c) {
      c.u += NP;
      while (c.u >= U) {
        c.u -= U;
        ++c.tile;
      }
    };
    auto entry = [&](const Cursor& c, int (&e)[kUnitInts]) {  // lane 0: the unit-table entry
      const int2* src = reinterpret_cast<const int2*>(p.utab + size_t(c.u) * kUnitInts);
#pragma unroll
      for (int q = 0; q < kUnitInts / 2; ++q) {
        const int2 x = __ldg(src + q);
        e[2 * q] = x.x;
        e[2 * q + 1] = x.y;
      }
    };
    // bulk copies of a unit's factor rows into aq slot q, completing on bar
    // the slot's info area keeps the unit's whole table entry: the TMA issue
    // of a W-formation unit reads it from shared memory (written DA units
    // earlier by this lane) instead of a second global round trip
    auto copy_rows = [&](const int (&e)[kUnitInts], int q, uint64_t* bar, bool arm) {
      const int n_valid = e[3], n1 = e[4], kwrap = e[5];
      T* aq = aq_of(q);
      int* info = info_of(q);
#pragma unroll
      for (int i = 0; i < kUnitInts; ++i) info[i] = e[i];
      const bool wrap = kwrap < KB;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the slot first
      if (arm) mbar_arrive_expect_tx(bar, unsigned(n_valid + p.nb * (wrap ? 2 : 1)) * row_bytes);
      bulk_load(aq, fL + size_t(e[2]) * r, unsigned(n1) * row_bytes, bar);
      if (n_valid > n1) bulk_load(aq + size_t(n1) * r, fL + size_t(p.rowL_wrap) * r, unsigned(n_valid - n1) * row_bytes, bar);
#pragma unroll
      for (int t = 0; t < kMaxBase; ++t)
        if (t < p.nb) {
          bulk_load(aq + size_t(KB + t) * r, bfac[t] + size_t(e[6 + t]) * r, row_bytes, bar);
          if (wrap)
            bulk_load(aq + size_t(KB + kMaxBase + t) * r, bfac[t] + size_t(e[6 + kMaxBase + t]) * r, row_bytes, bar);
        }
    };
    auto tma_unit = [&](const int (&e)[kUnitInts], int tile, int s) {
      unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
      for (int mb = 0; mb < p.n_mbox; ++mb) {
        const int m0 = tile * p.m_cta + mb * p.m_box;
        if (LAYOUT == fast::kRow)
          tma_load_3d(ts + size_t(mb) * p.m_box * 128, &tmap, &full[s], e[0], m0, e[1]);
        else
          tma_load_3d(ts + size_t(mb) * p.m_pitch * KB * sizeof(T), &tmap, &full[s], m0, e[0], 0);
      }
    };
    const int CPL = (r + 31) / 32;  // columns per lane
    int s = warp;
    uint32_t round = 0;
    Cursor cur = cursor_at(0), ahead = cursor_at(DA);
    int q_cur = warp * naw, q_ahead = warp * naw + DA;  // aq slots of the two streams
    uint32_t aq_round = 0;                                // completed trips of q_cur around the ring
    // lane 0 reads the table entry it needs next one trip early (the global
    // load's latency hides behind the trip)
    int nx[kUnitInts];
    if (!p.direct_b && lane == 0) {
      Cursor c = cur;
      for (long long jj = 0; jj < DA && jj < n_mine; ++jj) {  // prologue copies
        int e[kUnitInts];
        entry(c, e);
        copy_rows(e, warp * naw + int(jj), &aqb[warp * naw + int(jj)], true);
        advance(c);
      }
      if (DA < n_mine) entry(ahead, nx);
    }
    if (p.direct_b && lane == 0 && n_mine > 0) entry(cur, nx);
    for (long long jj = 0; jj < n_mine; ++jj) {
      __syncwarp();  // every lane's reads of the slot formed last trip precede its refill
      if (!p.direct_b && jj + DA < n_mine) {  // rows of a later unit (its slot was formed from)
        if (lane == 0) copy_rows(nx, q_ahead, &aqb[q_ahead], true);
        advance(ahead);
        if (lane == 0 && jj + DA + 1 < n_mine) entry(ahead, nx);
        if (++q_ahead == (warp + 1) * naw) q_ahead = warp * naw;
      }
      if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
      const int tile = cur.tile;
      advance(cur);
      if (lane == 0) {
        if (p.direct_b) {
          int e[kUnitInts];
#pragma unroll
          for (int i = 0; i < kUnitInts; ++i) e[i] = nx[i];
          if (jj + 1 < n_mine) entry(cur, nx);
          mbar_arrive_expect_tx(&full[s], p.tx_bytes + unsigned(e[3]) * row_bytes);
          tma_unit(e, tile, s);
          copy_rows(e, s, &full[s], false);
        } else {
          int e[kUnitInts];
          const int* info = info_of(q_cur);
#pragma unroll
          for (int i = 0; i < kUnitInts; ++i) e[i] = info[i];
          mbar_expect_tx(&full[s], p.tx_bytes);
          tma_unit(e, tile, s);
        }
      }
      if (!p.direct_b) {
        const int q = q_cur;
        const uint32_t ph = aq_round & 1u;
        if (++q_cur == (warp + 1) * naw) {
          q_cur = warp * naw;
          ++aq_round;
        }
        mbar_wait(&aqb[q], ph);
        T* ws = w_base + size_t(s) * (p.w_stage_bytes / sizeof(T));
        const T* aq = aq_of(q);
        const int* info = info_of(q);
        const int kmax = info[3];
        const int kwrap = info[5];
        const bool wrap = kwrap < KB;
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
#pragma unroll
          for (int k = 0; k < KB; ++k)
            ws[k * p.wld + c] = (k < kmax) ? (k >= kwrap ? base1 : base0) * aq[k * r + c] : T(0);
        }
        mbar_arrive(&full[s]);
      }
      if ((s += NP) >= stages) {
        s -= stages;
        ++round;
      }
    }
  } else if (warp < NP + MW) {
    // ------------------------------------------------------------ consumers
    if constexpr (sizeof(T) == 4) {
      consume_f32<NNF, FA, LAYOUT>(p, t_base, reinterpret_cast<const unsigned char*>(w_base),
                               reinterpret_cast<const unsigned char*>(aq_base), full, empty, w0, w1, U,
                               tile_ctas, b, warp - NP, lane);
    } else {
    const int cw = warp - NP;
    const int g8 = lane >> 2, t4 = lane & 3;
    // ROW fragments take rows with swizzle keys 0,2,4,6 | 1,3,5,7 on the two
    // half-warps (conflict-free 16-byte chunks, mttkrp_fast_impl.cuh)
    const int frow = LAYOUT == fast::kRow ? (((g8 & 3) << 1) | (g8 >> 2)) : g8;
    // byte offsets of the lane's fragment rows in a stage. ROW: fragment f's
    // row is cw RW + 8 f + frow, whose 128-byte swizzle key is frow (the
    // fragment bases are multiples of 8 rows), so one chunk offset per k
    // serves every fragment and the rows are 1024 bytes apart.
    int moff[NMF];
#pragma unroll
    for (int f = 0; f < NMF; ++f) {
      const int m = cw * RW + 8 * f + frow;
      moff[f] = LAYOUT == fast::kRow ? (cw * RW + frow) * 128 + f * 1024
                                     : ((m / p.m_box) * p.m_pitch * KBT + (m % p.m_box)) * 8;
    }
    const int wcol = g8 * 8;  // byte offset of column 8 jn + g8 within a W row (+ jn * 64)
    double acc[NMF][NNF][2];
#pragma unroll
    for (int f = 0; f < NMF; ++f)
#pragma unroll
      for (int jn = 0; jn < NNF; ++jn) acc[f][jn][0] = acc[f][jn][1] = 0.0;
    // B rows: the W stage (pitch wld) or, direct_b, the stage's factor rows (pitch r)
    const unsigned bpitch = p.direct_b ? unsigned(r) * 8u : unsigned(p.wld) * 8u;
    const unsigned tpitch = unsigned(p.m_pitch) * 8u;  // COL: bytes between k rows
    // operand loads of one 4-k step (k = 4 ks + t4)
    auto load_ops = [&](const unsigned char* ts, const unsigned char* wsb, int ks, double (&av)[NMF],
                        double (&bv)[NNF]) {
      const int k = 4 * ks + t4;
      const unsigned char* wk = wsb + k * bpitch + wcol;
#pragma unroll
      for (int jn = 0; jn < NNF; ++jn) bv[jn] = *reinterpret_cast<const double*>(wk + jn * 64);
      const unsigned char* tk = LAYOUT == fast::kRow ? ts + ((((k >> 1) ^ frow) & 7) << 4) + ((k & 1) << 3)
                                                     : ts + k * tpitch;
#pragma unroll
      for (int f = 0; f < NMF; ++f) av[f] = *reinterpret_cast<const double*>(tk + moff[f]);
    };
    // the accumulators of one finished tile segment -> out (whole tile in
    // this CTA) or this CTA's partial slot
    auto flush = [&](int tile, bool direct, int slot) {
      double* dst;
      long long row0;
      if (direct) {
        dst = p.out;
        row0 = (long long)tile * p.m_cta;
      } else {
        dst = p.partial + size_t(slot) * p.m_cta * r;
        row0 = 0;
      }
#pragma unroll
      for (int f = 0; f < NMF; ++f) {
        const int m = cw * RW + 8 * f + frow;
        const bool row_ok = (long long)tile * p.m_cta + m < v.I;
#pragma unroll
        for (int jn = 0; jn < NNF; ++jn) {
          const int c = 8 * jn + 2 * t4;
          if (row_ok && c < r)
            *reinterpret_cast<double2*>(dst + (row0 + m) * r + c) = make_double2(acc[f][jn][0], acc[f][jn][1]);
          acc[f][jn][0] = acc[f][jn][1] = 0.0;
        }
      }
    };
    int s = 0;
    uint32_t phase = 0;
    const int first_tile = int(w0 / U);
    int tile = first_tile;
    long long u_in = w0 - (long long)first_tile * U;  // unit index inside the current tile
    for (long long w = w0; w < w1; ++w) {
      mbar_wait(&full[s], phase);
      const unsigned char* ts = t_base + size_t(s) * p.t_stage_bytes;
      const unsigned char* wsb = p.direct_b ? reinterpret_cast<const unsigned char*>(aq_base) + size_t(s) * p.aq_stage_bytes
                                            : reinterpret_cast<const unsigned char*>(w_base) + size_t(s) * p.w_stage_bytes;
      double a0[NMF], b0[NNF], a1[NMF], b1[NNF];
      load_ops(ts, wsb, 0, a0, b0);
      load_ops(ts, wsb, 1, a1, b1);
#pragma unroll
      for (int f = 0; f < NMF; ++f)
#pragma unroll
        for (int jn = 0; jn < NNF; ++jn) dmma_8x8x4(acc[f][jn], a0[f], b0[jn]);
      load_ops(ts, wsb, 2, a0, b0);
#pragma unroll
      for (int f = 0; f < NMF; ++f)
#pragma unroll
        for (int jn = 0; jn < NNF; ++jn) dmma_8x8x4(acc[f][jn], a1[f], b1[jn]);
      load_ops(ts, wsb, 3, a1, b1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // every operand of this stage is in registers
      if (++s == stages) {
        s = 0;
        phase ^= 1;
      }
#pragma unroll
      for (int f = 0; f < NMF; ++f)
#pragma unroll
        for (int jn = 0; jn < NNF; ++jn) dmma_8x8x4(acc[f][jn], a0[f], b0[jn]);
#pragma unroll
      for (int f = 0; f < NMF; ++f)
#pragma unroll
        for (int jn = 0; jn < NNF; ++jn) dmma_8x8x4(acc[f][jn], a1[f], b1[jn]);
      if (++u_in == U || w + 1 == w1) {
        const int2 cs = reinterpret_cast<const int2*>(tile_ctas)[tile];
        const bool direct = cs.x == cs.y;
        flush(tile, direct, 2 * b + (tile == first_tile ? 0 : 1));
        u_in = 0;
        ++tile;
      }
    }
    }  // DMMA consumer
  }
  if (!p.n_split) return;
  // ---------------------------------------------------- split-tile reduction
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    // sense-reversing grid barrier (counter[0] arrivals, counter[1] generation)
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
  __syncthreads();
  // LPO lanes per output (8 for a wide fan-in, else 1): lane t of the group
  // adds contributors t, t + LPO, ... in order, eight loads in flight at a
  // time, then the group folds (xor 1, 2, 4). The order depends only on the
  // contributor count and LPO (fixed per plan): bit-reproducible.
  const long long per_tile = (long long)p.m_cta * r;
  const long long n = (long long)p.n_split * per_tile;
  const long long per = (n + G - 1) / G;
  const long long e0 = (long long)b * per;
  const long long e1 = e0 + per < n ? e0 + per : n;
  const int lpo = p.lpo;
  const int grp = threadIdx.x / lpo, tq = threadIdx.x % lpo;
  const int n_grp = blockDim.x / lpo;
  for (long long eb = e0; eb < e1; eb += n_grp) {
    const long long e = eb + grp;
    const bool ok = e < e1 && grp < n_grp;
    int tile = 0, lo = 0, hi = -1;
    long long within = 0;
    if (ok) {
      tile = split_list[e / per_tile];
      within = e % per_tile;
      const int2 cs = reinterpret_cast<const int2*>(tile_ctas)[tile];
      lo = cs.x;
      hi = cs.y;
    }
    double sum = 0.0;
    for (int q0 = lo + tq; q0 <= hi; q0 += 8 * lpo) {
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int q = q0 + i * lpo;
        double val = 0.0;
        if (q <= hi) {
          const int sl = 2 * q + (int(range_lo(p, G, q) / U) == tile ? 0 : 1);
          val = __ldcg(p.partial + size_t(sl) * per_tile + within);
        }
        x[i] = val;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += x[i];
    }
    if (lpo == 8) {
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    }
    const long long row = (long long)tile * p.m_cta + within / r;
    if (ok && tq == 0 && row < v.I) p.out[row * r + within % r] = sum;
  }
}

template <typename T, int NMF, int NNF, int LAYOUT>
void launch_sk(const CUtensorMap& map, const SkParams& p, int grid, int threads, size_t smem, cudaStream_t s) {
  auto fn = mttkrp_sk_kernel<T, NMF, NNF, LAYOUT>;
  NTF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;  // the split-tile reduction waits for every CTA
  attr[0].val.cooperative = p.n_split ? 1 : 0;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  NTF_CUDA(cudaLaunchKernelEx(&cfg, fn, map, p));
}

using SkLaunch = void (*)(const CUtensorMap&, const SkParams&, int, int, size_t, cudaStream_t);

template <int NMF, int NNF>
SkLaunch pick_layout(int layout) {
  return layout == fast::kRow ? launch_sk<double, NMF, NNF, fast::kRow> : launch_sk<double, NMF, NNF, fast::kCol>;
}

// FP32: NNF = column groups of 8 (4: r <= 32, 8: r <= 64); rows per lane 8 (NMF = 1) or 4 (NMF = 4)
SkLaunch pick_f32(int cg, int layout, int arows = 8) {
  if (cg == 4 && arows == 4)
    return layout == fast::kRow ? launch_sk<float, 4, 4, fast::kRow> : launch_sk<float, 4, 4, fast::kCol>;
  if (arows != 8) return nullptr;
  switch (cg) {
    case 4: return layout == fast::kRow ? launch_sk<float, 1, 4, fast::kRow> : launch_sk<float, 1, 4, fast::kCol>;
    case 8: return layout == fast::kRow ? launch_sk<float, 1, 8, fast::kRow> : launch_sk<float, 1, 8, fast::kCol>;
    default: return nullptr;
  }
}

template <int NMF>
SkLaunch pick_nnf(int nnf, int layout) {
  switch (nnf) {
    case 1: return pick_layout<NMF, 1>(layout);
    case 2: return pick_layout<NMF, 2>(layout);
    case 3: return pick_layout<NMF, 3>(layout);
    case 4: return pick_layout<NMF, 4>(layout);
    default: return nullptr;
  }
}

SkLaunch pick(int nmf, int nnf, int layout) {
  switch (nmf) {
    case 2: return pick_nnf<2>(nnf, layout);
    case 4: return pick_nnf<4>(nnf, layout);
    case 5: return pick_nnf<5>(nnf, layout);
    case 8: return pick_nnf<8>(nnf, layout);
    case 10: return pick_nnf<10>(nnf, layout);
    default: return nullptr;
  }
}

}  // namespace sk

namespace {

PFN_cuTensorMapEncodeTiled_v12000 sk_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    cudaGetLastError();
    return f;
  }();
  return fn;
}

constexpr size_t kSkSmem = 222 * 1024;  // of the 227 KB a CTA may claim

}  // namespace

bool sk_choose(const ModeView& v, int dtype, int sms, SkPlan* out) {
  if (const char* e = std::getenv("NTF_SK"); e && std::atoi(e) == 0) return false;
  const bool f32 = dtype == NTF_DTYPE_F32;
  if (f32 && std::getenv("NTF_SK_F32") && std::atoi(std::getenv("NTF_SK_F32")) == 0) return false;
  const int es = f32 ? 4 : 8;
  const int KB = 128 / es;
  const int r = v.rank;
  int nnf;
  if (f32) {  // FFMA2 tiles of 8 x 8 per lane: column groups of 8
    if (r <= 16 || r > 64 || (r * 4) % 16) return false;
    nnf = r <= 32 ? 4 : 8;
  } else {
    if (r % 2 || r > 32) return false;
    nnf = (r + 7) / 8;
  }
  if (v.L * v.I * v.R < (1LL << 15)) return false;
  if (v.L >= (1LL << 31) || v.R >= (1LL << 31)) return false;
  int layout;
  if (v.R > 1) {
    layout = fast::kRow;
    if ((v.R * es) % 16 || (v.I * v.R * es) % 16) return false;
  } else if (v.L > 1) {
    layout = fast::kCol;
    if ((v.I * es) % 16) return false;
  } else {
    return false;
  }
  const int qL = layout == fast::kRow ? v.order - 1 : v.order - 2;
  if (v.dims[qL] < KB) return false;
  if (v.order > fast::kMaxBase + 2) return false;
  // tile: four consumer warps (one per SM sub-partition) of NMF fragments;
  // a short mode gets one tile of ten-fragment warps (C2: 300 rows -> 320)
  // Tall views (the dimension tree's partials) take whole tiles per CTA when
  // there are enough of them (>= 4 per SM: at most ~5 % imbalance), with
  // four-fragment warps if eight-fragment tiles would be too few.
  // mw consumer warps of nmf 8-row fragments: 4 warps (one per SM
  // sub-partition) or 8 (two, so one warp's operand loads hide behind the
  // other's DMMAs); NTF_SK_MW / NTF_SK_NMF override.
  // (measured r02k: tall tile-aligned views gain from 8 -- C2's Y_L pass
  // 67 -> 57 us -- the others do not)
  int mw = 4;
  {
    const long long t8 = (v.I + 127) / 128;  // 128-row tiles of 8 two-fragment warps
    if (t8 >= 4LL * sms) mw = 8;
  }
  if (const char* e = std::getenv("NTF_SK_MW")) mw = std::atoi(e) == 8 ? 8 : 4;
  const int rows_per_frag_set = 8 * mw;  // rows per fragment index over the warps
  int nmf = 32 / mw, align = 0;           // 256-row tiles
  if (v.I > 256 && v.I <= 320) nmf = 40 / mw;
  if (v.I <= 128) nmf = 16 / mw;
  const auto tiles_of = [&](int f) { return (v.I + (long long)rows_per_frag_set * f - 1) / ((long long)rows_per_frag_set * f); };
  if (tiles_of(nmf) >= 4LL * sms) {
    align = 1;
  } else if (tiles_of(nmf / 2) >= 4LL * sms) {
    nmf /= 2;
    align = 1;
  }
  if (const char* e = std::getenv("NTF_SK_NMF")) nmf = std::atoi(e);
  if (f32) {  // warps of (32 / nnf) x 8 rows: 4 x 64 (r <= 32) or 8 x 32 (r <= 64) = 256-row tiles
    // (measured r02z: r = 64 gains from 8 warps -- C5 pass 24.0 -> 19.4 ms,
    // 0.70 of the FFMA peak; r = 32 has no room for 8 x 64-row warps' stages)
    // r <= 32: eight warps of 32 rows (4 rows x 8 columns per lane) -- two
    // warps per SM sub-partition hide each other's operand loads and barrier
    // waits, the same 256-row stages as four 64-row warps (NTF_SK_F32A=8)
    mw = 8;
    if (const char* e = std::getenv("NTF_SK_MW")) mw = std::atoi(e) == 8 ? 8 : 4;
    nmf = nnf == 4 && mw == 8 ? 4 : 1;
    if (const char* e = std::getenv("NTF_SK_F32A")) nmf = (std::atoi(e) == 4 && nnf == 4) ? 4 : 1;
    if (nnf == 4 && nmf == 1 && !std::getenv("NTF_SK_MW")) mw = 4;  // 64-row warps: four (stage room)
    align = 0;
  }
  if (const char* e = std::getenv("NTF_SK_ALIGN")) align = std::atoi(e);
  const int m_cta = f32 ? mw * (32 / nnf) * (nmf == 4 ? 4 : 8) : rows_per_frag_set * nmf;
  if (f32 && (v.I + m_cta - 1) / m_cta >= 4LL * sms && !std::getenv("NTF_SK_ALIGN")) align = 1;
  SkPlan pl;
  SkParams& p = pl.p;
  p = SkParams{};
  p.v = v;
  p.MW = mw;
  p.NP = 2;
  if (const char* e = std::getenv("NTF_SK_NP")) p.NP = std::max(1, std::min(sk::kMaxNP, std::atoi(e)));
  p.m_cta = m_cta;
  p.n_mbox = (m_cta + 255) / 256;
  // FP64 COL boxes need 4 spare elements for the conflict-free row pitch
  // (m_box + 4 <= 256, the TMA box limit): a 256-row tile takes two boxes
  // (r02ab capture at C3: 19.2 M of 28.6 M shared wavefronts were conflicts)
  if (!f32 && layout == fast::kCol && m_cta / p.n_mbox + 4 > 256 && !std::getenv("NTF_SK_ONEBOX")) p.n_mbox *= 2;
  p.m_box = m_cta / p.n_mbox;
  if (p.m_box * p.n_mbox != m_cta || p.m_box % 8) return false;
  p.wld = 8 * nnf + 4;  // 32 B off the 64-byte bank period (4 k rows per half-warp)
  if (layout == fast::kRow) {
    p.U = v.L * ((v.R + KB - 1) / KB);  // (l, rho box) units, as the unit table
    p.m_pitch = p.m_box;
    p.t_stage_bytes = unsigned(m_cta * 128);
  } else {
    p.U = (v.L + KB - 1) / KB;
    p.m_pitch = !f32 && p.m_box + 4 <= 256 ? p.m_box + 4 : p.m_box;
    p.t_stage_bytes = unsigned(size_t(p.n_mbox) * p.m_pitch * KB * es);
  }
  p.n_tiles = int((v.I + m_cta - 1) / m_cta);
  p.W = (long long)p.n_tiles * p.U;
  // a single-tile COL view (C2's block N-1 pass: 300 rows, K split over every
  // SM) stays on the k-split fast kernel: measured r02n/r02o, 75 us there
  // against 75-90 us here across stage / producer / warp counts
  if (layout == fast::kCol && p.n_tiles == 1 && !std::getenv("NTF_SK_FORCE")) return false;
  p.align = align && p.n_tiles >= sms ? 1 : 0;
  p.tx_bytes = p.t_stage_bytes;
  // no base modes (a single varying factor, e.g. the dimension tree's Y_L
  // at 3-way): the B operand is the factor rows themselves (direct_b)
  {
    int nbase = 0;
    for (int q = 0; q < v.order; ++q) {
      const bool vary = layout == fast::kRow ? q > v.mode : q < v.mode;
      const bool fixd = layout == fast::kRow && q < v.mode;
      if ((vary || fixd) && q != qL) ++nbase;
    }
    p.direct_b = nbase == 0 ? 1 : 0;
    if (const char* e = std::getenv("NTF_SK_DIRECTB")) p.direct_b = p.direct_b && std::atoi(e) != 0;
  }
  // aq slots per producer warp (copies run naw - 1 of its units ahead): 4,
  // fewer when the T stages would drop below four (C2's 300-row COL view)
  p.w_stage_bytes = p.direct_b ? 0u : unsigned((size_t(KB) * p.wld * es + 127) / 128 * 128);
  p.aq_stage_bytes = unsigned(((size_t(KB) + 2 * fast::kMaxBase) * r * es + fast::kUnitInts * sizeof(int) + 127) /
                              128 * 128);
  // FP32: no FP32 register sum over more than 16384 terms (512 units of 32)
  p.flush_units = f32 ? 16384 / KB : 0;
  const size_t per_stage = size_t(p.t_stage_bytes) + p.w_stage_bytes + (p.direct_b ? p.aq_stage_bytes : 0u);
  size_t fixed = 0;
  for (p.naw = 4; p.naw >= 2; --p.naw) {
    fixed = p.direct_b ? 0 : size_t(p.NP) * p.naw * p.aq_stage_bytes;
    if ((kSkSmem - fixed) / per_stage >= 4) break;
  }
  if (p.naw < 2) p.naw = 2;
  if (const char* e = std::getenv("NTF_SK_NAW")) p.naw = std::max(2, std::min(8, std::atoi(e)));
  fixed = p.direct_b ? 0 : size_t(p.NP) * p.naw * p.aq_stage_bytes;
  if (fixed >= kSkSmem) return false;
  p.stages = int(std::min<size_t>(8, (kSkSmem - fixed) / per_stage));
  if (const char* e = std::getenv("NTF_SK_STAGES")) p.stages = std::min(p.stages, std::max(2, std::atoi(e)));
  p.stages -= p.stages % p.NP;
  if (p.stages < 2 * p.NP) return false;
  pl.grid = int(std::min<long long>(sms, p.W));
  pl.threads = 32 * (p.NP + p.MW);
  pl.smem = size_t(p.stages) * per_stage + fixed + (2 * size_t(p.stages) + size_t(p.NP) * p.naw) * sizeof(uint64_t);
  pl.layout = layout;
  pl.nmf = nmf;
  pl.nnf = nnf;
  pl.f32 = f32;
  if (!(f32 ? sk::pick_f32(nnf, layout, nmf == 4 ? 4 : 8) : sk::pick(nmf, nnf, layout))) return false;
  // contributors per tile and the split tiles
  pl.tile_ctas.assign(size_t(2 * p.n_tiles), 0);
  for (int t = 0; t < p.n_tiles; ++t) {
    pl.tile_ctas[size_t(2 * t)] = -1;
    pl.tile_ctas[size_t(2 * t + 1)] = -1;
  }
  for (int bb = 0; bb < pl.grid; ++bb) {
    const long long a = sk::range_lo(p, pl.grid, bb), z = sk::range_lo(p, pl.grid, bb + 1);
    if (z <= a) continue;
    for (long long t = a / p.U; t <= (z - 1) / p.U; ++t) {
      if (pl.tile_ctas[size_t(2 * t)] < 0) pl.tile_ctas[size_t(2 * t)] = bb;
      pl.tile_ctas[size_t(2 * t + 1)] = bb;
    }
  }
  pl.split.clear();
  for (int t = 0; t < p.n_tiles; ++t)
    if (pl.tile_ctas[size_t(2 * t)] != pl.tile_ctas[size_t(2 * t + 1)]) pl.split.push_back(t);
  p.n_split = int(pl.split.size());
  int fan = 1;
  for (int t : pl.split) fan = std::max(fan, pl.tile_ctas[size_t(2 * t + 1)] - pl.tile_ctas[size_t(2 * t)] + 1);
  p.lpo = fan > 16 ? 8 : 1;
  *out = pl;
  return true;
}

size_t sk_partial_len(const ModeView& v, int dtype, int sms) {
  SkPlan pl;
  if (!sk_choose(v, dtype, sms, &pl)) return 0;
  return size_t(2 * pl.grid) * pl.p.m_cta * v.rank;
}

void sk_append_tables(const SkPlan& pl, std::vector<int>* tab) {
  tab->insert(tab->end(), pl.tile_ctas.begin(), pl.tile_ctas.end());
  tab->insert(tab->end(), pl.split.begin(), pl.split.end());
}

void sk_mttkrp(const void* t, const ModeView& v, const SkPlan& pl, const DevFactors* dF, const int* unit_table,
               double* partial, double* out, cudaStream_t s, unsigned* counter, const fast::Params& modes,
               bool pdl) {
  auto fn = sk_encode_fn();
  if (!fn) throw CudaError("cuTensorMapEncodeTiled is unavailable");
  const SkParams& p0 = pl.p;
  CUtensorMap map;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  CUtensorMapSwizzle sw;
  const size_t es = pl.f32 ? 4 : 8;
  const cuuint32_t KB = cuuint32_t(128 / es);
  if (pl.layout == fast::kRow) {
    dims[0] = cuuint64_t(v.R);
    dims[1] = cuuint64_t(v.I);
    dims[2] = cuuint64_t(v.L);
    strides[0] = cuuint64_t(v.R * es);
    strides[1] = cuuint64_t(v.I * v.R * es);
    box[0] = KB;
    box[1] = cuuint32_t(p0.m_box);
    box[2] = 1;
    sw = CU_TENSOR_MAP_SWIZZLE_128B;
  } else {
    dims[0] = cuuint64_t(v.I);
    dims[1] = cuuint64_t(v.L);
    dims[2] = 1;
    strides[0] = cuuint64_t(v.I * es);
    strides[1] = cuuint64_t(v.I * v.L * es);
    box[0] = cuuint32_t(p0.m_pitch);
    box[1] = KB;
    box[2] = 1;
    sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  }
  const CUresult rr = fn(&map, pl.f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                         const_cast<void*>(t), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rr != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(rr)) + ")");
  SkParams p = p0;
  p.F = dF;
  p.partial = partial;
  p.out = out;
  p.counter = counter;
  p.utab = unit_table;
  p.nb = modes.nb;
  for (int q = 0; q < fast::kMaxBase; ++q) p.bq[q] = modes.bq[q];
  p.qL = modes.qL;
  p.rowL_wrap = modes.rowL_wrap;
  p.pdl = pdl && !p.n_split ? 1 : 0;  // (a cooperative split-tile launch is never a dependent)
  if (p.n_split && !counter) throw LogicError("stream-K MTTKRP needs an arrival counter");
  (pl.f32 ? sk::pick_f32(pl.nnf, pl.layout, pl.nmf == 4 ? 4 : 8) : sk::pick(pl.nmf, pl.nnf, pl.layout))(
      map, p, pl.grid, pl.threads, pl.smem, s);
}

std::string sk_describe(const SkPlan& pl) {
  char buf[256];
  snprintf(buf, sizeof buf,
           "sk-%s+%s NMF=%d NNF=%d MW=%d NP=%d m_cta=%d stages=%d grid=%d threads=%d smem=%zu "
           "tiles=%d units/tile=%lld split=%d align=%d lpo=%d direct_b=%d naw=%d",
           pl.layout == fast::kRow ? "row" : "col", pl.f32 ? "ffma2" : "dmma", pl.nmf, pl.nnf, pl.p.MW, pl.p.NP,
           pl.p.m_cta, pl.p.stages, pl.grid, pl.threads, pl.smem, pl.p.n_tiles, pl.p.U, pl.p.n_split, pl.p.align,
           pl.p.lpo, pl.p.direct_b, pl.p.naw);
  return buf;
}

}  // namespace ntfb
