// Fast sm_100a MTTKRP: plan selection, TMA descriptors and dispatch.
// The kernel template lives in mttkrp_fast_impl.cuh; its instantiations are
// split over mttkrp_fast_f64.cu / mttkrp_fast_f32.cu to compile in parallel.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "mttkrp_fast.h"
#include "mttkrp_fast_launch.h"
#include "mttkrp_sk.h"

namespace ntfb {

namespace {

constexpr long long kMinElems = 1 << 15;  // below this the generic kernel is as fast
constexpr size_t kSmemBudget = 200 * 1024;
constexpr int kMaxMW = 11;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

struct Choice {
  fast::KernelCfg cfg;
  fast::Params p;
  int layout, grid, threads;
  size_t smem;
  bool mma = false;  // FP64 DMMA consumers
};

bool choose(const ModeView& v, int dtype, int sms, Choice* out) {
  const size_t es = dtype == NTF_DTYPE_F32 ? 4 : 8;
  if (v.L * v.I * v.R < kMinElems) return false;
  if (v.L >= (1LL << 31) || v.R >= (1LL << 31)) return false;  // 32-bit digit math in the producer
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
  // the producer bulk-copies KB consecutive rows of the last varying mode's
  // factor per unit (rows of r elements must be 16-byte multiples) and
  // assumes at most one wrap of that digit inside a unit
  const int kb = int(128 / es);
  if ((v.rank * es) % 16) return false;
  const int qL = layout == fast::kRow ? v.order - 1 : v.order - 2;
  if (v.dims[qL] < kb) return false;
  if (v.order > fast::kMaxBase + 2) return false;  // base rows per unit <= kMaxBase
  fast::KernelCfg cfg;
  if (!fast::lookup(dtype, v.rank, v.I, &cfg)) return false;
  const int RW = (32 / cfg.G) * cfg.A;
  const long long mw_total = (v.I + RW - 1) / RW;
  const int warp_cap = fast::max_threads_es(cfg.A, cfg.B, int(es)) / 32;
  // producer warps (each forms W for every NP-th unit): a short m range
  // (<= 128 rows, e.g. C3) means small units, so W formation and copy
  // issue, not the FMAs, bound the pipeline (r01: 4 producers 245 us vs
  // 2 producers 339 us per C3 mode)
  int NP = RW * mw_total <= 128 ? 4 : 2;
  if (const char* e = std::getenv("NTF_FAST_NP")) NP = std::max(1, std::atoi(e));  // tuning override
  const int cons_cap = std::min(kMaxMW, warp_cap - NP);
  if (cons_cap < 1) return false;
  int MW0, n_mtiles0;
  if (mw_total <= cons_cap) {
    MW0 = int(mw_total);
    n_mtiles0 = 1;
  } else {
    MW0 = std::min(cons_cap, 8);
    n_mtiles0 = int((v.I + (long long)MW0 * RW - 1) / ((long long)MW0 * RW));
  }
  // Tall views (the dimension tree's partials: Y_L has prod_{n<h} I_n rows)
  // need smaller m-tiles for a pipeline of >= 2 NP stages: fewer m-warps.
  // FP64: DMMA consumers when the blocking has them (NTF_FAST_MMA=0: DFMA)
  const char* mma_env = std::getenv("NTF_FAST_MMA");
  const bool mma_try = !(mma_env && std::atoi(mma_env) == 0) && dtype == NTF_DTYPE_F64 &&
                       (layout == fast::kRow ? cfg.row_mma : cfg.col_mma) != nullptr;
  for (int MW = MW0; MW >= 1; --MW) {
    const int n_mtiles = MW == MW0 ? n_mtiles0 : int((v.I + (long long)MW * RW - 1) / ((long long)MW * RW));
    // at least four consumer warps (one per SM sub-partition): split k
    const char* ce = std::getenv("NTF_FAST_CONS");  // tuning override
    const int cons_target = ce ? std::max(1, std::atoi(ce)) : cfg.cons;
    int KW = std::max(1, std::min(8, (cons_target + MW - 1) / MW));
    if (const char* e = std::getenv("NTF_FAST_KW")) KW = std::max(1, std::min(8, std::atoi(e)));
    while (MW * KW > cons_cap && KW > 1) --KW;
    const int m_cta = MW * RW;
    fast::Params& p = out->p;
    p = fast::Params{};
    p.v = v;
    p.MW = MW;
    p.KW = KW;
    p.NP = NP;
    p.m_cta = m_cta;
    p.n_mbox = (m_cta + 255) / 256;
    p.m_box = m_cta / p.n_mbox;
    if (p.m_box * p.n_mbox != m_cta || p.m_box % 8) continue;
    const int vec = int(16 / es);
    const int bp = (cfg.B + vec - 1) / vec * vec;
    p.wld = cfg.G * bp;
    // DMMA B fragments read 4 k rows per half-warp: a W row pitch that is a
    // multiple of 64 B puts two (or four) of them on the same banks; pad it
    // to 32 B off (the padding columns stay zero)
    if (mma_try && (p.wld * es) % 64 == 0) p.wld += int(32 / es);
    if (layout == fast::kRow) {
      p.kbox = int(128 / es);
      p.nbox_r = (v.R + p.kbox - 1) / p.kbox;
      p.units = v.L * p.nbox_r;
      p.m_pitch = p.m_box;
      p.t_stage_bytes = unsigned(m_cta * 128);
    } else {
      p.kbox = int(128 / es);  // 16 doubles / 32 floats of l per unit
      p.nbox_r = 0;
      p.units = (v.L + p.kbox - 1) / p.kbox;
      p.m_pitch = (mma_try && p.m_box + 4 <= 256) ? p.m_box + 4 : p.m_box;
      p.t_stage_bytes = unsigned(size_t(p.n_mbox) * p.m_pitch * p.kbox * es);
    }
    p.tx_bytes = p.t_stage_bytes;
    p.w_stage_bytes = unsigned((size_t(p.kbox) * p.wld * es + 127) / 128 * 128);
    // KB rows of the last varying mode, 2 x kMaxBase base rows, 2 info ints
    p.aq_stage_bytes =
        unsigned(((size_t(p.kbox) + 2 * fast::kMaxBase) * v.rank * es + 2 * sizeof(int) + 127) / 128 * 128);
    const size_t per_stage = size_t(p.t_stage_bytes) + p.w_stage_bytes + p.aq_stage_bytes;
    p.stages = int(std::min<size_t>(8, kSmemBudget / per_stage));
    if (const char* e = std::getenv("NTF_FAST_STAGES"))  // tuning override
      p.stages = std::min(p.stages, std::max(2, std::atoi(e)));
    // Producer warp w owns stages s == w (mod NP) and visits them in
    // consecutive rounds, so its parity waits never run more than one phase
    // ahead of an mbarrier; that needs NP | stages.
    p.stages -= p.stages % p.NP;
    if (p.stages < 2 * p.NP) continue;  // each producer looks at least one unit ahead
    // the k-split fold reuses the T stages as scratch
    if (size_t(m_cta) * cfg.G * cfg.B * es > size_t(p.stages) * p.t_stage_bytes) continue;
    p.ctas_per_mtile = int(std::max<long long>(1, std::min<long long>(p.units, std::max(1, sms / n_mtiles))));
    out->grid = n_mtiles * p.ctas_per_mtile;
    out->threads = 32 * (p.NP + MW * KW);
    out->smem = size_t(p.stages) * per_stage + 3 * size_t(p.stages) * sizeof(uint64_t);
    out->cfg = cfg;
    out->layout = layout;
    // FP64: DMMA consumers when the blocking has them and their fragment
    // scratch fits the stage buffers (NTF_FAST_MMA=0: DFMA consumers)
    {
      const size_t scr = size_t(MW) * KW * fast::mma_scratch_doubles(cfg.G, cfg.B, cfg.A) * sizeof(double);
      out->mma = mma_try && scr <= size_t(p.stages) * p.t_stage_bytes;
    }
    return true;
  }
  return false;
}

void make_map(const void* t, int dtype, const ModeView& v, const Choice& ch, CUtensorMap* map) {
  auto fn = encode_fn();
  if (!fn) throw CudaError("cuTensorMapEncodeTiled is unavailable");
  const size_t es = dtype == NTF_DTYPE_F32 ? 4 : 8;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  CUtensorMapSwizzle sw;
  if (ch.layout == fast::kRow) {
    dims[0] = cuuint64_t(v.R);
    dims[1] = cuuint64_t(v.I);
    dims[2] = cuuint64_t(v.L);
    strides[0] = cuuint64_t(v.R * es);
    strides[1] = cuuint64_t(v.I * v.R * es);
    box[0] = cuuint32_t(ch.p.kbox);
    box[1] = cuuint32_t(ch.p.m_box);
    box[2] = 1;
    sw = CU_TENSOR_MAP_SWIZZLE_128B;
  } else {
    dims[0] = cuuint64_t(v.I);
    dims[1] = cuuint64_t(v.L);
    dims[2] = 1;
    strides[0] = cuuint64_t(v.I * es);
    strides[1] = cuuint64_t(v.I * v.L * es);
    box[0] = cuuint32_t(ch.p.m_pitch);
    box[1] = cuuint32_t(ch.p.kbox);
    box[2] = 1;
    sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  }
  const CUresult r = fn(map, dtype == NTF_DTYPE_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                        3, const_cast<void*>(t), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

}  // namespace

bool fast_mttkrp_supported(const ModeView& v, int dtype) {
  if (!encode_fn()) return false;
  Choice ch;
  return choose(v, dtype, device_sm_count(), &ch);
}

int fast_mttkrp_kernels(const ModeView& v, int dtype) {
  SkPlan sp;
  if (sk_choose(v, dtype, device_sm_count(), &sp)) return 1;
  Choice ch;
  if (!choose(v, dtype, device_sm_count(), &ch)) return 2;
  return ch.p.ctas_per_mtile == 1 ? 1 : 2;  // upper bound (2 without an arrival counter)
}

size_t fast_mttkrp_partial_len(const ModeView& v, int dtype, int sms) {
  Choice ch;
  if (!choose(v, dtype, sms, &ch)) return 0;
  return std::max<size_t>(size_t(ch.p.ctas_per_mtile) * size_t(v.I) * size_t(v.rank), sk_partial_len(v, dtype, sms));
}

namespace {

// Modes whose digit varies with k inside a unit (ROW: after `mode`; COL:
// before it), the last of them (qL, fastest), and the base modes (every
// other contributing mode, ascending).
struct UnitModes {
  bool vary[kMaxOrder] = {}, fixd[kMaxOrder] = {};
  int qL = 0, nb = 0, bq[fast::kMaxBase] = {};
};

UnitModes unit_modes(const ModeView& v, int layout) {
  UnitModes m;
  for (int q = 0; q < v.order; ++q) {
    m.vary[q] = layout == fast::kRow ? q > v.mode : q < v.mode;
    m.fixd[q] = layout == fast::kRow && q < v.mode;
  }
  m.qL = layout == fast::kRow ? v.order - 1 : v.order - 2;
  for (int q = 0; q < v.order; ++q)
    if ((m.vary[q] || m.fixd[q]) && q != m.qL) m.bq[m.nb++] = q;
  return m;
}

void fill_params_modes(const ModeView& v, int layout, fast::Params& p) {
  const UnitModes m = unit_modes(v, layout);
  // factor index of view dim q (merged-row views: dims q >= 1 are shifted)
  const auto fac = [&](int q) { return q >= 1 ? q + v.fshift : q; };
  p.qL = fac(m.qL);
  p.nb = m.nb;
  for (int t = 0; t < fast::kMaxBase; ++t) p.bq[t] = t < m.nb ? fac(m.bq[t]) : m.bq[t];
  p.rowL_wrap = m.qL == 0 ? int(v.row0) : 0;
}

}  // namespace

std::vector<int> fast_mttkrp_unit_table(const ModeView& v, int dtype, int sms) {
  Choice ch;
  if (!choose(v, dtype, sms, &ch)) return {};
  const UnitModes m = unit_modes(v, ch.layout);
  const fast::Params& p = ch.p;
  const int kb = p.kbox;
  std::vector<int> tab(size_t(p.units) * fast::kUnitInts, 0);
  for (long long u = 0; u < p.units; ++u) {
    int* e = &tab[size_t(u) * fast::kUnitInts];
    long long l, first, kmax;
    if (ch.layout == fast::kRow) {
      l = u / p.nbox_r;
      first = (u - l * p.nbox_r) * kb;
      kmax = v.R - first;
      e[0] = int(first);
      e[1] = int(l);
    } else {
      l = 0;
      first = u * kb;
      kmax = v.L - first;
      e[0] = int(first);
      e[1] = 0;
    }
    int dig[kMaxOrder] = {};
    long long rem = first, lrem = l;
    for (int q = v.order - 1; q >= 0; --q) {
      if (m.vary[q]) {
        dig[q] = int(rem % v.dims[q]);
        rem /= v.dims[q];
      } else if (m.fixd[q]) {
        dig[q] = int(lrem % v.dims[q]);
        lrem /= v.dims[q];
      }
    }
    const int dimL = v.dims[m.qL];
    const int n_valid = int(std::min<long long>(kb, kmax));
    e[2] = dig[m.qL] + (m.qL == 0 ? int(v.row0) : 0);
    e[3] = n_valid;
    e[4] = std::min(n_valid, dimL - dig[m.qL]);
    e[5] = dimL - dig[m.qL];
    for (int t = 0; t < m.nb; ++t) e[6 + t] = dig[m.bq[t]] + (m.bq[t] == 0 ? int(v.row0) : 0);
    // carry of the wrap into the higher varying digits
    bool carry = true;
    for (int q = v.order - 1; q >= 0; --q)
      if (m.vary[q] && q < m.qL && carry) {
        if (++dig[q] < v.dims[q])
          carry = false;
        else
          dig[q] = 0;
      }
    for (int t = 0; t < m.nb; ++t) e[6 + fast::kMaxBase + t] = dig[m.bq[t]] + (m.bq[t] == 0 ? int(v.row0) : 0);
  }
  SkPlan sp;  // the stream-K kernel reads its tile tables after the units
  if (sk_choose(v, dtype, sms, &sp) && sp.layout == ch.layout) sk_append_tables(sp, &tab);
  return tab;
}

void fast_mttkrp(const void* t, int dtype, const ModeView& v, const DevFactors* dF, const int* unit_table,
                 double* partial, double* out, int sms, cudaStream_t s, unsigned* counter, bool pdl) {
  Choice ch;
  if (!choose(v, dtype, sms, &ch)) throw Unsupported("no fast MTTKRP plan for this view");
  if (!unit_table) throw LogicError("fast MTTKRP needs its unit table");
  {
    SkPlan sp;  // FP64: the persistent stream-K DMMA kernel (mttkrp_sk.cu)
    if (sk_choose(v, dtype, sms, &sp) && sp.layout == ch.layout) {
      fast::Params modes{};
      fill_params_modes(v, sp.layout, modes);
      sk_mttkrp(t, v, sp, dF, unit_table, partial, out, s, counter, modes, pdl);
      return;
    }
  }
  CUtensorMap map;
  make_map(t, dtype, v, ch, &map);
  ch.p.F = dF;
  // one CTA per m-tile: the kernel writes the result rows directly;
  // otherwise it reduces its split-K slabs itself (grid-wide arrival count)
  const bool direct = ch.p.ctas_per_mtile == 1;
  ch.p.partial = direct ? out : partial;
  ch.p.out = out;
  ch.p.counter = nullptr;
  if (!direct && counter && !std::getenv("NTF_FAST_SEPARATE_REDUCE")) ch.p.counter = counter;
  ch.p.utab = unit_table;
  ch.p.pdl = pdl && !ch.p.counter ? 1 : 0;  // (a cooperative split-K launch is never a dependent)
  fill_params_modes(v, ch.layout, ch.p);
  // FP32 register sums over more than ~16k terms drift past the 1e-5
  // relative bar at BASELINE config 5 (1.05e-5 measured at 2000^3, r = 64)
  ch.p.flush_units = 0;
  if (dtype == NTF_DTYPE_F32 && ch.p.KW == 1) {
    const long long per_cta = (ch.p.units + ch.p.ctas_per_mtile - 1) / ch.p.ctas_per_mtile;
    const int fu = std::max(1, 16384 / ch.p.kbox);
    if (per_cta > fu) ch.p.flush_units = fu;
  }
  // diagnostics: NTF_FAST_PROF=1 prints per-CTA-averaged pipeline wait cycles
  static unsigned long long* prof = nullptr;
  const bool profiling = std::getenv("NTF_FAST_PROF") != nullptr;
  if (profiling) {
    const size_t n = size_t(ch.grid) * fast::kProfSlots;
    if (!prof) NTF_CUDA(cudaMalloc(&prof, 4096 * fast::kProfSlots * sizeof(unsigned long long)));
    NTF_CUDA(cudaMemsetAsync(prof, 0, n * sizeof(unsigned long long), s));
    ch.p.prof = prof;
  }
  fast::LaunchFn fn = ch.layout == fast::kRow ? (ch.mma ? ch.cfg.row_mma : ch.cfg.row)
                                              : (ch.mma ? ch.cfg.col_mma : ch.cfg.col);
  fn(map, ch.p, ch.grid, ch.threads, ch.smem, s);
  if (profiling) {
    std::vector<unsigned long long> h(size_t(ch.grid) * fast::kProfSlots);
    NTF_CUDA(cudaMemcpyAsync(h.data(), prof, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    NTF_CUDA(cudaStreamSynchronize(s));
    double a[fast::kProfSlots] = {};
    unsigned long long g0 = ~0ull, g1 = 0, gs0 = 0, gs1 = ~0ull;
    double gspan = 0;
    for (int b = 0; b < ch.grid; ++b) {
      for (int q = 0; q < 6; ++q) a[q] += double(h[size_t(b) * fast::kProfSlots + q]) / ch.grid;
      const unsigned long long st = h[size_t(b) * fast::kProfSlots + 6], en = h[size_t(b) * fast::kProfSlots + 7];
      g0 = std::min(g0, st);
      g1 = std::max(g1, en);
      gs0 = std::max(gs0, st);
      gs1 = std::min(gs1, en);
      gspan += double(en - st) / ch.grid;
    }
    fprintf(stderr, "[fast-prof mode %d] CTA starts spread %.1f us, ends spread %.1f us, avg CTA span %.1f us, "
            "first start to last end %.1f us\n", v.mode, (gs0 - g0) * 1e-3, (g1 - gs1) * 1e-3, gspan * 1e-3,
            (g1 - g0) * 1e-3);
    double ep[3] = {0, 0, 0};
    unsigned long long gend = 0;
    for (int b = 0; b < ch.grid; ++b) {
      const unsigned long long* q = &h[size_t(b) * fast::kProfSlots];
      if (q[8]) ep[0] += double(q[8] - q[7]) / ch.grid;
      if (q[9]) ep[1] += double(q[9] - q[8]) / ch.grid;
      if (q[10]) ep[2] += double(q[10] - q[9]) / ch.grid;
      gend = std::max(gend, std::max(q[8], q[10]));
    }
    fprintf(stderr, "[fast-prof mode %d] epilogue: fold+partials %.1f us, grid barrier %.1f us, slab reduce %.1f us; "
            "first start to last epilogue end %.1f us\n", v.mode, ep[0] * 1e-3, ep[1] * 1e-3, ep[2] * 1e-3,
            (gend - g0) * 1e-3);
    fprintf(stderr,
            "[fast-prof mode %d] units/CTA %.1f | producer %.0f cyc (stage wait %.0f, copy wait %.0f) | "
            "consumer %.0f cyc (data wait %.0f) | %.0f cyc/unit\n",
            v.mode, a[5], a[0], a[1], a[2], a[3], a[4], a[5] > 0 ? a[3] / a[5] : 0.0);
  }
  if (!direct && !ch.p.counter) launch_reduce_partials(partial, ch.p.ctas_per_mtile, v.I * v.rank, out, s);
}

std::string fast_mttkrp_describe(const ModeView& v, int dtype, int sms) {
  Choice ch;
  if (!choose(v, dtype, sms, &ch)) return "generic";
  SkPlan sp;
  if (sk_choose(v, dtype, sms, &sp) && sp.layout == ch.layout) return sk_describe(sp);
  char buf[256];
  snprintf(buf, sizeof buf, "%s%s G=%d B=%d A=%d MW=%d KW=%d m_cta=%d stages=%d grid=%d threads=%d smem=%zu units=%lld",
           ch.layout == fast::kRow ? "row" : "col", ch.mma ? "+dmma" : "", ch.cfg.G, ch.cfg.B, ch.cfg.A, ch.p.MW, ch.p.KW, ch.p.m_cta,
           ch.p.stages, ch.grid, ch.threads, ch.smem, ch.p.units);
  return buf;
}

}  // namespace ntfb
