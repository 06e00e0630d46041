// Fast sm_100a MTTKRP: plan selection, TMA descriptors and dispatch.
// The kernel template lives in mttkrp_fast_impl.cuh; its instantiations are
// split over mttkrp_fast_f64.cu / mttkrp_fast_f32.cu to compile in parallel.
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "mttkrp_fast.h"
#include "mttkrp_fast_launch.h"

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
  fast::KernelCfg cfg;
  if (!fast::lookup(dtype, v.rank, v.I, &cfg)) return false;
  const int RW = (32 / cfg.G) * cfg.A;
  const long long mw_total = (v.I + RW - 1) / RW;
  int MW, n_mtiles;
  if (mw_total <= kMaxMW) {
    MW = int(mw_total);
    n_mtiles = 1;
  } else {
    MW = 8;
    n_mtiles = int((v.I + 8LL * RW - 1) / (8LL * RW));
  }
  const int KW = std::max(1, std::min(8, 8 / MW));
  const int m_cta = MW * RW;
  fast::Params& p = out->p;
  p = fast::Params{};
  p.v = v;
  p.MW = MW;
  p.KW = KW;
  p.NP = std::max(1, std::min(2, 12 - MW * KW));
  p.m_cta = m_cta;
  p.n_mbox = (m_cta + 255) / 256;
  p.m_box = m_cta / p.n_mbox;
  if (p.m_box * p.n_mbox != m_cta || p.m_box % 8) return false;
  const int vec = int(16 / es);
  const int bp = (cfg.B + vec - 1) / vec * vec;
  p.wld = cfg.G * bp;
  if (layout == fast::kRow) {
    p.kbox = int(128 / es);
    p.nbox_r = (v.R + p.kbox - 1) / p.kbox;
    p.units = v.L * p.nbox_r;
    p.t_stage_bytes = unsigned(m_cta * 128);
  } else {
    p.kbox = int(128 / es);  // 16 doubles / 32 floats of l per unit
    p.nbox_r = 0;
    p.units = (v.L + p.kbox - 1) / p.kbox;
    p.t_stage_bytes = unsigned(size_t(m_cta) * p.kbox * es);
  }
  p.tx_bytes = p.t_stage_bytes;
  p.w_stage_bytes = unsigned((size_t(p.kbox) * p.wld * es + 127) / 128 * 128);
  const size_t per_stage = size_t(p.t_stage_bytes) + p.w_stage_bytes;
  p.stages = int(std::min<size_t>(8, kSmemBudget / per_stage));
  if (p.stages < 2) return false;
  // the k-split fold reuses the T stages as scratch
  if (size_t(m_cta) * cfg.G * cfg.B * es > size_t(p.stages) * p.t_stage_bytes) return false;
  p.ctas_per_mtile = int(std::max<long long>(1, std::min<long long>(p.units, std::max(1, sms / n_mtiles))));
  out->cfg = cfg;
  out->layout = layout;
  out->grid = n_mtiles * p.ctas_per_mtile;
  out->threads = 32 * (p.NP + MW * KW);
  out->smem = size_t(p.stages) * per_stage + 2 * size_t(p.stages) * sizeof(uint64_t);
  return true;
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
    box[0] = cuuint32_t(ch.p.m_box);
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

int fast_mttkrp_kernels(const ModeView&, int) { return 2; }

size_t fast_mttkrp_partial_len(const ModeView& v, int dtype, int sms) {
  Choice ch;
  if (!choose(v, dtype, sms, &ch)) return 0;
  return size_t(ch.p.ctas_per_mtile) * v.I * v.rank;
}

void fast_mttkrp(const void* t, int dtype, const ModeView& v, const DevFactors* dF, double* partial, double* out,
                 int sms, cudaStream_t s) {
  Choice ch;
  if (!choose(v, dtype, sms, &ch)) throw Unsupported("no fast MTTKRP plan for this view");
  CUtensorMap map;
  make_map(t, dtype, v, ch, &map);
  ch.p.F = dF;
  ch.p.partial = partial;
  fast::LaunchFn fn = ch.layout == fast::kRow ? ch.cfg.row : ch.cfg.col;
  fn(map, ch.p, ch.grid, ch.threads, ch.smem, s);
  launch_reduce_partials(partial, ch.p.ctas_per_mtile, v.I * v.rank, out, s);
}

std::string fast_mttkrp_describe(const ModeView& v, int dtype, int sms) {
  Choice ch;
  if (!choose(v, dtype, sms, &ch)) return "generic";
  char buf[256];
  snprintf(buf, sizeof buf, "%s G=%d B=%d A=%d MW=%d KW=%d m_cta=%d stages=%d grid=%d threads=%d smem=%zu units=%lld",
           ch.layout == fast::kRow ? "row" : "col", ch.cfg.G, ch.cfg.B, ch.cfg.A, ch.p.MW, ch.p.KW, ch.p.m_cta,
           ch.p.stages, ch.grid, ch.threads, ch.smem, ch.p.units);
  return buf;
}

}  // namespace ntfb
