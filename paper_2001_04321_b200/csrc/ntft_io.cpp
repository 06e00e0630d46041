// The reference's binary dense-tensor container "NTFT" (tensor.cpp:56-96,
// README.md "File formats"): magic "NTFT", u32 version (1), u32 order, u64
// dims, then the FP64 payload, little-endian, last index fastest. Same
// checks and messages as DenseTensor::load (std::runtime_error -> status
// NTF_ERR_RUNTIME at the ABI).
//
// Beyond the reference: a mode-1 slab can be read on its own (a rank of a
// sharded context reads only its rows: one seek), FP32 storage is produced
// by round-to-nearest of the FP64 payload in chunks, and the device upload
// streams the slab through two pinned staging buffers so a 32 GB instance
// never sits whole in host memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "runtime.h"

namespace ntfb {

namespace {

constexpr char kMagic[4] = {'N', 'T', 'F', 'T'};
constexpr uint32_t kVersion = 1;
constexpr size_t kChunkValues = size_t(1) << 23;  // 64 MB of FP64 per staging chunk

struct File {
  FILE* f = nullptr;
  File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

void read_exact(FILE* f, void* dst, size_t bytes, const std::string& path, const char* what) {
  if (std::fread(dst, 1, bytes, f) != bytes) throw std::runtime_error(path + ": " + what);
}

}  // namespace

NtftHeader ntft_read_header(const std::string& path) {
  File in(path, "rb");
  if (!in.f) throw std::runtime_error("cannot open " + path);
  char magic[4];
  if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
    throw std::runtime_error(path + ": not a tensor container");
  uint32_t version = 0, order = 0;
  if (std::fread(&version, sizeof version, 1, in.f) != 1 || std::fread(&order, sizeof order, 1, in.f) != 1 ||
      version != kVersion)
    throw std::runtime_error(path + ": unsupported version");
  if (order < 1 || order > 64) throw std::runtime_error(path + ": bad order");
  if (order > uint32_t(kMaxOrder)) throw Unsupported(path + ": order above the GPU path's limit (8)");
  NtftHeader h;
  h.order = int(order);
  for (uint32_t l = 0; l < order; ++l) {
    uint64_t d = 0;
    read_exact(in.f, &d, sizeof d, path, "truncated header");
    if (d < 1 || d > uint64_t((1LL << 31) - 1)) throw std::runtime_error(path + ": bad dimension");
    h.shape[l] = int64_t(d);
  }
  h.payload_offset = int64_t(4 + 2 * sizeof(uint32_t) + order * sizeof(uint64_t));
  return h;
}

void ntft_write(const std::string& path, const void* data, int dtype, int order, const int64_t* shape) {
  if (order < 1 || order > kMaxOrder) throw InvalidArgument("tensor order must lie in 1..8");
  if (dtype != NTF_DTYPE_F64 && dtype != NTF_DTYPE_F32) throw InvalidArgument("unknown dtype");
  long long n = 1;
  for (int i = 0; i < order; ++i) {
    if (shape[i] < 1) throw InvalidArgument("tensor dimensions must be positive");
    n *= shape[i];
  }
  File out(path, "wb");
  if (!out.f) throw std::runtime_error("cannot open " + path + " for writing");
  const uint32_t version = kVersion, ord = uint32_t(order);
  bool ok = std::fwrite(kMagic, 1, 4, out.f) == 4 && std::fwrite(&version, sizeof version, 1, out.f) == 1 &&
            std::fwrite(&ord, sizeof ord, 1, out.f) == 1;
  for (int i = 0; ok && i < order; ++i) {
    const uint64_t d = uint64_t(shape[i]);
    ok = std::fwrite(&d, sizeof d, 1, out.f) == 1;
  }
  if (dtype == NTF_DTYPE_F64) {
    ok = ok && std::fwrite(data, sizeof(double), size_t(n), out.f) == size_t(n);
  } else {  // FP32 storage: the container always holds FP64 (exact upcast)
    std::vector<double> buf(std::min<size_t>(size_t(n), kChunkValues));
    const float* src = static_cast<const float*>(data);
    for (long long off = 0; ok && off < n; off += (long long)buf.size()) {
      const size_t m = size_t(std::min<long long>((long long)buf.size(), n - off));
      for (size_t e = 0; e < m; ++e) buf[e] = double(src[off + (long long)e]);
      ok = std::fwrite(buf.data(), sizeof(double), m, out.f) == m;
    }
  }
  if (!ok || std::fflush(out.f) != 0) throw std::runtime_error("write failed: " + path);
}

// Entries [first, first + count) of the payload, converted to `dtype`, in
// chunks of kChunkValues through `stage` (FP64 scratch of that size); each
// chunk is handed to sink(dst_offset_in_values, pointer, values).
template <typename Sink>
static void read_range(const std::string& path, const NtftHeader& h, long long first, long long count, int dtype,
                       std::vector<double>& stage, Sink&& sink) {
  File in(path, "rb");
  if (!in.f) throw std::runtime_error("cannot open " + path);
  if (std::fseek(in.f, long(h.payload_offset + first * 8), SEEK_SET) != 0)
    throw std::runtime_error(path + ": truncated payload");
  std::vector<float> f32;
  if (dtype == NTF_DTYPE_F32) f32.resize(stage.size());
  for (long long off = 0; off < count; off += (long long)stage.size()) {
    const size_t m = size_t(std::min<long long>((long long)stage.size(), count - off));
    read_exact(in.f, stage.data(), m * sizeof(double), path, "truncated payload");
    if (dtype == NTF_DTYPE_F32) {
      for (size_t e = 0; e < m; ++e) f32[e] = float(stage[e]);  // round to nearest
      sink(off, static_cast<const void*>(f32.data()), m);
    } else {
      sink(off, static_cast<const void*>(stage.data()), m);
    }
  }
}

void ntft_read_slab(const std::string& path, int dtype, int64_t slab_begin, int64_t slab_end, void* out) {
  const NtftHeader h = ntft_read_header(path);
  if (dtype != NTF_DTYPE_F64 && dtype != NTF_DTYPE_F32) throw InvalidArgument("unknown dtype");
  if (slab_begin < 0 && slab_end < 0) {
    slab_begin = 0;
    slab_end = h.shape[0];
  }
  if (slab_begin < 0 || slab_end < slab_begin || slab_end > h.shape[0])
    throw InvalidArgument("slab outside the first mode");
  long long stride0 = 1;
  for (int i = 1; i < h.order; ++i) stride0 *= h.shape[i];
  const long long count = (slab_end - slab_begin) * stride0;
  std::vector<double> stage(std::min<size_t>(size_t(std::max<long long>(count, 1)), kChunkValues));
  const size_t es = dtype == NTF_DTYPE_F32 ? 4 : 8;
  read_range(path, h, slab_begin * stride0, count, dtype, stage, [&](long long off, const void* p, size_t m) {
    std::memcpy(static_cast<char*>(out) + size_t(off) * es, p, m * es);
  });
}

// Stream [first, first + count) into device memory `dst` (dtype storage)
// through two pinned buffers: the copy of chunk c overlaps the file read
// (and FP32 rounding) of chunk c + 1.
void ntft_stream_to_device(const std::string& path, const NtftHeader& h, long long first, long long count,
                           int dtype, void* dst, cudaStream_t s) {
  const size_t es = dtype == NTF_DTYPE_F32 ? 4 : 8;
  std::vector<double> stage(std::min<size_t>(size_t(std::max<long long>(count, 1)), kChunkValues));
  void* pin[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  try {
    for (int b = 0; b < 2; ++b) {
      NTF_CUDA(cudaHostAlloc(&pin[b], stage.size() * es, cudaHostAllocDefault));
      NTF_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    }
    int b = 0;
    bool used[2] = {false, false};
    read_range(path, h, first, count, dtype, stage, [&](long long off, const void* p, size_t m) {
      if (used[b]) NTF_CUDA(cudaEventSynchronize(done[b]));  // the buffer's previous copy is done
      std::memcpy(pin[b], p, m * es);
      NTF_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + size_t(off) * es, pin[b], m * es, cudaMemcpyHostToDevice,
                               s));
      NTF_CUDA(cudaEventRecord(done[b], s));
      used[b] = true;
      b ^= 1;
    });
    NTF_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cudaStreamSynchronize(s);
    for (int b = 0; b < 2; ++b) {
      if (pin[b]) cudaFreeHost(pin[b]);
      if (done[b]) cudaEventDestroy(done[b]);
    }
    throw;
  }
  for (int b = 0; b < 2; ++b) {
    NTF_CUDA(cudaFreeHost(pin[b]));
    NTF_CUDA(cudaEventDestroy(done[b]));
  }
}

}  // namespace ntfb

// ---- "NTFK": TuckerFormat::save / load (tucker.cpp:106-165) -----------------
// magic "NTFK", u32 version (1), u32 order, u64 full dims, u64 core dims
// (ranks), the FP64 core payload (last index fastest), then every basis
// I_p x r_p row-major in mode order. Same messages as TuckerFormat::load.
namespace ntfb {

namespace {
constexpr char kMagicK[4] = {'N', 'T', 'F', 'K'};
}

NtfkHeader ntfk_read_header(const std::string& path) {
  File in(path, "rb");
  if (!in.f) throw std::runtime_error("cannot open " + path);
  char magic[4];
  if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, kMagicK, 4) != 0)
    throw std::runtime_error(path + ": not a tucker container");
  uint32_t version = 0, order = 0;
  if (std::fread(&version, sizeof version, 1, in.f) != 1 || std::fread(&order, sizeof order, 1, in.f) != 1 ||
      version != kVersion)
    throw std::runtime_error(path + ": unsupported version");
  if (order < 1 || order > 64) throw std::runtime_error(path + ": bad order");
  if (order > uint32_t(kMaxOrder)) throw Unsupported(path + ": order above the GPU path's limit (8)");
  NtfkHeader h;
  h.order = int(order);
  for (int pass = 0; pass < 2; ++pass)
    for (uint32_t l = 0; l < order; ++l) {
      uint64_t d = 0;
      read_exact(in.f, &d, sizeof d, path, "truncated payload");
      if (d < 1 || d > uint64_t((1LL << 31) - 1)) throw std::runtime_error(path + ": bad dimension");
      (pass == 0 ? h.shape : h.ranks)[l] = int64_t(d);
    }
  h.payload_offset = int64_t(4 + 2 * sizeof(uint32_t) + 2 * order * sizeof(uint64_t));
  return h;
}

void ntfk_read(const std::string& path, double* core, double* bases) {
  const NtfkHeader h = ntfk_read_header(path);
  long long nc = 1, nb = 0;
  for (int l = 0; l < h.order; ++l) {
    nc *= h.ranks[l];
    nb += h.shape[l] * h.ranks[l];
  }
  File in(path, "rb");
  if (!in.f) throw std::runtime_error("cannot open " + path);
  if (std::fseek(in.f, long(h.payload_offset), SEEK_SET) != 0) throw std::runtime_error(path + ": truncated payload");
  read_exact(in.f, core, size_t(nc) * sizeof(double), path, "truncated payload");
  read_exact(in.f, bases, size_t(nb) * sizeof(double), path, "truncated payload");
}

void ntfk_write(const std::string& path, const double* core, const double* bases, int order, const int64_t* shape,
                const int64_t* ranks) {
  if (order < 1 || order > kMaxOrder) throw InvalidArgument("tensor order must lie in 1..8");
  long long nc = 1, nb = 0;
  for (int l = 0; l < order; ++l) {
    if (shape[l] < 1 || ranks[l] < 1) throw InvalidArgument("tensor dimensions must be positive");
    nc *= ranks[l];
    nb += shape[l] * ranks[l];
  }
  File out(path, "wb");
  if (!out.f) throw std::runtime_error("cannot open " + path + " for writing");
  const uint32_t version = kVersion, ord = uint32_t(order);
  bool ok = std::fwrite(kMagicK, 1, 4, out.f) == 4 && std::fwrite(&version, sizeof version, 1, out.f) == 1 &&
            std::fwrite(&ord, sizeof ord, 1, out.f) == 1;
  for (int pass = 0; pass < 2; ++pass)
    for (int l = 0; ok && l < order; ++l) {
      const uint64_t d = uint64_t((pass == 0 ? shape : ranks)[l]);
      ok = std::fwrite(&d, sizeof d, 1, out.f) == 1;
    }
  ok = ok && std::fwrite(core, sizeof(double), size_t(nc), out.f) == size_t(nc);
  ok = ok && std::fwrite(bases, sizeof(double), size_t(nb), out.f) == size_t(nb);
  if (!ok || std::fflush(out.f) != 0) throw std::runtime_error("write failed: " + path);
}

}  // namespace ntfb
