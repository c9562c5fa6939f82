// SKYC dataset files straight to and from device memory.
//
// Format (the reference's write_bin / read_bin, datagen.cpp:163-221):
//   "SKYC" | u32 version = 1 | u32 d | u64 n | n*d f64 coordinates, all
//   little-endian, row-major.
// read_bin re-derives dim_min / dim_max from the data (Dataset::
// compute_minmax, dataset.cpp:10-20; NaN never wins a std::min / std::max
// against the +-inf seeds).
//
// B200 path: the file streams through two pinned chunks (the read of chunk
// i+1 overlaps the H2D copy of chunk i) into a caller-owned device buffer,
// and the per-dimension min / max is reduced on the device as each chunk
// lands (order-preserving integer keys, exact).  A dataset therefore reaches
// HBM without a host-side Dataset copy, ready for skycell_gpu_skyline_f64.
#include <cstdio>

#include "engine.cuh"

using sk::u64;

namespace skyeng {

struct FileCloser {
  FILE* f = nullptr;
  ~FileCloser() {
    if (f) std::fclose(f);
  }
};

constexpr size_t kIoChunk = 64ull << 20;  // bytes per pinned staging chunk

// mm[2k] = min key, mm[2k+1] = max key of dimension k over values
// v[0 .. count), the first of which belongs to dimension 0.  A thread's
// values all share one dimension (its stride is a multiple of d).
static __global__ void k_minmax_rows(const double* __restrict__ v, u64 count, int d, u64* __restrict__ mm) {
  sk::pdl_enter();
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  const u64 total = (u64)gridDim.x * blockDim.x;
  const u64 stride = total / d * d;
  if (tid >= stride) return;
  u64 lo = ~0ull, hi = 0;
  for (u64 i = tid; i < count; i += stride) {
    const double x = v[i];
    if (x != x) continue;  // NaN: never selected by std::min / std::max
    const u64 k = sk::dkey(x);
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
  }
  const int k = (int)(tid % d);
  if (lo != ~0ull) atomicMin(mm + 2 * k, lo);
  if (hi != 0) atomicMax(mm + 2 * k + 1, hi);
}

struct BinHeader {
  uint32_t version = 0, d = 0;
  u64 n = 0;
};

// Header checks in the reference's order (datagen.cpp:203-212).
inline BinHeader read_header(FILE* f, const std::string& path) {
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "SKYC", 4) != 0)
    throw ApiFail{SKYCELL_INPUT, path + ": bad magic, not a dataset file"};
  unsigned char h[16];
  if (std::fread(h, 1, 16, f) != 16) throw ApiFail{SKYCELL_INPUT, path + ": truncated file"};
  BinHeader b;
  for (int i = 0; i < 4; ++i) b.version |= (uint32_t)h[i] << (8 * i);
  for (int i = 0; i < 4; ++i) b.d |= (uint32_t)h[4 + i] << (8 * i);
  for (int i = 0; i < 8; ++i) b.n |= (u64)h[8 + i] << (8 * i);
  if (b.version != 1) throw ApiFail{SKYCELL_INPUT, path + ": unsupported version " + std::to_string(b.version)};
  if (b.d < 2 || b.d > (uint32_t)sk::kMaxD) throw ApiFail{SKYCELL_INPUT, path + ": bad dimensionality"};
  return b;
}

inline FILE* open_or_throw(const char* path, const char* mode, const char* verb) {
  if (!path) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null path"};
  FILE* f = std::fopen(path, mode);
  if (!f) throw ApiFail{SKYCELL_IO, std::string(verb) + " " + path};
  return f;
}

}  // namespace skyeng

using namespace skyeng;

extern "C" {

int skycell_bin_header(const char* path, uint64_t* n, int* d, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!n || !d) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null output pointer"};
    FileCloser fc{open_or_throw(path, "rb", "cannot open")};
    const BinHeader b = read_header(fc.f, path);
    *n = b.n;
    *d = (int)b.d;
  });
}

int skycell_gpu_read_bin(skycell_gpu_ctx* ctx, const char* path, double* dev_coords, uint64_t cap_values,
                         uint64_t* n_out, int* d_out, double* dim_min, double* dim_max, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx || !n_out || !d_out || !dim_min || !dim_max)
      throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null context or output pointer"};
    FileCloser fc{open_or_throw(path, "rb", "cannot open")};
    const BinHeader b = read_header(fc.f, path);
    const int d = (int)b.d;
    if (b.n > 0xffffffffull) throw ApiFail{SKYCELL_INPUT, "normalize: more than 2^32 - 1 records"};
    const u64 values = b.n * (u64)d;
    if (values > cap_values)
      throw ApiFail{SKYCELL_USAGE, "skycell_gpu: device buffer holds " + std::to_string(cap_values) + " values, the file " +
                                       std::to_string(values)};
    if (values && !dev_coords) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null device buffer"};
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = ctx->stream;
    ensure(ctx->q_mm, 2 * sk::kMaxD * 8);
    u64* mm = static_cast<u64*>(ctx->q_mm.p);
    std::vector<u64> init(2 * d);
    for (int k = 0; k < d; ++k) {
      init[2 * k] = ~0ull;
      init[2 * k + 1] = 0;
    }
    ck(cudaMemcpyAsync(mm, init.data(), init.size() * 8, cudaMemcpyHostToDevice, s), "mm init");
    // chunks hold whole rows, so every chunk starts at dimension 0
    const u64 per = std::max<u64>(1, kIoChunk / (8 * (u64)d)) * (u64)d;
    double* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    struct PinGuard {
      double** p;
      cudaEvent_t* e;
      ~PinGuard() {
        for (int i = 0; i < 2; ++i) {
          if (p[i]) cudaFreeHost(p[i]);
          if (e[i]) cudaEventDestroy(e[i]);
        }
      }
    } guard{pin, done};
    for (int i = 0; i < 2; ++i) {
      ck(cudaMallocHost(reinterpret_cast<void**>(&pin[i]), per * 8), "pinned");
      ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "event");
    }
    const unsigned g = (unsigned)std::max(1, ctx->num_sms * 4);
    u64 at = 0;
    int bi = 0;
    while (at < values) {
      const u64 cnt = std::min<u64>(per, values - at);
      ck(cudaEventSynchronize(done[bi]), "staging reuse");  // its previous copy has finished
      if (std::fread(pin[bi], 8, cnt, fc.f) != cnt) throw ApiFail{SKYCELL_INPUT, std::string(path) + ": truncated file"};
      ck(cudaMemcpyAsync(dev_coords + at, pin[bi], cnt * 8, cudaMemcpyHostToDevice, s), "H2D");
      ck(cudaEventRecord(done[bi], s), "event");
      sk::launch(k_minmax_rows, g, 256, 0, s, dev_coords + at, cnt, d, mm);
      at += cnt;
      bi ^= 1;
    }
    ck(cudaGetLastError(), "kernel launch");
    std::vector<u64> hm(2 * d);
    ck(cudaMemcpyAsync(hm.data(), mm, hm.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    for (int k = 0; k < d; ++k) {
      dim_min[k] = hm[2 * k] == ~0ull ? HUGE_VAL : sk::dkey_inv(hm[2 * k]);
      dim_max[k] = hm[2 * k + 1] == 0 ? -HUGE_VAL : sk::dkey_inv(hm[2 * k + 1]);
    }
    *n_out = b.n;
    *d_out = d;
  });
}

int skycell_gpu_write_bin(skycell_gpu_ctx* ctx, const char* path, const double* coords, uint64_t n, int d, char* err,
                          size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null context"};
    if (d < 0 || (n && !coords)) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: bad coordinate buffer"};
    FileCloser fc{open_or_throw(path, "wb", "cannot write")};
    const std::string fail = std::string("failed writing ") + path;
    unsigned char h[20] = {'S', 'K', 'Y', 'C'};
    const uint32_t version = 1, dd = (uint32_t)d;
    for (int i = 0; i < 4; ++i) h[4 + i] = (unsigned char)(version >> (8 * i));
    for (int i = 0; i < 4; ++i) h[8 + i] = (unsigned char)(dd >> (8 * i));
    for (int i = 0; i < 8; ++i) h[12 + i] = (unsigned char)((u64)n >> (8 * i));
    if (std::fwrite(h, 1, 20, fc.f) != 20) throw ApiFail{SKYCELL_IO, fail};
    const u64 values = n * (u64)d;
    cudaPointerAttributes a{};
    const bool dev = values && cudaPointerGetAttributes(&a, coords) == cudaSuccess &&
                     (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    if (!dev) {
      if (values && std::fwrite(coords, 8, values, fc.f) != values) throw ApiFail{SKYCELL_IO, fail};
    } else {
      ck(cudaSetDevice(ctx->device), "cudaSetDevice");
      cudaStream_t s = ctx->stream;
      const u64 per = kIoChunk / 8;
      double* pin[2] = {nullptr, nullptr};
      cudaEvent_t done[2] = {nullptr, nullptr};
      struct PinGuard {
        double** p;
        cudaEvent_t* e;
        ~PinGuard() {
          for (int i = 0; i < 2; ++i) {
            if (p[i]) cudaFreeHost(p[i]);
            if (e[i]) cudaEventDestroy(e[i]);
          }
        }
      } guard{pin, done};
      for (int i = 0; i < 2; ++i) {
        ck(cudaMallocHost(reinterpret_cast<void**>(&pin[i]), per * 8), "pinned");
        ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "event");
      }
      // D2H of chunk i+1 overlaps the fwrite of chunk i
      u64 at = 0, cnt0 = std::min<u64>(per, values);
      ck(cudaMemcpyAsync(pin[0], coords, cnt0 * 8, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaEventRecord(done[0], s), "event");
      int bi = 0;
      while (at < values) {
        const u64 cnt = std::min<u64>(per, values - at);
        const u64 nx = at + cnt;
        if (nx < values) {
          const u64 c2 = std::min<u64>(per, values - nx);
          ck(cudaMemcpyAsync(pin[bi ^ 1], coords + nx, c2 * 8, cudaMemcpyDeviceToHost, s), "D2H");
          ck(cudaEventRecord(done[bi ^ 1], s), "event");
        }
        ck(cudaEventSynchronize(done[bi]), "D2H");
        if (std::fwrite(pin[bi], 8, cnt, fc.f) != cnt) throw ApiFail{SKYCELL_IO, fail};
        at = nx;
        bi ^= 1;
      }
    }
    if (std::fflush(fc.f) != 0) throw ApiFail{SKYCELL_IO, fail};
  });
}

}  // extern "C"
