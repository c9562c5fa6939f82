// MultiLayerGrid drop-in (grid.hpp:33-70, grid.cpp:35-140).
//
// The query path never needs the reference's grid object -- its ids do not
// depend on the Morton order (grid.hpp:27-28) -- but a caller of
// MultiLayerGrid's accessors does.  The build is the reference's, on the
// device:
//   * points sorted by the Z-order key of their layer-rho cell
//     (morton_key, grid.cpp:18-28), ties by input position -- a stable LSD
//     radix sort of (key, position) gives exactly the reference's order;
//   * per non-empty layer-rho cell the contiguous range [begin, end) of the
//     sorted points (grid.cpp:66-72), held as arrays sorted by linear index
//     instead of an unordered_map;
//   * occupancy bitmaps of the layers below by child-OR (grid.cpp:76-102),
//     the same word-parallel downsampling K3 uses.
// Accessors: occupied / range lookups in batches on the device, non-empty
// cells per layer in enumeration order (ascending linear index = lex_less),
// non-empty counts, the sorted PointSet.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "engine.cuh"

using sk::u64;

struct skycell_gpu_grid {
  int device = 0;
  int d = 0, rho = 0;
  u64 n = 0, nleaf = 0;
  skyeng::DevBuf coords, ids;                  // sorted PointSet
  skyeng::DevBuf leaf_lin, leaf_begin, leaf_end;  // non-empty layer-rho cells, ascending linear index
  std::vector<skyeng::DevBuf> occ;            // layers 0 .. rho-1 (u32 words)
  std::vector<u64> nonempty;                  // layers 0 .. rho
};

namespace skyeng {

// Layer-L columns of a normalised point: (int32)(u * 2^L) (point_to_cell,
// grid.cpp:10-16).  The linear index has dim d-1 most significant
// (cell.hpp:102-107).
__device__ __forceinline__ int32_t grid_col(double u, double scale) { return (int32_t)(u * scale); }

static __global__ void k_grid_keys(const double* __restrict__ coords, u64 n, int d, int rho, u64* __restrict__ keys,
                                   uint32_t* __restrict__ vals) {
  sk::pdl_enter();
  const double scale = ldexp(1.0, rho);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 key = 0;
    for (int k = 0; k < d; ++k) {
      const uint32_t c = (uint32_t)grid_col(coords[i * d + k], scale);
      // bit b of dim k -> key bit b*d + k (morton_key, grid.cpp:18-28)
      for (int b = 0; b < rho; ++b) key |= (u64)((c >> b) & 1u) << (b * d + k);
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
  }
}

static __global__ void k_grid_gather(const double* __restrict__ coords, const uint32_t* __restrict__ ids,
                                     const uint32_t* __restrict__ order, u64 n, int d, double* __restrict__ scoords,
                                     uint32_t* __restrict__ sids) {
  sk::pdl_enter();
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    const uint32_t i = order[j];
    for (int k = 0; k < d; ++k) scoords[j * d + k] = coords[(u64)i * d + k];
    sids[j] = ids ? ids[i] : i;
  }
}

static __global__ void k_grid_heads(const u64* __restrict__ keys, u64 n, uint32_t* __restrict__ head) {
  sk::pdl_enter();
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x)
    head[j] = j == 0 || keys[j] != keys[j - 1];
}

// Run r = cpos[j] - 1 at each head j: its linear index (from the sorted
// point's columns) and its range.
static __global__ void k_grid_runs(const double* __restrict__ scoords, const uint32_t* __restrict__ head,
                                   const uint32_t* __restrict__ cpos, u64 n, int d, int rho, u64* __restrict__ lin,
                                   uint32_t* __restrict__ begin, uint32_t* __restrict__ end) {
  sk::pdl_enter();
  const double scale = ldexp(1.0, rho);
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < n; j += (u64)gridDim.x * blockDim.x) {
    const uint32_t r = cpos[j] - 1;
    if (j + 1 == n || head[j + 1]) end[r] = (uint32_t)(j + 1);
    if (!head[j]) continue;
    u64 li = 0;
    for (int k = d - 1; k >= 0; --k) li = (li << rho) | (u64)(uint32_t)grid_col(scoords[j * d + k], scale);
    lin[r] = li;
    begin[r] = (uint32_t)j;
  }
}

static __global__ void k_grid_iota(uint32_t* __restrict__ v, u64 m) {
  sk::pdl_enter();
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < m; r += (u64)gridDim.x * blockDim.x) v[r] = (uint32_t)r;
}

static __global__ void k_grid_permute(const uint32_t* __restrict__ src, const uint32_t* __restrict__ order, u64 m,
                                      uint32_t* __restrict__ dst) {
  sk::pdl_enter();
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < m; r += (u64)gridDim.x * blockDim.x)
    dst[r] = src[order[r]];
}

// Layer rho-1 occupancy: the parent of every non-empty leaf (grid.cpp:84-86).
static __global__ void k_grid_parents(const u64* __restrict__ lin, u64 m, int d, int rho, uint32_t* __restrict__ occ) {
  sk::pdl_enter();
  const u64 mask = (1ull << rho) - 1;
  for (u64 r = blockIdx.x * (u64)blockDim.x + threadIdx.x; r < m; r += (u64)gridDim.x * blockDim.x) {
    u64 p = 0;
    for (int k = d - 1; k >= 0; --k) p = (p << (rho - 1)) | (((lin[r] >> (rho * k)) & mask) >> 1);
    sk::set_bit_global(occ, p);
  }
}

static __global__ void k_grid_popc(const uint32_t* __restrict__ bits, u64 words, u64* __restrict__ out) {
  sk::pdl_enter();
  u64 c = 0;
  for (u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x; w < words; w += (u64)gridDim.x * blockDim.x)
    c += __popc(bits[w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(sk::kFull, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Batched lookups.  Layer rho: binary search of the sorted leaf indices
// (range / occupied); below: the bitmap.
static __global__ void k_grid_lookup(const u64* __restrict__ q, u64 nq, const u64* __restrict__ lin, u64 m,
                                     const uint32_t* __restrict__ begin, const uint32_t* __restrict__ end,
                                     const uint32_t* __restrict__ bits, uint32_t* __restrict__ out_begin,
                                     uint32_t* __restrict__ out_end, uint8_t* __restrict__ out_occ) {
  sk::pdl_enter();
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nq; i += (u64)gridDim.x * blockDim.x) {
    const u64 x = q[i];
    if (bits) {
      out_occ[i] = (bits[x >> 5] >> (x & 31)) & 1u;
      continue;
    }
    u64 lo = 0, hi = m;
    while (lo < hi) {
      const u64 mid = (lo + hi) >> 1;
      if (lin[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    const bool hit = lo < m && lin[lo] == x;
    if (out_occ) out_occ[i] = hit;
    if (out_begin) {
      out_begin[i] = hit ? begin[lo] : 0;
      out_end[i] = hit ? end[lo] : 0;
    }
  }
}

inline u64 words_of(int L, int d) { return std::max<u64>(1, ((1ull << (u64)(L * d)) + 31) / 32); }

inline void to_host_or_device(void* dst, const void* src, u64 bytes, cudaStream_t s) {
  cudaPointerAttributes a{};
  const bool dev = cudaPointerGetAttributes(&a, dst) == cudaSuccess &&
                   (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
  cudaGetLastError();
  ck(cudaMemcpyAsync(dst, src, bytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s), "copy out");
}

}  // namespace skyeng

using namespace skyeng;

extern "C" {

int skycell_gpu_grid_build(skycell_gpu_ctx* ctx, const double* coords, const uint32_t* ids, uint64_t n, int d, int rho,
                           skycell_gpu_grid** out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx || !out) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null context or output handle"};
    if (d < 1 || d > sk::kMaxD) throw ApiFail{SKYCELL_INPUT, "grid: dimensionality must be 1..16"};
    // the reference's constructor checks (grid.cpp:38-43)
    Status rs = validate_rho(rho, d);
    if (rs.code) throw ApiFail{rs.code, rs.msg};
    if (n > 0xffffffffull) throw ApiFail{SKYCELL_INPUT, "normalize: more than 2^32 - 1 records"};
    if (n && !coords) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null coordinates"};
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = ctx->stream;
    std::unique_ptr<skycell_gpu_grid> g(new skycell_gpu_grid());
    g->device = ctx->device;
    g->d = d;
    g->rho = rho;
    g->n = n;
    const u64 nn = std::max<u64>(n, 1);
    const int nsm = ctx->num_sms;
    const unsigned gr = (unsigned)std::max<u64>(1, std::min<u64>((nn + 255) / 256, (u64)nsm * 8));
    // inputs on the device
    DevBuf in_c, in_i, keys, keys2, vals, vals2, head, cpos, lin_r, beg_r, end_r, tmp;
    ensure(in_c, nn * d * 8);
    ck(cudaMemcpyAsync(in_c.p, coords, n * d * 8, cudaMemcpyDefault, s), "coords in");
    const uint32_t* dev_ids = nullptr;
    if (ids) {
      ensure(in_i, nn * 4);
      ck(cudaMemcpyAsync(in_i.p, ids, n * 4, cudaMemcpyDefault, s), "ids in");
      dev_ids = static_cast<const uint32_t*>(in_i.p);
    }
    ensure(keys, nn * 8);
    ensure(keys2, nn * 8);
    ensure(vals, nn * 4);
    ensure(vals2, nn * 4);
    ensure(g->coords, nn * d * 8);
    ensure(g->ids, nn * 4);
    if (n) {
      sk::launch(k_grid_keys, gr, 256, 0, s, static_cast<const double*>(in_c.p), n, d, rho, static_cast<u64*>(keys.p),
                                     static_cast<uint32_t*>(vals.p));
      size_t t1 = 0, t2 = 0;
      ck(cub::DeviceRadixSort::SortPairs(nullptr, t1, static_cast<u64*>(keys.p), static_cast<u64*>(keys2.p),
                                         static_cast<uint32_t*>(vals.p), static_cast<uint32_t*>(vals2.p), (int64_t)n, 0,
                                         rho * d, s),
         "cub");
      ck(cub::DeviceScan::InclusiveSum(nullptr, t2, static_cast<uint32_t*>(vals.p), static_cast<uint32_t*>(vals.p),
                                       (int64_t)n, s),
         "cub");
      ensure(tmp, std::max(t1, t2));
      // stable LSD sort: equal keys keep ascending input position (the
      // reference's (key, position) order, grid.cpp:47-54)
      ck(cub::DeviceRadixSort::SortPairs(tmp.p, t1, static_cast<u64*>(keys.p), static_cast<u64*>(keys2.p),
                                         static_cast<uint32_t*>(vals.p), static_cast<uint32_t*>(vals2.p), (int64_t)n, 0,
                                         rho * d, s),
         "cub sort");
      sk::launch(k_grid_gather, gr, 256, 0, s, static_cast<const double*>(in_c.p), dev_ids,
                                       static_cast<const uint32_t*>(vals2.p), n, d, static_cast<double*>(g->coords.p),
                                       static_cast<uint32_t*>(g->ids.p));
      ensure(head, nn * 4);
      ensure(cpos, nn * 4);
      sk::launch(k_grid_heads, gr, 256, 0, s, static_cast<const u64*>(keys2.p), n, static_cast<uint32_t*>(head.p));
      ck(cub::DeviceScan::InclusiveSum(tmp.p, t2, static_cast<uint32_t*>(head.p), static_cast<uint32_t*>(cpos.p),
                                       (int64_t)n, s),
         "cub scan");
      uint32_t runs = 0;
      ck(cudaMemcpyAsync(&runs, static_cast<uint32_t*>(cpos.p) + (n - 1), 4, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaStreamSynchronize(s), "sync");
      g->nleaf = runs;
      ensure(lin_r, (u64)runs * 8);
      ensure(beg_r, (u64)runs * 4);
      ensure(end_r, (u64)runs * 4);
      sk::launch(k_grid_runs, gr, 256, 0, s, static_cast<const double*>(g->coords.p), static_cast<const uint32_t*>(head.p),
                                     static_cast<const uint32_t*>(cpos.p), n, d, rho, static_cast<u64*>(lin_r.p),
                                     static_cast<uint32_t*>(beg_r.p), static_cast<uint32_t*>(end_r.p));
      // leaves by linear index (enumeration order): sort (lin, run)
      uint32_t* rid = static_cast<uint32_t*>(vals.p);
      uint32_t* rid2 = static_cast<uint32_t*>(head.p);
      const unsigned gl = (unsigned)std::max<u64>(1, std::min<u64>((runs + 255) / 256, (u64)nsm * 8));
      ensure(g->leaf_lin, (u64)runs * 8);
      ensure(g->leaf_begin, (u64)runs * 4);
      ensure(g->leaf_end, (u64)runs * 4);
      sk::launch(k_grid_iota, gl, 256, 0, s, rid, runs);
      size_t t3 = 0;
      ck(cub::DeviceRadixSort::SortPairs(nullptr, t3, static_cast<u64*>(lin_r.p), static_cast<u64*>(g->leaf_lin.p), rid,
                                         rid2, (int64_t)runs, 0, rho * d, s),
         "cub");
      ensure(tmp, t3);
      ck(cub::DeviceRadixSort::SortPairs(tmp.p, t3, static_cast<u64*>(lin_r.p), static_cast<u64*>(g->leaf_lin.p), rid,
                                         rid2, (int64_t)runs, 0, rho * d, s),
         "cub sort");
      sk::launch(k_grid_permute, gl, 256, 0, s, static_cast<const uint32_t*>(beg_r.p), rid2, runs,
                                        static_cast<uint32_t*>(g->leaf_begin.p));
      sk::launch(k_grid_permute, gl, 256, 0, s, static_cast<const uint32_t*>(end_r.p), rid2, runs,
                                        static_cast<uint32_t*>(g->leaf_end.p));
    }
    // occupancy of layers 0 .. rho-1 by child-OR
    g->occ.resize(rho);
    g->nonempty.assign(rho + 1, 0);
    ensure(tmp, std::max<size_t>(tmp.cap, 8 * (rho + 1)));
    u64* cnt = static_cast<u64*>(tmp.p);
    ck(cudaMemsetAsync(cnt, 0, 8 * (rho + 1), s), "memset");
    for (int L = rho - 1; L >= 0; --L) {
      const u64 words = words_of(L, d);
      ensure(g->occ[L], words * 4);
      uint32_t* dst = static_cast<uint32_t*>(g->occ[L].p);
      ck(cudaMemsetAsync(dst, 0, words * 4, s), "memset");
      if (!n) continue;
      if (L == rho - 1) {
        const unsigned gl = (unsigned)std::max<u64>(1, std::min<u64>((g->nleaf + 255) / 256, (u64)nsm * 8));
        sk::launch(k_grid_parents, gl, 256, 0, s, static_cast<const u64*>(g->leaf_lin.p), g->nleaf, d, rho, dst);
      } else {
        const uint32_t* src = static_cast<const uint32_t*>(g->occ[L + 1].p);
        const u64 sw = words_of(L + 1, d);
        if (L >= 5) {
          const unsigned gw = (unsigned)std::max<u64>(1, std::min<u64>((words + 255) / 256, (u64)nsm * 8));
          sk::launch(sk::k_downsample_words, gw, 256, 0, s, src, L, d, words, dst);
        } else {
          const unsigned gw = (unsigned)std::max<u64>(1, std::min<u64>((sw + 255) / 256, (u64)nsm * 8));
          sk::launch(sk::k_downsample, gw, 256, 0, s, src, L, d, sw, dst);
        }
      }
      const unsigned gp = (unsigned)std::max<u64>(1, std::min<u64>((words + 255) / 256, (u64)nsm * 8));
      sk::launch(k_grid_popc, gp, 256, 0, s, dst, words, cnt + L);
    }
    ck(cudaGetLastError(), "kernel launch");
    ck(cudaMemcpyAsync(g->nonempty.data(), cnt, 8 * rho, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    g->nonempty[rho] = g->nleaf;
    for (DevBuf* b : {&in_c, &in_i, &keys, &keys2, &vals, &vals2, &head, &cpos, &lin_r, &beg_r, &end_r, &tmp})
      if (b->p) cudaFree(b->p);
    *out = g.release();
  });
}

void skycell_gpu_grid_destroy(skycell_gpu_grid* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  for (DevBuf* b : {&g->coords, &g->ids, &g->leaf_lin, &g->leaf_begin, &g->leaf_end})
    if (b->p) cudaFree(b->p);
  for (auto& b : g->occ)
    if (b.p) cudaFree(b.p);
  delete g;
}

int skycell_gpu_grid_shape(const skycell_gpu_grid* g, uint64_t* n, int* d, int* rho) {
  if (!g) return SKYCELL_USAGE;
  if (n) *n = g->n;
  if (d) *d = g->d;
  if (rho) *rho = g->rho;
  return SKYCELL_OK;
}

uint64_t skycell_gpu_grid_nonempty_count(const skycell_gpu_grid* g, int layer) {
  if (!g || layer < 0 || layer > g->rho) return 0;
  return g->nonempty[layer];
}

int skycell_gpu_grid_points(skycell_gpu_grid* g, double* coords_out, uint32_t* ids_out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!g) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null grid"};
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    if (g->n && coords_out) to_host_or_device(coords_out, g->coords.p, g->n * g->d * 8, 0);
    if (g->n && ids_out) to_host_or_device(ids_out, g->ids.p, g->n * 4, 0);
    ck(cudaStreamSynchronize(0), "sync");
  });
}

int skycell_gpu_grid_nonempty_cells(skycell_gpu_grid* g, int layer, uint64_t* lin_out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!g || !lin_out) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null grid or output"};
    if (layer < 0 || layer > g->rho) throw ApiFail{SKYCELL_USAGE, "grid: layer out of range"};
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    const u64 m = g->nonempty[layer];
    if (!m) return;
    if (layer == g->rho) {
      ck(cudaMemcpy(lin_out, g->leaf_lin.p, m * 8, cudaMemcpyDefault), "copy");
      return;
    }
    // ascending set bits of the layer bitmap (K6's popcount scan)
    const u64 words = words_of(layer, g->d);
    const unsigned blocks = (unsigned)((words + sk::kBitsBlock - 1) / sk::kBitsBlock);
    DevBuf bc, tot, ids32;
    ensure(bc, (u64)blocks * 4);
    ensure(tot, 8);
    ensure(ids32, m * 4);
    sk::launch(sk::k_bits_count, blocks, sk::kBitsThreads, 0, 0, static_cast<const uint32_t*>(g->occ[layer].p), words,
                                                   static_cast<unsigned*>(bc.p));
    sk::launch(sk::k_bits_scan, 1, 1024, 0, 0, static_cast<unsigned*>(bc.p), blocks, static_cast<u64*>(tot.p));
    sk::launch(sk::k_bits_write, blocks, sk::kBitsThreads, 0, 0, static_cast<const uint32_t*>(g->occ[layer].p), words,
                                                   static_cast<const unsigned*>(bc.p),
                                                   static_cast<uint32_t*>(ids32.p), 0);
    ck(cudaGetLastError(), "kernel launch");
    std::vector<uint32_t> h(m);
    ck(cudaMemcpy(h.data(), ids32.p, m * 4, cudaMemcpyDeviceToHost), "copy");
    for (u64 i = 0; i < m; ++i) lin_out[i] = h[i];
    for (DevBuf* b : {&bc, &tot, &ids32}) cudaFree(b->p);
  });
}

int skycell_gpu_grid_lookup(skycell_gpu_grid* g, int layer, const uint64_t* lin, uint64_t count, uint8_t* occupied,
                            uint32_t* begin, uint32_t* end, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!g) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null grid"};
    if (layer < 0 || layer > g->rho) throw ApiFail{SKYCELL_USAGE, "grid: layer out of range"};
    if ((begin || end) && layer != g->rho) throw ApiFail{SKYCELL_USAGE, "range: only layer-rho cells carry point ranges"};
    if (!count) return;
    if (!lin) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null cell list"};
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    const u64 cells = 1ull << (u64)(layer * g->d);
    for (u64 i = 0; i < count; ++i)
      if (lin[i] >= cells) throw ApiFail{SKYCELL_USAGE, "grid: linear index outside the layer"};
    DevBuf q, ob, oe, oo;
    ensure(q, count * 8);
    ensure(oo, count);
    ck(cudaMemcpy(q.p, lin, count * 8, cudaMemcpyDefault), "copy");
    if (begin) {
      ensure(ob, count * 4);
      ensure(oe, count * 4);
    }
    const unsigned gq = (unsigned)std::max<u64>(1, std::min<u64>((count + 255) / 256, 1184));
    sk::launch(k_grid_lookup, gq, 256, 0, 0, static_cast<const u64*>(q.p), count, static_cast<const u64*>(g->leaf_lin.p), g->nleaf,
                               static_cast<const uint32_t*>(g->leaf_begin.p), static_cast<const uint32_t*>(g->leaf_end.p),
                               layer == g->rho ? nullptr : static_cast<const uint32_t*>(g->occ[layer].p),
                               static_cast<uint32_t*>(ob.p), static_cast<uint32_t*>(oe.p), static_cast<uint8_t*>(oo.p));
    ck(cudaGetLastError(), "kernel launch");
    if (occupied) ck(cudaMemcpy(occupied, oo.p, count, cudaMemcpyDefault), "copy");
    if (begin) ck(cudaMemcpy(begin, ob.p, count * 4, cudaMemcpyDefault), "copy");
    if (end) ck(cudaMemcpy(end, oe.p, count * 4, cudaMemcpyDefault), "copy");
    for (DevBuf* b : {&q, &ob, &oe, &oo})
      if (b->p) cudaFree(b->p);
  });
}

}  // extern "C"
