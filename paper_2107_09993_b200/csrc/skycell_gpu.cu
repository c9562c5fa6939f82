// Host orchestration + C ABI (include/skycell_gpu.h) of the B200 SkyCell path.
//
// One query = one pass of compute_skyline (refine.cpp:108-158) on one device:
//   validate (dataset.cpp:23-24, grid.cpp:38-43) -> K0 sample filter -> K1
//   streaming pass -> K3 cell tables + per-layer counts -> K4 candidate
//   filter -> K5 block-recursive exact dominance -> ids (ascending) + stats.
// Every data-dependent size stays on the device (kernels read their input
// counts from device memory), so the whole query is enqueued without a host
// round trip; the only synchronisation is the final read of the counters.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/skycell_gpu.h"
#include "kernels.cuh"
#include "datagen.cuh"

using sk::u64;

namespace {

constexpr int kMaxLayers = 64;
constexpr int kMaxLevels = 16;

struct DevCounters {
  u64 nonfinite;
  u64 s1, s2, examined;
  u64 zero;
  u64 zmid[kMaxLevels];
  u64 znext[kMaxLevels];
  u64 cand[kMaxLayers];
  u64 key[kMaxLayers];
};

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct Status {
  int code = SKYCELL_OK;
  std::string msg;
};

struct CudaFail {
  cudaError_t e;
  const char* what;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail{e, what};
}

void ensure(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  ck(cudaMalloc(&b.p, bytes), "cudaMalloc");
  b.cap = bytes;
}

}  // namespace

struct skycell_gpu_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  DevBuf reset, slabs, H, table, staging, out_ids;
  DevBuf s1_rows, s1_ids, s2_rows, s2_ids, s2_fsum, flags;
  DevBuf z_rows[2], z_ids[2], z_fsum[2];
  DevCounters* host_ctr = nullptr;  // pinned
  cudaEvent_t ev[6] = {};
  u64 launches = 0;
  int result_buf = 0;     // z buffer holding the last query's ids
  int result_level = 0;   // level whose znext counter is the skyline size
};

namespace {

void put_err(char* err, size_t len, const std::string& m) {
  if (!err || !len) return;
  std::strncpy(err, m.c_str(), len - 1);
  err[len - 1] = '\0';
}

// Bump allocator over the per-query zeroed region.
struct Carver {
  size_t off = 0;
  size_t take(size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) & ~size_t(255);
    return o;
  }
};

struct Slot {
  size_t claim_off, status_off;
};

// Validation in the reference's order: normalize() first (dataset.cpp:23-24),
// then the grid budget (grid.cpp:38-43).
Status validate_shape(u64 n, int d) {
  if (n < 1) return {SKYCELL_INPUT, "normalize: empty dataset"};
  if (d < 2) return {SKYCELL_INPUT, "normalize: dimensionality must be at least 2"};
  if (d > sk::kMaxD) return {SKYCELL_INPUT, "normalize: dimensionality must be at most 16"};
  if (n > 0xffffffffull) return {SKYCELL_INPUT, "normalize: more than 2^32 - 1 records"};
  return {};
}

Status validate_rho(int rho, int d) {
  if (rho < 1) return {SKYCELL_CONFIG, "grid: rho must be at least 1"};
  if (rho * d > 60)
    return {SKYCELL_CONFIG, "grid: rho*d = " + std::to_string(rho * d) + " exceeds the 60-bit cell index budget"};
  if ((rho - 1) * d > 32)
    return {SKYCELL_CONFIG, "grid: occupancy bit-sets for rho = " + std::to_string(rho) + ", d = " +
                                std::to_string(d) + " would exceed memory"};
  return {};
}

int default_rho(u64 n, int d) {
  u64 x = n > 0 ? n : 1;
  int bw = 0;
  while (x) {
    ++bw;
    x >>= 1;
  }
  return std::max(1, std::min(6, (bw - 1) / d));
}

template <typename TIn, typename TOut, bool IDENT>
struct Pipeline;

// ------------------------------------------------------------------ config
constexpr int kStreamThreads = 512;
constexpr int kThreads = 256;
constexpr u64 kLevel0 = 4096;
constexpr int kLevelGrowthLog2 = 4;

template <typename T, int D>
constexpr int ppt_for() {
  constexpr int words = D * (int)sizeof(T) / 4;
  constexpr int p = 32 / words;
  return p < 1 ? 1 : (p > 8 ? 8 : p);
}

// ----------------------------------------------------------------- query
struct Query {
  skycell_gpu_ctx* ctx;
  u64 n;
  int d, rho, mode, merge;
  bool ident;
  sk::Norm nm;
  const void* dev_coords;  // device-resident input (user's or staged)
  bool in_f32;
  bool out_f32;
  skycell_gpu_stats* stats;
  bool timed;
};

template <typename TT>
void launch_layer_tables(Query& q, uint32_t* bits, int L, TT* table, u64* cand, u64* key) {
  cudaStream_t s = q.ctx->stream;
  const int d = q.d;
  const u64 rows = 1ull << (u64)(L * (d - 1));
  const u64 words = std::max<u64>(1, (1ull << (u64)(L * d)) / 32);
  const int nsm = q.ctx->num_sms;
  auto grid_for = [&](u64 items) { return (unsigned)std::max<u64>(1, std::min<u64>((items + 255) / 256, (u64)nsm * 16)); };
  sk::k_rowmin<TT><<<grid_for(rows), 256, 0, s>>>(bits, L, rows, table);
  ++q.ctx->launches;
  for (int k = 1; k < d; ++k) {
    const u64 lines = rows >> L;
    sk::k_prefix_min<TT><<<grid_for(lines), 256, 0, s>>>(table, L, k, lines);
    ++q.ctx->launches;
  }
  sk::k_count_cells<TT><<<grid_for(words), 256, 0, s>>>(bits, L, d, words, table, cand, key);
  ++q.ctx->launches;
}

template <typename TIn, typename TOut, bool IDENT, int D>
void run_pipeline(Query& q) {
  skycell_gpu_ctx* ctx = q.ctx;
  cudaStream_t s = ctx->stream;
  const u64 n = q.n;
  const int rho = q.rho;
  const int nsm = ctx->num_sms;

  // ---- sizes
  const u64 words_rho = std::max<u64>(1, (1ull << (u64)(rho * D)) / 32);
  const int lrm1 = rho - 1;
  const u64 words_rm1 = lrm1 >= 1 ? std::max<u64>(1, (1ull << (u64)(lrm1 * D)) / 32) : 0;
  int rm1_mode = 0;
  if (lrm1 >= 1) rm1_mode = (words_rm1 * 4 <= 128 * 1024) ? 1 : 2;
  int lf = 0;
  for (int L = std::min(rho, 7); L >= 1; --L) {
    if ((1ull << (u64)(L * (D - 1))) <= 32768 && L * D <= 30) {
      lf = L;
      break;
    }
  }
  const u64 m_sample = std::min<u64>(n, 1ull << 20);
  const uint32_t h_entries = lf ? (uint32_t)(1ull << (u64)(lf * (D - 1))) : 0;
  const u64 words_lf = lf ? std::max<u64>(1, (1ull << (u64)(lf * D)) / 32) : 0;

  // ---- K1 launch geometry
  constexpr int PPT1 = ppt_for<TIn, D>();
  constexpr u64 TILE1 = (u64)kStreamThreads * PPT1;
  const u64 tiles1 = (n + TILE1 - 1) / TILE1;
  const size_t occ_smem = rm1_mode == 1 ? words_rm1 * 4 : 0;
  const size_t smem1 = occ_smem + ((h_entries + 15) & ~15u) + (PPT1 * (kStreamThreads / 32) + 1) * 4 + 16;
  auto kstream = sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1>;
  ck(cudaFuncSetAttribute(kstream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1), "smem attr");
  int occ_blocks = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_blocks, kstream, kStreamThreads, smem1), "occupancy");
  occ_blocks = std::max(1, occ_blocks);
  const int grid1 = (int)std::max<u64>(1, std::min<u64>(tiles1, (u64)nsm * occ_blocks));

  // ---- K4/K5 geometry
  constexpr int PPTc = ppt_for<TOut, D>();
  constexpr u64 TILEc = (u64)kThreads * PPTc;
  const u64 tilesc = (n + TILEc - 1) / TILEc + 1;
  std::vector<u64> bounds;
  for (u64 b = kLevel0;; b <<= kLevelGrowthLog2) {
    bounds.push_back(std::min(b, n));
    if (b >= n) break;
  }
  const int levels = (int)bounds.size();
  if (levels > kMaxLevels) throw CudaFail{cudaErrorInvalidValue, "too many levels"};
  const size_t rec = D * sizeof(TOut) + 12;
  const uint32_t f_max = (uint32_t)std::min<u64>(4096, (96 * 1024) / rec);
  const size_t smem_f = (((u64)f_max * D * sizeof(TOut) + 15) & ~15ull) + (u64)f_max * 12;

  // ---- zeroed region
  Carver cv;
  const size_t o_ctr = cv.take(sizeof(DevCounters));
  const size_t o_occ_rho = cv.take(words_rho * 4);
  const size_t o_occ_rm1 = cv.take(std::max<u64>(words_rm1, 1) * 4);
  std::vector<size_t> o_occ_layer(rho + 1, 0);
  for (int L = 1; L <= rho - 2; ++L) o_occ_layer[L] = cv.take(std::max<u64>(1, (1ull << (u64)(L * D)) / 32) * 4);
  const size_t o_occ_lf = cv.take(std::max<u64>(words_lf, 1) * 4);
  auto slot = [&](u64 tiles) { Slot sl; sl.claim_off = cv.take(8); sl.status_off = cv.take(tiles * 8); return sl; };
  const Slot sl_stream = slot(tiles1 + 1);
  const Slot sl_cand = slot(tilesc);
  std::vector<Slot> sl_filter, sl_compact;
  for (int k = 0; k < levels; ++k) {
    sl_filter.push_back(slot(tilesc));
    sl_compact.push_back(slot(tilesc));
  }
  ensure(ctx->reset, cv.off);
  char* R = static_cast<char*>(ctx->reset.p);
  auto at = [&](size_t off) { return reinterpret_cast<void*>(R + off); };
  DevCounters* ctr = static_cast<DevCounters*>(at(o_ctr));
  uint32_t* occ_rho = static_cast<uint32_t*>(at(o_occ_rho));
  uint32_t* occ_rm1 = static_cast<uint32_t*>(at(o_occ_rm1));
  uint32_t* occ_lf = static_cast<uint32_t*>(at(o_occ_lf));

  // ---- working buffers
  ensure(ctx->H, std::max<u64>(h_entries, 16));
  if (rm1_mode == 1) ensure(ctx->slabs, (size_t)grid1 * words_rm1 * 4);
  const bool small_table = rho <= 7;
  const size_t tt = small_table ? 1 : 4;
  ensure(ctx->table, (1ull << (u64)(rho * (D - 1))) * tt);
  ensure(ctx->s1_rows, n * D * sizeof(TOut));
  ensure(ctx->s1_ids, n * 4);
  ensure(ctx->s2_rows, n * D * sizeof(TOut));
  ensure(ctx->s2_ids, n * 4);
  ensure(ctx->s2_fsum, n * 8);
  ensure(ctx->flags, n);
  for (int b = 0; b < 2; ++b) {
    ensure(ctx->z_rows[b], n * D * sizeof(TOut));
    ensure(ctx->z_ids[b], n * 4);
    ensure(ctx->z_fsum[b], n * 8);
  }

  if (q.timed) ck(cudaEventRecord(ctx->ev[0], s), "event");
  ck(cudaMemsetAsync(ctx->reset.p, 0, cv.off, s), "memset");

  // ---- K0: sample filter
  if (lf > 0) {
    sk::SampleParams sp{};
    sp.coords = q.dev_coords;
    sp.m = m_sample;
    sp.rho = rho;
    sp.lf = lf;
    sp.nm = q.nm;
    sp.occ = occ_lf;
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((m_sample + 255) / 256, (u64)nsm * 8));
    sk::k_sample_occ<TIn, TOut, D, IDENT><<<g, 256, 0, s>>>(sp);
    sk::k_build_filter<<<1, 1024, h_entries, s>>>(occ_lf, lf, D, static_cast<uint8_t*>(ctx->H.p));
    ctx->launches += 2;
  }

  // ---- K1: the streaming pass
  sk::StreamParams p1{};
  p1.coords = q.dev_coords;
  p1.n = n;
  p1.rho = rho;
  p1.lf = lf;
  p1.rm1_mode = rm1_mode;
  p1.rm1_words = (uint32_t)words_rm1;
  p1.h_entries = h_entries;
  p1.nm = q.nm;
  p1.H = static_cast<const uint8_t*>(ctx->H.p);
  p1.occ_rho = occ_rho;
  p1.occ_rm1 = occ_rm1;
  p1.slabs = static_cast<uint32_t*>(ctx->slabs.p);
  p1.out_rows = ctx->s1_rows.p;
  p1.out_ids = static_cast<uint32_t*>(ctx->s1_ids.p);
  p1.status = static_cast<u64*>(at(sl_stream.status_off));
  p1.claim = static_cast<u64*>(at(sl_stream.claim_off));
  p1.out_count = &ctr->s1;
  p1.nonfinite = &ctr->nonfinite;
  kstream<<<grid1, kStreamThreads, smem1, s>>>(p1);
  ++ctx->launches;
  if (rm1_mode == 1) {
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((words_rm1 + 255) / 256, (u64)nsm * 8));
    sk::k_reduce_slabs<<<g, 256, 0, s>>>(static_cast<uint32_t*>(ctx->slabs.p), grid1, (uint32_t)words_rm1, occ_rm1);
    ++ctx->launches;
  }
  if (q.timed) ck(cudaEventRecord(ctx->ev[1], s), "event");

  // ---- K3: layer tables and per-layer counts (layers rho, rho-1, ..., 1)
  auto tables_at = [&](uint32_t* bits, int L) {
    if (L <= 7)
      launch_layer_tables<uint8_t>(q, bits, L, static_cast<uint8_t*>(ctx->table.p), &ctr->cand[L - 1], &ctr->key[L - 1]);
    else
      launch_layer_tables<uint32_t>(q, bits, L, static_cast<uint32_t*>(ctx->table.p), &ctr->cand[L - 1], &ctr->key[L - 1]);
  };
  {
    uint32_t* prev = occ_rm1;
    for (int L = rho - 2; L >= 1; --L) {
      uint32_t* dst = static_cast<uint32_t*>(at(o_occ_layer[L]));
      const u64 src_words = std::max<u64>(1, (1ull << (u64)((L + 1) * D)) / 32);
      const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((src_words + 255) / 256, (u64)nsm * 8));
      sk::k_downsample<<<g, 256, 0, s>>>(prev, L, D, src_words, dst);
      ++ctx->launches;
      prev = dst;
    }
  }
  for (int L = 1; L <= rho - 1; ++L) tables_at(L == rho - 1 ? occ_rm1 : static_cast<uint32_t*>(at(o_occ_layer[L])), L);
  tables_at(occ_rho, rho);  // last: K4 reads this table
  if (q.timed) ck(cudaEventRecord(ctx->ev[2], s), "event");

  // ---- K4: candidate-cell filter
  sk::CandParams pc{};
  pc.rows = ctx->s1_rows.p;
  pc.ids = static_cast<const uint32_t*>(ctx->s1_ids.p);
  pc.count = &ctr->s1;
  pc.rho = rho;
  pc.PM = ctx->table.p;
  pc.out_rows = ctx->s2_rows.p;
  pc.out_ids = static_cast<uint32_t*>(ctx->s2_ids.p);
  pc.out_fsum = static_cast<u64*>(ctx->s2_fsum.p);
  pc.status = static_cast<u64*>(at(sl_cand.status_off));
  pc.claim = static_cast<u64*>(at(sl_cand.claim_off));
  pc.out_count = &ctr->s2;
  pc.examined = &ctr->examined;
  const unsigned gc = (unsigned)std::max<u64>(1, std::min<u64>(tilesc, (u64)nsm * 4));
  if (small_table)
    sk::k_candidates<TOut, D, uint8_t, kThreads, PPTc><<<gc, kThreads, 0, s>>>(pc);
  else
    sk::k_candidates<TOut, D, uint32_t, kThreads, PPTc><<<gc, kThreads, 0, s>>>(pc);
  ++ctx->launches;

  // ---- K5: block-recursive exact dominance
  auto kfilter = sk::k_filter_append<TOut, D, kThreads, PPTc>;
  ck(cudaFuncSetAttribute(kfilter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f), "smem attr");
  int cur = 0;
  const u64* cnt_prev = &ctr->zero;
  for (int k = 0; k < levels; ++k) {
    const u64 b0 = k == 0 ? 0 : bounds[k - 1];
    const u64 b1 = bounds[k];
    sk::FilterParams pf{};
    pf.src_rows = ctx->s2_rows.p;
    pf.src_ids = static_cast<const uint32_t*>(ctx->s2_ids.p);
    pf.src_fsum = static_cast<const u64*>(ctx->s2_fsum.p);
    pf.src_count = &ctr->s2;
    pf.begin = b0;
    pf.end = b1;
    pf.f_rows = ctx->z_rows[cur].p;
    pf.f_ids = static_cast<const uint32_t*>(ctx->z_ids[cur].p);
    pf.f_fsum = static_cast<const u64*>(ctx->z_fsum[cur].p);
    pf.f_count = cnt_prev;
    pf.f_max = f_max;
    pf.dst_rows = ctx->z_rows[cur].p;
    pf.dst_ids = static_cast<uint32_t*>(ctx->z_ids[cur].p);
    pf.dst_fsum = static_cast<u64*>(ctx->z_fsum[cur].p);
    pf.dst_count_in = cnt_prev;
    pf.dst_count_out = &ctr->zmid[k];
    pf.status = static_cast<u64*>(at(sl_filter[k].status_off));
    pf.claim = static_cast<u64*>(at(sl_filter[k].claim_off));
    const u64 span = b1 - b0;
    const unsigned gf = (unsigned)std::max<u64>(1, std::min<u64>((span + TILEc - 1) / TILEc, (u64)nsm * 2));
    kfilter<<<gf, kThreads, smem_f, s>>>(pf);

    const u64 zmax = b1;  // |F_{k-1}| + |Y_k| <= b1
    const unsigned ga = (unsigned)std::max<u64>(1, std::min<u64>((zmax + kThreads - 1) / kThreads, (u64)nsm * 8));
    sk::k_allpairs<TOut, D, kThreads><<<ga, kThreads, 0, s>>>(
        static_cast<const TOut*>(ctx->z_rows[cur].p), static_cast<const uint32_t*>(ctx->z_ids[cur].p),
        static_cast<const u64*>(ctx->z_fsum[cur].p), &ctr->zmid[k], static_cast<uint8_t*>(ctx->flags.p));

    sk::CompactParams pk{};
    pk.src_rows = ctx->z_rows[cur].p;
    pk.src_ids = static_cast<const uint32_t*>(ctx->z_ids[cur].p);
    pk.src_fsum = static_cast<const u64*>(ctx->z_fsum[cur].p);
    pk.count = &ctr->zmid[k];
    pk.flag = static_cast<const uint8_t*>(ctx->flags.p);
    pk.dst_rows = ctx->z_rows[cur ^ 1].p;
    pk.dst_ids = static_cast<uint32_t*>(ctx->z_ids[cur ^ 1].p);
    pk.dst_fsum = static_cast<u64*>(ctx->z_fsum[cur ^ 1].p);
    pk.dst_count = &ctr->znext[k];
    pk.status = static_cast<u64*>(at(sl_compact[k].status_off));
    pk.claim = static_cast<u64*>(at(sl_compact[k].claim_off));
    const unsigned gk = (unsigned)std::max<u64>(1, std::min<u64>((zmax + TILEc - 1) / TILEc, (u64)nsm * 4));
    sk::k_compact<TOut, D, kThreads, PPTc><<<gk, kThreads, 0, s>>>(pk);
    ctx->launches += 3;
    cur ^= 1;
    cnt_prev = &ctr->znext[k];
  }
  ck(cudaGetLastError(), "kernel launch");
  if (q.timed) ck(cudaEventRecord(ctx->ev[3], s), "event");

  // ---- results
  ck(cudaMemcpyAsync(ctx->host_ctr, ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s), "counters D2H");
  ck(cudaStreamSynchronize(s), "query");
  // The skyline ids are in z_ids[cur]; their count is znext[levels - 1].
  ctx->result_buf = cur;
  ctx->result_level = levels - 1;
  const DevCounters& hc = *ctx->host_ctr;
  if (q.stats) {
    q.stats->n_layers = rho;
    for (int L = 1; L <= rho; ++L) {
      q.stats->keys[L - 1] = hc.key[L - 1] + (u64)D;
      q.stats->candidates[L - 1] = (q.mode == SKYCELL_SEQUENTIAL && L != rho) ? -1 : (int64_t)hc.cand[L - 1];
    }
    q.stats->points_examined = hc.examined;
    q.stats->survivors_stream = hc.s1;
    q.stats->survivors_filter = hc.zmid[levels - 1];
  }
}

template <typename TIn>
int run_query(skycell_gpu_ctx* ctx, const TIn* coords, u64 n, int d, const double* dmin, const double* dmax,
              int rho, int mode, int merge, uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats, char* err,
              size_t err_len) {
  try {
    Status st = validate_shape(n, d);
    if (st.code) {
      put_err(err, err_len, st.msg);
      return st.code;
    }
    if (!ctx) {
      put_err(err, err_len, "skycell_gpu: null context");
      return SKYCELL_USAGE;
    }
    if (!merge) {
      put_err(err, err_len, "skycell_gpu: merge_cross_cell=false is not implemented on the GPU path yet");
      return SKYCELL_UNSUPPORTED;
    }
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const auto t_begin = std::chrono::steady_clock::now();
    cudaStream_t s = ctx->stream;
    ctx->launches = 0;

    // Input residency: device pointers are used in place when 16-byte
    // aligned; host pointers (and misaligned device pointers) are staged.
    cudaPointerAttributes attr{};
    const bool on_device = cudaPointerGetAttributes(&attr, coords) == cudaSuccess &&
                           (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    const size_t bytes = n * (size_t)d * sizeof(TIn);
    const void* dev_coords = coords;
    if (!on_device || (reinterpret_cast<uintptr_t>(coords) & 15)) {
      ensure(ctx->staging, bytes);
      ck(cudaMemcpyAsync(ctx->staging.p, coords, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s),
         "input copy");
      dev_coords = ctx->staging.p;
    }

    Status rs = validate_rho(rho, d);
    if (rs.code) {
      // normalize() runs before the grid checks: a non-finite record wins.
      ensure(ctx->reset, 256);
      ck(cudaMemsetAsync(ctx->reset.p, 0, 8, s), "memset");
      sk::k_check_finite<TIn><<<ctx->num_sms * 4, 256, 0, s>>>(static_cast<const TIn*>(dev_coords), n * d, d,
                                                               static_cast<u64*>(ctx->reset.p));
      u64 nf = 0;
      ck(cudaMemcpyAsync(&nf, ctx->reset.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaStreamSynchronize(s), "sync");
      if (nf) {
        put_err(err, err_len, "normalize: non-finite coordinate in record " + std::to_string(~nf));
        return SKYCELL_INPUT;
      }
      put_err(err, err_len, rs.msg);
      return rs.code;
    }
    if ((u64)rho * d > 36 || (u64)rho * (d - 1) > 30) {
      put_err(err, err_len, "skycell_gpu: rho*d = " + std::to_string(rho * d) +
                                " needs the sparse cell index (dense bitmaps are limited to 2^36 cells)");
      return SKYCELL_UNSUPPORTED;
    }

    Query q{};
    q.ctx = ctx;
    q.n = n;
    q.d = d;
    q.rho = rho;
    q.mode = mode;
    q.merge = merge;
    q.stats = stats;
    q.timed = stats != nullptr;
    q.dev_coords = dev_coords;
    // scale[k] = range > 0 ? 1/range : 0, dataset.cpp:32-36 (host, FP64).
    bool ident = true;
    for (int k = 0; k < d; ++k) {
      const double range = dmax[k] - dmin[k];
      q.nm.mn[k] = dmin[k];
      q.nm.sc[k] = range > 0 ? 1.0 / range : 0.0;
      ident &= dmin[k] == 0.0 && dmax[k] == 1.0;
    }
    if (stats) std::memset(stats, 0, sizeof(*stats));

    constexpr bool kF32 = sizeof(TIn) == 4;
#define SKYCELL_CASE(DD)                                              \
  case DD:                                                            \
    if constexpr (kF32) {                                             \
      if (ident) run_pipeline<float, float, true, DD>(q);             \
      else run_pipeline<float, double, false, DD>(q);                 \
    } else {                                                          \
      run_pipeline<double, double, false, DD>(q);                     \
    }                                                                 \
    break;
    switch (d) {
      SKYCELL_CASE(2) SKYCELL_CASE(3) SKYCELL_CASE(4) SKYCELL_CASE(5) SKYCELL_CASE(6) SKYCELL_CASE(7)
      SKYCELL_CASE(8) SKYCELL_CASE(9) SKYCELL_CASE(10) SKYCELL_CASE(11) SKYCELL_CASE(12) SKYCELL_CASE(13)
      SKYCELL_CASE(14) SKYCELL_CASE(15) SKYCELL_CASE(16)
      default:
        put_err(err, err_len, "normalize: dimensionality must be at most 16");
        return SKYCELL_INPUT;
    }
#undef SKYCELL_CASE
    const DevCounters& hc = *ctx->host_ctr;
    if (hc.nonfinite) {
      put_err(err, err_len, "normalize: non-finite coordinate in record " + std::to_string(~hc.nonfinite));
      return SKYCELL_INPUT;
    }
    const u64 count = hc.znext[ctx->result_level];
    const int cur = ctx->result_buf;
    *n_out = count;
    cudaPointerAttributes oattr{};
    const bool out_dev = cudaPointerGetAttributes(&oattr, ids_out) == cudaSuccess &&
                         (oattr.type == cudaMemoryTypeDevice || oattr.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    if (count)
      ck(cudaMemcpyAsync(ids_out, ctx->z_ids[cur].p, count * 4, out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         s),
         "ids copy");
    ck(cudaStreamSynchronize(s), "sync");
    if (stats) {
      float a = 0, b = 0, c = 0;
      cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
      cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
      cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
      stats->normalize_ms = 0.0;  // fused into the streaming pass (grid_ms)
      stats->grid_ms = a;
      stats->shrink_ms = b;
      stats->refine_ms = c;
      stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
      stats->kernel_launches = ctx->launches;
    }
    return SKYCELL_OK;
  } catch (const CudaFail& f) {
    put_err(err, err_len, std::string("CUDA error in ") + f.what + ": " + cudaGetErrorString(f.e));
    cudaGetLastError();
    return SKYCELL_CUDA;
  } catch (const std::exception& e) {
    put_err(err, err_len, std::string("skycell_gpu: ") + e.what());
    return SKYCELL_CUDA;
  }
}

}  // namespace

extern "C" {

int skycell_gpu_create(int device, skycell_gpu_ctx** out, char* err, size_t err_len) {
  try {
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) {
      put_err(err, err_len, "skycell_gpu: no CUDA device " + std::to_string(device));
      return SKYCELL_CUDA;
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new skycell_gpu_ctx();
    ctx->device = device;
    ck(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
    ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    ck(cudaMallocHost(reinterpret_cast<void**>(&ctx->host_ctr), sizeof(DevCounters)), "pinned");
    for (auto& e : ctx->ev) ck(cudaEventCreate(&e), "event");
    *out = ctx;
    return SKYCELL_OK;
  } catch (const CudaFail& f) {
    put_err(err, err_len, std::string("CUDA error in ") + f.what + ": " + cudaGetErrorString(f.e));
    return SKYCELL_CUDA;
  }
}

void skycell_gpu_destroy(skycell_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  DevBuf* bufs[] = {&ctx->reset, &ctx->slabs, &ctx->H, &ctx->table, &ctx->staging, &ctx->s1_rows, &ctx->s1_ids,
                    &ctx->s2_rows, &ctx->s2_ids, &ctx->s2_fsum, &ctx->flags, &ctx->z_rows[0], &ctx->z_rows[1],
                    &ctx->z_ids[0], &ctx->z_ids[1], &ctx->z_fsum[0], &ctx->z_fsum[1]};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->host_ctr) cudaFreeHost(ctx->host_ctr);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int skycell_gpu_skyline_f64(skycell_gpu_ctx* ctx, const double* coords, uint64_t n, int d, const double* dim_min,
                            const double* dim_max, int rho, int mode, int merge_cross_cell, uint32_t* ids_out,
                            uint64_t* n_out, skycell_gpu_stats* stats, char* err, size_t err_len) {
  return run_query<double>(ctx, coords, n, d, dim_min, dim_max, rho, mode, merge_cross_cell, ids_out, n_out, stats,
                           err, err_len);
}

int skycell_gpu_skyline_f32(skycell_gpu_ctx* ctx, const float* coords, uint64_t n, int d, const double* dim_min,
                            const double* dim_max, int rho, int mode, int merge_cross_cell, uint32_t* ids_out,
                            uint64_t* n_out, skycell_gpu_stats* stats, char* err, size_t err_len) {
  return run_query<float>(ctx, coords, n, d, dim_min, dim_max, rho, mode, merge_cross_cell, ids_out, n_out, stats,
                          err, err_len);
}

int skycell_gpu_quadrant_f64(skycell_gpu_ctx*, const double*, uint64_t, int, const double*, int, int, int, uint32_t*,
                             uint64_t*, skycell_gpu_stats*, char* err, size_t err_len) {
  put_err(err, err_len, "skycell_gpu: quadrant_skyline not implemented yet");
  return SKYCELL_UNSUPPORTED;
}

int skycell_gpu_generate(skycell_gpu_ctx* ctx, int dist, uint64_t n, int d, uint64_t seed, int kind, void* dev_out,
                         char* err, size_t err_len) {
  // generate(): ConfigError on n < 1, d < 2, d > kMaxDims (datagen.cpp:63-65)
  if (n < 1) { put_err(err, err_len, "generate: n must be at least 1"); return SKYCELL_CONFIG; }
  if (d < 2) { put_err(err, err_len, "generate: d must be at least 2"); return SKYCELL_CONFIG; }
  if (d > sk::kMaxD) { put_err(err, err_len, "generate: d must be at most 16"); return SKYCELL_CONFIG; }
  if (dist < 0 || dist > 2 || kind < 0 || kind > 1 || !ctx) {
    put_err(err, err_len, "generate: bad distribution or output kind");
    return SKYCELL_USAGE;
  }
  try {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const u64 blocks = (n + 65535) / 65536;
    const unsigned g = (unsigned)std::max<u64>(1, (blocks + 127) / 128);
#define SKYCELL_GEN(DD) \
  case DD: sk::k_generate<DD><<<g, 128, 0, ctx->stream>>>(dist, n, seed, kind, dev_out); break;
    switch (d) {
      SKYCELL_GEN(2) SKYCELL_GEN(3) SKYCELL_GEN(4) SKYCELL_GEN(5) SKYCELL_GEN(6) SKYCELL_GEN(7) SKYCELL_GEN(8)
      SKYCELL_GEN(9) SKYCELL_GEN(10) SKYCELL_GEN(11) SKYCELL_GEN(12) SKYCELL_GEN(13) SKYCELL_GEN(14)
      SKYCELL_GEN(15) SKYCELL_GEN(16)
    }
#undef SKYCELL_GEN
    ck(cudaGetLastError(), "generate launch");
    ck(cudaStreamSynchronize(ctx->stream), "generate");
    return SKYCELL_OK;
  } catch (const CudaFail& f) {
    put_err(err, err_len, std::string("CUDA error in ") + f.what + ": " + cudaGetErrorString(f.e));
    cudaGetLastError();
    return SKYCELL_CUDA;
  }
}

int skycell_default_rho(uint64_t n, int d) { return default_rho(n, d); }

int skycell_validate(uint64_t n, int d, int rho, char* err, size_t err_len) {
  Status st = validate_shape(n, d);
  if (!st.code) st = validate_rho(rho, d);
  if (st.code) put_err(err, err_len, st.msg);
  return st.code;
}

const char* skycell_gpu_version(void) { return "skycell-b200 0.1 (sm_100a)"; }

}  // extern "C"
