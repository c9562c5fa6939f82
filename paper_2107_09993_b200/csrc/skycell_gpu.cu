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

struct DevCounters {
  u64 nonfinite;
  u64 s1, s2, examined;
  u64 zero;
  u64 m, xs, xs_kept, nf, fs, fin, s1_kept, s2_kept;
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
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevBuf reset, slabs, H, table, table2, table_s, staging;
  DevBuf smp_rows, smp_ids, smp_fsum, f_rows, f_fsum, f_lists, f_offs, lists, ids_dev;
  DevBuf s1_rows, s1_ids, s2_rows, s2_ids, s2_fsum, flags;
  DevCounters* host_ctr = nullptr;  // pinned
  cudaEvent_t ev[8] = {};
  u64 launches = 0;
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


// ------------------------------------------------------------------ config
constexpr int kThreads = 256;

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
  uint32_t* ids_dev;       // caller's device output buffer, or nullptr (use ctx->ids_dev)
  bool in_f32;
  bool out_f32;
  skycell_gpu_stats* stats;
  bool timed;
};

template <typename TT>
void launch_tables(skycell_gpu_ctx* ctx, cudaStream_t s, const uint32_t* bits, int L, int d, TT* table) {
  const u64 rows = 1ull << (u64)(L * (d - 1));
  const u64 lines1 = rows >> L;
  const int nsm = ctx->num_sms;
  auto grid_for = [&](u64 items) {
    return (unsigned)std::max<u64>(1, std::min<u64>((items + 127) / 128, (u64)nsm * 16));
  };
  sk::k_rowmin_prefix1<TT><<<grid_for(lines1), 128, 0, s>>>(bits, L, d, lines1, table);
  ++ctx->launches;
  for (int k = 2; k < d; ++k) {
    sk::k_prefix_min<TT><<<grid_for(lines1), 128, 0, s>>>(table, L, k, lines1);
    ++ctx->launches;
  }
}

template <typename TT>
void launch_count(skycell_gpu_ctx* ctx, cudaStream_t s, const uint32_t* bits, int L, int d, const TT* table, u64* cand,
                  u64* key) {
  const u64 words = std::max<u64>(1, (1ull << (u64)(L * d)) / 32);
  const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((words + 255) / 256, (u64)ctx->num_sms * 16));
  sk::k_count_cells<TT><<<g, 256, 0, s>>>(bits, L, d, words, table, cand, key);
  ++ctx->launches;
}

// Exact sort-first pass (refine.cpp:31-59 as applied in phase 2, :98-99) over
// a point set given as slots (ids == kNoId marks an empty slot): per-dimension
// column lists, then the list-pruned dominance test; flags[i] = 1 for members
// of the result.
template <typename TOut, int D>
void run_exact(skycell_gpu_ctx* ctx, cudaStream_t s, const void* rows, const uint32_t* ids, const u64* fsum,
               const u64* count, u64 cap, unsigned* hist, unsigned* cursor) {
  const int nsm = ctx->num_sms;
  const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((cap + 255) / 256, (u64)nsm * 8));
  const TOut* trows = static_cast<const TOut*>(rows);
  uint32_t* lists = static_cast<uint32_t*>(ctx->lists.p);
  sk::k_list_hist<TOut, D><<<g, 256, 0, s>>>(trows, ids, fsum, count, hist);
  sk::k_list_scan<<<D, 1024, 0, s>>>(hist, cursor);
  sk::k_list_scatter<TOut, D><<<g, 256, 0, s>>>(trows, ids, fsum, count, cursor, lists, cap);
  const unsigned gw = (unsigned)std::max<u64>(1, std::min<u64>((cap * 32 + 255) / 256, (u64)nsm * 8));
  sk::k_allpairs_lists<TOut, D><<<gw, 256, 0, s>>>(trows, ids, fsum, count, lists, hist, cap,
                                                   static_cast<uint8_t*>(ctx->flags.p));
  ctx->launches += 4;
}

template <typename TIn, typename TOut, bool IDENT, int D>
void run_pipeline(Query& q) {
  skycell_gpu_ctx* ctx = q.ctx;
  cudaStream_t s = ctx->stream;
  cudaStream_t s2 = ctx->side;
  const u64 n = q.n;
  const int rho = q.rho;
  const int nsm = ctx->num_sms;

  // ---- levels and sizes
  const int la = sk::filter_level(rho, D);
  const bool test_b = rho > la;
  const u64 m = std::min<u64>(n, 1ull << 20);
  const uint32_t h_entries = (uint32_t)(1ull << (u64)(la * (D - 1)));
  auto words_at = [&](int L) { return std::max<u64>(1, (1ull << (u64)(L * D)) / 32); };
  const uint32_t lo_words = la >= 2 ? (uint32_t)words_at(la - 1) : 0;
  const bool wide = rho > 7;
  const size_t tt = wide ? 4 : 1;
  const u64 table_entries = 1ull << (u64)(rho * (D - 1));

  // ---- K1 geometry: persistent warps over round-robin warp tiles
  constexpr int kStreamThreads = 256;
  constexpr int PPT1 = std::max(1, ppt_for<TIn, D>() / 2);
  const size_t smem1 = (size_t)lo_words * 4 + ((h_entries + 15) & ~15u) + 16;
  // f32 identity inputs with D <= 8 and rho <= 7 get a compile-time (rho, la) instance
  auto pick = [&]() {
    if constexpr (IDENT && D <= 8) {
      switch (rho) {
        case 1: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 1>;
        case 2: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 2>;
        case 3: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 3>;
        case 4: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 4>;
        case 5: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 5>;
        case 6: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 6>;
        case 7: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 7>;
        default: break;
      }
    }
    return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 0>;
  };
  auto kstream = pick();
  ck(cudaFuncSetAttribute(kstream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1), "smem attr");
  int occ_blocks = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_blocks, kstream, kStreamThreads, smem1), "occupancy");
  occ_blocks = std::max(1, occ_blocks);
  const u64 wtiles = (n + 32 * PPT1 - 1) / (32 * PPT1);
  const int grid1 = (int)std::max<u64>(1, std::min<u64>((wtiles + 7) / 8, (u64)nsm * occ_blocks));
  constexpr unsigned kChunk1 = 256, kChunk4 = 64;
  static_assert(kChunk1 >= 32 * PPT1, "a stream tile's survivors must fit one output chunk");
  const u64 slack1 = (u64)grid1 * (kStreamThreads / 32) * kChunk1;
  const u64 cap1 = n + slack1;

  // ---- K4 geometry
  const int grid4 = nsm * 4;
  const u64 slack4 = (u64)grid4 * (kThreads / 32) * kChunk4;
  const u64 cap4 = std::max(cap1, m) + slack4;
  const int pf_max = (int)std::min<u64>(1024, (32 * 1024) / (D * sizeof(TOut) + 8));  // K4 point filter
  const size_t smem_pf = (((u64)pf_max * D * sizeof(TOut) + 15) & ~15ull) + (u64)pf_max * 8 +
                         (u64)D * pf_max * 2 + (u64)D * (sk::kListCols + 1) * 2 + 16;
  const size_t list_words = (size_t)D * (sk::kListCols + 1);
  const size_t bin_words = (size_t)D * (sk::kListBins + 1);
  const u64 id_words = (n + 31) / 32;
  const unsigned bit_blocks = (unsigned)((id_words + sk::kBitsBlock - 1) / sk::kBitsBlock);

  // ---- zeroed region
  Carver cv;
  const size_t o_ctr = cv.take(sizeof(DevCounters));
  std::vector<size_t> o_occ(rho + 1, 0);
  for (int L = 1; L <= rho; ++L) o_occ[L] = cv.take(words_at(L) * 4);
  const size_t o_sla = cv.take(words_at(la) * 4);
  const size_t o_srho = test_b ? cv.take(words_at(rho) * 4) : 0;
  const size_t o_shist = cv.take(bin_words * 4), o_scur = cv.take(bin_words * 4);
  const size_t o_hist = cv.take(bin_words * 4), o_cur = cv.take(bin_words * 4);
  const size_t o_idbits = cv.take(id_words * 4);
  const size_t o_bcount = cv.take((size_t)bit_blocks * 4);
  ensure(ctx->reset, cv.off);
  char* R = static_cast<char*>(ctx->reset.p);
  auto at = [&](size_t off) { return reinterpret_cast<void*>(R + off); };
  auto occ = [&](int L) { return static_cast<uint32_t*>(at(o_occ[L])); };
  DevCounters* ctr = static_cast<DevCounters*>(at(o_ctr));

  // ---- working buffers
  ensure(ctx->H, std::max<u64>(h_entries, 16));
  if (lo_words) ensure(ctx->slabs, (size_t)grid1 * lo_words * 4);
  ensure(ctx->table, table_entries * tt);
  ensure(ctx->table2, table_entries * tt);
  if (test_b) ensure(ctx->table_s, table_entries * tt);
  ensure(ctx->smp_rows, m * D * sizeof(TOut));
  ensure(ctx->smp_ids, m * 4);
  ensure(ctx->smp_fsum, m * 8);
  ensure(ctx->f_rows, (size_t)pf_max * D * sizeof(TOut));
  ensure(ctx->f_fsum, (size_t)pf_max * 8);
  ensure(ctx->f_lists, (size_t)D * pf_max * 2);
  ensure(ctx->f_offs, list_words * 2);
  ensure(ctx->s1_rows, cap1 * D * sizeof(TOut));
  ensure(ctx->s1_ids, cap1 * 4);
  ensure(ctx->s2_rows, cap4 * D * sizeof(TOut));
  ensure(ctx->s2_ids, cap4 * 4);
  ensure(ctx->s2_fsum, cap4 * 8);
  ensure(ctx->flags, cap4);
  ensure(ctx->lists, (size_t)D * cap4 * 4);
  ensure(ctx->ids_dev, n * 4);

  if (q.timed) ck(cudaEventRecord(ctx->ev[0], s), "event");
  ck(cudaMemsetAsync(ctx->reset.p, 0, cv.off, s), "memset");

  // ---- K0: sample occupancy, filter tables, sample skyline -> filter points F
  {
    sk::SampleParams sp{};
    sp.coords = q.dev_coords;
    sp.m = m;
    sp.rho = rho;
    sp.la = la;
    sp.nm = q.nm;
    sp.occ_la = static_cast<uint32_t*>(at(o_sla));
    sp.occ_rho = test_b ? static_cast<uint32_t*>(at(o_srho)) : nullptr;
    sp.rows = ctx->smp_rows.p;
    sp.ids = static_cast<uint32_t*>(ctx->smp_ids.p);
    sp.fsum = static_cast<u64*>(ctx->smp_fsum.p);
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((m + 255) / 256, (u64)nsm * 8));
    sk::k_sample<TIn, TOut, D, IDENT><<<g, 256, 0, s>>>(sp);
    sk::k_build_filter<<<1, 1024, h_entries, s>>>(static_cast<uint32_t*>(at(o_sla)), la, D,
                                                  static_cast<uint8_t*>(ctx->H.p));
    ctx->launches += 2;
    if (test_b) {
      if (wide) launch_tables<uint32_t>(ctx, s, static_cast<uint32_t*>(at(o_srho)), rho, D, static_cast<uint32_t*>(ctx->table_s.p));
      else launch_tables<uint8_t>(ctx, s, static_cast<uint32_t*>(at(o_srho)), rho, D, static_cast<uint8_t*>(ctx->table_s.p));
    }
    // sample points not strictly dominated at layer rho -> X (s2 buffers)
    sk::CandParams pc{};
    pc.rows = ctx->smp_rows.p;
    pc.ids = static_cast<const uint32_t*>(ctx->smp_ids.p);
    pc.count = nullptr;
    pc.count_const = m;
    pc.rho = rho;
    pc.PM = test_b ? ctx->table_s.p : nullptr;
    pc.f_max = 0;
    pc.out_rows = ctx->s2_rows.p;
    pc.out_ids = static_cast<uint32_t*>(ctx->s2_ids.p);
    pc.out_fsum = static_cast<u64*>(ctx->s2_fsum.p);
    pc.out_reserved = &ctr->xs;
    pc.chunk = kChunk4;
    pc.kept = &ctr->xs_kept;
    pc.examined = nullptr;
    if (wide) sk::k_candidates<TOut, D, uint32_t, kThreads><<<grid4, kThreads, 16, s>>>(pc);
    else sk::k_candidates<TOut, D, uint8_t, kThreads><<<grid4, kThreads, 16, s>>>(pc);
    ++ctx->launches;
    run_exact<TOut, D>(ctx, s, ctx->s2_rows.p, static_cast<const uint32_t*>(ctx->s2_ids.p),
                       static_cast<const u64*>(ctx->s2_fsum.p), &ctr->xs, cap4, static_cast<unsigned*>(at(o_shist)),
                       static_cast<unsigned*>(at(o_scur)));
    sk::k_compact_members<TOut, D><<<nsm * 4, 256, 0, s>>>(
        static_cast<const TOut*>(ctx->s2_rows.p), static_cast<const uint32_t*>(ctx->s2_ids.p),
        static_cast<const uint8_t*>(ctx->flags.p), static_cast<const u64*>(ctx->s2_fsum.p), &ctr->xs,
        static_cast<TOut*>(ctx->smp_rows.p), static_cast<u64*>(ctx->smp_fsum.p), &ctr->fs);
    sk::k_strength_order<TOut, D><<<1, 1024, 0, s>>>(
        static_cast<const TOut*>(ctx->smp_rows.p), static_cast<const u64*>(ctx->smp_fsum.p), &ctr->fs,
        (uint32_t)pf_max, static_cast<TOut*>(ctx->f_rows.p), static_cast<u64*>(ctx->f_fsum.p), &ctr->nf,
        static_cast<uint16_t*>(ctx->f_lists.p), static_cast<uint16_t*>(ctx->f_offs.p));
    ++ctx->launches;
    ++ctx->launches;
  }

  // ---- K1: the streaming pass
  sk::StreamParams p1{};
  p1.coords = q.dev_coords;
  p1.n = n;
  p1.rho = rho;
  p1.la = la;
  p1.lo_words = lo_words;
  p1.h_entries = h_entries;
  p1.nm = q.nm;
  p1.H = static_cast<const uint8_t*>(ctx->H.p);
  p1.PMs = test_b ? ctx->table_s.p : nullptr;
  p1.pms_wide = wide;
  p1.occ_rho = occ(rho);
  p1.occ_rm1 = rho >= 2 ? occ(rho - 1) : nullptr;
  p1.slabs = static_cast<uint32_t*>(ctx->slabs.p);
  p1.out_rows = ctx->s1_rows.p;
  p1.out_ids = static_cast<uint32_t*>(ctx->s1_ids.p);
  p1.out_reserved = &ctr->s1;
  p1.chunk = kChunk1;
  p1.kept = &ctr->s1_kept;
  p1.nonfinite = &ctr->nonfinite;
  if (q.timed) ck(cudaEventRecord(ctx->ev[4], s), "event");
  kstream<<<grid1, kStreamThreads, smem1, s>>>(p1);
  ++ctx->launches;
  if (q.timed) ck(cudaEventRecord(ctx->ev[5], s), "event");
  if (lo_words) {
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((lo_words + 255) / 256, (u64)nsm * 8));
    sk::k_reduce_slabs<<<g, 256, 0, s>>>(static_cast<uint32_t*>(ctx->slabs.p), grid1, lo_words, occ(la - 1));
    ++ctx->launches;
  }
  if (q.timed) ck(cudaEventRecord(ctx->ev[1], s), "event");

  // ---- K3: layer-rho prefix-min table of the survivors' occupancy
  if (wide) launch_tables<uint32_t>(ctx, s, occ(rho), rho, D, static_cast<uint32_t*>(ctx->table.p));
  else launch_tables<uint8_t>(ctx, s, occ(rho), rho, D, static_cast<uint8_t*>(ctx->table.p));
  if (q.timed) ck(cudaEventRecord(ctx->ev[2], s), "event");

  // ---- side stream: per-layer |KS_i|, |CS_i| (refine.cpp:125-147), overlapped with K4/K5.
  // Layer rho from O'_rho; below, O'_rho is OR-ed down into the partial
  // occupancies recorded by the filter.
  ck(cudaEventRecord(ctx->ev_fork, s), "event");
  ck(cudaStreamWaitEvent(s2, ctx->ev_fork, 0), "wait");
  {
    if (wide) launch_count<uint32_t>(ctx, s2, occ(rho), rho, D, static_cast<const uint32_t*>(ctx->table.p), &ctr->cand[rho - 1], &ctr->key[rho - 1]);
    else launch_count<uint8_t>(ctx, s2, occ(rho), rho, D, static_cast<const uint8_t*>(ctx->table.p), &ctr->cand[rho - 1], &ctr->key[rho - 1]);
    for (int L = rho - 1; L >= 1; --L) {
      const u64 src_words = words_at(L + 1);
      const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((src_words + 255) / 256, (u64)nsm * 8));
      sk::k_downsample<<<g, 256, 0, s2>>>(occ(L + 1), L, D, src_words, occ(L));
      ++ctx->launches;
      if (L > 7) {
        launch_tables<uint32_t>(ctx, s2, occ(L), L, D, static_cast<uint32_t*>(ctx->table2.p));
        launch_count<uint32_t>(ctx, s2, occ(L), L, D, static_cast<const uint32_t*>(ctx->table2.p), &ctr->cand[L - 1], &ctr->key[L - 1]);
      } else {
        launch_tables<uint8_t>(ctx, s2, occ(L), L, D, static_cast<uint8_t*>(ctx->table2.p));
        launch_count<uint8_t>(ctx, s2, occ(L), L, D, static_cast<const uint8_t*>(ctx->table2.p), &ctr->cand[L - 1], &ctr->key[L - 1]);
      }
    }
  }
  ck(cudaEventRecord(ctx->ev_join, s2), "event");

  // ---- K4: candidate cells + sample-skyline point filter
  {
    sk::CandParams pc{};
    pc.rows = ctx->s1_rows.p;
    pc.ids = static_cast<const uint32_t*>(ctx->s1_ids.p);
    pc.count = &ctr->s1;
    pc.rho = rho;
    pc.PM = ctx->table.p;
    pc.f_rows = ctx->f_rows.p;
    pc.f_fsum = static_cast<const u64*>(ctx->f_fsum.p);
    pc.f_count = &ctr->nf;
    pc.f_max = (uint32_t)pf_max;
    pc.f_lists = static_cast<const uint16_t*>(ctx->f_lists.p);
    pc.f_offs = static_cast<const uint16_t*>(ctx->f_offs.p);
    pc.out_rows = ctx->s2_rows.p;
    pc.out_ids = static_cast<uint32_t*>(ctx->s2_ids.p);
    pc.out_fsum = static_cast<u64*>(ctx->s2_fsum.p);
    pc.out_reserved = &ctr->s2;
    pc.chunk = kChunk4;
    pc.kept = &ctr->s2_kept;
    pc.examined = &ctr->examined;
    if (wide) {
      auto kc = sk::k_candidates<TOut, D, uint32_t, kThreads>;
      ck(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pf), "smem attr");
      kc<<<grid4, kThreads, smem_pf, s>>>(pc);
    } else {
      auto kc = sk::k_candidates<TOut, D, uint8_t, kThreads>;
      ck(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pf), "smem attr");
      kc<<<grid4, kThreads, smem_pf, s>>>(pc);
    }
    ++ctx->launches;
  }

  // ---- K5: exact sort-first pass over the remaining points
  run_exact<TOut, D>(ctx, s, ctx->s2_rows.p, static_cast<const uint32_t*>(ctx->s2_ids.p),
                     static_cast<const u64*>(ctx->s2_fsum.p), &ctr->s2, cap4, static_cast<unsigned*>(at(o_hist)),
                     static_cast<unsigned*>(at(o_cur)));
  // ---- K6: ids in ascending order through the id bitmap
  {
    uint32_t* idbits = static_cast<uint32_t*>(at(o_idbits));
    unsigned* bcount = static_cast<unsigned*>(at(o_bcount));
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((cap4 + 255) / 256, (u64)nsm * 8));
    sk::k_mark_ids<<<g, 256, 0, s>>>(static_cast<const uint32_t*>(ctx->s2_ids.p),
                                     static_cast<const uint8_t*>(ctx->flags.p), &ctr->s2, idbits);
    sk::k_bits_count<<<bit_blocks, sk::kBitsThreads, 0, s>>>(idbits, id_words, bcount);
    sk::k_bits_scan<<<1, 1024, 0, s>>>(bcount, bit_blocks, &ctr->fin);
    sk::k_bits_write<<<bit_blocks, sk::kBitsThreads, 0, s>>>(idbits, id_words, bcount,
                                                              q.ids_dev ? q.ids_dev : static_cast<uint32_t*>(ctx->ids_dev.p));
    ctx->launches += 4;
  }
  ck(cudaGetLastError(), "kernel launch");
  if (q.timed) ck(cudaEventRecord(ctx->ev[3], s), "event");
  ck(cudaStreamWaitEvent(s, ctx->ev_join, 0), "join");

  // ---- results
  ck(cudaMemcpyAsync(ctx->host_ctr, ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s), "counters D2H");
  ck(cudaStreamSynchronize(s), "query");
  const DevCounters& hc = *ctx->host_ctr;
  if (q.stats) {
    q.stats->n_layers = rho;
    for (int L = 1; L <= rho; ++L) {
      q.stats->keys[L - 1] = hc.key[L - 1] + (u64)D;
      q.stats->candidates[L - 1] = (q.mode == SKYCELL_SEQUENTIAL && L != rho) ? -1 : (int64_t)hc.cand[L - 1];
    }
    q.stats->points_examined = hc.examined;
    q.stats->survivors_stream = hc.s1_kept;
    q.stats->survivors_filter = hc.s2_kept;
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
    cudaPointerAttributes oattr{};
    const bool out_dev = cudaPointerGetAttributes(&oattr, ids_out) == cudaSuccess &&
                         (oattr.type == cudaMemoryTypeDevice || oattr.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    q.ids_dev = out_dev ? ids_out : nullptr;
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
    const u64 count = hc.fin;
    *n_out = count;
    if (count && !out_dev) {
      ck(cudaMemcpyAsync(ids_out, ctx->ids_dev.p, count * 4, cudaMemcpyDeviceToHost, s), "ids copy");
      ck(cudaStreamSynchronize(s), "sync");
    }
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
      float k1 = 0;
      cudaEventElapsedTime(&k1, ctx->ev[4], ctx->ev[5]);
      stats->stream_kernel_ms = k1;
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
    ck(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming), "event");
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
  DevBuf* bufs[] = {&ctx->reset, &ctx->slabs, &ctx->H, &ctx->table, &ctx->table2, &ctx->table_s, &ctx->staging,
                    &ctx->smp_rows, &ctx->smp_ids, &ctx->smp_fsum, &ctx->f_rows, &ctx->f_fsum, &ctx->f_lists, &ctx->f_offs,
                    &ctx->lists, &ctx->ids_dev, &ctx->s1_rows, &ctx->s1_ids,
                    &ctx->s2_rows, &ctx->s2_ids, &ctx->s2_fsum, &ctx->flags};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->host_ctr) cudaFreeHost(ctx->host_ctr);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->side) cudaStreamDestroy(ctx->side);
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
