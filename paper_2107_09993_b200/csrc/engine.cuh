// Internal engine of the B200 SkyCell path: device context, scratch
// buffers and the per-query pipeline (Pipe).  Included by the C-ABI TU
// (skycell_gpu.cu) and by inst.cu, which instantiates the pipeline once per
// dimensionality (one TU per D, compiled in parallel).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/skycell_gpu.h"
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "kernels.cuh"
#include "sparse.cuh"
#include "datagen.cuh"

using sk::u64;

namespace skyeng {

constexpr int kMaxLayers = 64;

struct DevCounters {
  u64 nonfinite;
  u64 s1, s2, examined;
  u64 zero;
  u64 m, xs, xs_kept, nf, fs, fin, s1_kept, s2_kept;
  u64 lsky;       // local skyline size (sharded)
  u64 tvalid;     // valid slots of the set a dominance tree is built over
  u64 tkilled;    // ... removed by the champion prefilter (must follow tvalid)
  u64 dres;       // D-stream slots handed out (K1 filter-point head)
  u64 xd, xs_cap; // sample candidates (dense) / those entering the sample skyline (capped)
  u64 pres, pkept;  // K4a -> K4b pending stream: slots handed out / points written
  u64 un, qend;   // union slots and own-slice end (sharded finish)
  u64 fweak;      // the filter points kill little (k_filter_gate): K4a -> S2 directly
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

struct ApiFail {
  int code;
  std::string msg;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail{e, what};
}

// Grow-only scratch buffers.  Growth takes 25% headroom: data-dependent sizes
// (survivor slot counts) vary slightly from query to query, and a cudaFree /
// cudaMalloc pair inside a query would synchronise the device.
inline void ensure(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  const size_t want = bytes + bytes / 4;
  if (cudaMalloc(&b.p, want) == cudaSuccess) {
    b.cap = want;
    return;
  }
  cudaGetLastError();
  ck(cudaMalloc(&b.p, bytes), "cudaMalloc");
  b.cap = bytes;
}

// Small fills as a PDL kernel rather than cudaMemsetAsync: a memset node
// breaks the programmatic-launch chain (a 2-3 us gap on each side).
inline void fill_words(skycell_gpu_ctx* ctx, cudaStream_t s, void* p, u64 words, uint32_t v = 0);

struct PipeBase {
  virtual ~PipeBase() = default;
  virtual void local() = 0;
  virtual u64 occ_bytes() const = 0;
  virtual void export_occ(void* dst) = 0;
  virtual void or_gathered(const void* gathered, int world) = 0;
  virtual void or_peers(const void* const* dev_table, int world) = 0;
  virtual u64 prune_local_skyline() = 0;
  virtual u64 block_bytes(u64 maxc) const = 0;
  virtual void pack(void* dst, u64 maxc) = 0;
  virtual void finish(const void* recv, int world, u64 maxc, int rank, u64 own_count, uint32_t* ids_out,
                      uint64_t* n_out, skycell_gpu_stats* stats) = 0;
};

}  // namespace skyeng

struct skycell_gpu_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // the stream every kernel is enqueued on
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_k0 = nullptr;  // K0's sample-skyline chain done (side stream, overlapped with K1)
  cudaEvent_t ev_k0occ = nullptr;  // ... its first step: the sample's level-(la-1) occupancy OR-ed in
  skyeng::DevBuf reset, slabs, H, table, table2, table_s, staging;
  skyeng::DevBuf smp_rows, smp_ids, smp_fsum, f_rows, f_fsum, f_lists, f_offs, ids_dev;
  skyeng::DevBuf s1_rows, s1_ids, s2_rows, s2_ids, s2_fsum, flags;
  skyeng::DevBuf sky_rows, sky_ids, sky_fsum;  // local skyline (sharded)
  skyeng::DevBuf d_cells;                      // K1's D stream
  skyeng::DevBuf p_rows, p_ids, p_fsum;        // K4a -> K4b pending points
  skyeng::DevBuf q_bits, q_orig, q_sub, q_ids, q_mm;  // quadrant_skyline
  skyeng::DevBuf t_keys, t_keys2, t_vals, t_vals2, t_cub, t_rows, t_ids, t_fsum, t_lo, t_hi, t_cs, t_ci;  // K5 tree
  skyeng::DevBuf t_cm, t_kill;  // K5 tree champion prefilter
  skyeng::DevBuf k5dbg;         // SKYCELL_K5STATS visit counters
  skyeng::DevBuf sp_keys, sp_keys2, sp_vals, sp_vals2, sp_head, sp_cpos, sp_crows, sp_cfsum, sp_cids, sp_cstart,
      sp_kflag, sp_cflag, sp_n, sp_qrec;  // sparse layer rho (sparse.cuh)
  int k5_mode = -1;  // 0 lists, 1 tree (packet query), 2 auto, 3 tree (point query); SKYCELL_K5
  skyeng::DevBuf long_q, long_n;  // K5 phase-B queue
  skyeng::DevBuf l_rows, l_sums, l_ids;  // K5 column lists (entries materialised per dimension)
  skyeng::DevBuf scan_tot;        // K5 list-scan chunk totals
  skyeng::DevCounters* host_ctr = nullptr;  // pinned
  u64* host_param = nullptr;        // pinned H2D staging
  u64* host_ctr_dev = nullptr;      // device views of the two (mapped pinned)
  u64* host_param_dev = nullptr;
  cudaEvent_t ev[10] = {};
  u64 launches = 0;
  std::unique_ptr<skyeng::PipeBase> shard;  // sharded query in flight
};

namespace skyeng {

inline void fill_words(skycell_gpu_ctx* ctx, cudaStream_t s, void* p, u64 words, uint32_t v) {
  const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((words + 255) / 256, (u64)ctx->num_sms * 8));
  sk::launch(sk::k_fill_u32, g, 256, 0, s, static_cast<uint32_t*>(p), words, v);
  ++ctx->launches;
}


inline void put_err(char* err, size_t len, const std::string& m) {
  if (!err || !len) return;
  std::strncpy(err, m.c_str(), len - 1);
  err[len - 1] = '\0';
}

// Runs an entry point's body, mapping exceptions onto status codes + err.
template <typename F>
inline int guarded(char* err, size_t err_len, F&& body) {
  try {
    body();
    return SKYCELL_OK;
  } catch (const ApiFail& f) {
    put_err(err, err_len, f.msg);
    return f.code;
  } catch (const CudaFail& f) {
    put_err(err, err_len, std::string("CUDA error in ") + f.what + ": " + cudaGetErrorString(f.e));
    cudaGetLastError();
    return SKYCELL_CUDA;
  } catch (const std::exception& e) {
    put_err(err, err_len, std::string("skycell_gpu: ") + e.what());
    return SKYCELL_CUDA;
  }
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
inline Status validate_shape(u64 n, int d) {
  if (n < 1) return {SKYCELL_INPUT, "normalize: empty dataset"};
  if (d < 2) return {SKYCELL_INPUT, "normalize: dimensionality must be at least 2"};
  if (d > sk::kMaxD) return {SKYCELL_INPUT, "normalize: dimensionality must be at most 16"};
  if (n > 0xffffffffull) return {SKYCELL_INPUT, "normalize: more than 2^32 - 1 records"};
  return {};
}

inline Status validate_rho(int rho, int d) {
  if (rho < 1) return {SKYCELL_CONFIG, "grid: rho must be at least 1"};
  if (rho * d > 60)
    return {SKYCELL_CONFIG, "grid: rho*d = " + std::to_string(rho * d) + " exceeds the 60-bit cell index budget"};
  if ((rho - 1) * d > 32)
    return {SKYCELL_CONFIG, "grid: occupancy bit-sets for rho = " + std::to_string(rho) + ", d = " +
                                std::to_string(d) + " would exceed memory"};
  return {};
}

inline int default_rho(u64 n, int d) {
  u64 x = n > 0 ? n : 1;
  int bw = 0;
  while (x) {
    ++bw;
    x >>= 1;
  }
  return std::max(1, std::min(6, (bw - 1) / d));
}

// SKYCELL_TRACE=1: synchronise and print the host time of each phase to
// stderr (debugging only; it serialises the pipeline).
struct Tracer {
  bool on = std::getenv("SKYCELL_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(cudaStream_t s, const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "[skycell] %-24s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};
inline Tracer& tracer() {
  static thread_local Tracer t;
  return t;
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
  sk::Norm nm;
  const void* dev_coords;  // device-resident input (user's or staged)
  uint32_t* ids_dev;       // caller's device output buffer, or nullptr (use ctx->ids_dev)
  skycell_gpu_stats* stats;
  bool timed;
  uint32_t id_base;        // global id of local record 0 (sharded: the shard offset)
};

template <typename TT>
void launch_tables(skycell_gpu_ctx* ctx, cudaStream_t s, const uint32_t* bits, int L, int d, TT* table) {
  const u64 rows = 1ull << (u64)(L * (d - 1));
  const u64 lines1 = rows >> L;
  const int nsm = ctx->num_sms;
  auto grid_for = [&](u64 items) {
    return (unsigned)std::max<u64>(1, std::min<u64>((items + 127) / 128, (u64)nsm * 16));
  };
  // enough dimension-1 lines to fill the GPU: one thread per line; else
  // (d = 2, or d = 3 at fine layers) row minima per thread + a CTA per line
  if (lines1 >= (u64)nsm * 128 || L <= 6) {
    // one warp per dimension-1 line
    const unsigned gw = (unsigned)std::max<u64>(1, std::min<u64>((lines1 * 32 + 255) / 256, (u64)nsm * 16));
    sk::launch(sk::k_rowmin_prefix1w<TT>, gw, 256, 0, s, bits, L, lines1, table);
    ++ctx->launches;
    for (int k = 2; k < d; ++k) {
      // a thread per line when lines fill the GPU, else a warp per line
      if (lines1 >= (u64)nsm * 128 || L < 5) sk::launch(sk::k_prefix_min<TT>, grid_for(lines1), 128, 0, s, table, L, k, lines1);
      else sk::launch(sk::k_prefix_minw<TT>, gw, 256, 0, s, table, L, k, lines1);
      ++ctx->launches;
    }
    return;
  }
  sk::launch(sk::k_rowmin<TT>, grid_for(rows), 128, 0, s, bits, L, rows, table);
  ++ctx->launches;
  for (int k = 1; k < d; ++k) {
    const unsigned g = (unsigned)std::min<u64>(lines1, (u64)nsm * 2);
    if (lines1 >= (u64)nsm * 128) sk::launch(sk::k_prefix_min<TT>, grid_for(lines1), 128, 0, s, table, L, k, lines1);
    else sk::launch(sk::k_prefix_min_cta<TT>, g, 1024, 0, s, table, L, k, lines1);
    ++ctx->launches;
  }
}

template <typename TT>
void launch_count(skycell_gpu_ctx* ctx, cudaStream_t s, const uint32_t* bits, int L, int d, const TT* table, u64* cand,
                  u64* key) {
  const u64 rows = 1ull << (u64)(L * (d - 1));
  const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((rows + 255) / 256, (u64)ctx->num_sms * 16));
  sk::launch(sk::k_count_rows<TT>, g, 256, 0, s, bits, L, d, rows, table, cand, key);
  ++ctx->launches;
}

// Exact sort-first pass (refine.cpp:31-59 as applied in phase 2, :98-99) over
// a point set given as slots (ids == kNoId marks an empty slot): per-dimension
// column lists, then the list-pruned dominance test; flags[i] = 1 for members
// of the result, for the query slots [q_begin, *q_end) (all slots when q_end
// is null).  cell_level > 0 restricts dominators to p's own layer-rho cell
// (merge_cross_cell = false, refine.cpp:98).
template <typename TOut, int D>
void run_exact(skycell_gpu_ctx* ctx, cudaStream_t s, const void* rows, const uint32_t* ids, const u64* fsum,
               const u64* count, u64 cap, unsigned* hist, unsigned* cursor, u64 q_begin = 0,
               const u64* q_end = nullptr, int cell_level = 0, const u64* gate = nullptr, u64 lcap = 0) {
  const int nsm = ctx->num_sms;
  const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((cap + 255) / 256, (u64)nsm * 8));
  const TOut* trows = static_cast<const TOut*>(rows);
  // list entries: at most the set's points (gated: at most the gate's limit)
  if (lcap == 0 || lcap > cap) lcap = cap;
  lcap = std::max<u64>(lcap, 1);
  ensure(ctx->l_rows, (size_t)D * lcap * D * sizeof(TOut));
  ensure(ctx->l_sums, (size_t)D * lcap * 8);
  ensure(ctx->l_ids, (size_t)D * lcap * 4);
  sk::ListArrays<TOut, D> la{static_cast<TOut*>(ctx->l_rows.p), static_cast<u64*>(ctx->l_sums.p),
                             static_cast<uint32_t*>(ctx->l_ids.p), lcap};
  sk::launch(sk::k_list_hist<TOut, D>, g, 256, 0, s, trows, ids, fsum, count, hist);
  unsigned* totals = static_cast<unsigned*>(ctx->scan_tot.p);
  sk::launch(sk::k_list_scan_sums, dim3(sk::kScanChunks, D), sk::kScanThreads, 0, s, hist, D, totals, gate);
  sk::launch(sk::k_list_scan, dim3(sk::kScanChunks, D), sk::kScanThreads, 0, s, hist, cursor, D, totals, gate);
  ++ctx->launches;
  sk::launch(sk::k_list_scatter<TOut, D>, g, 256, 0, s, trows, ids, fsum, count, cursor, la);
  const unsigned gw = (unsigned)std::max<u64>(1, std::min<u64>((cap * 32 + 255) / 256, (u64)nsm * 8));
  ensure(ctx->long_q, cap * 4);
  u64* long_n = static_cast<u64*>(ctx->long_n.p);
  fill_words(ctx, s, long_n, 2);
  // phase A budget in 32-entry steps (4..64 swept: 4-8 best at C2 / C4 shards; SKYCELL_LIST_STEPS)
  static const unsigned kMaxSteps = [] {
    const char* e = std::getenv("SKYCELL_LIST_STEPS");
    return e ? (unsigned)std::max(2, std::atoi(e)) : 8u;
  }();
  sk::launch(sk::k_allpairs_lists<TOut, D>, gw, 256, 0, s, trows, ids, fsum, count, la, hist,
                                                   static_cast<uint8_t*>(ctx->flags.p), q_begin, q_end, cell_level,
                                                   kMaxSteps, static_cast<uint32_t*>(ctx->long_q.p), long_n, gate);
  static const int kLongPerSm = [] {
    const char* e = std::getenv("SKYCELL_LONG_CTAS");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  sk::launch(sk::k_allpairs_long<TOut, D>, nsm * kLongPerSm, 256, 0, s, trows, ids, fsum, la, hist,
                                                       static_cast<uint8_t*>(ctx->flags.p), cell_level,
                                                       static_cast<const uint32_t*>(ctx->long_q.p), long_n);
  ctx->launches += 5;
}

// Exact sort-first pass through the dominance tree (tree.cuh).  Needs the
// set's slot count on the host (CUB's item count), so it synchronises once.
template <typename TOut, int D>
void run_tree(skycell_gpu_ctx* ctx, cudaStream_t s, const void* rows, const uint32_t* ids, const u64* fsum,
              const u64* count, u64* valid_ctr, u64 q_begin, const u64* q_end, int cell_level,
              bool point_query = false, bool no_prefilter = false, sk::TreeShape* shape_out = nullptr) {
  if (shape_out) shape_out->m = 0;
  const int nsm = ctx->num_sms;
  u64 hv[2];
  ck(cudaMemcpyAsync(&hv[0], count, 8, cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "sync");
  const u64 nslots = hv[0];
  if (nslots == 0) return;
  ensure(ctx->t_keys, nslots * 8);
  ensure(ctx->t_keys2, nslots * 8);
  ensure(ctx->t_vals, nslots * 4);
  ensure(ctx->t_vals2, nslots * 4);
  fill_words(ctx, s, valid_ctr, 2);
  const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((nslots + 255) / 256, (u64)nsm * 8));
  tracer().mark(s, "tree: count read");
  // champion prefilter over a dense level-Lc grid (<= 2^24 cells)
  // at most 2^24 cells and about 4 cells per set slot (the table's memset and
  // d prefix passes are a fixed cost; small sets would not amortise them)
  int lg = 0;
  while ((1ull << (lg + 1)) <= 4 * nslots) ++lg;
  const int Lc = std::min(std::min(12, 24 / D), lg / D);
  const uint8_t* kill = nullptr;
  // Not with merge_cross_cell = false (cell_level > 0): a dominator strictly
  // below p's prefilter cell may sit in another layer-rho cell, which
  // phase-1-only semantics (refine.cpp:98) must not use.
  if (Lc >= 1 && nslots >= (1ull << 16) && cell_level == 0 && !no_prefilter) {
    const u64 cells = 1ull << (u64)(Lc * D);
    // the plain grid, then grids shifted by 1/2, 1/4, 3/4 (.. 7/8) of a
    // cell: 4 passes at d >= 5 (C3: 542 -> 499 ms with the round-1 tree), 2
    // below (anti d=4: 11.2 vs 11.8 ms with 4); all passes' tables are built
    // in one read of the set and tested in one more
    int passes = D >= 5 ? 4 : 2;
    if (const char* e = std::getenv("SKYCELL_PREPASSES")) passes = std::max(1, std::min(8, std::atoi(e)));
    ensure(ctx->t_cm, cells * 4 * passes);
    ensure(ctx->t_kill, nslots);
    uint32_t* cm = static_cast<uint32_t*>(ctx->t_cm.p);
    const u64 lines = cells >> Lc;
    const unsigned gp = (unsigned)std::max<u64>(1, std::min<u64>((lines + 127) / 128, (u64)nsm * 16));
    uint8_t* killb = static_cast<uint8_t*>(ctx->t_kill.p);
    fill_words(ctx, s, cm, (u64)cells * passes, 0xffffffffu);
    sk::launch(sk::k_cellmin_multi<TOut, D>, g, 256, 0, s, static_cast<const TOut*>(rows), ids, fsum, count, Lc, passes, cells,
                                                   cm);
    for (int pass = 0; pass < passes; ++pass) {
      uint32_t* t = cm + (u64)pass * cells;
      for (int k = 1; k <= D; ++k) {
        // few long lines (d = 2: 512 lines of 512 cells): one CTA per line,
        // else a thread per line
        if (lines >= (u64)nsm * 4 || Lc < 8) sk::launch(sk::k_prefix_min<uint32_t>, gp, 128, 0, s, t, Lc, k, lines);
        else
          sk::launch(sk::k_prefix_min_cta<uint32_t>, (unsigned)std::min<u64>(lines, (u64)nsm * 2), 1024, 0, s, t, Lc, k, lines);
      }
    }
    sk::launch(sk::k_champ_kill_multi<TOut, D>, g, 256, 0, s, static_cast<const TOut*>(rows), ids, fsum, count, Lc, passes,
                                                      cells, cm, q_begin, q_end, killb,
                                                      static_cast<uint8_t*>(ctx->flags.p), valid_ctr + 1);
    ctx->launches += 2 + passes * D;
    kill = static_cast<const uint8_t*>(ctx->t_kill.p);
    tracer().mark(s, "tree: champion prefilter");
  }
  sk::launch(sk::k_tree_keys<TOut, D>, g, 256, 0, s, static_cast<const TOut*>(rows), ids, count, kill,
                                            static_cast<u64*>(ctx->t_keys.p), static_cast<uint32_t*>(ctx->t_vals.p),
                                            valid_ctr);
  size_t temp = 0;
  // key bits (the Morton key is shifted right by one: empty slots sort last)
  constexpr int kKeyBits = sk::morton_bits<D>() * D;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const u64*>(ctx->t_keys.p),
                                     static_cast<u64*>(ctx->t_keys2.p), static_cast<const uint32_t*>(ctx->t_vals.p),
                                     static_cast<uint32_t*>(ctx->t_vals2.p), nslots, 0, kKeyBits, s),
     "cub temp");
  ensure(ctx->t_cub, temp);
  ck(cub::DeviceRadixSort::SortPairs(ctx->t_cub.p, temp, static_cast<const u64*>(ctx->t_keys.p),
                                     static_cast<u64*>(ctx->t_keys2.p), static_cast<const uint32_t*>(ctx->t_vals.p),
                                     static_cast<uint32_t*>(ctx->t_vals2.p), nslots, 0, kKeyBits, s),
     "cub sort");
  tracer().mark(s, "tree: keys + sort");
  ck(cudaMemcpyAsync(&hv[1], valid_ctr, 8, cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "sync");
  const u64 m = hv[1];
  ctx->launches += 2;
  if (m == 0) return;
  sk::TreeShape sh{};
  sh.m = m;
  sh.nleaf = (m + sk::kLeaf - 1) / sk::kLeaf;
  if (sh.nleaf >= (1ull << 27)) throw ApiFail{SKYCELL_UNSUPPORTED, "skycell_gpu: dominance tree too large"};
  constexpr u64 F = sk::tree_fanout<D>();
  u64 off = 0, cnt = sh.nleaf;
  int L = 0;
  while (true) {
    sh.off[L] = (uint32_t)off;
    sh.cnt[L] = (uint32_t)cnt;
    off += cnt;
    ++L;
    if (cnt == 1) break;
    cnt = (cnt + F - 1) / F;
  }
  sh.levels = L;
  if (shape_out) *shape_out = sh;
  const u64 nodes = off;
  const uint32_t* order = static_cast<const uint32_t*>(ctx->t_vals2.p);
  const unsigned gm = (unsigned)std::max<u64>(1, std::min<u64>((m + 255) / 256, (u64)nsm * 8));
  const unsigned gl = (unsigned)std::max<u64>(1, std::min<u64>((sh.nleaf * 32 + 255) / 256, (u64)nsm * 8));
  const bool dbg = std::getenv("SKYCELL_K5STATS") != nullptr;
  u64* vst = nullptr;
  if (dbg) {
    ensure(ctx->k5dbg, 128);
    vst = static_cast<u64*>(ctx->k5dbg.p);
    fill_words(ctx, s, vst, 32);
  }
  // packet query (one warp per leaf of query points) unless merge_cross_cell
  // = false, whose same-cell restriction the point query keeps
  const bool packet = cell_level == 0 && !point_query;
  if (packet) {
    typedef sk::PkLayout<TOut, D> PL;
    ensure(ctx->t_rows, m * PL::PW * 4);
    ensure(ctx->t_lo, nodes * PL::NW * 4);
    uint32_t* prec = static_cast<uint32_t*>(ctx->t_rows.p);
    uint32_t* nrec = static_cast<uint32_t*>(ctx->t_lo.p);
    sk::launch(sk::k_pk_gather<TOut, D>, gm, 256, 0, s, static_cast<const TOut*>(rows), ids, fsum, order, m, prec);
    sk::launch(sk::k_pk_leaves<TOut, D>, gl, 256, 0, s, prec, m, sh.nleaf, nrec);
    ctx->launches += 2;
    for (int l = 1; l < sh.levels; ++l) {
      const unsigned gn = (unsigned)std::max<u64>(1, std::min<u64>((sh.cnt[l] + 255) / 256, (u64)nsm * 8));
      sk::launch(sk::k_pk_level<TOut, D>, gn, 256, 0, s, nrec, sh.off[l - 1], sh.cnt[l - 1], sh.off[l], sh.cnt[l]);
      ++ctx->launches;
    }
    tracer().mark(s, "tree: build");
    const unsigned gq = (unsigned)std::max<u64>(1, std::min<u64>((sh.nleaf * 32 + 255) / 256, (u64)nsm * 8));
    // phase-1 search radius (levels above the own leaf); phase 2 re-packs the
    // undecided points (SKYCELL_PK_H1 overrides; >= levels: one phase)
    int h1 = D <= 6 ? 5 : D == 7 ? 6 : 7;  // measured best (profiles/k5_h1_sweep_*)
    if (const char* e = std::getenv("SKYCELL_PK_H1")) h1 = std::atoi(e);
    const bool two = h1 < sh.levels - 1;
    uint32_t* umask = static_cast<uint32_t*>(ctx->t_keys.p);       // free after the sort
    uint32_t* pcnt = static_cast<uint32_t*>(ctx->t_keys2.p);
    uint32_t* poff = pcnt + sh.nleaf;
    uint32_t* list = static_cast<uint32_t*>(ctx->t_vals.p);
    u64* list_n = static_cast<u64*>(ctx->long_n.p) + 1;
    sk::launch(sk::k_pk_query<TOut, D, 0>, gq, 256, 0, s, prec, nrec, order, sh, q_begin, q_end, h1, two ? umask : nullptr,
                                                  nullptr, nullptr, nullptr, static_cast<uint8_t*>(ctx->flags.p), vst);
    ++ctx->launches;
    if (two) {
      tracer().mark(s, "tree: packet phase 1");
      const unsigned gc = (unsigned)std::max<u64>(1, std::min<u64>((sh.nleaf + 255) / 256, (u64)nsm * 8));
      sk::launch(sk::k_pk_counts, gc, 256, 0, s, umask, sh.nleaf, pcnt);
      size_t temp = 0;
      ck(cub::DeviceScan::ExclusiveSum(nullptr, temp, pcnt, poff, (int64_t)sh.nleaf, s), "cub scan temp");
      ensure(ctx->t_cub, temp);
      ck(cub::DeviceScan::ExclusiveSum(ctx->t_cub.p, temp, pcnt, poff, (int64_t)sh.nleaf, s), "cub scan");
      sk::launch(sk::k_pk_list, gc, 256, 0, s, umask, poff, sh.nleaf, list, list_n);
      sk::launch(sk::k_pk_query<TOut, D, 1>, gq, 256, 0, s, prec, nrec, order, sh, q_begin, q_end, h1, nullptr, list, list_n,
                                                  nullptr, static_cast<uint8_t*>(ctx->flags.p), vst);
      ctx->launches += 4;
    }
    tracer().mark(s, "tree: packet query");
  } else {
    ensure(ctx->t_rows, m * D * sizeof(TOut));
    ensure(ctx->t_ids, m * 4);
    ensure(ctx->t_fsum, m * 8);
    ensure(ctx->t_lo, nodes * D * sizeof(TOut));
    ensure(ctx->t_hi, nodes * D * sizeof(TOut));
    ensure(ctx->t_cs, nodes * 8);
    ensure(ctx->t_ci, nodes * 4);
    TOut* srows = static_cast<TOut*>(ctx->t_rows.p);
    uint32_t* sids = static_cast<uint32_t*>(ctx->t_ids.p);
    u64* sfsum = static_cast<u64*>(ctx->t_fsum.p);
    sk::launch(sk::k_tree_gather<TOut, D>, gm, 256, 0, s, static_cast<const TOut*>(rows), ids, fsum, order, m, srows, sids, sfsum);
    sk::TreeView<TOut, D> tv{static_cast<TOut*>(ctx->t_lo.p), static_cast<TOut*>(ctx->t_hi.p),
                             static_cast<u64*>(ctx->t_cs.p), static_cast<uint32_t*>(ctx->t_ci.p)};
    sk::launch(sk::k_tree_leaves<TOut, D>, gl, 256, 0, s, srows, sids, sfsum, m, sh.nleaf, tv);
    ctx->launches += 2;
    for (int l = 1; l < sh.levels; ++l) {
      const unsigned gn = (unsigned)std::max<u64>(1, std::min<u64>((sh.cnt[l] + 255) / 256, (u64)nsm * 8));
      sk::launch(sk::k_tree_level<TOut, D>, gn, 256, 0, s, tv, sh.off[l - 1], sh.cnt[l - 1], sh.off[l], sh.cnt[l]);
      ++ctx->launches;
    }
    tracer().mark(s, "tree: build");
    const unsigned gq = (unsigned)std::max<u64>(1, std::min<u64>((m * 32 + 255) / 256, (u64)nsm * 8));
    sk::launch(sk::k_tree_query<TOut, D>, gq, 256, 0, s, srows, sids, sfsum, order, tv, sh, q_begin, q_end, cell_level,
                                                static_cast<uint8_t*>(ctx->flags.p), vst);
    ++ctx->launches;
    tracer().mark(s, "tree: query");
  }
  if (dbg) {
    u64 hs[13], killed = 0;
    ck(cudaMemcpyAsync(hs, vst, 104, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaMemcpyAsync(&killed, valid_ctr + 1, 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    if (packet) {
      u64 ln = 0;
      ck(cudaMemcpy(&ln, static_cast<u64*>(ctx->long_n.p) + 1, 8, cudaMemcpyDeviceToHost), "D2H");
      const double p2 = std::max<double>(1.0, (double)((ln + 31) / 32));
      std::fprintf(stderr,
                   "[k5stats] D=%d slots=%llu prefilter_killed=%llu tree=%llu nodes=%llu | phase 1: %llu packets, %.1f "
                   "nodes %.1f leaves %.1f staged points per packet | phase 2: %llu points, %.1f nodes %.1f leaves %.1f "
                   "staged points per packet\n",
                   D, (unsigned long long)nslots, (unsigned long long)killed, (unsigned long long)m,
                   (unsigned long long)nodes, (unsigned long long)sh.nleaf, (double)hs[6] / sh.nleaf,
                   (double)hs[7] / sh.nleaf, (double)hs[8] / sh.nleaf, (unsigned long long)ln, (double)hs[10] / p2,
                   (double)hs[11] / p2, (double)hs[12] / p2);
    }
    else
      std::fprintf(stderr,
                   "[k5stats] D=%d slots=%llu prefilter_killed=%llu tree=%llu nodes=%llu | dominated %llu: %.1f nodes "
                   "%.1f leaves | members %llu: %.1f nodes %.1f leaves\n",
                   D, (unsigned long long)nslots, (unsigned long long)killed, (unsigned long long)m,
                   (unsigned long long)nodes, (unsigned long long)hs[0], hs[0] ? (double)hs[1] / hs[0] : 0.0,
                   hs[0] ? (double)hs[2] / hs[0] : 0.0, (unsigned long long)hs[3], hs[3] ? (double)hs[4] / hs[3] : 0.0,
                   hs[3] ? (double)hs[5] / hs[3] : 0.0);
  }
}

// SKYCELL_K5 = lists | tree | tree-point | auto (default): which K5 variant
// runs (tree-point: the tree with the one-warp-per-point query).
inline int k5_mode(skycell_gpu_ctx* ctx) {
  if (ctx->k5_mode < 0) {
    const char* e = std::getenv("SKYCELL_K5");
    ctx->k5_mode = !e ? 2 : !std::strcmp(e, "lists") ? 0 : !std::strcmp(e, "tree") ? 1 : !std::strcmp(e, "tree-point") ? 3 : 2;
  }
  return ctx->k5_mode;
}

// Sets up to this many slots go through the column lists; larger ones
// (anti-correlated data: 8e6 at n=1e8 d=4, 5.4e7 at d=6) through the tree,
// whose cost grows with the skyline boundary instead of the list prefixes.
constexpr u64 kTreeMinSlots = 1ull << 20;
constexpr u64 kTreeMainMin = 1ull << 16;  // main K5: decided on the point count
// sample skyline (K0): lists up to this many candidates (SKYCELL_SAMPLE_TREE_MIN)
inline u64 sample_tree_min() {
  static const u64 v = [] {
    const char* e = std::getenv("SKYCELL_SAMPLE_TREE_MIN");
    return e ? (u64)std::strtoull(e, nullptr, 10) : (u64)(96 * 1024);
  }();
  return v;
}

// K5 dispatcher: flags[slot] for the query slots of the set.
template <typename TOut, int D>
void run_dominance(skycell_gpu_ctx* ctx, cudaStream_t s, const void* rows, const uint32_t* ids, const u64* fsum,
                   const u64* count, u64 cap, unsigned* hist, unsigned* cursor, u64* valid_ctr, u64 q_begin = 0,
                   const u64* q_end = nullptr, int cell_level = 0, u64 tree_min = kTreeMinSlots,
                   const u64* valid_count = nullptr) {
  int mode = k5_mode(ctx);
  if (mode == 2 && cell_level == 0) {
    // The column lists are enqueued at once, gated on the device by the
    // set's point count (valid_count when known, else slots) and by exact
    // origins (k_origin_count: a set holding one is decided in O(n)); the
    // host reads both counts meanwhile and adds the tree only for a large
    // set without origins -- no GPU bubble for the common small set.
    const u64* vc = valid_count ? valid_count : count;
    u64* lc = static_cast<u64*>(ctx->long_n.p) + 2;
    u64* org = static_cast<u64*>(ctx->long_n.p) + 3;
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((cap + 255) / 256, (u64)ctx->num_sms * 8));
    fill_words(ctx, s, org, 2);
    sk::launch(sk::k_origin_count, g, 256, 0, s, ids, fsum, count, org);
    sk::launch(sk::k_origin_flags, g, 256, 0, s, ids, fsum, count, q_begin, q_end, org, static_cast<uint8_t*>(ctx->flags.p));
    sk::launch(sk::k_gate_count, 1, 1, 0, s, vc, count, tree_min, org, lc, ctx->host_param_dev + 3);
    ck(cudaEventRecord(ctx->ev[8], s), "event");
    ctx->launches += 3;
    run_exact<TOut, D>(ctx, s, rows, ids, fsum, lc, cap, hist, cursor, q_begin, q_end, cell_level, lc, tree_min);
    ck(cudaEventSynchronize(ctx->ev[8]), "count");
    if (ctx->host_param[4] == 0 && ctx->host_param[3] > tree_min)
      run_tree<TOut, D>(ctx, s, rows, ids, fsum, count, valid_ctr, q_begin, q_end, cell_level, false);
    return;
  }
  if (mode == 2) mode = 0;  // cap <= tree_min: the lists
  if (mode == 0)
    run_exact<TOut, D>(ctx, s, rows, ids, fsum, count, cap, hist, cursor, q_begin, q_end, cell_level);
  else
    run_tree<TOut, D>(ctx, s, rows, ids, fsum, count, valid_ctr, q_begin, q_end, cell_level, mode == 3);
}

template <typename TIn, typename TOut, bool IDENT, int D>
struct Pipe final : PipeBase {
  Query q;
  skycell_gpu_ctx* ctx;
  cudaStream_t s, s2;
  u64 n;
  int rho, nsm;

  // ---- geometry
  int la;
  bool test_b, wide;
  u64 m;
  uint32_t h_entries, lo_words;
  size_t tt;
  u64 table_entries;
  static constexpr int kStreamThreads = 256;
  static constexpr int kRecLaThreads = 768;
  // the shape with a record-at-la K1 instance (the headline: d = 4, rho = 6, la = 5)
  static bool rec_la_shape(int r) {
    // measured slower than the 3 x 256-thread instance (516 vs 445 us at C2):
    // kept as an opt-in experiment (SKYCELL_RECLA=1)
    if constexpr (IDENT && D == 4) return r == 6 && std::getenv("SKYCELL_RECLA") != nullptr;
    return false;
  }
  int k1_threads = kStreamThreads;
  bool rec_la = false;
  static constexpr int PPT1 = std::max(1, ppt_for<TIn, D>() / 2);
  static constexpr unsigned kChunk1 = 256, kChunk4 = 64;
  static_assert(kChunk1 >= 32 * PPT1, "a stream tile's survivors must fit one output chunk");
  size_t smem1;
  void (*kstream)(sk::StreamParams);
  int grid1, grid4, pf_max;
  u64 cap1, cap4;
  size_t smem_pf;
  u64 id_words;
  unsigned bit_blocks;
  bool k0_side = false;  // K0's sample-skyline chain runs on the side stream (joined before K4)
  bool cover = false;    // H carries cover flags; the sample's level-(la-1) occupancy is OR-ed in (side stream)
  bool k1_head = false;  // K1 ran the filter-point head (its D stream feeds K4's points_examined)

  // ---- zeroed region
  size_t o_ctr, o_sla, o_srho, o_shist, o_scur, o_hist, o_cur, o_fhist, o_fcur, o_idbits, o_bcount, o_end, o_total;
  std::vector<size_t> o_occ;

  u64 words_at(int L) const { return std::max<u64>(1, (1ull << (u64)(L * D)) / 32); }
  void* at(size_t off) const { return static_cast<char*>(ctx->reset.p) + off; }
  uint32_t* occ(int L) const { return static_cast<uint32_t*>(at(o_occ[L])); }
  DevCounters* ctr() const { return static_cast<DevCounters*>(at(o_ctr)); }
  unsigned* U(size_t off) const { return static_cast<unsigned*>(at(off)); }
  // merge_cross_cell = false: dominators share p's cell at the QUERY's rho
  int cell_level() const { return q.merge ? 0 : rho_q; }
  // sparse layer rho (sparse.cuh): the dense pipeline runs up to rho - 1
  static bool sparse_top(int r) { return r * D > 36 || r * (D - 1) > 30; }

  // (64-point tiles in a 4-stage ring, the same shared memory: C2 K1 0.382 ->
  // 0.550 ms, profiles/ab_k1ring4_r9k.txt)
  // K1 tiles by cp.async.bulk into a shared-memory ring (identity f32 input at
  // d = 4, whose 16-byte rows make every tile a whole number of 16-byte
  // chunks): C2 K1 0.429 -> 0.404 ms, correlated 0.409 -> 0.375 ms
  // (profiles/ab_k1bulk_r9e.txt).  SKYCELL_K1_BULK=0: per-lane LDG.128 into
  // two register buffers.
  static bool k1_bulk_env() {
    static const bool v = [] { const char* e = std::getenv("SKYCELL_K1_BULK"); return !e || e[0] != '0'; }();
    return v;
  }
  bool k1_bulk() const {
    if constexpr (IDENT && D == 4) return k1_bulk_env() && !rec_la_shape(rho);
    return false;
  }
  template <bool B>
  static auto pick_stream_b(int rho) {
    if constexpr (IDENT && D <= 8) {
      switch (rho) {
        case 1: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 1, 3, false, B>;
        case 2: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 2, 3, false, B>;
        case 3: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 3, 3, false, B>;
        case 4: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 4, 3, false, B>;
        case 5: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 5, 3, false, B>;
        case 6: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 6, 3, false, B>;
        case 7: return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 7, 3, false, B>;
        default: break;
      }
    }
    return sk::k_stream<TIn, TOut, D, IDENT, kStreamThreads, PPT1, 0, 3, false, B>;
  }
  static auto pick_stream(int rho) {
    if constexpr (IDENT && D == 4) {
      if (rec_la_shape(rho)) return sk::k_stream<TIn, TOut, D, IDENT, kRecLaThreads, PPT1, 6, 1, true>;
      if (k1_bulk_env()) return pick_stream_b<true>(rho);
    }
    return pick_stream_b<false>(rho);
  }

  int rho_q;    // the query's rho (reported layers 1..rho_q)
  bool sparse;  // layer rho_q is sparse; `rho` (the dense top layer) = rho_q - 1

  explicit Pipe(const Query& qq)
      : q(qq), ctx(qq.ctx), s(qq.ctx->stream), s2(qq.ctx->side), n(qq.n),
        rho(sparse_top(qq.rho) ? qq.rho - 1 : qq.rho), rho_q(qq.rho), sparse(sparse_top(qq.rho)) {
    nsm = ctx->num_sms;
    la = sk::filter_level(rho, D);
    test_b = rho > la;
    m = std::min<u64>(n, 1ull << 20);
    h_entries = (uint32_t)(1ull << (u64)(la * (D - 1)));
    rec_la = rec_la_shape(rho);
    k1_threads = rec_la ? kRecLaThreads : kStreamThreads;
    lo_words = rec_la ? (uint32_t)words_at(la) : (la >= 2 ? (uint32_t)words_at(la - 1) : 0);
    wide = rho > 7;
    tt = wide ? 4 : 1;
    table_entries = 1ull << (u64)(rho * (D - 1));

    // K1 geometry: persistent warps over round-robin warp tiles
    smem1 = (((size_t)lo_words * 4 + 15) & ~(size_t)15) + ((h_entries + 15) & ~15u) + (size_t)k1_threads * PPT1 +
            (((size_t)sk::kK1Head * (D * sizeof(TOut) + 8) + 15) & ~(size_t)15) +
            (size_t)k1_threads * PPT1 * D * sizeof(TIn) * (k1_bulk() ? 2 : 1) + (size_t)(k1_threads / 32) * 32 + 16;
    kstream = pick_stream(rho);
    ck(cudaFuncSetAttribute(kstream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1), "smem attr");
    int occ_blocks = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_blocks, kstream, k1_threads, smem1), "occupancy");
    occ_blocks = std::max(1, occ_blocks);
    if (const char* e = std::getenv("SKYCELL_K1_CTAS")) occ_blocks = std::max(1, std::min(occ_blocks, std::atoi(e)));
    const u64 wtiles = (n + 32 * PPT1 - 1) / (32 * PPT1);
    const u64 wpc = (u64)k1_threads / 32;
    grid1 = (int)std::max<u64>(1, std::min<u64>((wtiles + wpc - 1) / wpc, (u64)nsm * occ_blocks));
    if (q.merge && k0_overlap() && !k1_head_wanted()) {
      // leave CTA slots free for K0's sample-skyline chain, which runs beside K1
      // (12 slots: C2 1.195 -> 1.175 ms; 24/48/96 measured slower)
      int free_slots = 12;
      if (const char* e = std::getenv("SKYCELL_K1_FREE")) free_slots = std::atoi(e);
      if (grid1 >= nsm * 2) grid1 = std::max(nsm, grid1 - free_slots);
    }
    cap1 = n + (u64)grid1 * (k1_threads / 32) * kChunk1;

    // K4 geometry
    grid4 = nsm * 4;
    cap4 = std::max(cap1, m) + (u64)grid4 * (kThreads / 32) * kChunk4;
    pf_max = (int)std::min<u64>(1024, (32 * 1024) / (D * sizeof(TOut) + 8));
    smem_pf = (((u64)pf_max * D * sizeof(TOut) + 15) & ~15ull) + (u64)pf_max * 8 + (u64)D * pf_max * 2 +
              (u64)D * (sk::kListCols + 1) * 2 + 16;
    const size_t bin_words = (size_t)D * sk::kListStride;
    id_words = (n + 31) / 32;
    bit_blocks = (unsigned)((id_words + sk::kBitsBlock - 1) / sk::kBitsBlock);

    // zeroed region: counters, occupancy layers 1..rho (contiguous: the
    // sharded exchange ships [o_occ[1], o_occ[rho] + words) as one block)
    Carver cv;
    o_ctr = cv.take(sizeof(DevCounters));
    o_occ.assign(rho + 1, 0);
    for (int L = 1; L <= rho; ++L) o_occ[L] = cv.take(words_at(L) * 4);
    o_end = cv.off;
    o_sla = cv.take(words_at(la) * 4);
    o_srho = test_b ? cv.take(words_at(rho) * 4) : 0;
    o_shist = cv.take(bin_words * 4);
    o_scur = cv.take(bin_words * 4);
    o_hist = cv.take(bin_words * 4);
    o_cur = cv.take(bin_words * 4);
    o_fhist = cv.take(bin_words * 4);
    o_fcur = cv.take(bin_words * 4);
    o_idbits = cv.take(id_words * 4);
    o_bcount = cv.take((size_t)bit_blocks * 4);
    o_total = cv.off;
    ensure(ctx->reset, o_total);

    // working buffers
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
    ensure(ctx->f_offs, (size_t)D * (sk::kListCols + 1) * 2);
    ensure(ctx->s1_rows, cap1 * D * sizeof(TOut));
    ensure(ctx->s1_ids, cap1 * 4);
    ensure(ctx->d_cells, cap1 * (rho * D >= 32 ? 8 : 4));
    ensure(ctx->s2_rows, cap4 * D * sizeof(TOut));
    ensure(ctx->s2_ids, cap4 * 4);
    ensure(ctx->s2_fsum, cap4 * 8);
    ensure(ctx->flags, cap4);
    ensure(ctx->ids_dev, n * 4);
  }

  // ---- K0 + K1 (+ slab reduction): everything that reads the input
  void local() override {
    DevCounters* c = ctr();
    if (q.timed) ck(cudaEventRecord(ctx->ev[0], s), "event");
    // a fill kernel, not a memset node: keeps the programmatic-launch chain into K0
    fill_words(ctx, s, ctx->reset.p, o_total / 4);

    // K0: sample occupancy, filter tables, sample skyline -> filter points F
    {
      sk::SampleParams sp{};
      sp.coords = q.dev_coords;
      sp.m = m;
      sp.rho = rho;
      sp.la = la;
      sp.nm = q.nm;
      sp.occ_la = U(o_sla);
      sp.occ_rho = test_b ? U(o_srho) : nullptr;
      sp.rows = ctx->smp_rows.p;
      sp.ids = static_cast<uint32_t*>(ctx->smp_ids.p);
      sp.fsum = static_cast<u64*>(ctx->smp_fsum.p);
      sp.id_base = q.id_base;
      const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((m + 255) / 256, (u64)nsm * 8));
      tracer().mark(s, "K0: memset");
      sk::launch(sk::k_sample<TIn, TOut, D, IDENT>, g, 256, 0, s, sp);
      tracer().mark(s, "K0: sample");
      // H = the strict-dominance height of the sample's level-la occupancy:
      // a level-la prefix-min table (multi-CTA) shifted by one cell per dim
      launch_tables<uint8_t>(ctx, s, U(o_sla), la, D, static_cast<uint8_t*>(ctx->table2.p));
      // cover flags (bit 7 of H) only when the sample's level-(la-1) occupancy
      // is OR-ed into layer la-1 (sample_skyline, side stream)
      cover = q.merge && !k1_head_wanted() && k0_overlap() && la >= 2 && !rec_la && IDENT && D <= 6 &&
              !(std::getenv("SKYCELL_COVER") && std::getenv("SKYCELL_COVER")[0] == '0');
      sk::launch(sk::k_filter_from_table, (unsigned)std::max<u64>(1, std::min<u64>((h_entries + 255) / 256, (u64)nsm * 4)), 256, 0, s, static_cast<const uint8_t*>(ctx->table2.p), la, D, h_entries,
                                     static_cast<uint8_t*>(ctx->H.p), cover ? static_cast<const uint32_t*>(U(o_sla)) : nullptr);
      tracer().mark(s, "K0: build_filter");
      ctx->launches += 2;
      // layer-rho prefix-min table of the sample: K1's test B
      if (test_b) {
        if (wide) launch_tables<uint32_t>(ctx, s, U(o_srho), rho, D, static_cast<uint32_t*>(ctx->table_s.p));
        else launch_tables<uint8_t>(ctx, s, U(o_srho), rho, D, static_cast<uint8_t*>(ctx->table_s.p));
      }
    }
    // The sample skyline only serves as K4's point filter, which phase-1
    // only semantics (merge_cross_cell = false) cannot use.  K1 does not
    // read it (unless its filter-point head is on), so with
    // SKYCELL_K0_OVERLAP=1 it runs on the side stream behind K1's launch.
    // Part A (X) stays on the main stream: on K1's few free CTA slots it
    // would hold up part B's host-read gate until K1's end.
    k0_side = q.merge && !k1_head_wanted() && k0_overlap();
    if (q.merge) sample_candidates();
    if (q.merge && !k0_side) sample_skyline(s);
    // fork point: K0's sample buffers and tables are complete here
    if (k0_side) ck(cudaEventRecord(ctx->ev_fork, s), "event");
    launch_k1(c);
    if (k0_side) sample_skyline(s2);
    if (cover) ck(cudaStreamWaitEvent(s, ctx->ev_k0occ, 0), "join occupancy");
    if (q.timed) ck(cudaEventRecord(ctx->ev[1], s), "event");
  }

  static bool k0_overlap() {
    static const bool v = [] { const char* e = std::getenv("SKYCELL_K0_OVERLAP"); return !e || e[0] != '0'; }();
    return v;
  }
  bool k1_head_wanted() const {
    const char* he = std::getenv("SKYCELL_K1HEAD");
    return q.merge && he && he[0] == '1';
  }

  // K0 part A (main stream): the sample's candidates X, packed and capped
  void sample_candidates() {
    DevCounters* c = ctr();
    {
      {
        tracer().mark(s, "K0: sample tables");
        // sample points not strictly dominated at layer rho -> X (s2 buffers)
        sk::CandParams pc{};
        pc.rows = ctx->smp_rows.p;
        pc.ids = static_cast<const uint32_t*>(ctx->smp_ids.p);
        pc.count = nullptr;
        // the filter points come from the skyline of the first mf sample
        // points (SKYCELL_FSAMPLE overrides; H uses all m)
        u64 mf = m;
        if (const char* e = std::getenv("SKYCELL_FSAMPLE")) mf = std::min<u64>(m, std::strtoull(e, nullptr, 10));
        pc.count_const = mf;
        pc.rho = rho;
        pc.PM = test_b ? ctx->table_s.p : nullptr;
        pc.f_max = 0;
        pc.out_rows = ctx->s2_rows.p;
        pc.out_ids = static_cast<uint32_t*>(ctx->s2_ids.p);
        pc.out_fsum = static_cast<u64*>(ctx->s2_fsum.p);
        pc.out_reserved = &c->xs;
        pc.chunk = kChunk4;
        pc.kept = &c->xs_kept;
        pc.examined = nullptr;
        if (wide) sk::launch(sk::k_candidates<TOut, D, uint32_t, kThreads>, grid4, kThreads, 16, s, pc);
        else sk::launch(sk::k_candidates<TOut, D, uint8_t, kThreads>, grid4, kThreads, 16, s, pc);
        ++ctx->launches;
        tracer().mark(s, "K0: sample X");
        // Filter points = the strongest points of the sample's skyline (the
        // whole skyline: its extremes filter the extremes of the data).  X
        // is capped at kXMax slots (a random subset: slots follow the sample
        // order): anti-correlated samples keep ~all points in X, and their
        // filter points remove little anyway.
        constexpr u64 kXMax = 1ull << 17;
        sk::launch(sk::k_pack_members<TOut, D>, nsm * 4, 256, 0, s, 
            static_cast<const TOut*>(ctx->s2_rows.p), static_cast<const uint32_t*>(ctx->s2_ids.p), nullptr,
            static_cast<const u64*>(ctx->s2_fsum.p), &c->xs, static_cast<TOut*>(ctx->smp_rows.p),
            static_cast<u64*>(ctx->smp_fsum.p), static_cast<uint32_t*>(ctx->smp_ids.p), &c->xd);
        sk::launch(sk::k_clamp_count, 1, 32, 0, s, &c->xd, kXMax, &c->xs_cap);
        ctx->launches += 2;
      }
    }
  }

  // K0 part B: the sample skyline of X -> filter points F (+ column lists)
  void sample_skyline(cudaStream_t st) {
    DevCounters* c = ctr();
    const bool side = st != s;
    cudaStream_t s = st;  // every launch below goes to st
    if (side) ck(cudaStreamWaitEvent(s, ctx->ev_fork, 0), "fork");
    if (cover) {
      // the sample's level-(la-1) occupancy into layer la-1: K1 skips the
      // dropped points of covered rows (H bit 7); the main stream joins here
      // before it reads the layer (ev_k0occ)
      const u64 sw = words_at(la);
      const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((sw + 255) / 256, (u64)nsm * 8));
      sk::launch(sk::k_downsample, g, 256, 0, s, static_cast<const uint32_t*>(U(o_sla)), la - 1, D, sw, occ(la - 1));
      ++ctx->launches;
      ck(cudaEventRecord(ctx->ev_k0occ, s), "event");
    }
    constexpr u64 kXMax = 1ull << 17;
    {
      {
        run_dominance<TOut, D>(ctx, s, ctx->smp_rows.p, static_cast<const uint32_t*>(ctx->smp_ids.p),
                               static_cast<const u64*>(ctx->smp_fsum.p), &c->xs_cap, std::min<u64>(m, kXMax),
                               U(o_shist), U(o_scur), &c->tvalid, 0, nullptr, 0, sample_tree_min());
        tracer().mark(s, "K0: sample skyline");
        sk::launch(sk::k_compact_members<TOut, D>, nsm * 4, 256, 0, s, 
            static_cast<const TOut*>(ctx->smp_rows.p), static_cast<const uint32_t*>(ctx->smp_ids.p),
            static_cast<const uint8_t*>(ctx->flags.p), static_cast<const u64*>(ctx->smp_fsum.p), &c->xs_cap,
            static_cast<TOut*>(ctx->s2_rows.p), static_cast<u64*>(ctx->s2_fsum.p), &c->fs);
        sk::launch(sk::k_strength_order<TOut, D>, 1, 256, 0, s, 
            static_cast<const TOut*>(ctx->s2_rows.p), static_cast<const u64*>(ctx->s2_fsum.p), nullptr, &c->fs,
            (uint32_t)pf_max, static_cast<TOut*>(ctx->f_rows.p), static_cast<u64*>(ctx->f_fsum.p), nullptr, &c->nf);
        sk::launch(sk::k_filter_gate, 1, 1, 0, s, &c->fs, &c->xs_cap, &c->fweak);
        ++ctx->launches;
        sk::launch(sk::k_filter_lists<TOut, D>, D, 256, 0, s, static_cast<const TOut*>(ctx->f_rows.p), &c->nf,
                                                        (uint32_t)pf_max, static_cast<uint16_t*>(ctx->f_lists.p),
                                                        static_cast<uint16_t*>(ctx->f_offs.p));
        ++ctx->launches;
        ctx->launches += 2;
      }
    }
    if (side) ck(cudaEventRecord(ctx->ev_k0, s), "event");
  }

  void launch_k1(DevCounters* c) {
    // K1: the streaming pass
    sk::StreamParams p1{};
    p1.coords = q.dev_coords;
    p1.n = n;
    p1.rho = rho;
    p1.la = la;
    p1.lo_words = lo_words;
    p1.h_entries = h_entries;
    p1.nm = q.nm;
    p1.H = static_cast<const uint8_t*>(ctx->H.p);
    // Test B costs two dependent L2 round trips per K1 survivor; it pays off
    // when the shared-memory filter level la is at least two layers coarser
    // than rho (SKYCELL_TESTB=0/1 overrides).
    bool use_b = test_b && rho - la >= 2;
    if (const char* e = std::getenv("SKYCELL_TESTB")) use_b = test_b && e[0] == '1';
    p1.PMs = use_b ? ctx->table_s.p : nullptr;
    p1.pms_wide = wide;
    p1.occ_rho = occ(rho);
    p1.occ_rm1 = rho >= 2 ? occ(rho - 1) : nullptr;
    p1.slabs = static_cast<uint32_t*>(ctx->slabs.p);
    p1.out_rows = ctx->s1_rows.p;
    p1.out_ids = static_cast<uint32_t*>(ctx->s1_ids.p);
    p1.out_reserved = &c->s1;
    p1.chunk = kChunk1;
    p1.kept = &c->s1_kept;
    p1.nonfinite = &c->nonfinite;
    p1.id_base = q.id_base;
    // K1's filter-point head (SKYCELL_K1HEAD=1): cuts S1 ~8x but costs K1
    // more than it saves K4 at the headline config
    const char* he = std::getenv("SKYCELL_K1HEAD");
    k1_head = q.merge && he && he[0] == '1';
    if (k1_head) {  // the filter points exist (K0) only with the phase-2 merge
      p1.f_rows = ctx->f_rows.p;
      p1.f_fsum = static_cast<const u64*>(ctx->f_fsum.p);
      p1.f_count = &c->nf;
      p1.d_cells = ctx->d_cells.p;
      p1.d_reserved = &c->dres;
    }
    if (q.timed) ck(cudaEventRecord(ctx->ev[4], s), "event");
    sk::launch(kstream, grid1, k1_threads, smem1, s, p1);
    ++ctx->launches;
    if (q.timed) ck(cudaEventRecord(ctx->ev[5], s), "event");
    if (lo_words) {
      const unsigned gx = (unsigned)std::max<u64>(1, std::min<u64>((lo_words + 255) / 256, (u64)nsm * 8));
      const unsigned gy = (unsigned)std::max<u64>(1, std::min<u64>(32, (u64)nsm * 4 / gx));
      sk::launch(sk::k_reduce_slabs, dim3(gx, gy), 256, 0, s, static_cast<uint32_t*>(ctx->slabs.p), grid1, lo_words,
                                                       occ(rec_la ? la : la - 1));
      ++ctx->launches;
    }
  }

  // ---- sharded exchange 1: the occupancy region of every layer
  u64 occ_bytes() const override { return o_end - o_occ[1]; }
  void export_occ(void* dst) override {
    ck(cudaMemcpyAsync(dst, at(o_occ[1]), occ_bytes(), cudaMemcpyDeviceToDevice, s), "occ export");
  }
  void or_gathered(const void* gathered, int world) override {
    const u64 w4 = occ_bytes() / 16;
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((w4 + 255) / 256, (u64)nsm * 8));
    sk::launch(sk::k_or_gather, g, 256, 0, s, static_cast<const uint4*>(gathered), world, w4,
                                      static_cast<uint4*>(at(o_occ[1])));
    ++ctx->launches;
  }

  void or_peers(const void* const* dev_table, int world) override {
    const u64 w4 = occ_bytes() / 16;
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((w4 + 255) / 256, (u64)nsm * 8));
    sk::launch(sk::k_or_peers, g, 256, 0, s, reinterpret_cast<const uint4* const*>(dev_table), world, w4,
                                     static_cast<uint4*>(at(o_occ[1])));
    ++ctx->launches;
  }

  // ---- K3 (tables + per-layer counts on the side stream) + K4
  void prune() {
    DevCounters* c = ctr();
    if (wide) launch_tables<uint32_t>(ctx, s, occ(rho), rho, D, static_cast<uint32_t*>(ctx->table.p));
    else launch_tables<uint8_t>(ctx, s, occ(rho), rho, D, static_cast<uint8_t*>(ctx->table.p));
    if (q.timed) ck(cudaEventRecord(ctx->ev[2], s), "event");

    // Per-layer |KS_i|, |CS_i| (refine.cpp:125-147), overlapped with K4/K5.
    // Layer rho from O'_rho; below, O'_rho is OR-ed down into the partial
    // occupancies recorded by the filter.
    ck(cudaEventRecord(ctx->ev_fork, s), "event");
    ck(cudaStreamWaitEvent(s2, ctx->ev_fork, 0), "wait");
    if (wide) launch_count<uint32_t>(ctx, s2, occ(rho), rho, D, static_cast<const uint32_t*>(ctx->table.p), &c->cand[rho - 1], &c->key[rho - 1]);
    else launch_count<uint8_t>(ctx, s2, occ(rho), rho, D, static_cast<const uint8_t*>(ctx->table.p), &c->cand[rho - 1], &c->key[rho - 1]);
    for (int L = rho - 1; L >= 1; --L) {
      const u64 src_words = words_at(L + 1);
      const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((src_words + 255) / 256, (u64)nsm * 8));
      if (L >= 5) {
        const u64 dst_words = words_at(L);
        const unsigned gw = (unsigned)std::max<u64>(1, std::min<u64>((dst_words + 255) / 256, (u64)nsm * 8));
        sk::launch(sk::k_downsample_words, gw, 256, 0, s2, occ(L + 1), L, D, dst_words, occ(L));
      } else {
        sk::launch(sk::k_downsample, g, 256, 0, s2, occ(L + 1), L, D, src_words, occ(L));
      }
      ++ctx->launches;
      if (L > 7) {
        launch_tables<uint32_t>(ctx, s2, occ(L), L, D, static_cast<uint32_t*>(ctx->table2.p));
        launch_count<uint32_t>(ctx, s2, occ(L), L, D, static_cast<const uint32_t*>(ctx->table2.p), &c->cand[L - 1], &c->key[L - 1]);
      } else {
        launch_tables<uint8_t>(ctx, s2, occ(L), L, D, static_cast<uint8_t*>(ctx->table2.p));
        launch_count<uint8_t>(ctx, s2, occ(L), L, D, static_cast<const uint8_t*>(ctx->table2.p), &c->cand[L - 1], &c->key[L - 1]);
      }
    }
    ck(cudaEventRecord(ctx->ev_join, s2), "event");

    // K4: candidate cells + sample-skyline point filter
    sk::CandParams pc{};
    pc.rows = ctx->s1_rows.p;
    pc.ids = static_cast<const uint32_t*>(ctx->s1_ids.p);
    pc.count = &c->s1;
    pc.rho = rho;
    pc.PM = ctx->table.p;
    pc.f_rows = ctx->f_rows.p;
    pc.f_fsum = static_cast<const u64*>(ctx->f_fsum.p);
    // sparse: K4 is the layer-(rho-1) cell test only; the filter points run
    // after the sparse layer-rho stage
    pc.f_count = q.merge && !sparse ? &c->nf : nullptr;
    pc.f_max = q.merge && !sparse ? (uint32_t)pf_max : 0;
    pc.f_lists = static_cast<const uint16_t*>(ctx->f_lists.p);
    pc.f_offs = static_cast<const uint16_t*>(ctx->f_offs.p);
    pc.out_rows = ctx->s2_rows.p;
    pc.out_ids = static_cast<uint32_t*>(ctx->s2_ids.p);
    pc.out_fsum = static_cast<u64*>(ctx->s2_fsum.p);
    pc.out_reserved = &c->s2;
    pc.chunk = kChunk4;
    pc.kept = &c->s2_kept;
    pc.examined = &c->examined;
    if (k1_head) {
      pc.d_cells = ctx->d_cells.p;
      pc.d_count = &c->dres;
      pc.d_wide = rho * D >= 32;
    }
    auto kc = wide ? sk::k_candidates<TOut, D, uint32_t, kThreads> : sk::k_candidates<TOut, D, uint8_t, kThreads>;
    ck(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pf), "smem attr");
    if (k0_side) ck(cudaStreamWaitEvent(s, ctx->ev_k0, 0), "join K0");
    if (q.merge && !sparse) {
      // K4a: cell test + the 8 strongest filter points over S1 -> P (dense
      // pending points, in the S1 buffers' twin); K4b: the rest of the filter
      // over P, whose lanes are all pending (no idle lanes in the head test)
      ensure(ctx->p_rows, cap1 * D * sizeof(TOut));
      ensure(ctx->p_ids, cap1 * 4);
      ensure(ctx->p_fsum, cap1 * 8);
      sk::CandParams pa = pc;
      pa.out_rows = ctx->p_rows.p;
      pa.out_ids = static_cast<uint32_t*>(ctx->p_ids.p);
      pa.out_fsum = static_cast<u64*>(ctx->p_fsum.p);
      pa.out_reserved = &c->pres;
      pa.kept = &c->pkept;
      pa.coop = 0;
      // weak filter (anti-correlated data): K4a's survivors go straight to S2
      pa.gate = std::getenv("SKYCELL_NOGATE") ? nullptr : &c->fweak;
      pa.alt_rows = ctx->s2_rows.p;
      pa.alt_ids = static_cast<uint32_t*>(ctx->s2_ids.p);
      pa.alt_fsum = static_cast<u64*>(ctx->s2_fsum.p);
      pa.alt_reserved = &c->s2;
      pa.alt_kept = &c->s2_kept;
      if (!k1_head && !std::getenv("SKYCELL_K4A_OLD")) {
        auto ka = wide ? sk::k_cand_head<TOut, D, uint32_t, kThreads> : sk::k_cand_head<TOut, D, uint8_t, kThreads>;
        const size_t sa = ((sk::kK4aHead * D * sizeof(TOut) + 15) & ~(size_t)15) + sk::kK4aHead * 8 +
                          (size_t)(kThreads / 32) * 64 * (D * sizeof(TOut) + 8 + 4) + 16;
        ck(cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa), "smem attr");
        // K4a CTAs per SM (SKYCELL_K4A_CTAS; its output slack is covered by cap1)
        static const int k4a_per_sm = [] {
          const char* e = std::getenv("SKYCELL_K4A_CTAS");
          return e ? std::max(1, std::min(8, std::atoi(e))) : 4;
        }();
        sk::launch(ka, nsm * k4a_per_sm, kThreads, sa, s, pa);
      } else {
        sk::launch(kc, grid4, kThreads, smem_pf, s, pa);
      }
      sk::CandParams pb = pc;
      pb.rows = ctx->p_rows.p;
      pb.ids = static_cast<const uint32_t*>(ctx->p_ids.p);
      pb.count = &c->pres;
      pb.PM = nullptr;
      pb.examined = nullptr;
      pb.d_cells = nullptr;
      pb.head_start = sk::kK4aHead;
      pb.coop = 1;
      pb.coop_mid = 16;  // measured: 16 best at C2 / C4 shards (8..64 swept)
      if (const char* e = std::getenv("SKYCELL_K4B_MID")) pb.coop_mid = (uint32_t)std::max(0, std::atoi(e));
      sk::launch(kc, grid4, kThreads, smem_pf, s, pb);
      ctx->launches += 2;
    } else {
      sk::launch(kc, grid4, kThreads, smem_pf, s, pc);
      ++ctx->launches;
    }
    if (q.timed) ck(cudaEventRecord(ctx->ev[6], s), "event");
  }

  // ---- sparse layer rho (sparse.cuh): U = the layer-rho cells of K4's
  // layer-(rho-1) candidates, classified through the dominance tree; the
  // points of U's candidate cells then meet the filter points -> S2
  void sparse_layer() {
    DevCounters* c = ctr();
    u64 nslots = 0;
    ck(cudaMemcpyAsync(&nslots, &c->s2, 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    fill_words(ctx, s, &c->examined, 2);
    const u64 ns = std::max<u64>(nslots, 1);
    ensure(ctx->sp_keys, ns * 8);
    ensure(ctx->sp_keys2, ns * 8);
    ensure(ctx->sp_vals, ns * 4);
    ensure(ctx->sp_vals2, ns * 4);
    ensure(ctx->sp_head, ns * 4);
    ensure(ctx->sp_cpos, ns * 4);
    ensure(ctx->sp_crows, ns * D * 4);
    ensure(ctx->sp_cfsum, ns * 8);
    ensure(ctx->sp_cids, ns * 4);
    ensure(ctx->sp_cstart, ns * 4);
    ensure(ctx->sp_kflag, ns);
    ensure(ctx->sp_cflag, ns);
    ensure(ctx->sp_n, 64);
    u64* keys = static_cast<u64*>(ctx->sp_keys.p);
    u64* keys2 = static_cast<u64*>(ctx->sp_keys2.p);
    uint32_t* vals = static_cast<uint32_t*>(ctx->sp_vals.p);
    uint32_t* vals2 = static_cast<uint32_t*>(ctx->sp_vals2.p);
    uint32_t* head = static_cast<uint32_t*>(ctx->sp_head.p);
    uint32_t* cpos = static_cast<uint32_t*>(ctx->sp_cpos.p);
    float* crows = static_cast<float*>(ctx->sp_crows.p);
    u64* cfsum = static_cast<u64*>(ctx->sp_cfsum.p);
    uint32_t* cids = static_cast<uint32_t*>(ctx->sp_cids.p);
    uint32_t* cstart = static_cast<uint32_t*>(ctx->sp_cstart.p);
    uint8_t* kflag = static_cast<uint8_t*>(ctx->sp_kflag.p);
    uint8_t* cflag = static_cast<uint8_t*>(ctx->sp_cflag.p);
    u64* spn = static_cast<u64*>(ctx->sp_n.p);  // [ncells, nvalid, queries]
    fill_words(ctx, s, spn, 16);
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((ns + 255) / 256, (u64)nsm * 8));
    sk::launch(sk::k_sp_keys<TOut, D>, g, 256, 0, s, static_cast<const TOut*>(ctx->s2_rows.p),
                                             static_cast<const uint32_t*>(ctx->s2_ids.p), &c->s2, rho_q, keys, vals);
    size_t temp = 0, temp2 = 0;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys, keys2, vals, vals2, (int64_t)ns, 0, rho_q * D, s), "cub");
    ck(cub::DeviceScan::InclusiveSum(nullptr, temp2, head, cpos, (int64_t)ns, s), "cub");
    ensure(ctx->t_cub, std::max(temp, temp2));
    ck(cub::DeviceRadixSort::SortPairs(ctx->t_cub.p, temp, keys, keys2, vals, vals2, (int64_t)ns, 0, rho_q * D, s),
       "cub sort");
    sk::launch(sk::k_sp_heads, g, 256, 0, s, keys2, ns, head);
    ck(cub::DeviceScan::InclusiveSum(ctx->t_cub.p, temp2, head, cpos, (int64_t)ns, s), "cub scan");
    sk::launch(sk::k_sp_cells<D>, g, 256, 0, s, keys2, head, cpos, ns, rho_q, crows, cfsum, cids, cstart, spn, spn + 1);
    ctx->launches += 5;
    // key test: corners dominated by another corner of U (no prefilter, so
    // the tree holds every cell for the strict test below)
    sk::TreeShape sh{};
    run_tree<float, D>(ctx, s, crows, cids, cfsum, spn, &c->tvalid, 0, nullptr, 0, false, true, &sh);
    ck(cudaMemcpyAsync(kflag, ctx->flags.p, ns, cudaMemcpyDeviceToDevice, s), "flags");
    ck(cudaMemsetAsync(cflag, 0, ns, s), "memset");
    if (sh.m) {
      typedef sk::PkLayout<float, D> PL;
      ensure(ctx->sp_qrec, sh.m * PL::PW * 4);
      uint32_t* qrec = static_cast<uint32_t*>(ctx->sp_qrec.p);
      const uint32_t* prec = static_cast<const uint32_t*>(ctx->t_rows.p);
      const uint32_t* nrec = static_cast<const uint32_t*>(ctx->t_lo.p);
      const uint32_t* order = static_cast<const uint32_t*>(ctx->t_vals2.p);
      ctx->host_param[2] = sh.m;
      ck(cudaMemcpyAsync(spn + 2, ctx->host_param + 2, 8, cudaMemcpyHostToDevice, s), "param");
      const unsigned gm = (unsigned)std::max<u64>(1, std::min<u64>((sh.m + 255) / 256, (u64)nsm * 8));
      sk::launch(sk::k_sp_queries<D>, gm, 256, 0, s, prec, sh.m, rho_q, qrec);
      const unsigned gq = (unsigned)std::max<u64>(1, std::min<u64>((sh.nleaf * 32 + 255) / 256, (u64)nsm * 8));
      sk::launch(sk::k_pk_query<float, D, 2>, gq, 256, 0, s, prec, nrec, order, sh, 0, nullptr, 0, nullptr, nullptr, spn + 2,
                                                    qrec, static_cast<uint8_t*>(ctx->flags.p), nullptr);
      sk::launch(sk::k_sp_cand, gm, 256, 0, s, static_cast<const uint8_t*>(ctx->flags.p), qrec + PL::KW + 2, PL::PW, order,
                                      sh.m, cflag);
      ctx->launches += 3;
    }
    sk::launch(sk::k_sp_classify<D>, g, 256, 0, s, crows, kflag, cflag, cstart, spn, spn + 1, rho_q, &c->key[rho_q - 1],
                                          &c->cand[rho_q - 1], &c->examined);
    // the points of candidate cells -> P, then the filter points -> S2
    ensure(ctx->p_rows, cap4 * D * sizeof(TOut));
    ensure(ctx->p_ids, cap4 * 4);
    ensure(ctx->p_fsum, cap4 * 8);
    fill_words(ctx, s, &c->pres, 2);
    sk::launch(sk::k_sp_points<TOut, D>, grid4, kThreads, 0, s, 
        static_cast<const TOut*>(ctx->s2_rows.p), static_cast<const uint32_t*>(ctx->s2_ids.p),
        static_cast<const u64*>(ctx->s2_fsum.p), vals2, keys2, cpos, cflag, ns, static_cast<TOut*>(ctx->p_rows.p),
        static_cast<uint32_t*>(ctx->p_ids.p), static_cast<u64*>(ctx->p_fsum.p), &c->pres, kChunk4);
    fill_words(ctx, s, &c->s2, 2);
    fill_words(ctx, s, &c->s2_kept, 2);
    sk::CandParams pb{};
    pb.rows = ctx->p_rows.p;
    pb.ids = static_cast<const uint32_t*>(ctx->p_ids.p);
    pb.count = &c->pres;
    pb.rho = rho;
    pb.PM = nullptr;
    pb.f_rows = ctx->f_rows.p;
    pb.f_fsum = static_cast<const u64*>(ctx->f_fsum.p);
    pb.f_count = q.merge ? &c->nf : nullptr;
    pb.f_max = q.merge ? (uint32_t)pf_max : 0;
    pb.f_lists = static_cast<const uint16_t*>(ctx->f_lists.p);
    pb.f_offs = static_cast<const uint16_t*>(ctx->f_offs.p);
    pb.out_rows = ctx->s2_rows.p;
    pb.out_ids = static_cast<uint32_t*>(ctx->s2_ids.p);
    pb.out_fsum = static_cast<u64*>(ctx->s2_fsum.p);
    pb.out_reserved = &c->s2;
    pb.chunk = kChunk4;
    pb.kept = &c->s2_kept;
    pb.head_start = 0;
    pb.coop = 1;
    pb.coop_mid = 16;
    auto kc = sk::k_candidates<TOut, D, uint8_t, kThreads>;
    ck(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pf), "smem attr");
    sk::launch(kc, grid4, kThreads, smem_pf, s, pb);
    ctx->launches += 3;
  }

  // ---- K5 over S2 (the local point set)
  void exact_local() {
    DevCounters* c = ctr();
    // the tree above 64K points: measured on one B200, lists win at C2's 50K
    // (1.45 vs 1.9 ms per query), the tree at anti d=3's 84K (K5 1.3 vs 2.6 ms)
    run_dominance<TOut, D>(ctx, s, ctx->s2_rows.p, static_cast<const uint32_t*>(ctx->s2_ids.p),
                           static_cast<const u64*>(ctx->s2_fsum.p), &c->s2, cap4, U(o_hist), U(o_cur), &c->tvalid, 0,
                           nullptr, cell_level(), kTreeMainMin, &c->s2_kept);
    if (q.timed) ck(cudaEventRecord(ctx->ev[7], s), "event");
  }

  // ---- K6: members' ids in ascending order through the id bitmap
  void ids_out(const uint32_t* ids, const u64* count, u64 cap, uint32_t* dst) {
    DevCounters* c = ctr();
    uint32_t* idbits = U(o_idbits);
    unsigned* bcount = U(o_bcount);
    const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((cap + 255) / 256, (u64)nsm * 8));
    sk::launch(sk::k_mark_ids, g, 256, 0, s, ids, static_cast<const uint8_t*>(ctx->flags.p), count, idbits, q.id_base);
    sk::launch(sk::k_bits_count, bit_blocks, sk::kBitsThreads, 0, s, idbits, id_words, bcount);
    sk::launch(sk::k_bits_scan, 1, 1024, 0, s, bcount, bit_blocks, &c->fin);
    sk::launch(sk::k_bits_write, bit_blocks, sk::kBitsThreads, 0, s, idbits, id_words, bcount, dst, q.id_base);
    ctx->launches += 4;
  }

  uint32_t* id_dst() const { return q.ids_dev ? q.ids_dev : static_cast<uint32_t*>(ctx->ids_dev.p); }

  void read_counters() {
    ck(cudaStreamWaitEvent(s, ctx->ev_join, 0), "join");
    static_assert(sizeof(DevCounters) % 8 == 0, "counters are whole words");
    sk::launch(sk::k_copy_words, 1, 64, 0, s, reinterpret_cast<const u64*>(ctr()), ctx->host_ctr_dev,
               (unsigned)(sizeof(DevCounters) / 8));
    ++ctx->launches;
    ck(cudaStreamSynchronize(s), "query");
    if (tracer().on) {
      const DevCounters& h = *ctx->host_ctr;
      std::fprintf(stderr,
                   "[skycell] counters: S1 %llu | sample X %llu (capped %llu), sample skyline %llu, filter points %llu, "
                   "weak filter %llu | K4a pending %llu | S2 %llu | examined %llu\n",
                   (unsigned long long)h.s1_kept, (unsigned long long)h.xd, (unsigned long long)h.xs_cap,
                   (unsigned long long)h.fs, (unsigned long long)h.nf, (unsigned long long)h.fweak,
                   (unsigned long long)h.pkept, (unsigned long long)h.s2_kept, (unsigned long long)h.examined);
    }
  }

  void fill_stats(skycell_gpu_stats* st) const {
    if (!st) return;
    const DevCounters& hc = *ctx->host_ctr;
    st->n_layers = rho_q;
    for (int L = 1; L <= rho_q; ++L) {
      st->keys[L - 1] = hc.key[L - 1] + (u64)D;
      st->candidates[L - 1] = (q.mode == SKYCELL_SEQUENTIAL && L != rho_q) ? -1 : (int64_t)hc.cand[L - 1];
    }
    st->points_examined = hc.examined;
    st->survivors_stream = hc.s1_kept;
    st->survivors_filter = hc.s2_kept;
  }

  void check_finite() const {
    const DevCounters& hc = *ctx->host_ctr;
    if (hc.nonfinite)
      throw ApiFail{SKYCELL_INPUT,
                    "normalize: non-finite coordinate in record " + std::to_string((u64)q.id_base + ~hc.nonfinite)};
  }

  // ---- the single-device query
  void run_single() {
    DevCounters* c = ctr();
    tracer().t0 = std::chrono::steady_clock::now();
    local();
    tracer().mark(s, "K0+K1");
    prune();
    tracer().mark(s, "K3+K4");
    if (sparse) {
      sparse_layer();
      tracer().mark(s, "sparse layer rho");
    }
    exact_local();
    tracer().mark(s, "K5");
    ids_out(static_cast<const uint32_t*>(ctx->s2_ids.p), &c->s2, cap4, id_dst());
    tracer().mark(s, "K6");
    ck(cudaGetLastError(), "kernel launch");
    if (q.timed) ck(cudaEventRecord(ctx->ev[3], s), "event");
    read_counters();
    fill_stats(q.stats);
  }

  // ---- sharded phase 2: prune against the global occupancy, local skyline
  u64 prune_local_skyline() override {
    DevCounters* c = ctr();
    prune();
    exact_local();
    ensure(ctx->sky_rows, cap4 * D * sizeof(TOut));
    ensure(ctx->sky_fsum, cap4 * 8);
    ensure(ctx->sky_ids, cap4 * 4);
    sk::launch(sk::k_pack_members<TOut, D>, nsm * 4, 256, 0, s, 
        static_cast<const TOut*>(ctx->s2_rows.p), static_cast<const uint32_t*>(ctx->s2_ids.p),
        static_cast<const uint8_t*>(ctx->flags.p), static_cast<const u64*>(ctx->s2_fsum.p), &c->s2,
        static_cast<TOut*>(ctx->sky_rows.p), static_cast<u64*>(ctx->sky_fsum.p),
        static_cast<uint32_t*>(ctx->sky_ids.p), &c->lsky);
    ++ctx->launches;
    ck(cudaGetLastError(), "kernel launch");
    read_counters();
    check_finite();
    return ctx->host_ctr->lsky;
  }

  // Block layout of one rank's local skyline in the exchange buffer:
  // [rows maxc x D x TOut][fsum maxc x u64][ids maxc x u32], 256-B aligned.
  static u64 al(u64 b) { return (b + 255) & ~255ull; }
  u64 rows_bytes(u64 maxc) const { return al(maxc * D * sizeof(TOut)); }
  u64 block_bytes(u64 maxc) const override { return rows_bytes(maxc) + al(maxc * 8) + al(maxc * 4); }

  void pack(void* dst, u64 maxc) override {
    const u64 cnt = ctx->host_ctr->lsky;
    char* b = static_cast<char*>(dst);
    if (cnt) {
      ck(cudaMemcpyAsync(b, ctx->sky_rows.p, cnt * D * sizeof(TOut), cudaMemcpyDeviceToDevice, s), "pack");
      ck(cudaMemcpyAsync(b + rows_bytes(maxc), ctx->sky_fsum.p, cnt * 8, cudaMemcpyDeviceToDevice, s), "pack");
      ck(cudaMemcpyAsync(b + rows_bytes(maxc) + al(maxc * 8), ctx->sky_ids.p, cnt * 4, cudaMemcpyDeviceToDevice, s),
         "pack");
    }
    if (maxc > cnt) {
      uint32_t* ids = reinterpret_cast<uint32_t*>(b + rows_bytes(maxc) + al(maxc * 8));
      sk::launch(sk::k_fill_u32, nsm, 256, 0, s, ids + cnt, maxc - cnt, sk::kNoId);
      ++ctx->launches;
    }
  }

  // ---- sharded phase 3: own local skyline against the union -> ids
  void finish(const void* recv, int world, u64 maxc, int rank, u64 own_count, uint32_t* ids_dst, uint64_t* n_out,
              skycell_gpu_stats* st) override {
    DevCounters* c = ctr();
    const u64 un = (u64)world * maxc;
    const u64 cap = std::max<u64>(un, 1);
    // the union, unpacked into flat slot arrays (S2's buffers are free now)
    ensure(ctx->s2_rows, cap * D * sizeof(TOut));
    ensure(ctx->s2_fsum, cap * 8);
    ensure(ctx->s2_ids, cap * 4);
    ensure(ctx->flags, cap);
    const char* r = static_cast<const char*>(recv);
    const u64 bb = block_bytes(maxc);
    if (maxc) {
      ck(cudaMemcpy2DAsync(ctx->s2_rows.p, maxc * D * sizeof(TOut), r, bb, maxc * D * sizeof(TOut), world,
                           cudaMemcpyDeviceToDevice, s), "unpack rows");
      ck(cudaMemcpy2DAsync(ctx->s2_fsum.p, maxc * 8, r + rows_bytes(maxc), bb, maxc * 8, world,
                           cudaMemcpyDeviceToDevice, s), "unpack sums");
      ck(cudaMemcpy2DAsync(ctx->s2_ids.p, maxc * 4, r + rows_bytes(maxc) + al(maxc * 8), bb, maxc * 4, world,
                           cudaMemcpyDeviceToDevice, s), "unpack ids");
    }
    ctx->host_param[0] = un;
    ctx->host_param[1] = (u64)rank * maxc + own_count;
    ck(cudaMemcpyAsync(&c->un, ctx->host_param, 16, cudaMemcpyHostToDevice, s), "params");
    ck(cudaMemsetAsync(ctx->flags.p, 0, cap, s), "flags");
    run_dominance<TOut, D>(ctx, s, ctx->s2_rows.p, static_cast<const uint32_t*>(ctx->s2_ids.p),
                           static_cast<const u64*>(ctx->s2_fsum.p), &c->un, cap, U(o_fhist), U(o_fcur), &c->tvalid,
                           (u64)rank * maxc, &c->qend, cell_level());
    ids_out(static_cast<const uint32_t*>(ctx->s2_ids.p), &c->un, cap, ids_dst ? ids_dst : id_dst());
    ck(cudaGetLastError(), "kernel launch");
    if (q.timed) ck(cudaEventRecord(ctx->ev[3], s), "event");
    read_counters();
    *n_out = ctx->host_ctr->fin;
    fill_stats(st);
  }
};


  // per-dimensionality pipeline instances (inst.cu, compiled once per D):
  // kind 0 = f32 input with the identity range (the benchmark path), 1 = f32
  // input with a general range, 2 = f64 input
  template <int D>
  void run_single_d(const Query& q, int kind);
  template <int D>
  void make_shard_d(const Query& q, int kind, std::unique_ptr<PipeBase>* out);

}  // namespace skyeng
