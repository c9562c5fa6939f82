// Host orchestration + C ABI (include/skycell_gpu.h) of the B200 SkyCell path.
//
// One query = one pass of compute_skyline (refine.cpp:108-158) on one device:
//   validate (dataset.cpp:23-24, grid.cpp:38-43) -> K0 sample filter -> K1
//   streaming pass -> K3 cell tables + per-layer counts -> K4 candidate
//   filter -> K5 exact sort-first dominance -> K6 ids (ascending) + stats.
// Data-dependent sizes stay on the device (kernels read their input counts
// from device memory).  The host synchronises only where a count must reach
// it: before a K5 whose set may exceed the list threshold (lists or tree,
// and CUB's item count), in the sparse layer-rho stage, and for the final
// read of the counters.
//
// The same pipeline object runs the sharded (multi-GPU) query in phases
// (DESIGN.md §4): local (K0+K1) | occupancy exchange (K2) | prune + local
// skyline (K3-K5) | local-skyline exchange | finish (K5 over the union, K6).
// The collectives themselves are issued by the caller (NCCL through
// torch.distributed in paper_2107_09993_b200/dist.py) on the stream the
// context is bound to (skycell_gpu_set_stream), so no phase needs a host
// synchronisation except where a count must reach the host.
#include "engine.cuh"

using sk::u64;

namespace skyeng {

// --------------------------------------------------------- query plumbing
template <typename TIn>
const void* stage_input(skycell_gpu_ctx* ctx, const TIn* coords, u64 n, int d) {
  // Input residency: device pointers are used in place when 16-byte
  // aligned; host pointers (and misaligned device pointers) are staged.
  cudaPointerAttributes attr{};
  const bool on_device = cudaPointerGetAttributes(&attr, coords) == cudaSuccess &&
                         (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged);
  cudaGetLastError();
  if (on_device && !(reinterpret_cast<uintptr_t>(coords) & 15)) return coords;
  const size_t bytes = n * (size_t)d * sizeof(TIn);
  ensure(ctx->staging, bytes);
  ck(cudaMemcpyAsync(ctx->staging.p, coords, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     ctx->stream),
     "input copy");
  return ctx->staging.p;
}

inline bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  const bool dev = p && cudaPointerGetAttributes(&a, p) == cudaSuccess &&
                   (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
  cudaGetLastError();
  return dev;
}

// normalize() runs before the grid checks (refine.cpp:113 then :117): with an
// invalid rho a non-finite record still wins.
template <typename TIn>
void reject_rho(skycell_gpu_ctx* ctx, const void* dev_coords, u64 n, int d, const Status& rs, u64 id_base) {
  ensure(ctx->reset, 256);
  ck(cudaMemsetAsync(ctx->reset.p, 0, 8, ctx->stream), "memset");
  sk::launch(sk::k_check_finite<TIn>, ctx->num_sms * 4, 256, 0, ctx->stream, static_cast<const TIn*>(dev_coords), n * d, d,
                                                                      static_cast<u64*>(ctx->reset.p));
  u64 nf = 0;
  ck(cudaMemcpyAsync(&nf, ctx->reset.p, 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  ck(cudaStreamSynchronize(ctx->stream), "sync");
  if (nf) throw ApiFail{SKYCELL_INPUT, "normalize: non-finite coordinate in record " + std::to_string(id_base + ~nf)};
  throw ApiFail{rs.code, rs.msg};
}

// Builds the Query (validation, staging, normalisation constants).
template <typename TIn>
Query make_query(skycell_gpu_ctx* ctx, const TIn* coords, u64 n, int d, const double* dmin, const double* dmax,
                 int rho, int mode, int merge, uint32_t* ids_out, skycell_gpu_stats* stats, u64 id_base) {
  Status st = validate_shape(n, d);
  if (st.code) throw ApiFail{st.code, st.msg};
  if (!ctx) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null context"};
  if (!coords || !dmin || !dmax) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null coordinate or range pointer"};
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  ctx->launches = 0;
  const void* dev_coords = stage_input<TIn>(ctx, coords, n, d);
  Status rs = validate_rho(rho, d);
  if (rs.code) reject_rho<TIn>(ctx, dev_coords, n, d, rs, id_base);
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
  q.ids_dev = is_device_ptr(ids_out) ? ids_out : nullptr;
  q.id_base = (uint32_t)id_base;
  // scale[k] = range > 0 ? 1/range : 0, dataset.cpp:32-36 (host, FP64).
  for (int k = 0; k < d; ++k) {
    const double range = dmax[k] - dmin[k];
    q.nm.mn[k] = dmin[k];
    q.nm.sc[k] = range > 0 ? 1.0 / range : 0.0;
  }
  if (stats) std::memset(stats, 0, sizeof(*stats));
  return q;
}

template <typename TIn>
bool identity_range(const Query& q, const double* dmin, const double* dmax) {
  if constexpr (sizeof(TIn) != 4) {
    return false;
  } else {
    for (int k = 0; k < q.d; ++k)
      if (!(dmin[k] == 0.0 && dmax[k] == 1.0)) return false;
    return true;
  }
}

// Dispatch on (input type, identity range, d) to a Pipe instance (inst.cu).
inline int kind_of(bool f32, bool ident) { return f32 ? (ident ? 0 : 1) : 2; }

#define SKYCELL_DCASES(CALL)                                                                          \
  switch (q.d) {                                                                                    \
    case 2: CALL(2); break; case 3: CALL(3); break; case 4: CALL(4); break; case 5: CALL(5); break; \
    case 6: CALL(6); break; case 7: CALL(7); break; case 8: CALL(8); break; case 9: CALL(9); break; \
    case 10: CALL(10); break; case 11: CALL(11); break; case 12: CALL(12); break;                   \
    case 13: CALL(13); break; case 14: CALL(14); break; case 15: CALL(15); break;                  \
    case 16: CALL(16); break;                                                                       \
    default: throw ApiFail{SKYCELL_INPUT, "normalize: dimensionality must be at most 16"};         \
  }

template <typename TIn>
void dispatch_single(const Query& q, bool ident) {
  const int kind = kind_of(sizeof(TIn) == 4, ident);
#define SKYCELL_RUN(DD) run_single_d<DD>(q, kind)
  SKYCELL_DCASES(SKYCELL_RUN)
#undef SKYCELL_RUN
}

template <typename TIn>
void dispatch_shard(const Query& q, bool ident, std::unique_ptr<PipeBase>* out) {
  const int kind = kind_of(sizeof(TIn) == 4, ident);
#define SKYCELL_MAKE(DD) make_shard_d<DD>(q, kind, out)
  SKYCELL_DCASES(SKYCELL_MAKE)
#undef SKYCELL_MAKE
}

template <typename TIn>
int run_query(skycell_gpu_ctx* ctx, const TIn* coords, u64 n, int d, const double* dmin, const double* dmax,
              int rho, int mode, int merge, uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats, char* err,
              size_t err_len) {
  return guarded(err, err_len, [&] {
    const auto t_begin = std::chrono::steady_clock::now();
    if (!n_out || !ids_out) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null output pointer"};
    Query q = make_query<TIn>(ctx, coords, n, d, dmin, dmax, rho, mode, merge, ids_out, stats, 0);
    dispatch_single<TIn>(q, identity_range<TIn>(q, dmin, dmax));
    const DevCounters& hc = *ctx->host_ctr;
    if (hc.nonfinite)
      throw ApiFail{SKYCELL_INPUT, "normalize: non-finite coordinate in record " + std::to_string(~hc.nonfinite)};
    const u64 count = hc.fin;
    *n_out = count;
    if (count && !q.ids_dev) {
      ck(cudaMemcpyAsync(ids_out, ctx->ids_dev.p, count * 4, cudaMemcpyDeviceToHost, ctx->stream), "ids copy");
      ck(cudaStreamSynchronize(ctx->stream), "sync");
    }
    if (stats) {
      float a = 0, b = 0, c = 0, k1 = 0, k4 = 0, k5 = 0;
      cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
      cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
      cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
      cudaEventElapsedTime(&k1, ctx->ev[4], ctx->ev[5]);
      cudaEventElapsedTime(&k4, ctx->ev[2], ctx->ev[6]);
      cudaEventElapsedTime(&k5, ctx->ev[6], ctx->ev[7]);
      stats->filter_kernel_ms = k4;
      stats->dominance_ms = k5;
      stats->normalize_ms = 0.0;  // fused into the streaming pass (grid_ms)
      stats->grid_ms = a;
      stats->shrink_ms = b;
      stats->refine_ms = c;
      stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
      stats->kernel_launches = ctx->launches;
      stats->stream_kernel_ms = k1;
    }
  });
}

template <int D>
void quadrant_launch(skycell_gpu_ctx* ctx, const double* dev, u64 n, const sk::Norm& org, u64 id_words,
                     unsigned blocks, u64* d_count) {
  cudaStream_t s = ctx->stream;
  const int nsm = ctx->num_sms;
  uint32_t* bits = static_cast<uint32_t*>(ctx->q_bits.p);
  unsigned* bcount = reinterpret_cast<unsigned*>(bits + id_words);
  const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((n + 255) / 256, (u64)nsm * 8));
  sk::launch(sk::k_quadrant_mark<D>, g, 256, 0, s, dev, n, org, bits);
  sk::launch(sk::k_bits_count, blocks, sk::kBitsThreads, 0, s, bits, id_words, bcount);
  sk::launch(sk::k_bits_scan, 1, 1024, 0, s, bcount, blocks, d_count);
  sk::launch(sk::k_bits_write, blocks, sk::kBitsThreads, 0, s, bits, id_words, bcount, static_cast<uint32_t*>(ctx->q_orig.p), 0);
  sk::launch(sk::k_quadrant_gather<D>, g, 256, 0, s, dev, static_cast<const uint32_t*>(ctx->q_orig.p), d_count,
                                             static_cast<double*>(ctx->q_sub.p), static_cast<u64*>(ctx->q_mm.p) + 2);
  ctx->launches += 5;
}

}  // namespace skyeng

using namespace skyeng;

extern "C" {

int skycell_gpu_create(int device, skycell_gpu_ctx** out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!out) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null output handle"};
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) throw ApiFail{SKYCELL_CUDA, "skycell_gpu: no CUDA device " + std::to_string(device)};
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new skycell_gpu_ctx();
    ctx->device = device;
    ck(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
    ck(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
    ctx->stream = ctx->own_stream;
    ck(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ctx->ev_k0, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ctx->ev_k0occ, cudaEventDisableTiming), "event");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->host_ctr), sizeof(DevCounters), cudaHostAllocMapped), "pinned");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&ctx->host_param), 64, cudaHostAllocMapped), "pinned");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->host_ctr_dev), ctx->host_ctr, 0), "mapped");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->host_param_dev), ctx->host_param, 0), "mapped");
    ensure(ctx->long_n, 64);
    ensure(ctx->scan_tot, (size_t)2 * sk::kMaxD * sk::kScanChunks * 4);
    for (auto& e : ctx->ev) ck(cudaEventCreate(&e), "event");
    *out = ctx;
  });
}

void skycell_gpu_destroy(skycell_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  ctx->shard.reset();
  DevBuf* bufs[] = {&ctx->reset, &ctx->slabs, &ctx->H, &ctx->table, &ctx->table2, &ctx->table_s, &ctx->staging,
                    &ctx->smp_rows, &ctx->smp_ids, &ctx->smp_fsum, &ctx->f_rows, &ctx->f_fsum, &ctx->f_lists,
                    &ctx->f_offs, &ctx->l_rows, &ctx->l_sums, &ctx->l_ids, &ctx->ids_dev, &ctx->s1_rows, &ctx->s1_ids, &ctx->s2_rows,
                    &ctx->s2_ids, &ctx->s2_fsum, &ctx->flags, &ctx->sky_rows, &ctx->sky_ids, &ctx->sky_fsum,
                    &ctx->q_bits, &ctx->q_orig, &ctx->q_sub, &ctx->q_ids, &ctx->q_mm, &ctx->t_keys,
                    &ctx->t_keys2, &ctx->t_vals, &ctx->t_vals2, &ctx->t_cub, &ctx->t_rows, &ctx->t_ids,
                    &ctx->t_fsum, &ctx->t_lo, &ctx->t_hi, &ctx->t_cs, &ctx->t_ci, &ctx->long_q, &ctx->long_n, &ctx->scan_tot, &ctx->d_cells, &ctx->t_cm, &ctx->t_kill, &ctx->p_rows, &ctx->p_ids, &ctx->p_fsum, &ctx->k5dbg, &ctx->sp_keys, &ctx->sp_keys2, &ctx->sp_vals, &ctx->sp_vals2, &ctx->sp_head, &ctx->sp_cpos, &ctx->sp_crows, &ctx->sp_cfsum, &ctx->sp_cids, &ctx->sp_cstart, &ctx->sp_kflag, &ctx->sp_cflag, &ctx->sp_n, &ctx->sp_qrec};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->host_ctr) cudaFreeHost(ctx->host_ctr);
  if (ctx->host_param) cudaFreeHost(ctx->host_param);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_k0) cudaEventDestroy(ctx->ev_k0);
  if (ctx->ev_k0occ) cudaEventDestroy(ctx->ev_k0occ);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int skycell_gpu_set_stream(skycell_gpu_ctx* ctx, void* stream, int use_own) {
  if (!ctx) return SKYCELL_USAGE;
  ctx->stream = use_own ? ctx->own_stream : static_cast<cudaStream_t>(stream);  // 0 = the legacy default stream
  return SKYCELL_OK;
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

int skycell_gpu_quadrant_f64(skycell_gpu_ctx* ctx, const double* coords, uint64_t n, int d, const double* origin,
                             int origin_len, int rho, int mode, uint32_t* ids_out, uint64_t* n_out,
                             skycell_gpu_stats* stats, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null context"};
    if (!n_out || !ids_out) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null output pointer"};
    // refine.cpp:162-163
    if (origin_len != d)
      throw ApiFail{SKYCELL_USAGE, "quadrant_skyline: origin arity does not match the dataset dimensionality"};
    if (stats) std::memset(stats, 0, sizeof(*stats));
    *n_out = 0;
    if (n == 0) return;  // empty quadrant -> empty result (refine.cpp:176)
    if (d < 1 || d > sk::kMaxD) throw ApiFail{SKYCELL_INPUT, "normalize: dimensionality must be at most 16"};
    if (d < 2) throw ApiFail{SKYCELL_INPUT, "normalize: dimensionality must be at least 2"};
    if (n > 0xffffffffull) throw ApiFail{SKYCELL_INPUT, "normalize: more than 2^32 - 1 records"};
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    ctx->launches = 0;
    cudaStream_t s = ctx->stream;
    const double* dev = static_cast<const double*>(stage_input<double>(ctx, coords, n, d));
    const u64 id_words = (n + 31) / 32;
    const unsigned blocks = (unsigned)((id_words + sk::kBitsBlock - 1) / sk::kBitsBlock);
    ensure(ctx->q_bits, id_words * 4 + (u64)blocks * 4);
    ensure(ctx->q_orig, n * 4);
    ensure(ctx->q_sub, n * (u64)d * 8);
    ensure(ctx->q_mm, (2 + 2 * (u64)d) * 8);
    ck(cudaMemsetAsync(ctx->q_bits.p, 0, id_words * 4, s), "memset");
    // q_mm = [count, pad, (min key, max key) x d]
    ck(cudaMemsetAsync(ctx->q_mm.p, 0, 16, s), "memset");
    std::vector<u64> init(2 * d);
    for (int k = 0; k < d; ++k) {
      init[2 * k] = ~0ull;
      init[2 * k + 1] = 0;
    }
    ck(cudaMemcpyAsync(static_cast<u64*>(ctx->q_mm.p) + 2, init.data(), 16 * (u64)d, cudaMemcpyHostToDevice, s),
       "mm init");
    sk::Norm org{};
    for (int k = 0; k < d; ++k) org.mn[k] = origin[k];
    u64* d_count = static_cast<u64*>(ctx->q_mm.p);
#define SKYCELL_Q(DD) \
  case DD: quadrant_launch<DD>(ctx, dev, n, org, id_words, blocks, d_count); break;
    switch (d) {
      SKYCELL_Q(2) SKYCELL_Q(3) SKYCELL_Q(4) SKYCELL_Q(5) SKYCELL_Q(6) SKYCELL_Q(7) SKYCELL_Q(8) SKYCELL_Q(9)
      SKYCELL_Q(10) SKYCELL_Q(11) SKYCELL_Q(12) SKYCELL_Q(13) SKYCELL_Q(14) SKYCELL_Q(15) SKYCELL_Q(16)
    }
#undef SKYCELL_Q
    ck(cudaGetLastError(), "kernel launch");
    std::vector<u64> mm(2 + 2 * d);
    ck(cudaMemcpyAsync(mm.data(), ctx->q_mm.p, mm.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    const u64 sub_n = mm[0];
    if (sub_n == 0) return;  // refine.cpp:176
    std::vector<double> mn(d), mx(d);
    for (int k = 0; k < d; ++k) {
      mn[k] = sk::dkey_inv(mm[2 + 2 * k]);
      mx[k] = sk::dkey_inv(mm[2 + 2 * k + 1]);
    }
    // refine.cpp:179: sub_rho = min(rho, max(1, default_rho(sub.n, d)))
    const int sub_rho = std::min(rho, std::max(1, default_rho(sub_n, d)));
    ensure(ctx->q_ids, sub_n * 4);
    uint32_t* sub_ids = static_cast<uint32_t*>(ctx->q_ids.p);
    const u64 prior = ctx->launches;
    uint64_t k = 0;
    const int rc = run_query<double>(ctx, static_cast<const double*>(ctx->q_sub.p), sub_n, d, mn.data(), mx.data(),
                                     sub_rho, mode, 1, sub_ids, &k, stats, err, err_len);
    if (rc != SKYCELL_OK) throw ApiFail{rc, std::string(err ? err : "")};
    ctx->launches += prior;
    if (k) {
      const unsigned g = (unsigned)std::max<u64>(1, std::min<u64>((k + 255) / 256, (u64)ctx->num_sms * 8));
      sk::launch(sk::k_map_ids, g, 256, 0, s, sub_ids, static_cast<const uint32_t*>(ctx->q_orig.p), k);
      ++ctx->launches;
      ck(cudaGetLastError(), "kernel launch");
      if (is_device_ptr(ids_out)) ck(cudaMemcpyAsync(ids_out, sub_ids, k * 4, cudaMemcpyDeviceToDevice, s), "ids");
      else ck(cudaMemcpyAsync(ids_out, sub_ids, k * 4, cudaMemcpyDeviceToHost, s), "ids");
      ck(cudaStreamSynchronize(s), "sync");
    }
    *n_out = k;
    if (stats) stats->kernel_launches = ctx->launches;
  });
}

// ------------------------------------------------------ sharded query (§4)
int skycell_gpu_shard_begin(skycell_gpu_ctx* ctx, const void* coords, int coords_f32, uint64_t n, int d,
                            const double* dim_min, const double* dim_max, int rho, int mode, uint64_t id_base,
                            uint64_t* occ_bytes, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx || !occ_bytes) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null context or output pointer"};
    ctx->shard.reset();
    if (id_base + n > 0xffffffffull) throw ApiFail{SKYCELL_INPUT, "normalize: more than 2^32 - 1 records"};
    if ((u64)rho * d > 36 || (u64)rho * (d - 1) > 30)
      throw ApiFail{SKYCELL_UNSUPPORTED, "skycell_gpu: sharded query with rho*d = " + std::to_string(rho * d) +
                                             ": the sparse layer-rho index is single-device only"};
    if (coords_f32) {
      Query q = make_query<float>(ctx, static_cast<const float*>(coords), n, d, dim_min, dim_max, rho, mode, 1,
                                  nullptr, nullptr, id_base);
      q.timed = true;  // K1 events: stream_kernel_ms of the finish stats
      dispatch_shard<float>(q, identity_range<float>(q, dim_min, dim_max), &ctx->shard);
    } else {
      Query q = make_query<double>(ctx, static_cast<const double*>(coords), n, d, dim_min, dim_max, rho, mode, 1,
                                   nullptr, nullptr, id_base);
      q.timed = true;
      dispatch_shard<double>(q, false, &ctx->shard);
    }
    ck(cudaGetLastError(), "kernel launch");
    *occ_bytes = ctx->shard->occ_bytes();
  });
}

int skycell_gpu_shard_export_occ(skycell_gpu_ctx* ctx, void* dev_dst, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx || !ctx->shard) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: no sharded query in flight"};
    ctx->shard->export_occ(dev_dst);
  });
}

int skycell_gpu_shard_prune(skycell_gpu_ctx* ctx, const void* dev_gathered, int world, uint64_t* local_count,
                            char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx || !ctx->shard) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: no sharded query in flight"};
    if (world < 1 || !dev_gathered || !local_count) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: bad exchange buffer"};
    ctx->shard->or_gathered(dev_gathered, world);
    *local_count = ctx->shard->prune_local_skyline();
  });
}

uint64_t skycell_gpu_shard_block_bytes(skycell_gpu_ctx* ctx, uint64_t max_count) {
  if (!ctx || !ctx->shard) return 0;
  return ctx->shard->block_bytes(max_count);
}

int skycell_gpu_shard_pack(skycell_gpu_ctx* ctx, void* dev_dst, uint64_t max_count, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx || !ctx->shard) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: no sharded query in flight"};
    ctx->shard->pack(dev_dst, max_count);
  });
}

int skycell_gpu_shard_finish(skycell_gpu_ctx* ctx, const void* dev_recv, int world, uint64_t max_count, int rank,
                             uint64_t own_count, uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats,
                             char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!ctx || !ctx->shard) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: no sharded query in flight"};
    if (rank < 0 || rank >= world || !n_out) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: bad rank or output pointer"};
    if (stats) std::memset(stats, 0, sizeof(*stats));
    const bool dev_out = is_device_ptr(ids_out);
    ctx->shard->finish(dev_recv, world, max_count, rank, own_count, dev_out ? ids_out : nullptr, n_out, stats);
    if (!dev_out && *n_out) {
      if (!ids_out) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null output pointer"};
      ck(cudaMemcpyAsync(ids_out, ctx->ids_dev.p, *n_out * 4, cudaMemcpyDeviceToHost, ctx->stream), "ids copy");
      ck(cudaStreamSynchronize(ctx->stream), "sync");
    }
    if (stats) {
      stats->kernel_launches = ctx->launches;
      float k1 = 0, k4 = 0, k5 = 0;
      cudaEventElapsedTime(&k1, ctx->ev[4], ctx->ev[5]);
      cudaEventElapsedTime(&k4, ctx->ev[2], ctx->ev[6]);
      cudaEventElapsedTime(&k5, ctx->ev[6], ctx->ev[7]);
      stats->stream_kernel_ms = k1;
      stats->filter_kernel_ms = k4;
      stats->dominance_ms = k5;
    }
    ctx->shard.reset();
  });
}

int skycell_gpu_generate(skycell_gpu_ctx* ctx, int dist, uint64_t n, int d, uint64_t seed, int kind, void* dev_out,
                         char* err, size_t err_len) {
  return skycell_gpu_generate_range(ctx, dist, n, d, seed, kind, 0, n, dev_out, err, err_len);
}

int skycell_gpu_generate_range(skycell_gpu_ctx* ctx, int dist, uint64_t n, int d, uint64_t seed, int kind,
                               uint64_t begin, uint64_t count, void* dev_out, char* err, size_t err_len) {
  // generate(): ConfigError on n < 1, d < 2, d > kMaxDims (datagen.cpp:63-65)
  if (n < 1) { put_err(err, err_len, "generate: n must be at least 1"); return SKYCELL_CONFIG; }
  if (d < 2) { put_err(err, err_len, "generate: d must be at least 2"); return SKYCELL_CONFIG; }
  if (d > sk::kMaxD) { put_err(err, err_len, "generate: d must be at most 16"); return SKYCELL_CONFIG; }
  if (dist < 0 || dist > 2 || kind < 0 || kind > 1 || !ctx || begin > n || count > n - begin) {
    put_err(err, err_len, "generate: bad distribution, output kind or record range");
    return SKYCELL_USAGE;
  }
  return guarded(err, err_len, [&] {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (count == 0) return;
    const u64 b0 = begin / 65536, b1 = (begin + count + 65535) / 65536;
    const unsigned g = (unsigned)std::max<u64>(1, (b1 - b0 + 127) / 128);
#define SKYCELL_GEN(DD) \
  case DD: sk::launch(sk::k_generate<DD>, g, 128, 0, ctx->stream, dist, n, seed, kind, begin, count, dev_out); break;
    switch (d) {
      SKYCELL_GEN(2) SKYCELL_GEN(3) SKYCELL_GEN(4) SKYCELL_GEN(5) SKYCELL_GEN(6) SKYCELL_GEN(7) SKYCELL_GEN(8)
      SKYCELL_GEN(9) SKYCELL_GEN(10) SKYCELL_GEN(11) SKYCELL_GEN(12) SKYCELL_GEN(13) SKYCELL_GEN(14)
      SKYCELL_GEN(15) SKYCELL_GEN(16)
    }
#undef SKYCELL_GEN
    ck(cudaGetLastError(), "generate launch");
    ck(cudaStreamSynchronize(ctx->stream), "generate");
  });
}

int skycell_default_rho(uint64_t n, int d) { return default_rho(n, d); }

int skycell_validate(uint64_t n, int d, int rho, char* err, size_t err_len) {
  Status st = validate_shape(n, d);
  if (!st.code) st = validate_rho(rho, d);
  if (st.code) put_err(err, err_len, st.msg);
  return st.code;
}

const char* skycell_gpu_version(void) { return "skycell-b200 0.2 (sm_100a)"; }

}  // extern "C"
