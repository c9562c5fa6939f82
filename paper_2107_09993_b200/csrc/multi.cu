// Single-process multi-device query (SURVEY.md §8(b) "skycell_gpu_create(int
// n_gpus, ...)", §8(e)): one handle owns G device contexts, shards the
// records by index and runs the sharded protocol of DESIGN.md §4 itself, so
// skycell::gpu::compute_skyline (the drop-in for refine.hpp:61-62) uses every
// GPU of the box from plain C++ -- no MPI, no NCCL communicator to set up.
//
// The two exchanges run device to device, ordered by cross-device events,
// with no host round trip except the two counts the protocol needs anyway:
//   exchange 1: every device ORs all occupancy regions in one kernel that
//               reads the peers' regions in place over NVLink / NVSwitch
//               (k_or_peers; peer access) -- or, without peer access, gathers
//               them with cudaMemcpyPeerAsync and ORs the gather buffer;
//   exchange 2: every device gathers all padded local skylines
//               (cudaMemcpyPeerAsync).
// Each phase runs on one host thread per device, so the devices' H2D
// staging, K0-K5 and finish passes overlap.
#include <thread>

#include "engine.cuh"

using sk::u64;

struct skycell_gpu_multi {
  std::vector<skycell_gpu_ctx*> ctx;
  std::vector<skyeng::DevBuf> occ, gath, send, recv, tbl;  // per device
  std::vector<cudaEvent_t> ev;                             // per device: "my exchange buffer is ready"
  bool peer = true;  // every device reads every other's memory (peer access or the same device)
};

namespace skyeng {

// Runs fn(g) for every device g on its own thread (device set); collects the
// first failure in rank order (the reference reports the lowest record).
template <typename F>
void per_device(skycell_gpu_multi* m, F&& fn) {
  const int G = (int)m->ctx.size();
  std::vector<int> code(G, SKYCELL_OK);
  std::vector<std::string> msg(G);
  std::vector<std::thread> th;
  for (int g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      char err[512] = {0};
      code[g] = guarded(err, sizeof err, [&] {
        ck(cudaSetDevice(m->ctx[g]->device), "cudaSetDevice");
        fn(g);
      });
      msg[g] = err;
    });
  for (auto& t : th) t.join();
  for (int g = 0; g < G; ++g)
    if (code[g] != SKYCELL_OK) throw ApiFail{code[g], msg[g]};
}

// dst[dev] <- src[sdev], after src's event; on the destination's stream.
inline void peer_copy(skycell_gpu_ctx* dst, void* d, skycell_gpu_ctx* src, const void* sp, u64 bytes,
                      cudaEvent_t ready) {
  ck(cudaStreamWaitEvent(dst->stream, ready, 0), "wait");
  if (!bytes) return;
  if (dst->device == src->device)
    ck(cudaMemcpyAsync(d, sp, bytes, cudaMemcpyDeviceToDevice, dst->stream), "copy");
  else
    ck(cudaMemcpyPeerAsync(d, dst->device, sp, src->device, bytes, dst->stream), "peer copy");
}

template <typename TIn>
int multi_query(skycell_gpu_multi* m, const TIn* coords, u64 n, int d, const double* dmin, const double* dmax,
                int rho, int mode, int merge, uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats, char* err,
                size_t err_len) {
  if (!m || m->ctx.empty()) {
    put_err(err, err_len, "skycell_gpu: null multi-device handle");
    return SKYCELL_USAGE;
  }
  // One device does the whole query when sharding cannot apply: a single
  // device, fewer records than devices, merge_cross_cell = false (a
  // test-only superset mode, refine.hpp:50-56) or a sparse layer rho.
  const int G0 = (int)m->ctx.size();
  if (G0 == 1 || n < (u64)G0 || !merge || (u64)rho * d > 36 || (u64)rho * (d - 1) > 30) {
    if constexpr (sizeof(TIn) == 4)
      return skycell_gpu_skyline_f32(m->ctx[0], coords, n, d, dmin, dmax, rho, mode, merge, ids_out, n_out, stats, err,
                                     err_len);
    else
      return skycell_gpu_skyline_f64(m->ctx[0], coords, n, d, dmin, dmax, rho, mode, merge, ids_out, n_out, stats, err,
                                     err_len);
  }
  return guarded(err, err_len, [&] {
    if (!n_out || !ids_out || !coords || !dmin || !dmax)
      throw ApiFail{SKYCELL_USAGE, "skycell_gpu: null coordinate, range or output pointer"};
    Status st = validate_shape(n, d);
    if (st.code) throw ApiFail{st.code, st.msg};
    const int G = G0;
    if (stats) std::memset(stats, 0, sizeof(*stats));
    // shard g owns records [b_g, b_g + n_g): contiguous, the first n % G one longer
    std::vector<u64> b(G), cnt(G);
    for (int g = 0; g < G; ++g) {
      b[g] = g * (n / G) + std::min<u64>(g, n % G);
      cnt[g] = n / G + (g < (int)(n % G) ? 1 : 0);
    }
    const auto t0 = std::chrono::steady_clock::now();
    // phase 1: K0 + K1 per shard; each device exports its occupancy region
    std::vector<uint64_t> occ_bytes(G);
    per_device(m, [&](int g) {
      char e[512] = {0};
      const int rc = skycell_gpu_shard_begin(m->ctx[g], coords + b[g] * d, sizeof(TIn) == 4, cnt[g], d, dmin, dmax,
                                             rho, mode, b[g], &occ_bytes[g], e, sizeof e);
      if (rc) throw ApiFail{rc, e};
      ensure(m->occ[g], occ_bytes[g]);
      if (!m->peer) ensure(m->gath[g], occ_bytes[g] * G);
      m->ctx[g]->shard->export_occ(m->occ[g].p);
      ck(cudaEventRecord(m->ev[g], m->ctx[g]->stream), "event");
    });
    const u64 ob = occ_bytes[0];
    // exchange 1 + phase 2: OR every region, prune, local skyline.  With
    // peer access the OR kernel reads the peers' regions in place (one pass
    // over NVLink / NVSwitch, k_or_peers); otherwise the regions are copied
    // into a gather buffer first.
    std::vector<uint64_t> local(G);
    std::vector<const void*> srcs(G);
    for (int h = 0; h < G; ++h) srcs[h] = m->occ[h].p;
    per_device(m, [&](int g) {
      if (m->peer) {
        ensure(m->tbl[g], sizeof(void*) * G);
        ck(cudaMemcpyAsync(m->tbl[g].p, srcs.data(), sizeof(void*) * G, cudaMemcpyHostToDevice, m->ctx[g]->stream),
           "peer table");
        for (int h = 0; h < G; ++h) ck(cudaStreamWaitEvent(m->ctx[g]->stream, m->ev[h], 0), "wait");
        m->ctx[g]->shard->or_peers(static_cast<const void* const*>(m->tbl[g].p), G);
        local[g] = m->ctx[g]->shard->prune_local_skyline();
      } else {
        for (int h = 0; h < G; ++h)
          peer_copy(m->ctx[g], static_cast<char*>(m->gath[g].p) + h * ob, m->ctx[h], m->occ[h].p, ob, m->ev[h]);
        char e[512] = {0};
        const int rc = skycell_gpu_shard_prune(m->ctx[g], m->gath[g].p, G, &local[g], e, sizeof e);
        if (rc) throw ApiFail{rc, e};
      }
    });
    u64 maxc = 0;
    for (int g = 0; g < G; ++g) maxc = std::max<u64>(maxc, local[g]);
    const u64 bb = skycell_gpu_shard_block_bytes(m->ctx[0], maxc);
    per_device(m, [&](int g) {
      ensure(m->send[g], bb);
      ensure(m->recv[g], bb * G);
      char e[512] = {0};
      const int rc = skycell_gpu_shard_pack(m->ctx[g], m->send[g].p, maxc, e, sizeof e);
      if (rc) throw ApiFail{rc, e};
      ck(cudaEventRecord(m->ev[g], m->ctx[g]->stream), "event");
    });
    // exchange 2 + phase 3: gather the local skylines, own part vs the union
    std::vector<uint64_t> got(G);
    std::vector<skycell_gpu_stats> gst(G);
    per_device(m, [&](int g) {
      for (int h = 0; h < G; ++h)
        peer_copy(m->ctx[g], static_cast<char*>(m->recv[g].p) + h * bb, m->ctx[h], m->send[h].p, bb, m->ev[h]);
      ensure(m->ctx[g]->ids_dev, std::max<u64>(cnt[g], 1) * 4);
      char e[512] = {0};
      const int rc = skycell_gpu_shard_finish(m->ctx[g], m->recv[g].p, G, maxc, g, local[g],
                                              static_cast<uint32_t*>(m->ctx[g]->ids_dev.p), &got[g], &gst[g], e,
                                              sizeof e);
      if (rc) throw ApiFail{rc, e};
    });
    // ids: rank order is ascending global id order
    u64 off = 0;
    const bool dev_out = [&] {
      cudaPointerAttributes a{};
      const bool r = cudaPointerGetAttributes(&a, ids_out) == cudaSuccess &&
                     (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
      cudaGetLastError();
      return r;
    }();
    for (int g = 0; g < G; ++g) {
      if (got[g]) {
        ck(cudaSetDevice(m->ctx[g]->device), "cudaSetDevice");
        ck(cudaMemcpy(ids_out + off, m->ctx[g]->ids_dev.p, got[g] * 4,
                      dev_out ? cudaMemcpyDefault : cudaMemcpyDeviceToHost),
           "ids copy");
      }
      off += got[g];
    }
    *n_out = off;
    if (stats) {
      *stats = gst[0];  // per-layer counts come from the global occupancy
      stats->points_examined = 0;
      stats->survivors_stream = stats->survivors_filter = stats->kernel_launches = 0;
      for (int g = 0; g < G; ++g) {
        stats->points_examined += gst[g].points_examined;
        stats->survivors_stream += gst[g].survivors_stream;
        stats->survivors_filter += gst[g].survivors_filter;
        stats->kernel_launches += gst[g].kernel_launches;
      }
      stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

}  // namespace skyeng

using namespace skyeng;

extern "C" {

int skycell_gpu_multi_create(const int* devices, int n_devices, skycell_gpu_multi** out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    if (!out || !devices || n_devices < 1) throw ApiFail{SKYCELL_USAGE, "skycell_gpu: bad device list"};
    auto* m = new skycell_gpu_multi();
    std::unique_ptr<skycell_gpu_multi, void (*)(skycell_gpu_multi*)> guard(m, skycell_gpu_multi_destroy);
    for (int g = 0; g < n_devices; ++g) {
      skycell_gpu_ctx* c = nullptr;
      char e[512] = {0};
      const int rc = skycell_gpu_create(devices[g], &c, e, sizeof e);
      if (rc) throw ApiFail{rc, e};
      m->ctx.push_back(c);
      cudaEvent_t ev;
      ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
      m->ev.push_back(ev);
    }
    // peer access between distinct devices (NVLink / NVSwitch); copies work
    // without it too, staged by the driver
    for (int a = 0; a < n_devices; ++a)
      for (int b = 0; b < n_devices; ++b) {
        if (devices[a] == devices[b]) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices[a], devices[b]);
        if (!can) {
          m->peer = false;
          continue;
        }
        ck(cudaSetDevice(devices[a]), "cudaSetDevice");
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "peer access");
        cudaGetLastError();
      }
    if (std::getenv("SKYCELL_MULTI_COPY")) m->peer = false;  // force the gather-copy exchange (tests)
    m->occ.resize(n_devices);
    m->tbl.resize(n_devices);
    m->gath.resize(n_devices);
    m->send.resize(n_devices);
    m->recv.resize(n_devices);
    *out = guard.release();
  });
}

void skycell_gpu_multi_destroy(skycell_gpu_multi* m) {
  if (!m) return;
  for (size_t g = 0; g < m->ctx.size(); ++g) {
    cudaSetDevice(m->ctx[g]->device);
    for (auto* v : {&m->occ, &m->gath, &m->send, &m->recv, &m->tbl})
      if (g < v->size() && (*v)[g].p) cudaFree((*v)[g].p);
    if (g < m->ev.size()) cudaEventDestroy(m->ev[g]);
    skycell_gpu_destroy(m->ctx[g]);
  }
  delete m;
}

int skycell_gpu_multi_size(const skycell_gpu_multi* m) { return m ? (int)m->ctx.size() : 0; }

skycell_gpu_ctx* skycell_gpu_multi_context(skycell_gpu_multi* m, int g) {
  return m && g >= 0 && g < (int)m->ctx.size() ? m->ctx[g] : nullptr;
}

int skycell_gpu_multi_skyline_f64(skycell_gpu_multi* m, const double* coords, uint64_t n, int d,
                                  const double* dim_min, const double* dim_max, int rho, int mode,
                                  int merge_cross_cell, uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats,
                                  char* err, size_t err_len) {
  return multi_query<double>(m, coords, n, d, dim_min, dim_max, rho, mode, merge_cross_cell, ids_out, n_out, stats,
                             err, err_len);
}

int skycell_gpu_multi_skyline_f32(skycell_gpu_multi* m, const float* coords, uint64_t n, int d,
                                  const double* dim_min, const double* dim_max, int rho, int mode,
                                  int merge_cross_cell, uint32_t* ids_out, uint64_t* n_out, skycell_gpu_stats* stats,
                                  char* err, size_t err_len) {
  return multi_query<float>(m, coords, n, d, dim_min, dim_max, rho, mode, merge_cross_cell, ids_out, n_out, stats,
                            err, err_len);
}

}  // extern "C"
