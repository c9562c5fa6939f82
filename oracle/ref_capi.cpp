// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI shim over the *unmodified* reference library, compiled together with
// /root/reference/proj/src/*.cpp into oracle/_ref/libskycell_ref.so by
// oracle/Makefile.  It lets the Python tests, tests/golden/make_golden.py and
// bench.py's reference arm (`--impl reference`, `cpu_baseline`) call the
// reference's own entry points through ctypes:
//
//   skycell::generate            proj/src/datagen.cpp:62-87
//   skycell::compute_skyline     proj/src/refine.cpp:108-158
//   skycell::quadrant_skyline    proj/src/refine.cpp:160-184
//   skycell::brute_force_skyline proj/src/baseline.cpp:32-58
//   MultiLayerGrid::default_rho  proj/src/grid.cpp:30-33
//   skycell::write_bin/read_bin  proj/src/datagen.cpp:185-221
//
// Exceptions are mapped onto the same status codes the product C-ABI uses
// (include/skycell_gpu.h) so that error parity can be asserted code-for-code
// and message-for-message.

#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "skycell/baseline.hpp"
#include "skycell/datagen.hpp"
#include "skycell/grid.hpp"
#include "skycell/refine.hpp"

namespace {

enum Status { kOk = 0, kInput = 1, kConfig = 2, kUsage = 3, kIo = 4, kInternal = 9 };

void put_err(char* err, size_t len, const char* msg) {
  if (err == nullptr || len == 0) return;
  std::strncpy(err, msg, len - 1);
  err[len - 1] = '\0';
}

template <typename F>
int guarded(char* err, size_t len, F&& body) {
  try {
    body();
    return kOk;
  } catch (const skycell::InputError& e) {
    put_err(err, len, e.what());
    return kInput;
  } catch (const skycell::ConfigError& e) {
    put_err(err, len, e.what());
    return kConfig;
  } catch (const skycell::UsageError& e) {
    put_err(err, len, e.what());
    return kUsage;
  } catch (const skycell::IoError& e) {
    put_err(err, len, e.what());
    return kIo;
  } catch (const std::exception& e) {
    put_err(err, len, e.what());
    return kInternal;
  }
}

skycell::Dataset make_ds(const double* coords, uint64_t n, int d, const double* dmin,
                         const double* dmax) {
  skycell::Dataset ds;
  ds.n = static_cast<uint32_t>(n);
  ds.d = d;
  ds.coords.assign(coords, coords + n * static_cast<uint64_t>(d));
  ds.dim_min.assign(dmin, dmin + d);
  ds.dim_max.assign(dmax, dmax + d);
  return ds;
}

}  // namespace

extern "C" {

// Mirrors SkylineResult (refine.hpp:19-38); layer arrays hold rho entries.
struct ref_stats {
  double normalize_ms, grid_ms, shrink_ms, refine_ms, total_ms;
  uint64_t points_examined;
  int32_t n_layers;
  int32_t pad_;
  uint64_t keys[64];
  int64_t candidates[64];
};

int ref_generate(int dist, uint64_t n, int d, uint64_t seed, int workers, double* out, char* err,
                 size_t err_len) {
  return guarded(err, err_len, [&] {
    skycell::GenSpec spec{static_cast<skycell::Distribution>(dist), n, d, seed};
    skycell::Dataset ds;
    if (workers == 1) {
      ds = skycell::generate(spec);
    } else {
      skycell::ThreadPool pool(workers < 0 ? 0u : static_cast<unsigned>(workers));
      ds = skycell::generate(spec, &pool);
    }
    std::memcpy(out, ds.coords.data(), ds.coords.size() * sizeof(double));
  });
}

int ref_default_rho(uint64_t n, int d) { return skycell::MultiLayerGrid::default_rho(n, d); }

// MultiLayerGrid over a normalised PointSet (ids 0..n-1): the sorted ids,
// the non-empty counts of layers 0..rho, the non-empty leaf cells (linear
// index, range) in enumeration order, and the non-empty cells of `layer`.
int ref_grid(const double* coords, uint64_t n, int d, int rho, int layer, uint32_t* sorted_ids, uint64_t* counts,
             uint64_t* leaf_lin, uint32_t* leaf_begin, uint32_t* leaf_end, uint64_t* layer_lin, char* err,
             size_t err_len) {
  return guarded(err, err_len, [&] {
    skycell::PointSet ps;
    ps.n = static_cast<uint32_t>(n);
    ps.d = d;
    ps.coords.assign(coords, coords + n * static_cast<uint64_t>(d));
    ps.ids.resize(n);
    for (uint32_t i = 0; i < n; ++i) ps.ids[i] = i;
    skycell::MultiLayerGrid g(std::move(ps), rho);
    std::memcpy(sorted_ids, g.points().ids.data(), n * sizeof(uint32_t));
    for (int L = 0; L <= rho; ++L) counts[L] = g.nonempty_count(L);
    const auto leaves = g.nonempty_cells(rho);
    for (size_t i = 0; i < leaves.size(); ++i) {
      leaf_lin[i] = leaves[i].linear_index();
      const skycell::CellRange r = g.range(leaves[i]);
      leaf_begin[i] = r.begin;
      leaf_end[i] = r.end;
    }
    const auto cells = g.nonempty_cells(layer);
    for (size_t i = 0; i < cells.size(); ++i) layer_lin[i] = cells[i].linear_index();
  });
}

int ref_write_bin(const char* path, const double* coords, uint64_t n, int d, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const std::vector<double> lo(d, 0.0), hi(d, 1.0);
    skycell::write_bin(make_ds(coords, n, d, lo.data(), hi.data()), path);
  });
}

// read_bin in two calls: the header (n, d), then the data and min/max into
// caller buffers (out may be null on the first call).
int ref_read_bin(const char* path, uint64_t* n, int* d, double* out, double* dmin, double* dmax, char* err,
                 size_t err_len) {
  return guarded(err, err_len, [&] {
    const skycell::Dataset ds = skycell::read_bin(path);
    *n = ds.n;
    *d = ds.d;
    if (out) {
      std::memcpy(out, ds.coords.data(), ds.coords.size() * sizeof(double));
      std::memcpy(dmin, ds.dim_min.data(), ds.d * sizeof(double));
      std::memcpy(dmax, ds.dim_max.data(), ds.d * sizeof(double));
    }
  });
}

static void fill_stats(const skycell::SkylineResult& r, ref_stats* st) {
  if (st == nullptr) return;
  std::memset(st, 0, sizeof(*st));
  st->normalize_ms = r.times.normalize_ms;
  st->grid_ms = r.times.grid_ms;
  st->shrink_ms = r.times.shrink_ms;
  st->refine_ms = r.times.refine_ms;
  st->total_ms = r.times.total_ms;
  st->points_examined = r.points_examined;
  st->n_layers = static_cast<int32_t>(r.layers.keys.size());
  for (size_t i = 0; i < r.layers.keys.size() && i < 64; ++i) st->keys[i] = r.layers.keys[i];
  for (size_t i = 0; i < r.layers.candidates.size() && i < 64; ++i)
    st->candidates[i] = r.layers.candidates[i];
}

// ids_out must hold n entries.
int ref_compute_skyline(const double* coords, uint64_t n, int d, const double* dmin,
                        const double* dmax, int rho, int mode, int merge_cross_cell, int workers,
                        uint32_t* ids_out, uint64_t* n_out, ref_stats* stats, char* err,
                        size_t err_len) {
  return guarded(err, err_len, [&] {
    const skycell::Dataset ds = make_ds(coords, n, d, dmin, dmax);
    skycell::ThreadPool pool(workers < 0 ? 0u : static_cast<unsigned>(workers));
    const skycell::SkylineResult r =
        skycell::compute_skyline(ds, rho, static_cast<skycell::Mode>(mode), pool, merge_cross_cell != 0);
    std::memcpy(ids_out, r.ids.data(), r.ids.size() * sizeof(uint32_t));
    *n_out = r.ids.size();
    fill_stats(r, stats);
  });
}

int ref_quadrant_skyline(const double* coords, uint64_t n, int d, const double* dmin,
                         const double* dmax, const double* origin, int origin_len, int rho,
                         int mode, int workers, uint32_t* ids_out, uint64_t* n_out,
                         ref_stats* stats, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const skycell::Dataset ds = make_ds(coords, n, d, dmin, dmax);
    skycell::ThreadPool pool(workers < 0 ? 0u : static_cast<unsigned>(workers));
    const skycell::SkylineResult r = skycell::quadrant_skyline(
        ds, std::span<const double>(origin, static_cast<size_t>(origin_len)), rho,
        static_cast<skycell::Mode>(mode), pool);
    std::memcpy(ids_out, r.ids.data(), r.ids.size() * sizeof(uint32_t));
    *n_out = r.ids.size();
    fill_stats(r, stats);
  });
}

// brute_force_skyline(normalize(ds)) -- the reference's all-pairs oracle.
int ref_brute_force(const double* coords, uint64_t n, int d, const double* dmin, const double* dmax,
                    uint32_t cap, int workers, uint32_t* ids_out, uint64_t* n_out, char* err,
                    size_t err_len) {
  return guarded(err, err_len, [&] {
    const skycell::Dataset ds = make_ds(coords, n, d, dmin, dmax);
    skycell::ThreadPool pool(workers < 0 ? 0u : static_cast<unsigned>(workers));
    const auto ids = skycell::brute_force_skyline(skycell::normalize(ds), cap, &pool);
    std::memcpy(ids_out, ids.data(), ids.size() * sizeof(uint32_t));
    *n_out = ids.size();
  });
}

// normalize(ds) (dataset.cpp:22-50): out holds n*d normalized doubles.
int ref_normalize(const double* coords, uint64_t n, int d, const double* dmin, const double* dmax,
                  double* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const skycell::Dataset ds = make_ds(coords, n, d, dmin, dmax);
    const skycell::PointSet ps = skycell::normalize(ds);
    std::memcpy(out, ps.coords.data(), ps.coords.size() * sizeof(double));
  });
}

// Dataset::compute_minmax (dataset.cpp:10-20).
void ref_compute_minmax(const double* coords, uint64_t n, int d, double* dmin, double* dmax) {
  skycell::Dataset ds;
  ds.n = static_cast<uint32_t>(n);
  ds.d = d;
  ds.coords.assign(coords, coords + n * static_cast<uint64_t>(d));
  ds.compute_minmax();
  std::memcpy(dmin, ds.dim_min.data(), d * sizeof(double));
  std::memcpy(dmax, ds.dim_max.data(), d * sizeof(double));
}

}  // extern "C"
