// skycell_gpu.hpp -- the reference's C++ signature over the B200 C ABI.
//
// Header-only.  Include it from code that already uses the reference headers
// (proj/include/skycell/*.hpp) and link libskycell_gpu.so next to the
// reference library.  The functions live in skycell::gpu so they never clash
// with skycell::compute_skyline (one-definition rule).
//
//   skycell::gpu::compute_skyline   replaces  skycell::compute_skyline
//                                   (proj/include/skycell/refine.hpp:61-62,
//                                    proj/src/refine.cpp:108-158)
//   skycell::gpu::quadrant_skyline  replaces  skycell::quadrant_skyline
//                                   (refine.hpp:66-68, refine.cpp:160-184)
//   skycell::gpu::MultiDevice       compute_skyline sharded over several
//                                   GPUs of one process
//   skycell::gpu::MultiLayerGrid    replaces  skycell::MultiLayerGrid
//                                   (grid.hpp:33-70, grid.cpp:35-140)
//
// Status codes are rethrown as the reference's exception types
// (proj/include/skycell/error.hpp:9-26) with the reference's message text.
// The ThreadPool argument is accepted for signature parity and unused: the
// GPU path runs no host worker threads.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "skycell/dataset.hpp"
#include "skycell/error.hpp"
#include "skycell/grid.hpp"
#include "skycell/parallel.hpp"
#include "skycell/refine.hpp"
#include "skycell_gpu.h"

namespace skycell::gpu {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::logic_error {
  using std::logic_error::logic_error;
};

inline void throw_status(int code, const char* msg) {
  switch (code) {
    case SKYCELL_OK: return;
    case SKYCELL_INPUT: throw skycell::InputError(msg);
    case SKYCELL_CONFIG: throw skycell::ConfigError(msg);
    case SKYCELL_USAGE: throw skycell::UsageError(msg);
    case SKYCELL_IO: throw skycell::IoError(msg);
    case SKYCELL_UNSUPPORTED: throw Unsupported(msg);
    default: throw CudaError(msg);
  }
}

// One context per device, created on first use and kept for the process
// lifetime (scratch buffers are reused across calls).  Calls on one context
// are serialised by a mutex, matching the reference's reentrancy contract.
class Device {
 public:
  explicit Device(int device = 0) {
    char err[512] = {0};
    throw_status(skycell_gpu_create(device, &ctx_, err, sizeof err), err);
  }
  ~Device() { skycell_gpu_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  skycell_gpu_ctx* context() { return ctx_; }
  std::mutex& mutex() { return mu_; }

  SkylineResult compute_skyline(const Dataset& ds, int rho, Mode mode, bool merge_cross_cell = true) {
    SkylineResult r;
    r.ids.resize(ds.n > 0 ? ds.n : 1);
    skycell_gpu_stats st{};
    uint64_t n_out = 0;
    char err[512] = {0};
    int rc;
    {
      std::lock_guard<std::mutex> lock(mu_);
      rc = skycell_gpu_skyline_f64(ctx_, ds.coords.data(), ds.n, ds.d, ds.dim_min.data(), ds.dim_max.data(), rho,
                                   mode == Mode::kSequential ? SKYCELL_SEQUENTIAL : SKYCELL_PARALLEL,
                                   merge_cross_cell ? 1 : 0, r.ids.data(), &n_out, &st, err, sizeof err);
    }
    throw_status(rc, err);
    r.ids.resize(n_out);
    fill(r, st);
    return r;
  }

  SkylineResult quadrant_skyline(const Dataset& ds, std::span<const double> origin, int rho, Mode mode) {
    SkylineResult r;
    r.ids.resize(ds.n > 0 ? ds.n : 1);
    skycell_gpu_stats st{};
    uint64_t n_out = 0;
    char err[512] = {0};
    int rc;
    {
      std::lock_guard<std::mutex> lock(mu_);
      rc = skycell_gpu_quadrant_f64(ctx_, ds.coords.data(), ds.n, ds.d, origin.data(), (int)origin.size(), rho,
                                    mode == Mode::kSequential ? SKYCELL_SEQUENTIAL : SKYCELL_PARALLEL, r.ids.data(),
                                    &n_out, &st, err, sizeof err);
    }
    throw_status(rc, err);
    r.ids.resize(n_out);
    fill(r, st);
    return r;
  }

 private:
  static void fill(SkylineResult& r, const skycell_gpu_stats& st) {
    r.times.normalize_ms = st.normalize_ms;
    r.times.grid_ms = st.grid_ms;
    r.times.shrink_ms = st.shrink_ms;
    r.times.refine_ms = st.refine_ms;
    r.times.total_ms = st.total_ms;
    r.points_examined = st.points_examined;
    r.layers.keys.assign(st.keys, st.keys + st.n_layers);
    r.layers.candidates.assign(st.candidates, st.candidates + st.n_layers);
  }
  skycell_gpu_ctx* ctx_ = nullptr;
  std::mutex mu_;
};

// Several devices in one process (skycell_gpu_multi_*): records are sharded
// by index over the listed devices and the library runs both exchanges
// itself (device-to-device copies over NVLink / NVSwitch).  Same results as
// Device::compute_skyline.
class MultiDevice {
 public:
  explicit MultiDevice(const std::vector<int>& devices) {
    char err[512] = {0};
    throw_status(skycell_gpu_multi_create(devices.data(), (int)devices.size(), &m_, err, sizeof err), err);
  }
  ~MultiDevice() { skycell_gpu_multi_destroy(m_); }
  MultiDevice(const MultiDevice&) = delete;
  MultiDevice& operator=(const MultiDevice&) = delete;

  SkylineResult compute_skyline(const Dataset& ds, int rho, Mode mode, bool merge_cross_cell = true) {
    SkylineResult r;
    r.ids.resize(ds.n > 0 ? ds.n : 1);
    skycell_gpu_stats st{};
    uint64_t n_out = 0;
    char err[512] = {0};
    int rc;
    {
      std::lock_guard<std::mutex> lock(mu_);
      rc = skycell_gpu_multi_skyline_f64(m_, ds.coords.data(), ds.n, ds.d, ds.dim_min.data(), ds.dim_max.data(), rho,
                                         mode == Mode::kSequential ? SKYCELL_SEQUENTIAL : SKYCELL_PARALLEL,
                                         merge_cross_cell ? 1 : 0, r.ids.data(), &n_out, &st, err, sizeof err);
    }
    throw_status(rc, err);
    r.ids.resize(n_out);
    r.times.normalize_ms = st.normalize_ms;
    r.times.grid_ms = st.grid_ms;
    r.times.shrink_ms = st.shrink_ms;
    r.times.refine_ms = st.refine_ms;
    r.times.total_ms = st.total_ms;
    r.points_examined = st.points_examined;
    r.layers.keys.assign(st.keys, st.keys + st.n_layers);
    r.layers.candidates.assign(st.candidates, st.candidates + st.n_layers);
    return r;
  }

 private:
  skycell_gpu_multi* m_ = nullptr;
  std::mutex mu_;
};

inline Device& default_device() {
  static Device dev(0);
  return dev;
}

// Same signature and semantics as skycell::compute_skyline (refine.hpp:61-62).
inline SkylineResult compute_skyline(const Dataset& ds, int rho, Mode mode, ThreadPool& /*pool*/,
                                     bool merge_cross_cell = true) {
  return default_device().compute_skyline(ds, rho, mode, merge_cross_cell);
}

// Same signature and semantics as skycell::quadrant_skyline (refine.hpp:66-68).
inline SkylineResult quadrant_skyline(const Dataset& ds, std::span<const double> origin, int rho, Mode mode,
                                      ThreadPool& /*pool*/) {
  return default_device().quadrant_skyline(ds, origin, rho, mode);
}

// Same interface as skycell::MultiLayerGrid (grid.hpp:33-70), built on the
// device (skycell_gpu_grid_*): the sorted PointSet, layer-rho ranges,
// occupancy of every layer.  Needs the reference headers and library for
// CellIndex / point_to_cell, like the rest of this header.
class MultiLayerGrid {
 public:
  MultiLayerGrid(PointSet points, int rho, Device& dev = default_device()) : rho_(rho) {
    char err[512] = {0};
    int rc;
    {
      std::lock_guard<std::mutex> lock(dev.mutex());
      rc = skycell_gpu_grid_build(dev.context(), points.coords.data(), points.ids.data(), points.n, points.d, rho, &g_,
                                  err, sizeof err);
    }
    throw_status(rc, err);
    points_.n = points.n;
    points_.d = points.d;
    points_.coords.resize(points.coords.size());
    points_.ids.resize(points.n);
    throw_status(skycell_gpu_grid_points(g_, points_.coords.data(), points_.ids.data(), err, sizeof err), err);
  }
  ~MultiLayerGrid() { skycell_gpu_grid_destroy(g_); }
  MultiLayerGrid(const MultiLayerGrid&) = delete;
  MultiLayerGrid& operator=(const MultiLayerGrid&) = delete;

  int rho() const { return rho_; }
  int dims() const { return points_.d; }
  uint32_t size() const { return points_.n; }
  const PointSet& points() const { return points_; }
  CellIndex cell_of(uint32_t position, int layer) const { return point_to_cell(points_.point(position), layer); }

  bool occupied(const CellIndex& c) const {
    if (c.is_auxiliary()) return true;
    if (!c.in_grid() || c.layer() > rho_) return false;
    for (int k = 0; k < c.dims(); ++k)
      if (c.col(k) > c.top_column()) return false;
    const uint64_t lin = c.linear_index();
    uint8_t occ = 0;
    char err[512] = {0};
    throw_status(skycell_gpu_grid_lookup(g_, c.layer(), &lin, 1, &occ, nullptr, nullptr, err, sizeof err), err);
    return occ != 0;
  }

  CellRange range(const CellIndex& leaf_cell) const {
    if (leaf_cell.layer() != rho_) throw UsageError("range: only layer-rho cells carry point ranges");
    const uint64_t lin = leaf_cell.linear_index();
    uint32_t b = 0, e = 0;
    char err[512] = {0};
    throw_status(skycell_gpu_grid_lookup(g_, rho_, &lin, 1, nullptr, &b, &e, err, sizeof err), err);
    return CellRange{b, e};
  }

  std::vector<CellIndex> nonempty_cells(int layer) const {
    std::vector<uint64_t> lin(skycell_gpu_grid_nonempty_count(g_, layer));
    char err[512] = {0};
    if (!lin.empty()) throw_status(skycell_gpu_grid_nonempty_cells(g_, layer, lin.data(), err, sizeof err), err);
    std::vector<CellIndex> out;
    out.reserve(lin.size());
    for (uint64_t x : lin) out.push_back(CellIndex::from_linear_index(x, layer, points_.d));
    return out;
  }

  uint64_t nonempty_count(int layer) const { return skycell_gpu_grid_nonempty_count(g_, layer); }
  CellIndex origin_cell() const { return CellIndex(0, points_.d); }
  static int default_rho(uint64_t n, int d) { return skycell_default_rho(n, d); }

 private:
  skycell_gpu_grid* g_ = nullptr;
  PointSet points_;
  int rho_;
};

}  // namespace skycell::gpu
