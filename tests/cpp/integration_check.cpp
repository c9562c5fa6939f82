// Integration check of include/skycell_gpu.hpp against the reference itself.
//
// TEST INFRASTRUCTURE.  Compiled (oracle/Makefile, target `integration`)
// against the reference's own headers and linked with BOTH the unmodified
// reference library (oracle/_ref/libskycell_ref.so) and the product
// (paper_2107_09993_b200/lib/libskycell_gpu.so) -- exactly what a reference
// maintainer would do.  On a GPU it runs the same inputs
// through skycell::compute_skyline (refine.cpp:108-158) and
// skycell::gpu::compute_skyline and requires identical results; exceptions
// must have the same type and message.  Exit code 0 = all equal.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "skycell/datagen.hpp"
#include "skycell/error.hpp"
#include "skycell/refine.hpp"
#include "skycell_gpu.hpp"

namespace {

int failures = 0;

void expect(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
  if (!ok) ++failures;
}

bool same(const skycell::SkylineResult& a, const skycell::SkylineResult& b) {
  return a.ids == b.ids && a.points_examined == b.points_examined && a.layers.keys == b.layers.keys &&
         a.layers.candidates == b.layers.candidates;
}

skycell::Dataset quantised(skycell::Distribution dist, uint32_t n, int d, uint64_t seed) {
  skycell::GenSpec spec;
  spec.distribution = dist;
  spec.n = n;
  spec.d = d;
  spec.seed = seed;
  skycell::Dataset ds = skycell::generate(spec);
  for (double& v : ds.coords) v = (double)(float)(std::floor(v * 16777216.0) / 16777216.0);
  ds.dim_min.assign(d, 0.0);
  ds.dim_max.assign(d, 1.0);
  return ds;
}

// skycell::gpu::MultiLayerGrid against skycell::MultiLayerGrid on the same
// normalised PointSet (grid.cpp:35-140).
bool same_grid(const skycell::PointSet& ps, int rho) {
  skycell::MultiLayerGrid want(ps, rho);
  skycell::gpu::MultiLayerGrid got(ps, rho);
  if (want.points().ids != got.points().ids || want.points().coords != got.points().coords) return false;
  if (want.rho() != got.rho() || want.dims() != got.dims() || want.size() != got.size()) return false;
  for (int L = 0; L <= rho; ++L) {
    if (want.nonempty_count(L) != got.nonempty_count(L)) return false;
    const auto a = want.nonempty_cells(L), b = got.nonempty_cells(L);
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i) {
      if (a[i].linear_index() != b[i].linear_index()) return false;
      if (!got.occupied(a[i])) return false;
      if (L == rho) {
        const auto ra = want.range(a[i]), rb = got.range(b[i]);
        if (ra.begin != rb.begin || ra.end != rb.end) return false;
      }
    }
    // auxiliary cells are always occupied; a cell past the top is not
    if (!got.occupied(skycell::CellIndex::auxiliary(L, ps.d, 0))) return false;
  }
  for (uint32_t pos = 0; pos < ps.n; pos += 97)
    if (!(want.cell_of(pos, rho) == got.cell_of(pos, rho))) return false;
  return true;
}

template <typename F>
std::string what_of(F&& f, int* kind) {
  try {
    f();
  } catch (const skycell::InputError& e) {
    *kind = 1;
    return e.what();
  } catch (const skycell::ConfigError& e) {
    *kind = 2;
    return e.what();
  } catch (const skycell::UsageError& e) {
    *kind = 3;
    return e.what();
  }
  *kind = 0;
  return "";
}

}  // namespace

int main() {
  skycell::ThreadPool pool(0);
  // three contexts on device 0: the multi-device handle's sharded protocol
  skycell::gpu::MultiDevice multi({0, 0, 0});
  const skycell::Distribution dists[] = {skycell::Distribution::kIndependent, skycell::Distribution::kCorrelated,
                                         skycell::Distribution::kAnticorrelated};
  int di = 0;
  for (auto dist : dists) {
    for (int d = 2; d <= 5; ++d) {
      const uint32_t n = 20000 + 3000 * d;
      skycell::Dataset ds = quantised(dist, n, d, 40 + d);
      const int rho = skycell::MultiLayerGrid::default_rho(n, d);
      for (auto mode : {skycell::Mode::kSequential, skycell::Mode::kParallel}) {
        auto want = skycell::compute_skyline(ds, rho, mode, pool);
        auto got = skycell::gpu::compute_skyline(ds, rho, mode, pool);
        expect(same(want, got), "compute_skyline dist=" + std::to_string(di) + " d=" + std::to_string(d) +
                                    " mode=" + std::to_string((int)mode) + " |S|=" + std::to_string(want.ids.size()));
        auto gm = multi.compute_skyline(ds, rho, mode);
        expect(same(want, gm), "MultiDevice compute_skyline dist=" + std::to_string(di) + " d=" + std::to_string(d));
      }
      // general FP64 path: raw generator output, observed min/max
      skycell::GenSpec spec;
      spec.distribution = dist;
      spec.n = n / 4;
      spec.d = d;
      spec.seed = 7;
      skycell::Dataset raw = skycell::generate(spec);
      for (double& v : raw.coords) v = v * 5.0 - 2.0;
      raw.compute_minmax();
      auto w2 = skycell::compute_skyline(raw, 3, skycell::Mode::kParallel, pool);
      auto g2 = skycell::gpu::compute_skyline(raw, 3, skycell::Mode::kParallel, pool);
      expect(same(w2, g2), "compute_skyline f64 dist=" + std::to_string(di) + " d=" + std::to_string(d));
      auto w3 = skycell::compute_skyline(raw, 2, skycell::Mode::kParallel, pool, false);
      auto g3 = skycell::gpu::compute_skyline(raw, 2, skycell::Mode::kParallel, pool, false);
      expect(same(w3, g3), "compute_skyline merge_cross_cell=false d=" + std::to_string(d));
      {
        const skycell::PointSet ps = skycell::normalize(raw);
        expect(same_grid(ps, std::min(3, skycell::MultiLayerGrid::default_rho(ps.n, d) + 1)),
               "MultiLayerGrid d=" + std::to_string(d));
      }
      std::vector<double> origin(d, 0.2);
      auto wq = skycell::quadrant_skyline(raw, origin, 4, skycell::Mode::kParallel, pool);
      auto gq = skycell::gpu::quadrant_skyline(raw, origin, 4, skycell::Mode::kParallel, pool);
      expect(same(wq, gq), "quadrant_skyline d=" + std::to_string(d));
    }
    ++di;
  }
  // error taxonomy and message text
  skycell::Dataset bad = quantised(skycell::Distribution::kIndependent, 100, 3, 1);
  bad.coords[3 * 57 + 2] = std::nan("");
  int k1 = 0, k2 = 0;
  const std::string m1 = what_of([&] { skycell::compute_skyline(bad, 2, skycell::Mode::kParallel, pool); }, &k1);
  const std::string m2 = what_of([&] { skycell::gpu::compute_skyline(bad, 2, skycell::Mode::kParallel, pool); }, &k2);
  expect(k1 == 1 && k1 == k2 && m1 == m2, "InputError: " + m2);
  skycell::Dataset ok = quantised(skycell::Distribution::kIndependent, 100, 4, 1);
  const std::string m3 = what_of([&] { skycell::compute_skyline(ok, 16, skycell::Mode::kParallel, pool); }, &k1);
  const std::string m4 = what_of([&] { skycell::gpu::compute_skyline(ok, 16, skycell::Mode::kParallel, pool); }, &k2);
  expect(k1 == 2 && k1 == k2 && m3 == m4, "ConfigError: " + m4);
  std::vector<double> o2(2, 0.0);
  const std::string m5 = what_of([&] { skycell::quadrant_skyline(ok, o2, 3, skycell::Mode::kParallel, pool); }, &k1);
  const std::string m6 = what_of([&] { skycell::gpu::quadrant_skyline(ok, o2, 3, skycell::Mode::kParallel, pool); }, &k2);
  expect(k1 == 3 && k1 == k2 && m5 == m6, "UsageError: " + m6);
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL EQUAL", failures);
  return failures ? 1 : 0;
}
