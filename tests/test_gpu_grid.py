"""MultiLayerGrid drop-in (csrc/grid.cu) against the
unmodified reference's MultiLayerGrid (grid.cpp:35-140) on the same
normalised PointSet: the sorted point order (Z-order of the layer-rho cell,
ties by position), the range of every non-empty leaf cell, the non-empty
cells and counts of every layer, occupancy lookups, and the constructor's
ConfigError messages."""
import numpy as np
import pytest

import paper_2107_09993_b200 as sky

pytestmark = pytest.mark.gpu

CASES = [(0, 20000, 2, 6), (0, 30000, 3, 5), (1, 40000, 4, 4), (2, 25000, 4, 6), (2, 8000, 6, 3), (0, 5000, 8, 2),
         (2, 3000, 8, 5), (1, 1, 3, 2), (0, 200_000, 4, 6)]


@pytest.mark.parametrize("dist,n,d,rho", CASES, ids=lambda v: str(v))
def test_gpu_grid_matches_reference(engine, reference, oracle, dist, n, d, rho):
    v = oracle.generate(dist, n, d, 60 + d)
    x = v * 4.0 - 1.0
    pts = oracle.normalize(x, x.min(0), x.max(0))  # the PointSet compute_skyline builds (dataset.cpp:22-50)
    g = engine.grid(pts, rho)
    assert (g.rho(), g.dims(), g.size()) == (rho, d, n)
    for layer in range(rho + 1):
        ref = reference.grid(pts, rho, layer)
        if layer == 0:
            coords, ids = g.points()
            assert np.array_equal(ids, ref["ids"])
            assert np.array_equal(coords.view(np.uint64), pts[ref["ids"]].view(np.uint64))
            assert [g.nonempty_count(L) for L in range(rho + 1)] == ref["counts"]
            b, e = g.range(ref["leaf_lin"])
            assert np.array_equal(b, ref["leaf_begin"]) and np.array_equal(e, ref["leaf_end"])
            assert np.array_equal(g.nonempty_cells(rho), ref["leaf_lin"])
        cells = g.nonempty_cells(layer)
        assert np.array_equal(cells, ref["layer_lin"]), layer
        # occupancy of random in-grid cells (and every non-empty one)
        total = 1 << (layer * d)
        rng = np.random.default_rng(layer + 7 * d)
        q = np.unique(np.concatenate([rng.integers(0, total, size=min(total, 4000), dtype=np.uint64), cells]))
        want = np.isin(q, cells)
        assert np.array_equal(g.occupied(layer, q), want)
        if layer == rho:
            b, e = g.range(q[~want])
            assert not b.any() and not e.any()  # empty cells: begin == end == 0
    g.close()


def test_gpu_grid_config_errors(engine, reference, oracle):
    """The constructor's rho budget (grid.cpp:38-43): same type, same text."""
    from oracle.oracle import CpuError
    pts = oracle.normalize(oracle.generate(0, 100, 8, 1), np.zeros(8), np.ones(8))
    for rho in (0, 8, 6):
        with pytest.raises(CpuError) as r:
            reference.grid(pts, rho, 0)
        with pytest.raises(sky.ConfigError) as e:
            engine.grid(pts, rho)
        assert r.value.code == 2 and str(e.value) == str(r.value)
