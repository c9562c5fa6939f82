"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the CPU oracle on the same inputs.  Bit-exact ids,
points_examined and per-layer |KS_i| / |CS_i|."""
import numpy as np
import pytest

import paper_2107_09993_b200 as sky
from golden_io import inputs_for, load_ids, load_json

pytestmark = pytest.mark.gpu
MODES = {0: "seq", 1: "par"}


def check(res, ids=None, examined=None, keys=None, cands=None):
    if ids is not None:
        assert np.array_equal(np.asarray(res.ids), np.asarray(ids, dtype=np.uint32)), (len(res.ids), len(ids))
    if examined is not None:
        assert res.points_examined == examined
    if keys is not None:
        assert res.layers.keys == list(keys)
    if cands is not None:
        assert res.layers.candidates == list(cands)


@pytest.mark.parametrize("case", load_json("kat.json")["cases"], ids=lambda c: c["name"])
def test_gpu_kats(engine, case):
    x = np.asarray(case["rows"], dtype=np.float64)
    ds = sky.Dataset(x, np.asarray(case["dim_min"], float), np.asarray(case["dim_max"], float))
    for mode, key in MODES.items():
        w = case[key]
        check(engine.compute_skyline(ds, case["rho"], sky.Mode(mode), merge_cross_cell=case["merge"]), w["ids"],
              w["points_examined"], w["keys"], w["candidates"])


@pytest.mark.parametrize("case", load_json("kat.json")["errors"], ids=lambda c: c["name"])
def test_gpu_errors(engine, case):
    x = np.asarray(case["rows"], dtype=np.float64)
    ds = sky.Dataset(x, np.asarray(case["dim_min"], float), np.asarray(case["dim_max"], float))
    exc = {1: sky.InputError, 2: sky.ConfigError, 3: sky.UsageError}[case["code"]]
    with pytest.raises(exc) as ei:
        engine.compute_skyline(ds, case["rho"])
    assert str(ei.value) == case["message"]


def test_gpu_random_small_golden(engine, oracle):
    ids = load_ids("random_small_ids.npz")
    for rec in load_json("random_small.json")["records"]:
        x, mn, mx = inputs_for(oracle, rec)
        r = engine.compute_skyline(sky.Dataset(x, mn, mx), rec["rho"], sky.Mode(rec["mode"]))
        check(r, ids[rec["key"]], rec["points_examined"], rec["keys"], rec["candidates"])


@pytest.mark.parametrize("rec", load_json("c1.json")["records"], ids=lambda r: r["key"])
def test_gpu_c1_golden(engine, oracle, rec):
    x, mn, mx = inputs_for(oracle, rec)
    r = engine.compute_skyline(sky.Dataset(x, mn, mx), rec["rho"])
    check(r, load_ids("c1_ids.npz")[rec["key"]], rec["points_examined"], rec["keys"], rec["candidates"])


@pytest.mark.parametrize("seed", range(30))
def test_gpu_vs_oracle_random(engine, oracle, seed):
    from oracle.oracle import quantize_f32
    rng = np.random.default_rng(seed)
    dist = seed % 3
    d = int(rng.integers(2, 9))
    n = int(rng.integers(1, 6000)) if seed % 5 else int(rng.integers(1, 40))
    rho_max = max(r for r in range(1, 9) if r * d <= 36 and (r - 1) * d <= 32 and r * (d - 1) <= 30)
    rho = int(rng.integers(1, min(rho_max, 7) + 1))
    v = oracle.generate(dist, n, d, 1000 + seed)
    cases = [(quantize_f32(v), np.zeros(d), np.ones(d)),
             (v * 7.0 - 3.0, (v * 7.0 - 3.0).min(0), (v * 7.0 - 3.0).max(0)),
             (quantize_f32(v) * np.float32(3) - np.float32(1), np.full(d, -0.5), np.full(d, 1.5))]
    for x, mn, mx in cases:
        want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho, 1)
        got = engine.compute_skyline(sky.Dataset(np.ascontiguousarray(x), mn, mx), rho)
        check(got, want.ids, want.points_examined, want.keys, want.candidates)


def test_gpu_device_tensor_input(engine, oracle):
    import torch
    from oracle.oracle import quantize_f32
    x = quantize_f32(oracle.generate(0, 50000, 4, 3))
    t = torch.from_numpy(x).cuda()
    out = torch.empty(50000, dtype=torch.int32, device="cuda")
    r = engine.skyline_raw(t, 50000, 4, np.zeros(4), np.ones(4), 4, ids_out=out)
    want = oracle.compute_skyline(x.astype(np.float64), np.zeros(4), np.ones(4), 4)
    assert np.array_equal(r.ids.cpu().numpy().astype(np.uint32), want.ids)


def test_gpu_generator_matches_host(engine, oracle):
    from oracle.oracle import quantize_f32
    for dist in range(3):
        g = engine.generate(dist, 200_000, 4, 42, quantized=True).cpu().numpy()
        h = quantize_f32(oracle.generate(dist, 200_000, 4, 42))
        mism = int((g != h).sum())
        if dist == 0:
            assert mism == 0
        else:
            assert mism <= 4, mism  # CUDA log/cos vs glibc: ulp-level, see datagen.cuh
        r = engine.generate(dist, 70_000, 3, 7, quantized=False).cpu().numpy()
        hr = oracle.generate(dist, 70_000, 3, 7)
        if dist == 0:
            assert np.array_equal(r, hr)
        else:
            assert np.abs(r - hr).max() < 1e-12


def test_gpu_repeat_deterministic(engine, oracle):
    from oracle.oracle import quantize_f32
    x = quantize_f32(oracle.generate(2, 100_000, 5, 11))
    ds = sky.Dataset(x, np.zeros(5), np.ones(5))
    a = engine.compute_skyline(ds, 3)
    for _ in range(3):
        b = engine.compute_skyline(ds, 3)
        assert np.array_equal(a.ids, b.ids) and a.points_examined == b.points_examined


@pytest.mark.parametrize("rec", load_json("large.json")["records"], ids=lambda r: r["key"])
def test_gpu_large_skyline_golden(engine, oracle, rec):
    """Large-S anchors: anti-correlated d=6/8 where 59-99% of points are
    skyline points (the reference needs 40-290 s for these)."""
    x, mn, mx = inputs_for(oracle, rec)
    r = engine.compute_skyline(sky.Dataset(x, mn, mx), rec["rho"])
    check(r, load_ids("large_ids.npz")[rec["key"]], rec["points_examined"], rec["keys"], rec["candidates"])


@pytest.mark.parametrize("seed", range(8))
def test_gpu_phase1_only_vs_oracle(engine, oracle, seed):
    """merge_cross_cell = false (refine.hpp:50-56): union of per-cell SFS."""
    from oracle.oracle import quantize_f32
    rng = np.random.default_rng(100 + seed)
    dist, d = seed % 3, int(rng.integers(2, 6))
    n = int(rng.integers(50, 4000))
    rho = int(rng.integers(1, 4))
    v = oracle.generate(dist, n, d, 300 + seed)
    for x, mn, mx in ((quantize_f32(v), np.zeros(d), np.ones(d)), (v * 2 - 1, (v * 2 - 1).min(0), (v * 2 - 1).max(0))):
        want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho, 1, False)
        got = engine.compute_skyline(sky.Dataset(np.ascontiguousarray(x), mn, mx), rho, merge_cross_cell=False)
        check(got, want.ids, want.points_examined, want.keys, want.candidates)


@pytest.mark.parametrize("seed", range(6))
def test_gpu_quadrant_vs_oracle(engine, oracle, seed):
    """quadrant_skyline (refine.cpp:160-184): filter, renormalise, sub_rho."""
    rng = np.random.default_rng(seed)
    d = 2 + seed % 4
    v = oracle.generate(seed % 3, 3000 + 500 * seed, d, 40 + seed)
    for _ in range(4):
        origin = rng.uniform(-0.1, 0.7, d)
        want = oracle.quadrant_skyline(v, origin, 4)
        got = engine.quadrant_skyline(sky.Dataset(v, v.min(0), v.max(0)), origin, 4)
        check(got, want.ids, want.points_examined, want.keys, want.candidates)


def test_gpu_quadrant_edges(engine, oracle):
    v = oracle.generate(0, 500, 3, 1)
    ds = sky.Dataset(v, v.min(0), v.max(0))
    # empty quadrant -> empty result, no layers (refine.cpp:176)
    r = engine.quadrant_skyline(ds, np.full(3, 2.0), 3)
    assert r.ids.size == 0 and r.layers.keys == []
    # arity mismatch -> UsageError with the reference's message (refine.cpp:162-163)
    with pytest.raises(sky.UsageError, match="origin arity does not match"):
        engine.quadrant_skyline(ds, np.zeros(2), 3)
    # NaN records are outside every quadrant (the >= test is false)
    w = v.copy()
    w[7, 1] = np.nan
    want = oracle.quadrant_skyline(w, np.zeros(3), 3)
    got = engine.quadrant_skyline(sky.Dataset(w, np.zeros(3), np.ones(3)), np.zeros(3), 3)
    check(got, want.ids, want.points_examined)
    # a single record inside
    o = v[np.argmax(v.sum(1))]
    want = oracle.quadrant_skyline(v, o, 3)
    got = engine.quadrant_skyline(ds, o, 3)
    check(got, want.ids, want.points_examined)


@pytest.fixture(scope="module", params=["tree", "tree-point", "lists"])
def forced_engine(request):
    """An engine pinned to one K5 variant (SKYCELL_K5 is read once per context)."""
    import os
    old = os.environ.get("SKYCELL_K5")
    os.environ["SKYCELL_K5"] = request.param
    e = sky.Engine(0)
    e.compute_skyline(sky.Dataset(np.zeros((1, 2)), np.zeros(2), np.ones(2)), 1)  # latch the mode
    if old is None:
        del os.environ["SKYCELL_K5"]
    else:
        os.environ["SKYCELL_K5"] = old
    yield e
    e.close()


@pytest.mark.parametrize("seed", range(12))
def test_gpu_k5_variants_vs_oracle(forced_engine, oracle, seed):
    """Every K5 variant (column lists, dominance tree with the packet or the
    point query) on every path:
    identity f32, general f64, merge_cross_cell = false."""
    from oracle.oracle import quantize_f32
    rng = np.random.default_rng(500 + seed)
    dist, d = seed % 3, int(rng.integers(2, 9))
    n = int(rng.integers(1, 8000))
    rho = int(rng.integers(1, 4))
    v = oracle.generate(dist, n, d, 900 + seed)
    for x, mn, mx in ((quantize_f32(v), np.zeros(d), np.ones(d)), (v * 4 - 1, (v * 4 - 1).min(0), (v * 4 - 1).max(0))):
        for merge in (True, False):
            want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho, 1, merge)
            got = forced_engine.compute_skyline(sky.Dataset(np.ascontiguousarray(x), mn, mx), rho,
                                                merge_cross_cell=merge)
            check(got, want.ids, want.points_examined, want.keys, want.candidates)


@pytest.mark.parametrize("rec", load_json("large.json")["records"], ids=lambda r: r["key"])
def test_gpu_k5_variants_large_golden(forced_engine, oracle, rec):
    x, mn, mx = inputs_for(oracle, rec)
    r = forced_engine.compute_skyline(sky.Dataset(x, mn, mx), rec["rho"])
    check(r, load_ids("large_ids.npz")[rec["key"]], rec["points_examined"], rec["keys"], rec["candidates"])


@pytest.mark.parametrize("d,rho", [(2, 8), (2, 11), (2, 14), (3, 8), (3, 10), (4, 8), (5, 7), (6, 5)])
def test_gpu_fine_grids_vs_oracle(engine, oracle, d, rho):
    """Layers above 7 (u32 prefix-min tables) and the largest grids of the
    reference's budget that the dense bitmaps cover (grid.cpp:38-43)."""
    from oracle.oracle import quantize_f32
    for dist in range(3):
        v = oracle.generate(dist, 3000, d, 70 + rho)
        for x, mn, mx in ((quantize_f32(v), np.zeros(d), np.ones(d)), (v * 3 - 1, (v * 3 - 1).min(0), (v * 3 - 1).max(0))):
            want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho)
            got = engine.compute_skyline(sky.Dataset(np.ascontiguousarray(x), mn, mx), rho)
            check(got, want.ids, want.points_examined, want.keys, want.candidates)


@pytest.mark.parametrize("dist", [0, 1])
def test_gpu_f64_general_path_large(engine, oracle, dist):
    """The general FP64 path (device-side normalisation with the host's
    scale, dataset.cpp:32-45) at a size where every kernel runs at scale."""
    v = oracle.generate(dist, 3_000_000, 4, 21)
    x = v * 10.0 - 3.0
    mn, mx = x.min(0), x.max(0)
    want = oracle.compute_skyline(x, mn, mx, 5)
    got = engine.compute_skyline(sky.Dataset(x, mn, mx), 5)
    check(got, want.ids, want.points_examined, want.keys, want.candidates)


@pytest.mark.parametrize("d", [9, 11, 13, 16])
def test_gpu_high_dimensions(engine, oracle, d):
    """d up to the reference's kMaxDims = 16 (cell.hpp:15), both K5 variants'
    dispatch sizes, identity and general paths."""
    from oracle.oracle import quantize_f32
    for dist, n in ((0, 3000), (2, 1500)):
        v = oracle.generate(dist, n, d, 13 + d)
        rho_max = max(r for r in range(1, 8) if r * d <= 60 and (r - 1) * d <= 32)  # grid.cpp:38-43
        for rho in sorted({1, rho_max}):
            for x, mn, mx in ((quantize_f32(v), np.zeros(d), np.ones(d)), (v * 2 - 1, (v * 2 - 1).min(0), (v * 2 - 1).max(0))):
                want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho)
                got = engine.compute_skyline(sky.Dataset(np.ascontiguousarray(x), mn, mx), rho)
                check(got, want.ids, want.points_examined, want.keys, want.candidates)


# every (d, rho) of the reference's budget (rho*d <= 60, (rho-1)*d <= 32,
# grid.cpp:38-43) whose layer rho exceeds the dense bitmaps (sparse.cuh)
SPARSE = [(8, 5), (9, 4), (10, 4), (11, 3), (12, 3), (13, 3), (14, 3), (15, 3), (16, 3)]


@pytest.mark.parametrize("d,rho", SPARSE)
def test_gpu_sparse_layer_vs_oracle(engine, oracle, d, rho):
    """Layer rho as sorted unique cells classified through the dominance tree
    (sparse.cuh) instead of a 2^(rho d)-bit bitmap: ids, points_examined and
    |KS_i|, |CS_i| of every layer, both merge modes, identity and general
    normalisation."""
    from oracle.oracle import quantize_f32
    for dist in range(3):
        v = oracle.generate(dist, 3000, d, 90 + d)
        for x, mn, mx in ((quantize_f32(v), np.zeros(d), np.ones(d)), (v * 3 - 1, (v * 3 - 1).min(0), (v * 3 - 1).max(0))):
            for merge in (True, False):
                want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho, 1, merge)
                got = engine.compute_skyline(sky.Dataset(np.ascontiguousarray(x), mn, mx), rho, merge_cross_cell=merge)
                check(got, want.ids, want.points_examined, want.keys, want.candidates)


@pytest.mark.parametrize("dist,n", [(0, 400_000), (1, 400_000), (2, 25_000)])
def test_gpu_sparse_layer_large(engine, oracle, dist, n):
    """d = 8, rho = 5 at sizes where the cell tree is large (>64K cells:
    multi-level tree, two-phase packet query)."""
    from oracle.oracle import quantize_f32
    d, rho = 8, 5
    x = quantize_f32(oracle.generate(dist, n, d, 5))
    want = oracle.compute_skyline(x.astype(np.float64), np.zeros(d), np.ones(d), rho)
    got = engine.compute_skyline(sky.Dataset(x, np.zeros(d), np.ones(d)), rho)
    check(got, want.ids, want.points_examined, want.keys, want.candidates)


@pytest.mark.parametrize("d,rho", [(3, 1), (4, 2)])
def test_gpu_phase1_only_large_tree(forced_engine, oracle, d, rho):
    """merge_cross_cell = false with more than 64K points in the K5 set (the
    size at which the tree's champion prefilter would run): dominators must
    stay inside p's layer-rho cell, so the prefilter must not run."""
    from oracle.oracle import quantize_f32
    v = oracle.generate(2, 150_000, d, 77)
    x = quantize_f32(v)
    want = oracle.compute_skyline(x.astype(np.float64), np.zeros(d), np.ones(d), rho, 1, False)
    got = forced_engine.compute_skyline(sky.Dataset(x, np.zeros(d), np.ones(d)), rho, merge_cross_cell=False)
    check(got, want.ids, want.points_examined, want.keys, want.candidates)
