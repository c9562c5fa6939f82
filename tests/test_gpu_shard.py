"""Device phases of the sharded query on one B200: G shards,
each with its own context, exchanging through an in-process loopback (the
same byte buffers the NCCL all-gathers carry), must reproduce the
single-device query and the oracle bit-exactly -- ids, points_examined and
per-layer key/candidate counts.  Plus the real NCCL path at world_size 1."""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2107_09993_b200 as sky
from paper_2107_09993_b200.dist import ShardedSkyline, shard_range

pytestmark = pytest.mark.gpu


def loopback_query(engines, x, d, mn, mx, rho, mode=1):
    G = len(engines)
    n = x.shape[0]
    stream = torch.cuda.current_stream()
    spans = [shard_range(n, g, G) for g in range(G)]
    occ = []
    for eng, (b, e) in zip(engines, spans):
        eng.set_stream(stream)
        nb = eng.shard_begin(x[b:e], e - b, d, mn, mx, rho, mode, b)
        t = torch.empty(nb, dtype=torch.uint8, device="cuda")
        eng.shard_export_occ(t)
        occ.append(t)
    gathered = torch.cat(occ)
    counts = [eng.shard_prune(gathered, G) for eng in engines]
    maxc = max(counts)
    blocks = []
    for eng in engines:
        t = torch.empty(eng.shard_block_bytes(maxc), dtype=torch.uint8, device="cuda")
        eng.shard_pack(t, maxc)
        blocks.append(t)
    recv = torch.cat(blocks)
    ids, examined, res0 = [], 0, None
    for g, (eng, (b, e)) in enumerate(zip(engines, spans)):
        out = np.empty(max(e - b, 1), dtype=np.uint32)
        r = eng.shard_finish(recv, G, maxc, g, counts[g], out)
        ids.append(np.asarray(r.ids).copy())
        examined += r.points_examined
        if res0 is None:
            res0 = r
        else:
            assert r.layers.keys == res0.layers.keys and r.layers.candidates == res0.layers.candidates
    return np.concatenate(ids), examined, res0


@pytest.fixture(scope="module")
def engines():
    es = [sky.Engine(0) for _ in range(4)]
    yield es
    for e in es:
        e.close()


CASES = [(0, 200_000, 4, None), (1, 150_000, 4, None), (2, 60_000, 3, None), (2, 20_000, 6, 3), (0, 5_000, 2, None),
         (1, 30_000, 8, 2), (0, 3, 3, 1)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"dist{c[0]}-n{c[1]}-d{c[2]}")
@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_loopback_shards_match_single(engines, oracle, case, G):
    from oracle.oracle import quantize_f32
    dist_id, n, d, rho = case
    if n < G:
        pytest.skip("every shard must hold at least one record")
    x = quantize_f32(oracle.generate(dist_id, n, d, 99 + n))
    rho = rho or sky.default_rho(n, d)
    mn, mx = np.zeros(d), np.ones(d)
    single = engines[0].compute_skyline(sky.Dataset(x, mn, mx), rho)
    want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho)
    assert np.array_equal(single.ids, want.ids)
    xd = torch.from_numpy(x).cuda()
    ids, examined, r0 = loopback_query(engines[:G], xd, d, mn, mx, rho)
    assert np.array_equal(ids, want.ids), (G, len(ids), len(want.ids))
    assert examined == want.points_examined
    assert r0.layers.keys == want.keys and r0.layers.candidates == want.candidates


def test_loopback_shards_f64_general_range(engines, oracle):
    v = oracle.generate(2, 40_000, 4, 5)
    x = v * 3.0 - 1.0
    mn, mx = x.min(0), x.max(0)
    want = oracle.compute_skyline(x, mn, mx, 4)
    ids, examined, r0 = loopback_query(engines[:3], torch.from_numpy(x).cuda(), 4, mn, mx, 4)
    assert np.array_equal(ids, want.ids)
    assert examined == want.points_examined


def test_nccl_world1(oracle):
    import torch.distributed as dist
    from oracle.oracle import quantize_f32
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        eng = sky.Engine(0)
        x = quantize_f32(oracle.generate(0, 300_000, 4, 3))
        want = oracle.compute_skyline(x.astype(np.float64), np.zeros(4), np.ones(4), 4)
        res = ShardedSkyline(eng).skyline(torch.from_numpy(x).cuda(), 300_000, 4, np.zeros(4), np.ones(4), 4, 0)
        assert np.array_equal(res.ids, want.ids)
        assert res.points_examined == want.points_examined
        eng.close()
    finally:
        dist.destroy_process_group()


def _real_worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle, quantize_f32
        torch.cuda.set_device(0)
        orc = Oracle()
        eng = sky.Engine(0)
        runner = ShardedSkyline(eng, device="cuda:0", coll_device="cpu")
        for dist_id, n, d in cases:
            x = quantize_f32(orc.generate(dist_id, n, d, 11 + n))
            rho = sky.default_rho(n, d)
            b, e = shard_range(n, rank, world)
            res = runner.skyline(x[b:e].copy(), e - b, d, np.zeros(d), np.ones(d), rho, b)
            if rank == 0:
                want = orc.compute_skyline(x.astype(np.float64), np.zeros(d), np.ones(d), rho)
                q.put((bool(np.array_equal(res.ids, want.ids)), res.points_examined == want.points_examined,
                       res.layers.keys == want.keys and res.layers.candidates == want.candidates))
        eng.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_real_engines_multi_process(world):
    """The whole multi-rank protocol with real engines (one process per rank,
    all on cuda:0) -- dist.py's collectives over gloo with staged buffers."""
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cases = [(0, 300_000, 4), (1, 200_000, 4), (2, 50_000, 5)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_real_worker, args=(world, port, cases, q), nprocs=world, start_method="spawn")
    for case in cases:
        ok_ids, ok_ex, ok_layers = q.get(timeout=120)
        assert ok_ids and ok_ex and ok_layers, case


# ---- the single-process multi-device handle (skycell_gpu_multi_*): the
# library runs the sharded protocol itself, exchanges included.
@pytest.fixture(scope="module", params=[(2, "peer"), (3, "peer"), (4, "peer"), (3, "copy")], ids=str)
def multi(request):
    """G contexts on device 0; exchange 1 through the in-place peer-read OR
    (k_or_peers) or the gather-copy path (SKYCELL_MULTI_COPY, read at create)."""
    G, how = request.param
    if how == "copy":
        os.environ["SKYCELL_MULTI_COPY"] = "1"
    try:
        m = sky.MultiEngine([0] * G)
    finally:
        os.environ.pop("SKYCELL_MULTI_COPY", None)
    yield m
    m.close()


@pytest.mark.parametrize("dist,n,d", [(0, 200_000, 4), (1, 150_000, 4), (2, 60_000, 5), (2, 20_000, 3), (0, 7, 2)])
def test_multi_device_handle_matches_single(multi, oracle, dist, n, d):
    from oracle.oracle import quantize_f32
    v = oracle.generate(dist, n, d, 31 + dist)
    rho = sky.default_rho(n, d)
    cases = [(quantize_f32(v), np.zeros(d), np.ones(d)),
             (v * 6.0 - 2.0, (v * 6.0 - 2.0).min(0), (v * 6.0 - 2.0).max(0))]
    for x, mn, mx in cases:
        want = oracle.compute_skyline(x.astype(np.float64), mn, mx, rho)
        got = multi.compute_skyline(sky.Dataset(np.ascontiguousarray(x), mn, mx), rho)
        assert np.array_equal(np.asarray(got.ids), want.ids)
        assert got.points_examined == want.points_examined
        assert got.layers.keys == want.keys and got.layers.candidates == want.candidates


def test_multi_device_handle_routes_and_errors(multi, engine, oracle):
    """Queries sharding cannot serve run on the first device (merge_cross_cell
    = false, a sparse layer rho); a non-finite record in a later shard is
    reported with its global record index, as by the single-device query."""
    from oracle.oracle import quantize_f32
    x = quantize_f32(oracle.generate(2, 4000, 8, 3))
    for rho, merge in ((3, False), (5, True)):
        want = oracle.compute_skyline(x.astype(np.float64), np.zeros(8), np.ones(8), rho, 1, merge)
        got = multi.compute_skyline(sky.Dataset(x, np.zeros(8), np.ones(8)), rho, merge_cross_cell=merge)
        assert np.array_equal(np.asarray(got.ids), want.ids)
        assert got.points_examined == want.points_examined and got.layers.keys == want.keys
    y = oracle.generate(0, 9000, 3, 4)
    y[7777, 1] = np.nan
    with pytest.raises(sky.InputError) as e1:
        engine.compute_skyline(sky.Dataset(y, np.zeros(3), np.ones(3)), 3)
    with pytest.raises(sky.InputError) as e2:
        multi.compute_skyline(sky.Dataset(y, np.zeros(3), np.ones(3)), 3)
    assert str(e1.value) == str(e2.value) and "7777" in str(e2.value)
