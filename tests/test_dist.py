"""Host side of the sharded query (paper_2107_09993_b200/dist.py) at
world_size 2 and 3 over gloo on CPU.

The device phases are replaced by a CPU stand-in with the same phase API
(test infrastructure, brute force, small n): it exercises everything the
orchestrator owns -- shard ranges, the occupancy all-gather + OR, count
exchange, padding, rank-order concatenation, global ids, the error
handshake -- and the result is compared with the oracle over the whole
dataset.  The device phases themselves are covered on one GPU by
tests/test_gpu_shard.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_09993_b200.dist import ShardedSkyline, shard_range
from paper_2107_09993_b200.skycell import InputError, SkylineResult


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class CpuShardEngine:
    """Stand-in for Engine's shard_* phases (reference semantics, brute force)."""

    def shard_begin(self, coords, n, d, dim_min, dim_max, rho, mode, id_base):
        x = np.asarray(coords, dtype=np.float64).reshape(n, d)
        if not np.isfinite(x).all():
            bad = int(np.nonzero(~np.isfinite(x).all(axis=1))[0][0])
            raise InputError(f"normalize: non-finite coordinate in record {id_base + bad}")
        rng = np.asarray(dim_max, float) - np.asarray(dim_min, float)
        scale = np.where(rng > 0, 1.0 / np.where(rng > 0, rng, 1.0), 0.0)
        self.u = np.clip((x - dim_min) * scale, 0.0, 1.0 - 2.0**-32)
        self.ids = np.arange(id_base, id_base + n, dtype=np.uint32)
        self.d, self.rho = d, rho
        cols = np.minimum((self.u * (1 << rho)).astype(np.int64), (1 << rho) - 1)
        self.cols = cols
        lin = np.zeros(n, dtype=np.int64)
        for k in range(d - 1, -1, -1):
            lin = (lin << rho) | cols[:, k]
        occ = np.zeros(1 << (rho * d), dtype=bool)
        occ[lin] = True
        self.occ = np.packbits(occ)
        return int(self.occ.size)

    def shard_export_occ(self, dst):
        dst.copy_(torch.from_numpy(self.occ))

    def _sums(self, u):
        s = np.zeros(len(u))
        for k in range(u.shape[1]):
            s = s + u[:, k]
        return s

    @staticmethod
    def _dominated(qu, qs, qid, pu, ps, pid):
        prec = (qs < ps) | ((qs == ps) & (qid < pid))
        dom = (qu <= pu).all(axis=1) & (qu < pu).any(axis=1)
        return bool((prec & dom).any())

    def shard_prune(self, gathered, world):
        g = gathered.numpy().reshape(world, -1)
        occ = np.unpackbits(np.bitwise_or.reduce(g, axis=0))[: 1 << (self.rho * self.d)].astype(bool)
        cells = np.array(np.nonzero(occ)[0])
        ccols = np.stack([(cells >> (self.rho * k)) & ((1 << self.rho) - 1) for k in range(self.d)], axis=1)
        # candidate cell: not strictly dominated by an occupied cell (Def. 5)
        cand = {}
        for i, c in enumerate(cells):
            cand[int(c)] = not (ccols < ccols[i]).all(axis=1).any()
        lin = np.zeros(len(self.u), dtype=np.int64)
        for k in range(self.d - 1, -1, -1):
            lin = (lin << self.rho) | self.cols[:, k]
        keep = np.array([cand[int(c)] for c in lin], dtype=bool)
        self.examined = int(keep.sum())
        u, ids = self.u[keep], self.ids[keep]
        s = self._sums(u)
        sky = [i for i in range(len(u)) if not self._dominated(u, s, ids, u[i], s[i], ids[i])]
        self.sky_u, self.sky_s, self.sky_ids = u[sky], s[sky], ids[sky]
        return len(sky)

    def shard_block_bytes(self, maxc):
        return maxc * (self.d * 8 + 8 + 4)

    def shard_pack(self, dst, maxc):
        c = len(self.sky_ids)
        rows = np.zeros((maxc, self.d))
        rows[:c] = self.sky_u
        sums = np.zeros(maxc)
        sums[:c] = self.sky_s
        ids = np.full(maxc, 0xFFFFFFFF, dtype=np.uint32)
        ids[:c] = self.sky_ids
        blob = np.concatenate([rows.view(np.uint8).ravel(), sums.view(np.uint8), ids.view(np.uint8)])
        dst.copy_(torch.from_numpy(blob))

    def shard_finish(self, recv, world, maxc, rank, own_count, ids_out):
        r = recv.numpy().reshape(world, -1)
        rb, sb = maxc * self.d * 8, maxc * 8
        U = np.concatenate([r[g, :rb].view(np.float64).reshape(maxc, self.d) for g in range(world)])
        S = np.concatenate([r[g, rb:rb + sb].view(np.float64) for g in range(world)])
        I = np.concatenate([r[g, rb + sb:].view(np.uint32) for g in range(world)])
        live = I != 0xFFFFFFFF
        U, S, I = U[live], S[live], I[live]
        mine = [i for i in range(len(self.sky_ids))
                if not self._dominated(U, S, I, self.sky_u[i], self.sky_s[i], self.sky_ids[i])]
        out = np.sort(self.sky_ids[mine]).astype(np.uint32)
        ids_out[: len(out)] = out
        return SkylineResult(ids=ids_out[: len(out)], points_examined=self.examined)


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle, quantize_f32
        orc = Oracle()
        for dist_id, n, d, rho, bad in cases:
            x = quantize_f32(orc.generate(dist_id, n, d, 7 + n)).astype(np.float64)
            if bad is not None:
                x[bad, 1] = np.nan
            b, e = shard_range(n, rank, world)
            runner = ShardedSkyline(CpuShardEngine(), device="cpu")
            try:
                res = runner.skyline(x[b:e], e - b, d, np.zeros(d), np.ones(d), rho, b)
            except InputError as err:
                q.put((rank, "input-error", str(err)))
                continue
            if rank == 0:
                want = orc.compute_skyline(x, np.zeros(d), np.ones(d), rho)
                q.put((rank, "ok", bool(np.array_equal(res.ids, want.ids)), res.points_examined,
                       want.points_examined, len(want.ids)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_matches_oracle(world):
    cases = [(0, 1500, 3, 3, None), (1, 1200, 2, 4, None), (2, 900, 4, 2, None), (2, 1001, 3, 2, None),
             (0, 7, 2, 1, None)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), cases, q), nprocs=world, start_method="spawn")
    got = [q.get(timeout=60) for _ in cases]
    for (_, status, equal, ex, want_ex, size), case in zip(got, cases):
        assert status == "ok"
        assert equal, case
        assert ex == want_ex, case


def test_sharded_error_reaches_every_rank():
    world = 2
    cases = [(0, 400, 3, 2, 350)]  # NaN in a record owned by rank 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), cases, q), nprocs=world, start_method="spawn")
    got = sorted(q.get(timeout=60) for _ in range(world))
    assert [g[1] for g in got] == ["input-error", "input-error"]
    assert got[1][2] == "normalize: non-finite coordinate in record 350"


def test_shard_range_partition():
    for n in (1, 7, 100, 10**9 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
