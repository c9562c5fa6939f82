"""Sharded skyline query over G devices: one process per GPU, points sharded
by index, NCCL over NVLink for the two exchanges (SURVEY.md
§8(e)).  No reference equivalent: the reference is single-process; the result
equals ``compute_skyline`` (refine.cpp:108-158) over the concatenation of all
shards, ids and per-layer counts included.

Protocol (each arrow is one collective on the engine's stream):

    shard_begin (K0+K1 on the local shard)
      -> all_gather(occupancy regions)         NCCL has no bitwise OR
    shard_prune (K2 OR, K3, K4, local K5)      (nccl.h:260-275), so the OR
      -> all_gather(local skyline counts)      is fused into the library
    shard_pack                                 after an all-gather
      -> all_gather(padded local skylines)
    shard_finish (own points vs the union, K6)
      -> all_gather(counts), all_gather(padded ids) -> rank 0 concatenates
         in rank order (ids are global and ascending per rank)

The engine only needs the ``shard_*`` methods of
:class:`paper_2107_09993_b200.skycell.Engine`; the collectives are plain
``torch.distributed`` calls, so the same code runs over NCCL on B200s and
over gloo on CPU tensors (tests/test_dist.py drives it with a CPU stand-in
engine at world_size 2).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .skycell import InputError, SkylineResult, UsageError


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Records [begin, end) owned by `rank`: contiguous index ranges, the
    first n_total % world ranks one record longer."""
    base, extra = divmod(n_total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


class ShardedSkyline:
    """Runs the phase API of one engine against the other ranks of `group`."""

    def __init__(self, engine, group=None, device=None, coll_device=None):
        """`device` holds the engine's exchange buffers; `coll_device` (default:
        the same) is where the collectives run.  They differ only in tests that
        drive real engines over gloo (CPU collectives, buffers staged)."""
        self.eng = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
        self.device = torch.device(device)
        self.coll_device = torch.device(coll_device) if coll_device is not None else self.device
        self._bufs: dict[str, torch.Tensor] = {}

    def _all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        if self.coll_device == out.device:
            dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        o = torch.empty(out.shape, dtype=out.dtype, device=self.coll_device)
        dist.all_gather_into_tensor(o, inp.to(self.coll_device), group=self.group)
        out.copy_(o)

    def _buf(self, name: str, nbytes: int) -> torch.Tensor:
        b = self._bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=self.device)
            self._bufs[name] = b
        return b[:nbytes]

    def _gather_counts(self, value: int) -> list[int]:
        t = torch.tensor([value], dtype=torch.int64, device=self.coll_device)
        out = torch.empty(self.world, dtype=torch.int64, device=self.coll_device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return [int(v) for v in out.cpu().tolist()]

    def skyline(self, coords, n_local: int, d: int, dim_min, dim_max, rho: int, id_base: int, mode: int = 1,
                ids_out=None, gather_to: int | None = 0) -> SkylineResult:
        """Skyline of the global dataset of which this rank holds records
        [id_base, id_base + n_local).  Returns, on rank `gather_to`, the whole
        skyline (ascending global ids) with global stats; on other ranks this
        rank's part.  With gather_to=None every rank returns its own part."""
        world, rank = self.world, self.rank
        if self.device.type == "cuda" and hasattr(self.eng, "set_stream"):
            # kernels and NCCL collectives share torch's current stream
            self.eng.set_stream(torch.cuda.current_stream(self.device))
        # Every step that can fail on one rank (a rejected shard, a failed
        # kernel, an allocation) runs through _together: the rank reports -1
        # in the next count exchange instead of skipping it, so every rank
        # raises and none blocks in a collective.
        # phase 1: local streaming pass, and the export of the occupancy
        # region (one status exchange for both)
        def begin():
            nb = self.eng.shard_begin(coords, n_local, d, dim_min, dim_max, rho, mode, id_base)
            self._export(nb)
            return nb

        sizes = self._together(begin)
        if len(set(sizes)) != 1:
            # ranks built different grids (rho or d differ): the all-gather
            # below would mis-align, so every rank refuses the query
            raise UsageError(f"sharded skyline: ranks disagree on the occupancy size {sizes} (rho or d differ)")
        occ_bytes = sizes[0]
        gathered = self._bufs["occ_all"][: world * occ_bytes]
        self._all_gather(gathered, self._bufs["occ"][:occ_bytes])

        # phase 2: prune against the global occupancy, local skyline
        counts = self._together(lambda: self.eng.shard_prune(gathered, world))
        maxc = max(counts)
        bb = self.eng.shard_block_bytes(maxc)
        self._together(lambda: self._pack(bb, maxc, world))
        recv = self._bufs["recv"][: world * bb]
        self._all_gather(recv, self._bufs["send"][:bb])

        # phase 3: own local skyline against the union
        if ids_out is None:
            ids_out = np.empty(max(n_local, 1), dtype=np.uint32)
        # the finish status and the three summed statistics in one exchange
        res, err = None, None
        try:
            res = self.eng.shard_finish(recv, world, maxc, rank, counts[rank], ids_out)
            vec = [0, res.points_examined, res.survivors_stream, res.survivors_filter]
        except Exception as e:  # noqa: BLE001 -- re-raised below, after the exchange
            err, vec = e, [-1, 0, 0, 0]
        stats = self._gather_vec(vec)
        self._reraise(err, [int(v) for v in stats[:, 0]])
        res.points_examined, res.survivors_stream, res.survivors_filter = (int(v) for v in stats[:, 1:].sum(axis=0))
        if gather_to is None:
            return res
        res.ids = self._gather_ids(res.ids, gather_to)
        return res

    def _together(self, fn) -> list[int]:
        """Run fn on every rank and exchange its (non-negative int) result;
        a rank whose fn raised contributes -1 and re-raises, the others raise
        InputError.  Returns every rank's value."""
        err, val = None, 0
        try:
            r = fn()
            val = int(r) if isinstance(r, (int, np.integer)) else 0
        except Exception as e:  # noqa: BLE001 -- re-raised below, after the exchange
            err = e
        values = self._gather_counts(val if err is None else -1)
        self._reraise(err, values)
        return values

    def _export(self, occ_bytes: int) -> None:
        occ = self._buf("occ", occ_bytes)
        self._buf("occ_all", self.world * occ_bytes)
        self.eng.shard_export_occ(occ)

    def _pack(self, bb: int, maxc: int, world: int) -> None:
        send = self._buf("send", bb)
        self._buf("recv", world * bb)
        self.eng.shard_pack(send, maxc)

    def _gather_vec(self, values) -> np.ndarray:
        t = torch.tensor(values, dtype=torch.int64, device=self.coll_device)
        out = torch.empty(self.world * len(values), dtype=torch.int64, device=self.coll_device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy().reshape(self.world, len(values))

    def _reraise(self, err, values) -> None:
        if err is not None:
            raise err
        if any(v < 0 for v in values):
            raise InputError("sharded skyline: another rank rejected its shard")

    def _gather_ids(self, ids, root: int):
        """Concatenate every rank's ids on `root`, in rank order."""
        if isinstance(ids, torch.Tensor):
            local = ids.to(self.device).view(torch.int32)
        else:
            local = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.uint32).view(np.int32)).to(self.device)
        counts = self._gather_counts(int(local.numel()))
        maxk = max(counts)
        pad = torch.full((max(maxk, 1),), -1, dtype=torch.int32, device=self.device)
        pad[: local.numel()] = local
        allp = torch.empty(self.world * pad.numel(), dtype=torch.int32, device=self.device)
        self._all_gather(allp, pad)
        if self.rank != root:
            return ids
        allp = allp.view(self.world, -1)
        parts = [allp[g, : counts[g]] for g in range(self.world)]
        out = torch.cat(parts).cpu().numpy().view(np.uint32)
        return out


__all__ = ["ShardedSkyline", "shard_range"]
