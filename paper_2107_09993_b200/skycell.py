"""Python mirror of the reference's public skyline API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/skycell/{dataset,refine,grid,error}.hpp):

    Dataset                 dataset.hpp:20-32   (coords n x d row-major, dim_min/dim_max)
    compute_skyline(...)    refine.hpp:61-62    -> SkylineResult (refine.hpp:33-38)
    quadrant_skyline(...)   refine.hpp:66-68
    default_rho(n, d)       grid.cpp:30-33
    InputError / ConfigError / UsageError / IoError   error.hpp:9-26

Every call goes through ``libskycell_gpu.so`` (include/skycell_gpu.h).  There
is no CPU fallback: if the library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libskycell_gpu.so")


# ------------------------------------------------------------------ errors
class SkycellError(Exception):
    """Base of the status-code exceptions."""


class InputError(SkycellError, RuntimeError):
    """Bad input data (dataset.cpp:23-43)."""


class ConfigError(SkycellError, RuntimeError):
    """Partition ratio out of budget (grid.cpp:38-43)."""


class UsageError(SkycellError):
    """API misuse (refine.cpp:162-163)."""


class IoError(SkycellError, RuntimeError):
    pass


class CudaError(SkycellError, RuntimeError):
    """CUDA runtime failure (no reference equivalent)."""


class UnsupportedError(SkycellError):
    """Valid for the reference but not implemented by this build."""


_ERRORS = {1: InputError, 2: ConfigError, 3: UsageError, 4: IoError, 5: CudaError, 6: CudaError, 7: UnsupportedError}


class Mode(enum.IntEnum):
    """refine.hpp:40."""
    kSequential = 0
    kParallel = 1


# ----------------------------------------------------------------- records
@dataclass
class Dataset:
    """dataset.hpp:20-32: n records of d coordinates, row-major, plus the
    declared normalisation range per dimension."""
    coords: np.ndarray
    dim_min: np.ndarray
    dim_max: np.ndarray

    @property
    def n(self) -> int:
        return int(self.coords.shape[0])

    @property
    def d(self) -> int:
        return int(self.coords.shape[1]) if self.coords.ndim == 2 else 0

    @staticmethod
    def from_coords(coords, dim_min=None, dim_max=None) -> "Dataset":
        x = np.asarray(coords)
        if x.dtype not in (np.float32, np.float64):
            x = x.astype(np.float64)
        x = np.ascontiguousarray(x)
        d = x.shape[1] if x.ndim == 2 else 0
        ds = Dataset(x, np.zeros(d), np.ones(d))
        if dim_min is None or dim_max is None:
            ds.compute_minmax()
        else:
            ds.dim_min = np.asarray(dim_min, dtype=np.float64)
            ds.dim_max = np.asarray(dim_max, dtype=np.float64)
        return ds

    def compute_minmax(self) -> None:
        """Dataset::compute_minmax (dataset.cpp:10-20)."""
        x = np.asarray(self.coords, dtype=np.float64)
        if x.shape[0] == 0:
            self.dim_min = np.full(self.d, np.inf)
            self.dim_max = np.full(self.d, -np.inf)
        else:
            self.dim_min = x.min(axis=0)
            self.dim_max = x.max(axis=0)


@dataclass
class StageTimes:
    normalize_ms: float = 0.0
    grid_ms: float = 0.0
    shrink_ms: float = 0.0
    refine_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class LayerCounts:
    keys: list = field(default_factory=list)        # |KS_i|, i = 1..rho (auxiliary included)
    candidates: list = field(default_factory=list)  # |CS_i|; -1 when not materialised


@dataclass
class SkylineResult:
    ids: np.ndarray
    times: StageTimes = field(default_factory=StageTimes)
    layers: LayerCounts = field(default_factory=LayerCounts)
    points_examined: int = 0
    survivors_stream: int = 0
    survivors_filter: int = 0
    kernel_launches: int = 0
    stream_kernel_ms: float = 0.0
    filter_kernel_ms: float = 0.0
    dominance_ms: float = 0.0


class _Stats(C.Structure):
    _fields_ = [
        ("normalize_ms", C.c_double), ("grid_ms", C.c_double), ("shrink_ms", C.c_double),
        ("refine_ms", C.c_double), ("total_ms", C.c_double),
        ("points_examined", C.c_uint64), ("n_layers", C.c_int32), ("pad_", C.c_int32),
        ("keys", C.c_uint64 * 64), ("candidates", C.c_int64 * 64),
        ("survivors_stream", C.c_uint64), ("survivors_filter", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("stream_kernel_ms", C.c_double), ("filter_kernel_ms", C.c_double), ("dominance_ms", C.c_double),
    ]


# ----------------------------------------------------------------- library
_lib = None
_lib_lock = threading.Lock()

EXPORTS = (
    "skycell_gpu_create", "skycell_gpu_destroy", "skycell_gpu_set_stream", "skycell_gpu_skyline_f64",
    "skycell_gpu_skyline_f32", "skycell_gpu_quadrant_f64", "skycell_gpu_shard_begin", "skycell_gpu_shard_export_occ",
    "skycell_gpu_shard_prune", "skycell_gpu_shard_block_bytes", "skycell_gpu_shard_pack", "skycell_gpu_shard_finish",
    "skycell_gpu_generate", "skycell_gpu_generate_range", "skycell_default_rho", "skycell_validate",
    "skycell_gpu_version", "skycell_bin_header", "skycell_gpu_read_bin", "skycell_gpu_write_bin",
    "skycell_gpu_multi_create", "skycell_gpu_multi_destroy", "skycell_gpu_multi_size", "skycell_gpu_multi_context",
    "skycell_gpu_multi_skyline_f64", "skycell_gpu_multi_skyline_f32",
    "skycell_gpu_grid_build", "skycell_gpu_grid_destroy", "skycell_gpu_grid_shape", "skycell_gpu_grid_nonempty_count",
    "skycell_gpu_grid_points", "skycell_gpu_grid_nonempty_cells", "skycell_gpu_grid_lookup",
)


def load_library(path: str = LIB_PATH):
    """Load libskycell_gpu.so (fails loudly: there is no fallback path)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"libskycell_gpu.so not built at {path}; run __graft_entry__.build()")
        lib = C.CDLL(path)
        vp, u64, i32, dp, fp, u32p = C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_double), C.c_void_p, C.c_void_p
        lib.skycell_gpu_create.argtypes = [i32, C.POINTER(vp), C.c_char_p, C.c_size_t]
        lib.skycell_gpu_destroy.argtypes = [vp]
        lib.skycell_gpu_destroy.restype = None
        for fn in (lib.skycell_gpu_skyline_f64, lib.skycell_gpu_skyline_f32):
            fn.argtypes = [vp, fp, u64, i32, dp, dp, i32, i32, i32, u32p, C.POINTER(C.c_uint64),
                           C.POINTER(_Stats), C.c_char_p, C.c_size_t]
        lib.skycell_gpu_quadrant_f64.argtypes = [vp, fp, u64, i32, dp, i32, i32, i32, u32p, C.POINTER(C.c_uint64),
                                                 C.POINTER(_Stats), C.c_char_p, C.c_size_t]
        lib.skycell_gpu_generate.argtypes = [vp, i32, u64, i32, u64, i32, vp, C.c_char_p, C.c_size_t]
        lib.skycell_gpu_generate_range.argtypes = [vp, i32, u64, i32, u64, i32, u64, u64, vp, C.c_char_p, C.c_size_t]
        lib.skycell_gpu_set_stream.argtypes = [vp, vp, i32]
        u64p, cp, sz = C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t
        lib.skycell_gpu_shard_begin.argtypes = [vp, vp, i32, u64, i32, dp, dp, i32, i32, u64, u64p, cp, sz]
        lib.skycell_gpu_shard_export_occ.argtypes = [vp, vp, cp, sz]
        lib.skycell_gpu_shard_prune.argtypes = [vp, vp, i32, u64p, cp, sz]
        lib.skycell_gpu_shard_block_bytes.argtypes = [vp, u64]
        lib.skycell_gpu_shard_block_bytes.restype = C.c_uint64
        lib.skycell_gpu_shard_pack.argtypes = [vp, vp, u64, cp, sz]
        lib.skycell_gpu_shard_finish.argtypes = [vp, vp, i32, u64, i32, u64, u32p, u64p, C.POINTER(_Stats), cp, sz]
        lib.skycell_default_rho.argtypes = [u64, i32]
        lib.skycell_validate.argtypes = [u64, i32, i32, C.c_char_p, C.c_size_t]
        lib.skycell_gpu_version.restype = C.c_char_p
        lib.skycell_bin_header.argtypes = [cp, u64p, C.POINTER(C.c_int), cp, sz]
        lib.skycell_gpu_read_bin.argtypes = [vp, cp, vp, u64, u64p, C.POINTER(C.c_int), dp, dp, cp, sz]
        lib.skycell_gpu_write_bin.argtypes = [vp, cp, vp, u64, i32, cp, sz]
        lib.skycell_gpu_multi_create.argtypes = [C.POINTER(C.c_int), i32, C.POINTER(vp), cp, sz]
        lib.skycell_gpu_multi_destroy.argtypes = [vp]
        lib.skycell_gpu_multi_destroy.restype = None
        lib.skycell_gpu_multi_size.argtypes = [vp]
        lib.skycell_gpu_multi_context.argtypes = [vp, i32]
        lib.skycell_gpu_multi_context.restype = vp
        for fn in (lib.skycell_gpu_multi_skyline_f64, lib.skycell_gpu_multi_skyline_f32):
            fn.argtypes = [vp, fp, u64, i32, dp, dp, i32, i32, i32, u32p, u64p, C.POINTER(_Stats), cp, sz]
        lib.skycell_gpu_grid_build.argtypes = [vp, vp, vp, u64, i32, i32, C.POINTER(vp), cp, sz]
        lib.skycell_gpu_grid_destroy.argtypes = [vp]
        lib.skycell_gpu_grid_destroy.restype = None
        lib.skycell_gpu_grid_shape.argtypes = [vp, u64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.skycell_gpu_grid_nonempty_count.argtypes = [vp, i32]
        lib.skycell_gpu_grid_nonempty_count.restype = C.c_uint64
        lib.skycell_gpu_grid_points.argtypes = [vp, vp, vp, cp, sz]
        lib.skycell_gpu_grid_nonempty_cells.argtypes = [vp, i32, vp, cp, sz]
        lib.skycell_gpu_grid_lookup.argtypes = [vp, i32, vp, u64, vp, vp, vp, cp, sz]
        _lib = lib
        return lib


def _raise(code: int, err) -> None:
    if code != 0:
        raise _ERRORS.get(code, SkycellError)(err.value.decode(errors="replace"))


def bin_header(path: str) -> tuple[int, int]:
    """(n, d) of a SKYC file, with read_bin's header checks (datagen.cpp:201-212)."""
    lib = load_library()
    n, d = C.c_uint64(0), C.c_int(0)
    err = C.create_string_buffer(512)
    _raise(lib.skycell_bin_header(os.fsencode(path), C.byref(n), C.byref(d), err, 512), err)
    return int(n.value), int(d.value)


def default_rho(n: int, d: int) -> int:
    """MultiLayerGrid::default_rho (grid.cpp:30-33)."""
    return int(load_library().skycell_default_rho(n, d))


def validate(n: int, d: int, rho: int) -> None:
    """Host-side argument checks in the reference's order (no device needed)."""
    err = C.create_string_buffer(512)
    _raise(load_library().skycell_validate(n, d, rho, err, 512), err)


# ------------------------------------------------------------------ engine
class Engine:
    """One device context (include/skycell_gpu.h: skycell_gpu_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.device = device
        self._ctx = C.c_void_p()
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_create(device, C.byref(self._ctx), err, 512), err)
        self._lock = threading.Lock()

    def close(self) -> None:
        if self._ctx:
            self.lib.skycell_gpu_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # raw entry point: coords may be a numpy array (host) or a CUDA tensor
    # (device pointer, used in place); ids_out likewise.
    def skyline_raw(self, coords, n: int, d: int, dim_min, dim_max, rho: int, mode: int = 1,
                    merge_cross_cell: bool = True, ids_out=None, with_stats: bool = True):
        ptr, is_f32 = _data_ptr(coords, n, d, self.device)
        mn = np.ascontiguousarray(dim_min, dtype=np.float64)
        mx = np.ascontiguousarray(dim_max, dtype=np.float64)
        if mn.shape[0] < d or mx.shape[0] < d:
            raise UsageError("dim_min/dim_max must hold d values")
        own = ids_out is None
        if own:
            ids_out = np.empty(max(n, 1), dtype=np.uint32)
        out_ptr, _ = _data_ptr(ids_out, n, None, self.device, "ids_out", itemsize=4)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(512)
        fn = self.lib.skycell_gpu_skyline_f32 if is_f32 else self.lib.skycell_gpu_skyline_f64
        with self._lock:
            rc = fn(self._ctx, ptr, n, d, mn.ctypes.data_as(C.POINTER(C.c_double)),
                    mx.ctypes.data_as(C.POINTER(C.c_double)), rho, int(mode), int(bool(merge_cross_cell)),
                    out_ptr, C.byref(n_out), C.byref(st) if with_stats else None, err, 512)
        _raise(rc, err)
        k = int(n_out.value)
        ids = ids_out[:k].copy() if own else ids_out[:k]
        return _to_result(ids, st if with_stats else None)

    def generate(self, dist: int, n: int, d: int, seed: int, quantized: bool = True, out=None,
                 begin: int = 0, count: int | None = None):
        """Synthetic data on the device (skycell_gpu_generate_range).  Returns a
        CUDA tensor of shape (count, d) holding records [begin, begin + count)
        of the n-record dataset: float32 on the 2^-24 grid, or raw float64."""
        import torch
        count = n - begin if count is None else count
        if out is None:
            out = torch.empty((count, d), dtype=torch.float32 if quantized else torch.float64,
                              device=f"cuda:{self.device}")
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_generate_range(self._ctx, int(dist), n, d, seed, 1 if quantized else 0, begin,
                                                   count, C.c_void_p(out.data_ptr()), err, 512), err)
        return out

    def grid(self, coords, rho: int, ids=None) -> "MultiLayerGrid":
        """MultiLayerGrid(PointSet, rho) on this device (grid.cpp:35-103)."""
        return MultiLayerGrid(self, coords, rho, ids)

    def read_bin(self, path: str):
        """skycell::read_bin (datagen.cpp:201-221) straight into device memory:
        returns (CUDA float64 tensor (n, d), dim_min, dim_max)."""
        import torch
        n, d = bin_header(path)
        out = torch.empty((max(n, 1), d), dtype=torch.float64, device=f"cuda:{self.device}")
        mn, mx = np.empty(d), np.empty(d)
        n_out, d_out = C.c_uint64(0), C.c_int(0)
        err = C.create_string_buffer(512)
        with self._lock:
            rc = self.lib.skycell_gpu_read_bin(self._ctx, os.fsencode(path), C.c_void_p(out.data_ptr()), n * d,
                                               C.byref(n_out), C.byref(d_out),
                                               mn.ctypes.data_as(C.POINTER(C.c_double)),
                                               mx.ctypes.data_as(C.POINTER(C.c_double)), err, 512)
        _raise(rc, err)
        return out[:n], mn, mx

    def write_bin(self, path: str, coords) -> None:
        """skycell::write_bin (datagen.cpp:185-199) from a float64 host array or
        CUDA tensor of shape (n, d)."""
        if isinstance(coords, np.ndarray):
            if coords.dtype != np.float64 or coords.ndim != 2 or not coords.flags.c_contiguous:
                raise UsageError("write_bin: coords must be a C-contiguous float64 (n, d) array")
            ptr, (n, d) = coords.ctypes.data, coords.shape
        else:
            import torch
            if coords.dtype != torch.float64 or coords.dim() != 2 or not coords.is_contiguous():
                raise UsageError("write_bin: coords must be a contiguous float64 (n, d) tensor")
            ptr, (n, d) = coords.data_ptr(), tuple(coords.shape)
        err = C.create_string_buffer(512)
        with self._lock:
            rc = self.lib.skycell_gpu_write_bin(self._ctx, os.fsencode(path), C.c_void_p(ptr), n, d, err, 512)
        _raise(rc, err)

    def set_stream(self, stream) -> None:
        """Enqueue all later work on `stream` (a torch.cuda.Stream, a raw
        cudaStream_t int, or None for the context's own stream)."""
        if stream is None:
            self.lib.skycell_gpu_set_stream(self._ctx, None, 1)
        else:
            h = int(getattr(stream, "cuda_stream", stream))  # 0 = legacy default stream
            self.lib.skycell_gpu_set_stream(self._ctx, C.c_void_p(h), 0)

    # ---- sharded query phases (include/skycell_gpu.h); the
    # exchanges between them are issued by paper_2107_09993_b200.dist.
    def shard_begin(self, coords, n: int, d: int, dim_min, dim_max, rho: int, mode: int, id_base: int) -> int:
        ptr, is_f32 = _data_ptr(coords, n, d, self.device)
        mn = np.ascontiguousarray(dim_min, dtype=np.float64)
        mx = np.ascontiguousarray(dim_max, dtype=np.float64)
        occ = C.c_uint64(0)
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_shard_begin(self._ctx, ptr, int(is_f32), n, d,
                                                mn.ctypes.data_as(C.POINTER(C.c_double)),
                                                mx.ctypes.data_as(C.POINTER(C.c_double)), rho, int(mode), id_base,
                                                C.byref(occ), err, 512), err)
        return int(occ.value)

    def shard_export_occ(self, dst) -> None:
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_shard_export_occ(self._ctx, C.c_void_p(dst.data_ptr()), err, 512), err)

    def shard_prune(self, gathered, world: int) -> int:
        cnt = C.c_uint64(0)
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_shard_prune(self._ctx, C.c_void_p(gathered.data_ptr()), world, C.byref(cnt),
                                                err, 512), err)
        return int(cnt.value)

    def shard_block_bytes(self, max_count: int) -> int:
        return int(self.lib.skycell_gpu_shard_block_bytes(self._ctx, max_count))

    def shard_pack(self, dst, max_count: int) -> None:
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_shard_pack(self._ctx, C.c_void_p(dst.data_ptr()), max_count, err, 512), err)

    def shard_finish(self, recv, world: int, max_count: int, rank: int, own_count: int, ids_out):
        out_ptr, _ = _data_ptr(ids_out, own_count, None, self.device, "ids_out", itemsize=4)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_shard_finish(self._ctx, C.c_void_p(recv.data_ptr()), world, max_count, rank,
                                                 own_count, out_ptr, C.byref(n_out), C.byref(st), err, 512), err)
        return _to_result(ids_out[: n_out.value], st)

    def compute_skyline(self, ds: Dataset, rho: int, mode: Mode = Mode.kParallel, pool=None,
                        merge_cross_cell: bool = True) -> SkylineResult:
        """compute_skyline (refine.hpp:61-62).  `pool` is accepted for
        signature parity and ignored: the GPU does not use host threads."""
        x = np.asarray(ds.coords)
        if x.ndim != 2:
            x = x.reshape(0, 0) if x.size == 0 else x.reshape(x.shape[0], -1)
        if x.dtype not in (np.float32, np.float64):
            x = x.astype(np.float64)
        x = np.ascontiguousarray(x)
        n, d = x.shape
        return self.skyline_raw(x, n, d, ds.dim_min, ds.dim_max, rho, int(mode), merge_cross_cell)

    def quadrant_skyline(self, ds: Dataset, origin, rho: int, mode: Mode = Mode.kParallel, pool=None) -> SkylineResult:
        """quadrant_skyline (refine.hpp:66-68, refine.cpp:160-184)."""
        x = np.ascontiguousarray(ds.coords, dtype=np.float64)
        n, d = x.shape
        o = np.ascontiguousarray(origin, dtype=np.float64)
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(512)
        with self._lock:
            rc = self.lib.skycell_gpu_quadrant_f64(self._ctx, x.ctypes.data, n, d,
                                                   o.ctypes.data_as(C.POINTER(C.c_double)), int(o.shape[0]),
                                                   rho, int(mode), ids.ctypes.data, C.byref(n_out), C.byref(st),
                                                   err, 512)
        _raise(rc, err)
        return _to_result(ids[: n_out.value].copy(), st)


class MultiLayerGrid:
    """skycell::MultiLayerGrid (grid.hpp:33-70) built on the device
    (skycell_gpu_grid_*).  Cells are named by their linear index
    (CellIndex::linear_index, dim d-1 most significant)."""

    def __init__(self, engine: "Engine", coords, rho: int, ids=None):
        self.lib = engine.lib
        x = np.ascontiguousarray(coords, dtype=np.float64)
        if x.ndim != 2:
            raise UsageError("MultiLayerGrid: coords must be (n, d)")
        n, d = x.shape
        idp = None
        if ids is not None:
            ids = np.ascontiguousarray(ids, dtype=np.uint32)
            if ids.shape != (n,):
                raise UsageError("MultiLayerGrid: ids must hold n values")
            idp = C.c_void_p(ids.ctypes.data)
        self._g = C.c_void_p()
        err = C.create_string_buffer(512)
        with engine._lock:
            rc = self.lib.skycell_gpu_grid_build(engine._ctx, C.c_void_p(x.ctypes.data), idp, n, d, rho,
                                                 C.byref(self._g), err, 512)
        _raise(rc, err)
        self.n, self.d, self._rho = n, d, rho

    def close(self) -> None:
        if self._g:
            self.lib.skycell_gpu_grid_destroy(self._g)
            self._g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rho(self) -> int:
        return self._rho

    def dims(self) -> int:
        return self.d

    def size(self) -> int:
        return self.n

    def points(self):
        """The sorted PointSet: (coords (n, d) float64, ids uint32)."""
        x = np.empty((self.n, self.d), dtype=np.float64)
        ids = np.empty(self.n, dtype=np.uint32)
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_grid_points(self._g, C.c_void_p(x.ctypes.data), C.c_void_p(ids.ctypes.data),
                                                err, 512), err)
        return x, ids

    def nonempty_count(self, layer: int) -> int:
        return int(self.lib.skycell_gpu_grid_nonempty_count(self._g, layer))

    def nonempty_cells(self, layer: int) -> np.ndarray:
        out = np.empty(max(self.nonempty_count(layer), 1), dtype=np.uint64)
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_grid_nonempty_cells(self._g, layer, C.c_void_p(out.ctypes.data), err, 512), err)
        return out[: self.nonempty_count(layer)]

    def _lookup(self, layer: int, lins, ranges: bool):
        q = np.ascontiguousarray(lins, dtype=np.uint64)
        occ = np.empty(max(q.size, 1), dtype=np.uint8)
        b = np.empty(max(q.size, 1), dtype=np.uint32) if ranges else None
        e = np.empty(max(q.size, 1), dtype=np.uint32) if ranges else None
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_grid_lookup(self._g, layer, C.c_void_p(q.ctypes.data), q.size,
                                                C.c_void_p(occ.ctypes.data), C.c_void_p(b.ctypes.data) if ranges else None,
                                                C.c_void_p(e.ctypes.data) if ranges else None, err, 512), err)
        return occ[: q.size].astype(bool), (b[: q.size] if ranges else None), (e[: q.size] if ranges else None)

    def occupied(self, layer: int, lins) -> np.ndarray:
        """MultiLayerGrid::occupied for in-grid cells of one layer (batch)."""
        return self._lookup(layer, lins, False)[0]

    def range(self, lins):
        """MultiLayerGrid::range for layer-rho cells (batch): (begin, end)."""
        _, b, e = self._lookup(self._rho, lins, True)
        return b, e


class MultiEngine:
    """One process, several devices (include/skycell_gpu.h: skycell_gpu_multi):
    the records are sharded by index over the devices and the sharded
    protocol runs inside the library (device-to-device exchanges).  Same
    results as Engine.compute_skyline; `devices` may repeat a device."""

    def __init__(self, devices):
        self.lib = load_library()
        self.devices = [int(x) for x in devices]
        arr = (C.c_int * len(self.devices))(*self.devices)
        self._m = C.c_void_p()
        err = C.create_string_buffer(512)
        _raise(self.lib.skycell_gpu_multi_create(arr, len(self.devices), C.byref(self._m), err, 512), err)
        self._lock = threading.Lock()

    def close(self) -> None:
        if self._m:
            self.lib.skycell_gpu_multi_destroy(self._m)
            self._m = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def skyline_raw(self, coords, n: int, d: int, dim_min, dim_max, rho: int, mode: int = 1,
                    merge_cross_cell: bool = True):
        if not isinstance(coords, np.ndarray):
            raise UsageError("MultiEngine: coords must be a host numpy array (sharded over the devices)")
        ptr, is_f32 = _data_ptr(coords, n, d)
        mn = np.ascontiguousarray(dim_min, dtype=np.float64)
        mx = np.ascontiguousarray(dim_max, dtype=np.float64)
        if mn.shape[0] < d or mx.shape[0] < d:
            raise UsageError("dim_min/dim_max must hold d values")
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(512)
        fn = self.lib.skycell_gpu_multi_skyline_f32 if is_f32 else self.lib.skycell_gpu_multi_skyline_f64
        with self._lock:
            rc = fn(self._m, ptr, n, d, mn.ctypes.data_as(C.POINTER(C.c_double)),
                    mx.ctypes.data_as(C.POINTER(C.c_double)), rho, int(mode), int(bool(merge_cross_cell)),
                    C.c_void_p(ids.ctypes.data), C.byref(n_out), C.byref(st), err, 512)
        _raise(rc, err)
        return _to_result(ids[: n_out.value].copy(), st)

    def compute_skyline(self, ds: Dataset, rho: int, mode: Mode = Mode.kParallel, pool=None,
                        merge_cross_cell: bool = True) -> SkylineResult:
        """compute_skyline (refine.hpp:61-62) over every device of the handle."""
        x = np.asarray(ds.coords)
        if x.dtype not in (np.float32, np.float64):
            x = x.astype(np.float64)
        x = np.ascontiguousarray(x.reshape(x.shape[0], -1) if x.ndim != 2 and x.size else x)
        n, d = x.shape if x.ndim == 2 else (0, 0)
        return self.skyline_raw(x, n, d, ds.dim_min, ds.dim_max, rho, int(mode), merge_cross_cell)


def _data_ptr(a, n: int | None = None, d: int | None = None, device: int | None = None, what: str = "coords",
              itemsize: int | None = None):
    """(pointer, is_f32) of a numpy array or a torch tensor (host or CUDA).

    Coordinates must be float32 or float64 (the two C ABI entry points); an
    output id buffer must be 4-byte integers.  With n (and d) given, the
    buffer must hold at least n * d elements; a CUDA tensor must live on the
    engine's device.  Anything else raises UsageError before the C ABI reads
    out of bounds."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise UsageError("arrays must be C-contiguous")
        dt, size = a.dtype, a.size
        ok = dt.itemsize == itemsize and dt.kind in "iu" if itemsize else dt in (np.float32, np.float64)
        is_f32 = dt == np.float32
        ptr = C.c_void_p(a.ctypes.data)
    elif hasattr(a, "data_ptr"):
        import torch
        if not a.is_contiguous():
            raise UsageError("tensors must be contiguous")
        if a.is_cuda and device is not None and a.device.index != device:
            raise UsageError(f"{what} tensor is on {a.device}, the engine on cuda:{device}")
        dt, size = a.dtype, a.numel()
        if itemsize:
            ok = dt in (torch.int32, torch.uint32) if hasattr(torch, "uint32") else dt == torch.int32
        else:
            ok = dt in (torch.float32, torch.float64)
        is_f32 = dt == torch.float32
        ptr = C.c_void_p(a.data_ptr())
    else:
        raise UsageError(f"unsupported array type {type(a)!r}")
    if not ok:
        raise UsageError(f"{what}: unsupported element type {dt} "
                         + ("(expected 32-bit integers)" if itemsize else "(expected float32 or float64)"))
    if n is not None and size < n * (d or 1):
        raise UsageError(f"{what}: buffer holds {size} elements, needs {n * (d or 1)}")
    return ptr, is_f32


def _to_result(ids, st) -> SkylineResult:
    r = SkylineResult(ids=ids)
    if st is not None:
        L = st.n_layers
        r.times = StageTimes(st.normalize_ms, st.grid_ms, st.shrink_ms, st.refine_ms, st.total_ms)
        r.layers = LayerCounts([int(st.keys[i]) for i in range(L)], [int(st.candidates[i]) for i in range(L)])
        r.points_examined = int(st.points_examined)
        r.survivors_stream = int(st.survivors_stream)
        r.survivors_filter = int(st.survivors_filter)
        r.kernel_launches = int(st.kernel_launches)
        r.stream_kernel_ms = float(st.stream_kernel_ms)
        r.filter_kernel_ms = float(st.filter_kernel_ms)
        r.dominance_ms = float(st.dominance_ms)
    return r


_default_engines: dict[int, Engine] = {}


def engine(device: int = 0) -> Engine:
    e = _default_engines.get(device)
    if e is None:
        e = _default_engines[device] = Engine(device)
    return e


def compute_skyline(ds: Dataset, rho: int, mode: Mode = Mode.kParallel, pool=None,
                    merge_cross_cell: bool = True) -> SkylineResult:
    """Drop-in for skycell::compute_skyline (refine.hpp:61-62) on cuda:0."""
    return engine(0).compute_skyline(ds, rho, mode, pool, merge_cross_cell)


def quadrant_skyline(ds: Dataset, origin, rho: int, mode: Mode = Mode.kParallel, pool=None) -> SkylineResult:
    """Drop-in for skycell::quadrant_skyline (refine.hpp:66-68) on cuda:0."""
    return engine(0).quadrant_skyline(ds, origin, rho, mode, pool)
