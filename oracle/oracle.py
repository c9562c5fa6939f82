"""TEST INFRASTRUCTURE ONLY -- ctypes loaders for the CPU checkers.

* :class:`Oracle` wraps ``oracle/_oracle/libskycell_oracle.so``, our plain-C
  restatement of the reference hot path (``oracle/skycell_oracle.c``).
* :class:`Reference` wraps ``oracle/_ref/libskycell_ref.so``, the unmodified
  reference library (``/root/reference/proj/src``) behind ``oracle/ref_capi.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
as the checker / CPU baseline -- never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_oracle", "libskycell_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libskycell_ref.so")
REF_SRC = "/root/reference/proj/src"


class _Stats(C.Structure):
    _fields_ = [
        ("normalize_ms", C.c_double), ("grid_ms", C.c_double), ("shrink_ms", C.c_double),
        ("refine_ms", C.c_double), ("total_ms", C.c_double),
        ("points_examined", C.c_uint64), ("n_layers", C.c_int32), ("pad_", C.c_int32),
        ("keys", C.c_uint64 * 64), ("candidates", C.c_int64 * 64),
    ]


@dataclass
class CpuResult:
    ids: np.ndarray
    points_examined: int = 0
    keys: list = field(default_factory=list)
    candidates: list = field(default_factory=list)
    times: dict = field(default_factory=dict)


class CpuError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(with_reference: bool | None = None) -> None:
    """Compile the oracle (always) and the reference (when its tree exists)."""
    targets = ["oracle"]
    if with_reference is None:
        with_reference = os.path.isdir(REF_SRC)
    if with_reference:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def _result(ids, n_out, st: _Stats | None) -> CpuResult:
    r = CpuResult(ids=ids[: n_out.value].copy())
    if st is not None:
        L = st.n_layers
        r.points_examined = int(st.points_examined)
        r.keys = [int(st.keys[i]) for i in range(L)]
        r.candidates = [int(st.candidates[i]) for i in range(L)]
        r.times = dict(normalize_ms=st.normalize_ms, grid_ms=st.grid_ms, shrink_ms=st.shrink_ms,
                       refine_ms=st.refine_ms, total_ms=st.total_ms)
    return r


class Oracle:
    """Our C restatement (oracle/skycell_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(with_reference=False)
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_generate.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
        L.orc_compute_skyline.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int,
                                          C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(_Stats),
                                          C.c_char_p, C.c_size_t]
        L.orc_brute_force.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                      C.c_char_p, C.c_size_t]
        L.orc_normalize.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
        L.orc_quadrant_skyline.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                           C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint32),
                                           C.POINTER(C.c_uint64), C.POINTER(_Stats), C.c_char_p, C.c_size_t]
        L.orc_compute_minmax.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
        L.orc_default_rho.argtypes = [C.c_uint64, C.c_int]

    def _check(self, rc, err):
        if rc != 0:
            raise CpuError(rc, err.value.decode())

    def generate(self, dist: int, n: int, d: int, seed: int) -> np.ndarray:
        out = np.empty((n, d), dtype=np.float64)
        err = C.create_string_buffer(256)
        self._check(self.lib.orc_generate(dist, n, d, seed, _ptr(out, C.c_double), err, 256), err)
        return out

    def normalize(self, coords, dmin, dmax) -> np.ndarray:
        x = _f64(coords)
        n, d = x.shape
        out = np.empty_like(x)
        err = C.create_string_buffer(256)
        self._check(self.lib.orc_normalize(_ptr(x, C.c_double), n, d, _ptr(_f64(dmin), C.c_double),
                                           _ptr(_f64(dmax), C.c_double), _ptr(out, C.c_double), err, 256), err)
        return out

    def compute_skyline(self, coords, dmin, dmax, rho: int, mode: int = 1, merge: bool = True) -> CpuResult:
        x = _f64(coords)
        n, d = x.shape
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(256)
        self._check(self.lib.orc_compute_skyline(_ptr(x, C.c_double), n, d, _ptr(_f64(dmin), C.c_double),
                                                 _ptr(_f64(dmax), C.c_double), rho, mode, int(merge),
                                                 _ptr(ids, C.c_uint32), C.byref(n_out), C.byref(st), err, 256), err)
        return _result(ids, n_out, st)

    def quadrant_skyline(self, coords, origin, rho: int, mode: int = 1) -> CpuResult:
        x = _f64(coords)
        n, d = x.shape
        o = _f64(origin)
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(256)
        self._check(self.lib.orc_quadrant_skyline(_ptr(x, C.c_double), n, d, _ptr(o, C.c_double), len(o), rho,
                                                  mode, _ptr(ids, C.c_uint32), C.byref(n_out), C.byref(st),
                                                  err, 256), err)
        return _result(ids, n_out, st)

    def brute_force(self, coords, dmin, dmax) -> np.ndarray:
        x = _f64(coords)
        n, d = x.shape
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        err = C.create_string_buffer(256)
        self._check(self.lib.orc_brute_force(_ptr(x, C.c_double), n, d, _ptr(_f64(dmin), C.c_double),
                                             _ptr(_f64(dmax), C.c_double), _ptr(ids, C.c_uint32),
                                             C.byref(n_out), err, 256), err)
        return ids[: n_out.value].copy()

    def compute_minmax(self, coords):
        x = _f64(coords)
        n, d = x.shape
        mn = np.empty(d)
        mx = np.empty(d)
        self.lib.orc_compute_minmax(_ptr(x, C.c_double), n, d, _ptr(mn, C.c_double), _ptr(mx, C.c_double))
        return mn, mx

    def default_rho(self, n: int, d: int) -> int:
        return int(self.lib.orc_default_rho(n, d))


class Reference:
    """The unmodified reference library (oracle/_ref/libskycell_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REF_SRC):
                build(with_reference=True)
            else:
                raise FileNotFoundError(f"{path} not built and {REF_SRC} absent")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                   C.c_char_p, C.c_size_t]
        L.ref_default_rho.argtypes = [C.c_uint64, C.c_int]
        L.ref_compute_skyline.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(_Stats),
                                          C.c_char_p, C.c_size_t]
        L.ref_quadrant_skyline.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                           C.POINTER(_Stats), C.c_char_p, C.c_size_t]
        L.ref_brute_force.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.c_uint32, C.c_int, C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_normalize.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
        L.ref_grid.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint32),
                               C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                               C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]
        L.ref_write_bin.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_uint64, C.c_int, C.c_char_p, C.c_size_t]
        L.ref_read_bin.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p, C.c_size_t]

    def _check(self, rc, err):
        if rc != 0:
            raise CpuError(rc, err.value.decode())

    def grid(self, coords, rho: int, layer: int):
        """skycell::MultiLayerGrid (grid.cpp:35-103) over a normalised PointSet
        with ids 0..n-1: dict(ids, counts, leaf_lin, leaf_begin, leaf_end,
        layer_lin) -- layer_lin = nonempty_cells(layer) as linear indices."""
        x = _f64(coords)
        n, d = x.shape
        ids = np.empty(max(n, 1), dtype=np.uint32)
        counts = np.zeros(rho + 1, dtype=np.uint64)
        lin, beg, end = np.empty(max(n, 1), dtype=np.uint64), np.empty(max(n, 1), dtype=np.uint32), np.empty(max(n, 1), dtype=np.uint32)
        cells = np.empty(max(n, 1 << min(24, layer * d)), dtype=np.uint64)
        err = C.create_string_buffer(512)
        self._check(self.lib.ref_grid(_ptr(x, C.c_double), n, d, rho, layer, _ptr(ids, C.c_uint32),
                                      _ptr(counts, C.c_uint64), _ptr(lin, C.c_uint64), _ptr(beg, C.c_uint32),
                                      _ptr(end, C.c_uint32), _ptr(cells, C.c_uint64), err, 512), err)
        nl, nc = int(counts[rho]), int(counts[layer])
        return dict(ids=ids[:n], counts=[int(c) for c in counts], leaf_lin=lin[:nl], leaf_begin=beg[:nl],
                    leaf_end=end[:nl], layer_lin=cells[:nc])

    def write_bin(self, path: str, coords) -> None:
        """skycell::write_bin (datagen.cpp:185-199)."""
        x = _f64(coords)
        err = C.create_string_buffer(512)
        self._check(self.lib.ref_write_bin(path.encode(), _ptr(x, C.c_double), x.shape[0], x.shape[1], err, 512), err)

    def read_bin(self, path: str):
        """skycell::read_bin (datagen.cpp:201-221): (coords, dim_min, dim_max)."""
        n, d = C.c_uint64(0), C.c_int(0)
        err = C.create_string_buffer(512)
        null = C.POINTER(C.c_double)()
        self._check(self.lib.ref_read_bin(path.encode(), C.byref(n), C.byref(d), null, null, null, err, 512), err)
        x = np.empty((n.value, d.value), dtype=np.float64)
        mn, mx = np.empty(d.value), np.empty(d.value)
        self._check(self.lib.ref_read_bin(path.encode(), C.byref(n), C.byref(d), _ptr(x, C.c_double),
                                          _ptr(mn, C.c_double), _ptr(mx, C.c_double), err, 512), err)
        return x, mn, mx

    def generate(self, dist: int, n: int, d: int, seed: int, workers: int = 0) -> np.ndarray:
        out = np.empty((n, d), dtype=np.float64)
        err = C.create_string_buffer(256)
        self._check(self.lib.ref_generate(dist, n, d, seed, workers, _ptr(out, C.c_double), err, 256), err)
        return out

    def default_rho(self, n: int, d: int) -> int:
        return int(self.lib.ref_default_rho(n, d))

    def compute_skyline(self, coords, dmin, dmax, rho: int, mode: int = 1, merge: bool = True,
                        workers: int = 0) -> CpuResult:
        x = _f64(coords)
        n, d = x.shape
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(256)
        self._check(self.lib.ref_compute_skyline(_ptr(x, C.c_double), n, d, _ptr(_f64(dmin), C.c_double),
                                                 _ptr(_f64(dmax), C.c_double), rho, mode, int(merge), workers,
                                                 _ptr(ids, C.c_uint32), C.byref(n_out), C.byref(st), err, 256), err)
        return _result(ids, n_out, st)

    def quadrant_skyline(self, coords, dmin, dmax, origin, rho: int, mode: int = 1, workers: int = 0) -> CpuResult:
        x = _f64(coords)
        n, d = x.shape
        o = _f64(origin)
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        st = _Stats()
        err = C.create_string_buffer(256)
        self._check(self.lib.ref_quadrant_skyline(_ptr(x, C.c_double), n, d, _ptr(_f64(dmin), C.c_double),
                                                  _ptr(_f64(dmax), C.c_double), _ptr(o, C.c_double), len(o), rho,
                                                  mode, workers, _ptr(ids, C.c_uint32), C.byref(n_out),
                                                  C.byref(st), err, 256), err)
        return _result(ids, n_out, st)

    def brute_force(self, coords, dmin, dmax, cap: int = 50000, workers: int = 0) -> np.ndarray:
        x = _f64(coords)
        n, d = x.shape
        ids = np.empty(max(n, 1), dtype=np.uint32)
        n_out = C.c_uint64(0)
        err = C.create_string_buffer(256)
        self._check(self.lib.ref_brute_force(_ptr(x, C.c_double), n, d, _ptr(_f64(dmin), C.c_double),
                                             _ptr(_f64(dmax), C.c_double), cap, workers, _ptr(ids, C.c_uint32),
                                             C.byref(n_out), err, 256), err)
        return ids[: n_out.value].copy()


def reference_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)


def quantize_f32(v: np.ndarray) -> np.ndarray:
    """BASELINE.md §2 input rule: x = (float)(floor(v * 2^24) * 2^-24)."""
    return (np.floor(v * 16777216.0) * (1.0 / 16777216.0)).astype(np.float32)


def fnv1a64_ids(ids: np.ndarray) -> str:
    """FNV-1a 64 over ascending ids as little-endian u32 bytes."""
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(ids, dtype="<u4").tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
