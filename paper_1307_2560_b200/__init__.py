"""B200-native yCHG hot path (arXiv 1307.2560): Python mirror of the reference API.

The reference's hot path is the C++ runscan API (proj/include/ychg/runscan.hpp):
``cut_vertex_counts(image, strategy)``, ``detect_boundary_columns(counts)`` and,
for hyperedge totals, ``hyperedge_count(decompose(build_profile(image)))``.
This module exposes the same names with the same argument meaning and error
behaviour, executed by the sm_100a kernels in ``libychg_b200.so`` through its C
ABI (``include/ychg_b200.h``).  PyTorch is not needed by this module; bench.py
uses it only for streams, events and torch.distributed plumbing.

There is no CPU fallback: if the native library is missing the import fails,
and on a machine without a CUDA device every compute call raises ``Error``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# YCHG_LIB selects an experimental launch-shape build (see _build.build_variant).
LIB_PATH = os.environ.get("YCHG_LIB") or os.path.join(_PKG, "libychg_b200.so")
CXX_LIB_PATH = os.path.join(_PKG, "libychg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()').  There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

# ---------------------------------------------------------------- C ABI
OK, ERR_INVALID, ERR_CUDA, ERR_OOM, ERR_NO_DEVICE, ERR_INTERNAL, ERR_PARSE = 0, -1, -2, -3, -4, -5, -6
STRATEGY_SERIAL, STRATEGY_PARALLEL = 0, 1
PATTERNS = {"full": 0, "empty": 1, "frame": 2, "hbands": 3, "checker": 4, "random": 5}


class Totals(ctypes.Structure):
    _fields_ = [("total_runs", ctypes.c_int64), ("links", ctypes.c_int64),
                ("hyperedges", ctypes.c_int64), ("n_boundaries", ctypes.c_int64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n_strips", ctypes.c_int32), ("n_blocks", ctypes.c_int32),
                ("seg_per_strip", ctypes.c_int32), ("n_segments", ctypes.c_int32),
                ("grid", ctypes.c_int32), ("kernels_per_scan", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64)]


_vp, _i32, _i64, _u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
_SIGS = {
    "ychg_last_error": (ctypes.c_char_p, []),
    "ychg_abi_version": (ctypes.c_int, []),
    "ychg_last_error_offset": (ctypes.c_int64, []),
    "ychg_pnm_info": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "ychg_load_pnm": (ctypes.c_int, [_vp, _i64, _i32, _vp, _i64]),
    "ychg_load_pnm_device": (ctypes.c_int, [_vp, _i64, _i32, _vp, _i64, _vp]),
    "ychg_scan_pnm": (ctypes.c_int, [_vp, _i64, _i32, _i32, _vp, _vp, ctypes.POINTER(Totals)]),
    "ychg_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "ychg_set_device": (ctypes.c_int, [ctypes.c_int]),
    "ychg_cut_vertex_counts": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _i32, _vp]),
    "ychg_detect_boundary_columns": (ctypes.c_int, [_vp, _i64, _vp, ctypes.POINTER(_i64)]),
    "ychg_scan_host": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _vp, _vp, ctypes.POINTER(Totals)]),
    "ychg_scan_host_sharded": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _vp, _i32, _i32, _vp, _vp,
                                              ctypes.POINTER(Totals)]),
    "ychg_build_profile_host": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _i32, _vp, _vp, _i64, ctypes.POINTER(_i64)]),
    "ychg_column_runs_host": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _vp, _i64, ctypes.POINTER(_i64)]),
    "ychg_build_profile_host_alloc": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _i32, _vp, _vp, _vp,
                                                     ctypes.POINTER(_i64)]),
    "ychg_decompose_image": (ctypes.c_int, [_vp, _i32, _i32, _i64, _i32, _i32, ctypes.POINTER(_vp)]),
    "ychg_decompose_profile": (ctypes.c_int, [_i32, _i32, _vp, _vp, _i64, ctypes.POINTER(_vp)]),
    "ychg_hypergraph_info": (ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                            ctypes.POINTER(ctypes.c_float)]),
    "ychg_hypergraph_copy": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "ychg_hypergraph_destroy": (None, [_vp]),
    "ychg_plan_create": (ctypes.c_int, [ctypes.c_int, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    "ychg_plan_create_ex": (ctypes.c_int, [ctypes.c_int, _i32, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    "ychg_plan_destroy": (None, [_vp]),
    "ychg_plan_get_info": (ctypes.c_int, [_vp, ctypes.POINTER(PlanInfo)]),
    "ychg_scan_device": (ctypes.c_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "ychg_plan_set_timing": (ctypes.c_int, [_vp, _i32]),
    "ychg_plan_last_ms": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
    "ychg_plan_debug_stamps": (ctypes.c_int, [_vp, _i32, _vp, _i32, ctypes.POINTER(_i32)]),
    "ychg_plan_debug_peek": (ctypes.c_int, [_vp, _vp, _i32]),
    "ychg_synth_device": (ctypes.c_int, [_i32, _i32, _i32, _i32, _i32, ctypes.c_double, _u64, _vp, _i64, _vp]),
    "ychg_boundary_flag_words": (_i64, [_i64]),
    "ychg_detect_boundaries_device": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp]),
    "ychg_assemble_strips_device": (ctypes.c_int, [_vp, _i32, _i32, _i32, ctypes.POINTER(_i32), _i64, _vp, _vp,
                                                   _vp, _vp, _vp, _vp]),
    "ychg_synth_device_window": (ctypes.c_int, [_i32, _i32, _i32, _i32, _i32, _i32, _i32, ctypes.c_double, _u64,
                                                _vp, _i64, _vp]),
    "ychg_device_alloc": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.POINTER(_vp)]),
    "ychg_device_free": (ctypes.c_int, [ctypes.c_int, _vp]),
    "ychg_host_alloc_pinned": (ctypes.c_int, [_i64, ctypes.POINTER(_vp)]),
    "ychg_host_free_pinned": (ctypes.c_int, [_vp]),
    "ychg_memcpy": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "ychg_memcpy_2d": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp]),
    "ychg_memset": (ctypes.c_int, [_vp, _i32, _i64, _vp]),
    "ychg_stream_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "ychg_stream_destroy": (ctypes.c_int, [_vp]),
    "ychg_stream_synchronize": (ctypes.c_int, [_vp]),
}
for _name, (_res, _args) in _SIGS.items():
    if not hasattr(_lib, _name) and os.environ.get("YCHG_LIB"):
        continue  # an older experimental build (A/B timing): only the entry points it has
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED_SYMBOLS = tuple(_SIGS)


# ---------------------------------------------------------------- errors (errors.hpp:11-40)
class Error(RuntimeError):
    """Base of everything the library raises on purpose (ychg::Error)."""


class ValidationError(Error):
    """Precondition violation (ychg::ValidationError)."""


class ParseError(Error):
    """Malformed input bytes (ychg::ParseError); `offset` is the byte offset."""

    def __init__(self, msg: str, offset: int = 0):
        super().__init__(msg)
        self.offset = offset


def _check(rc: int, what: str) -> None:
    if rc == OK:
        return
    msg = f"{what}: {_lib.ychg_last_error().decode(errors='replace')}"
    if rc == ERR_PARSE:
        off = int(_lib.ychg_last_error_offset())
        raise ParseError(f"{msg} (byte offset {off})", off)
    if rc == ERR_INVALID:
        raise ValidationError(msg)
    raise Error(msg)


def device_count() -> int:
    n = ctypes.c_int(0)
    _lib.ychg_device_count(ctypes.byref(n))
    return n.value


# ---------------------------------------------------------------- data model
class BinaryImage:
    """Bit-per-pixel raster with the reference layout (image.hpp:10-22,35-36):
    row-major, MSB-first bytes, rows of ceil(width/8) bytes, padding bits zero."""

    __slots__ = ("width", "height", "_bits")

    def __init__(self, width: int, height: int, bits: np.ndarray | None = None):
        if width < 0 or height < 0:
            raise ValidationError(f"negative dimensions {width}x{height}")
        self.width, self.height = int(width), int(height)
        stride = (self.width + 7) // 8
        if bits is None:
            self._bits = np.zeros((self.height, stride), dtype=np.uint8)
        else:
            bits = np.asarray(bits, dtype=np.uint8)
            if bits.shape != (self.height, stride):
                raise ValidationError(f"bits shape {bits.shape} != {(self.height, stride)}")
            self._bits = np.ascontiguousarray(bits)

    @property
    def row_stride(self) -> int:
        return (self.width + 7) // 8

    def bytes(self) -> np.ndarray:
        return self._bits

    def get(self, x: int, y: int) -> bool:
        return bool((self._bits[y, x >> 3] >> (7 - (x & 7))) & 1)

    def set(self, x: int, y: int, value: bool) -> None:
        m = np.uint8(0x80 >> (x & 7))
        if value:
            self._bits[y, x >> 3] |= m
        else:
            self._bits[y, x >> 3] &= np.uint8(~m & 0xFF)

    def __eq__(self, other) -> bool:
        return (isinstance(other, BinaryImage) and self.width == other.width
                and self.height == other.height and np.array_equal(self._bits, other._bits))

    def _ptr(self):
        return self._bits.ctypes.data_as(_vp) if self._bits.size else None


@dataclass(frozen=True)
class ScanStrategy:
    """runscan.hpp:26-36.  Validated, then irrelevant: every strategy runs the
    same GPU pass, so results are strategy-independent by construction."""
    kind: int = STRATEGY_SERIAL
    threads: int = 1

    @staticmethod
    def serial() -> "ScanStrategy":
        return ScanStrategy(STRATEGY_SERIAL, 1)

    @staticmethod
    def parallel(threads: int) -> "ScanStrategy":
        return ScanStrategy(STRATEGY_PARALLEL, int(threads))


@dataclass
class ScanResult:
    counts: np.ndarray
    boundaries: np.ndarray
    total_runs: int
    links: int
    hyperedges: int
    n_boundaries: int = field(default=0)


# ---------------------------------------------------------------- the runscan API
def cut_vertex_counts(image: BinaryImage, strategy: ScanStrategy = ScanStrategy.serial()) -> np.ndarray:
    """Paper §2 step 1 (runscan.cpp:122-128): runs per column, int32[width]."""
    out = np.zeros(max(image.width, 1), dtype=np.int32)
    _check(_lib.ychg_cut_vertex_counts(image._ptr(), image.width, image.height, image.row_stride,
                                       strategy.kind, strategy.threads, out.ctypes.data_as(_vp)),
           "cut_vertex_counts")
    return out[: image.width]


def detect_boundary_columns(counts) -> np.ndarray:
    """Paper §2 step 2 (runscan.cpp:145-153): ascending c with counts[c] != counts[c-1]."""
    counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int32))
    out = np.zeros(max(counts.size, 1), dtype=np.int32)
    n = _i64(0)
    _check(_lib.ychg_detect_boundary_columns(counts.ctypes.data_as(_vp) if counts.size else None,
                                             counts.size, out.ctypes.data_as(_vp), ctypes.byref(n)),
           "detect_boundary_columns")
    return out[: n.value].copy()


def scan(image: BinaryImage, with_hyperedges: bool = True) -> ScanResult:
    """Counts, boundaries and the hyperedge total from one pass over the mask.
    hyperedges == hyperedge_count(decompose(build_profile(image))) (hypergraph.cpp:192)."""
    counts = np.zeros(max(image.width, 1), dtype=np.int32)
    bounds = np.zeros(max(image.width, 1), dtype=np.int32)
    t = Totals()
    _check(_lib.ychg_scan_host(image._ptr(), image.width, image.height, image.row_stride,
                               int(with_hyperedges), counts.ctypes.data_as(_vp),
                               bounds.ctypes.data_as(_vp), ctypes.byref(t)), "scan")
    return ScanResult(counts[: image.width], bounds[: t.n_boundaries].copy(), t.total_runs,
                      t.links, t.hyperedges, t.n_boundaries)


# ---------------------------------------------------------------- PNM input (pnm.hpp, §8f row 3)
def pnm_info(data: bytes) -> tuple[int, int, int]:
    """(kind 1/2/4/5, width, height) of a PNM file's bytes (header parse only)."""
    buf = np.frombuffer(data, dtype=np.uint8)
    k, w, h = _i32(0), _i32(0), _i32(0)
    _check(_lib.ychg_pnm_info(buf.ctypes.data_as(_vp), buf.size, ctypes.byref(k), ctypes.byref(w), ctypes.byref(h)),
           "load_pnm")
    return k.value, w.value, h.value


def load_pnm(data: bytes, threshold: int = 128) -> BinaryImage:
    """load_pnm (pnm.cpp:124-153): P4 as is, P5 thresholded on the device, P1/P2 parsed."""
    buf = np.frombuffer(data, dtype=np.uint8)
    if not 0 <= threshold <= 255:
        raise ValidationError(f"load_pnm: pnm: threshold must lie in [0, 255], got {threshold}")
    _, w, h = pnm_info(data)
    img = BinaryImage(w, h)
    _check(_lib.ychg_load_pnm(buf.ctypes.data_as(_vp), buf.size, int(threshold), img._ptr(), img.row_stride),
           "load_pnm")
    return img


def save_pnm(image: BinaryImage) -> bytes:
    """save_pnm (pnm.cpp:155-163): binary P4 whose payload is the image buffer."""
    return f"P4\n{image.width} {image.height}\n".encode() + image.bytes().tobytes()


def scan_pnm(data: bytes, threshold: int = 128, with_hyperedges: bool = True) -> ScanResult:
    """scan() of a PNM file's bytes: the P4 raster goes to the device untouched, P5 is
    thresholded and packed on the device."""
    buf = np.frombuffer(data, dtype=np.uint8)
    if not 0 <= threshold <= 255:
        raise ValidationError(f"scan_pnm: pnm: threshold must lie in [0, 255], got {threshold}")
    _, w, _ = pnm_info(data)
    counts = np.zeros(max(w, 1), dtype=np.int32)
    bounds = np.zeros(max(w, 1), dtype=np.int32)
    t = Totals()
    _check(_lib.ychg_scan_pnm(buf.ctypes.data_as(_vp), buf.size, int(threshold), int(with_hyperedges),
                              counts.ctypes.data_as(_vp), bounds.ctypes.data_as(_vp), ctypes.byref(t)), "scan_pnm")
    return ScanResult(counts[:w], bounds[: t.n_boundaries].copy(), t.total_runs, t.links, t.hyperedges,
                      t.n_boundaries)


def scan_sharded(image: BinaryImage, n_parts: int, devices=None, with_hyperedges: bool = True) -> ScanResult:
    """scan() over several devices of this process: n_parts column strips (multiples of
    1024 columns, 8-column right halos) spread round-robin over `devices` (default:
    the current device), one host thread per device (ychg_scan_host_sharded)."""
    counts = np.zeros(max(image.width, 1), dtype=np.int32)
    bounds = np.zeros(max(image.width, 1), dtype=np.int32)
    t = Totals()
    devs = None if devices is None else np.ascontiguousarray(devices, dtype=np.int32)
    _check(_lib.ychg_scan_host_sharded(image._ptr(), image.width, image.height, image.row_stride, int(n_parts),
                                       devs.ctypes.data_as(_vp) if devs is not None else None,
                                       0 if devs is None else int(devs.size), int(with_hyperedges),
                                       counts.ctypes.data_as(_vp), bounds.ctypes.data_as(_vp), ctypes.byref(t)),
           "scan_sharded")
    return ScanResult(counts[: image.width], bounds[: t.n_boundaries].copy(), t.total_runs, t.links, t.hyperedges,
                      t.n_boundaries)


def hyperedge_count(image: BinaryImage) -> int:
    """hyperedge_count(decompose(build_profile(image))) without materialising runs."""
    return scan(image).hyperedges


@dataclass
class ColumnProfile:
    """runscan.hpp:40-50: per-column runs + counts.  `runs_flat` is the (n, 3) int32
    array {col, y_top, y_bot}, column-major, sorted by y_top inside a column."""
    width: int
    height: int
    counts: np.ndarray
    runs_flat: np.ndarray

    @property
    def col_off(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.counts, dtype=np.int64)])

    def runs(self, col: int) -> np.ndarray:
        o = self.col_off
        return self.runs_flat[o[col]:o[col + 1]]

    def total_runs(self) -> int:
        return int(self.counts.sum())


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


def build_profile(image: BinaryImage, strategy: ScanStrategy = ScanStrategy.serial()) -> ColumnProfile:
    """build_profile (runscan.cpp:130-143) on the GPU: count -> scan -> fill, in ONE
    library call (the run buffer is requested once the total is known)."""
    counts = np.zeros(max(image.width, 1), dtype=np.int32)
    n = _i64(0)
    holder = []

    def alloc(_ctx, n_runs):
        holder.append(np.empty((n_runs, 3), dtype=np.int32))
        return holder[-1].ctypes.data

    cb = _ALLOC_FN(alloc)
    _check(_lib.ychg_build_profile_host_alloc(image._ptr(), image.width, image.height, image.row_stride,
                                              strategy.kind, strategy.threads, counts.ctypes.data_as(_vp),
                                              ctypes.cast(cb, _vp), None, ctypes.byref(n)), "build_profile")
    runs = holder[-1] if holder else np.zeros((0, 3), dtype=np.int32)
    return ColumnProfile(image.width, image.height, counts[: image.width].copy(), runs[: n.value])


def column_runs(image: BinaryImage, col: int) -> np.ndarray:
    """column_runs (runscan.cpp:104-120): (n, 3) int32 {col, y_top, y_bot}; moves one
    byte column (O(height)) to the device, one call for columns of <= 65536 runs."""
    n = _i64(0)
    cap = max(1, min(image.height // 2 + 1, 1 << 16))
    out = np.zeros((cap, 3), dtype=np.int32)
    _check(_lib.ychg_column_runs_host(image._ptr(), image.width, image.height, image.row_stride, int(col),
                                      out.ctypes.data_as(_vp), cap, ctypes.byref(n)), "column_runs")
    if n.value > cap:
        out = np.zeros((n.value, 3), dtype=np.int32)
        _check(_lib.ychg_column_runs_host(image._ptr(), image.width, image.height, image.row_stride, int(col),
                                          out.ctypes.data_as(_vp), n.value, ctypes.byref(n)), "column_runs")
    return out[: n.value].copy()


class Hypergraph:
    """decompose's result (hypergraph.hpp:27-71) as flat arrays: `edge_runs` (n, 3)
    int32 grouped by hyperedge in canonical order, `edge_offsets` (E+1,) uint32,
    `run_to_edge` (n,) uint32 in profile order.  `device_ms` is the device time of
    the decomposition kernels."""

    def __init__(self, width: int, height: int, edge_runs: np.ndarray, edge_offsets: np.ndarray,
                 run_to_edge: np.ndarray, device_ms: float = 0.0):
        self.width, self.height = width, height
        self.edge_runs, self.edge_offsets, self.run_to_edge = edge_runs, edge_offsets, run_to_edge
        self.device_ms = device_ms

    @property
    def edge_count(self) -> int:
        return len(self.edge_offsets) - 1

    def edge(self, i: int) -> np.ndarray:
        """Runs of hyperedge i (HyperedgeView::runs)."""
        return self.edge_runs[self.edge_offsets[i]:self.edge_offsets[i + 1]]

    def all_runs(self) -> np.ndarray:
        return self.edge_runs

    def __eq__(self, other) -> bool:  # Hypergraph::operator== (hypergraph.hpp:62-65)
        return (self.width == other.width and self.height == other.height
                and np.array_equal(self.edge_runs, other.edge_runs)
                and np.array_equal(self.edge_offsets, other.edge_offsets))


class HypergraphBuffers:
    """Reusable pinned host arrays for decompose(..., out=...): the result arrays
    are copied straight into page-locked memory (full PCIe rate, no first-touch
    page faults) and returned as views -- valid until the next call that uses
    the same buffers."""

    def __init__(self, max_runs: int):
        self.capacity = int(max(max_runs, 1))
        self._ptrs = []
        self.edge_runs = self._pinned((self.capacity, 3), np.int32)
        self.edge_offsets = self._pinned((self.capacity + 1,), np.uint32)
        self.run_to_edge = self._pinned((self.capacity,), np.uint32)

    def _pinned(self, shape, dtype):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = _vp()
        _check(_lib.ychg_host_alloc_pinned(nbytes, ctypes.byref(p)), "host_alloc_pinned")
        self._ptrs.append(p.value)
        buf = (ctypes.c_uint8 * nbytes).from_address(p.value)
        return np.frombuffer(buf, dtype=dtype).reshape(shape)

    def close(self) -> None:
        for p in getattr(self, "_ptrs", []):
            if _lib is not None:
                _lib.ychg_host_free_pinned(p)
        self._ptrs = []

    __del__ = close


def _take_hypergraph(h: ctypes.c_void_p, width: int, height: int, out: "HypergraphBuffers | None" = None) -> Hypergraph:
    try:
        n, e, ms = _i64(0), _i64(0), ctypes.c_float(0)
        _check(_lib.ychg_hypergraph_info(h, ctypes.byref(n), ctypes.byref(e), ctypes.byref(ms)), "decompose")
        if out is not None and n.value <= out.capacity:
            er, eo, r2e = out.edge_runs, out.edge_offsets[: e.value + 1], out.run_to_edge
        else:
            er = np.empty((max(n.value, 1), 3), dtype=np.int32)
            eo = np.empty(e.value + 1, dtype=np.uint32)
            r2e = np.empty(max(n.value, 1), dtype=np.uint32)
        _check(_lib.ychg_hypergraph_copy(h, er.ctypes.data_as(_vp), eo.ctypes.data_as(_vp), r2e.ctypes.data_as(_vp)),
               "decompose")
        return Hypergraph(width, height, er[: n.value], eo, r2e[: n.value], float(ms.value))
    finally:
        _lib.ychg_hypergraph_destroy(h)


def decompose(source, strategy: ScanStrategy = ScanStrategy.serial(),
              out: "HypergraphBuffers | None" = None) -> Hypergraph:
    """decompose (hypergraph.cpp:94-170) on the GPU.  `source` is a ColumnProfile
    (validated like validate_profile, :62-90) or a BinaryImage (build_profile +
    decompose without leaving the device).  With `out` (HypergraphBuffers large
    enough for the run count) the result arrays are views into those pinned
    buffers; otherwise fresh arrays are allocated."""
    h = _vp()
    if isinstance(source, BinaryImage):
        _check(_lib.ychg_decompose_image(source._ptr(), source.width, source.height, source.row_stride,
                                         strategy.kind, strategy.threads, ctypes.byref(h)), "decompose")
        return _take_hypergraph(h, source.width, source.height, out)
    prof = source
    runs = np.ascontiguousarray(prof.runs_flat, dtype=np.int32).reshape(-1, 3)
    sizes = np.ascontiguousarray(prof.counts, dtype=np.int32)
    if prof.width >= 0 and sizes.shape[0] != prof.width:
        raise ValidationError(f"decompose: profile arrays do not match width {prof.width}")
    _check(_lib.ychg_decompose_profile(prof.width, prof.height, sizes.ctypes.data_as(_vp) if sizes.size else None,
                                       runs.ctypes.data_as(_vp) if runs.size else None, runs.shape[0],
                                       ctypes.byref(h)), "decompose")
    return _take_hypergraph(h, prof.width, prof.height, out)


# ---------------------------------------------------------------- device-resident plumbing
STAMP_RING = 64  # ychg_device.cuh kStampRing: scans kept in the diagnostics stamp ring


class Plan:
    """Geometry-specific launch plan + workspace on one device (ychg_plan_*)."""

    def __init__(self, width_img: int, height: int, width_cnt: int | None = None, device: int = 0,
                 latency: bool = False, sync_inputs: bool = False, skip: bool = True):
        """latency=True (YCHG_PLAN_LATENCY) sizes the launch for isolated scans (one CTA
        per SM); the default favours back-to-back scans.  sync_inputs=True (YCHG_PLAN_SYNC_INPUTS):
        the scan kernel waits for the kernel launched just before it, for images
        written by that kernel.  skip=False (YCHG_PLAN_NO_SKIP): never skip 32-row
        blocks identical to the row above (same results; A/B timing)."""
        self.device = device
        self.width_img, self.height = int(width_img), int(height)
        self.width_cnt = self.width_img if width_cnt is None else int(width_cnt)
        h = _vp()
        _check(_lib.ychg_plan_create_ex(device, self.width_img, self.width_cnt, self.height,
                                        int(bool(latency)) | 2 * int(bool(sync_inputs)) | 4 * int(not skip),
                                        ctypes.byref(h)), "plan_create")
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ychg_plan_destroy(self._h)
        self._h = None

    __del__ = close

    def info(self) -> PlanInfo:
        i = PlanInfo()
        _check(_lib.ychg_plan_get_info(self._h, ctypes.byref(i)), "plan_get_info")
        return i

    def set_timing(self, on: bool) -> None:
        _check(_lib.ychg_plan_set_timing(self._h, int(on)), "plan_set_timing")

    def last_ms(self) -> tuple[float, float]:
        a, b = ctypes.c_float(0), ctypes.c_float(0)
        _check(_lib.ychg_plan_last_ms(self._h, ctypes.byref(a), ctypes.byref(b)), "plan_last_ms")
        return a.value, b.value

    def debug_stamps(self, enable: bool = True):
        """Per-CTA %globaltimer stamps (ns) of the last STAMP_RING scans, shape (STAMP_RING, grid, 32),
        indexed by scan number % STAMP_RING; slots in ychg_scan.cu."""
        n = _i32(0)
        _check(_lib.ychg_plan_debug_stamps(self._h, int(enable), None, 0, ctypes.byref(n)), "debug_stamps")
        if not enable:
            return None
        out = np.zeros((STAMP_RING, max(n.value, 1), 32), dtype=np.uint64)
        _check(_lib.ychg_plan_debug_stamps(self._h, 1, out.ctypes.data_as(_vp), out.size, ctypes.byref(n)),
               "debug_stamps")
        return out[:, : n.value]

    def debug_peek(self):
        """The stamp ring (STAMP_RING, max(grid, n_strips), 32) read without synchronising (diagnostics)."""
        rows = max(self.info().grid, self.info().n_strips)
        out = np.zeros((STAMP_RING, rows, 32), dtype=np.uint64)
        _check(_lib.ychg_plan_debug_peek(self._h, out.ctypes.data_as(_vp), out.size), "debug_peek")
        return out

    def scan_device(self, d_bits: int, pitch: int, d_counts: int, d_flags: int, d_boundaries: int,
                    d_totals: int, stream: int = 0, with_hyperedges: bool = True) -> None:
        """Enqueue the fused scan on `stream` (raw cudaStream_t); all pointers are device addresses."""
        _check(_lib.ychg_scan_device(self._h, d_bits, int(pitch), int(with_hyperedges), d_counts, d_flags,
                                     d_boundaries, d_totals, stream or None), "scan_device")


def boundary_flag_words(n: int) -> int:
    """uint32 words of flags + scratch that detect_boundaries_device needs for n columns."""
    return int(_lib.ychg_boundary_flag_words(int(n)))


def detect_boundaries_device(d_counts: int, n: int, d_flags: int, d_boundaries: int, d_n: int,
                             stream: int = 0) -> None:
    """detect_boundary_columns (runscan.cpp:145-153) on device-resident counts (e.g. all-gathered
    from column strips), asynchronous on `stream`; *d_n (int64, device) = boundary count."""
    _check(_lib.ychg_detect_boundaries_device(d_counts, int(n), d_flags, d_boundaries, d_n, stream or None),
           "detect_boundaries_device")


def assemble_strips_device(d_gathered: int, c0: list[int], seg_stride: int, totals_off: int, d_counts: int,
                           d_flags: int, d_boundaries: int, d_n: int, d_sums: int, stream: int = 0) -> None:
    """All-gathered column strips (segment r: counts, then ychg_totals at int offset
    totals_off) -> global counts, flags, boundary list, *d_n and d_sums = (runs, links)."""
    arr = (_i32 * len(c0))(*c0)
    _check(_lib.ychg_assemble_strips_device(d_gathered, len(c0) - 1, int(seg_stride), int(totals_off), arr,
                                            int(c0[-1]), d_counts, d_flags, d_boundaries, d_n, d_sums,
                                            stream or None), "assemble_strips_device")


def pitch_for(width: int) -> int:
    """Device row pitch used by the library: ceil(width/8) rounded up to 16 B (TMA stride rule)."""
    return ((width + 7) // 8 + 15) // 16 * 16


def synth_device(pattern: str, width: int, height: int, d_bits: int, pitch: int, *, bands: int = 0,
                 cell: int = 0, density: float = 0.0, seed: int = 0, stream: int = 0,
                 x0: int = 0, win: int | None = None) -> None:
    """K0: bit-exact reference synth() (synth.cpp:38-104) written straight into device memory;
    with x0 / win only the column window [x0, x0 + win) of the width x height image
    (a multi-GPU column strip, x0 a multiple of 8)."""
    if x0 == 0 and win is None:
        _check(_lib.ychg_synth_device(PATTERNS[pattern], width, height, bands, cell, float(density),
                                      int(seed) & 0xFFFFFFFFFFFFFFFF, d_bits, int(pitch), stream or None),
               "synth_device")
        return
    win = width - x0 if win is None else int(win)
    _check(_lib.ychg_synth_device_window(PATTERNS[pattern], width, height, int(x0), win, bands, cell, float(density),
                                         int(seed) & 0xFFFFFFFFFFFFFFFF, d_bits, int(pitch), stream or None),
           "synth_device_window")


class DeviceBuffer:
    """Minimal owning device allocation (for hosts without torch)."""

    def __init__(self, nbytes: int, device: int = 0):
        self.device, self.nbytes = device, int(nbytes)
        p = _vp()
        _check(_lib.ychg_device_alloc(device, self.nbytes, ctypes.byref(p)), "device_alloc")
        self.ptr = p.value

    def close(self) -> None:
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.ychg_device_free(self.device, self.ptr)
        self.ptr = None

    __del__ = close

    def to_host(self, out: np.ndarray) -> np.ndarray:
        _check(_lib.ychg_memcpy(out.ctypes.data_as(_vp), self.ptr, out.nbytes, None), "memcpy")
        _check(_lib.ychg_stream_synchronize(None), "sync")
        return out

    def from_host(self, src: np.ndarray) -> None:
        src = np.ascontiguousarray(src)
        _check(_lib.ychg_memcpy(self.ptr, src.ctypes.data_as(_vp), src.nbytes, None), "memcpy")
        _check(_lib.ychg_stream_synchronize(None), "sync")


def synth(pattern: str, width: int, height: int, *, bands: int = 0, cell: int = 0, density: float = 0.0,
          seed: int = 0, device: int = 0) -> BinaryImage:
    """Generate a reference synthetic image on the GPU (K0) and return it on the host."""
    img = BinaryImage(width, height)
    if width == 0 or height == 0:
        synth_device(pattern, width, height, 0, max(1, pitch_for(width)), bands=bands, cell=cell,
                     density=density, seed=seed)
        return img
    pitch = pitch_for(width)
    buf = DeviceBuffer(pitch * height, device)
    try:
        synth_device(pattern, width, height, buf.ptr, pitch, bands=bands, cell=cell, density=density, seed=seed)
        dev = np.zeros((height, pitch), dtype=np.uint8)
        buf.to_host(dev)
        img._bits[:] = dev[:, : img.row_stride]
    finally:
        buf.close()
    return img


__all__ = [
    "BinaryImage", "ScanStrategy", "ScanResult", "ColumnProfile", "build_profile", "column_runs", "Error",
    "Hypergraph", "HypergraphBuffers", "decompose", "scan_sharded", "ParseError", "pnm_info", "load_pnm", "save_pnm", "scan_pnm",
    "ValidationError", "cut_vertex_counts",
    "detect_boundary_columns", "scan", "hyperedge_count", "Plan", "DeviceBuffer", "synth", "synth_device",
    "pitch_for", "device_count", "Totals", "PlanInfo", "LIB_PATH", "CXX_LIB_PATH", "EXPORTED_SYMBOLS",
]
