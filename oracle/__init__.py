"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the parity oracle.

Two libraries live here, both CPU-only checkers, never the product:

* ``liboracle.so`` -- our plain-C restatement of the reference algorithm
  (``oracle/ychg_oracle.c``; every function cites the reference file:line it
  follows).
* ``_ref/libychg_ref.so`` -- the UNMODIFIED reference CPU implementation compiled
  from ``/root/reference/proj/src`` by ``oracle/Makefile`` (namespace renamed to
  ``ychg_ref``).  Built in the dev container, shipped to the GPU box as a binary.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference leg may import this package.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libychg_ref.so")

# Pattern ids in the reference enum order (synth.hpp:27-34).
FULL, EMPTY, FRAME, HBANDS, CHECKER, RANDOM = range(6)
PATTERN_IDS = {"full": FULL, "empty": EMPTY, "frame": FRAME, "hbands": HBANDS,
               "checker": CHECKER, "random": RANDOM}

_u8p = ctypes.POINTER(ctypes.c_uint8)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u32p = ctypes.POINTER(ctypes.c_uint32)


class Decomposition(tuple):
    """decompose() as flat arrays: (edge_runs (n,3) int32 in hyperedge order,
    edge_offsets (E+1,) uint32, run_to_edge (n,) uint32 in profile order) --
    the members of the reference Hypergraph (hypergraph.hpp:68-71)."""

    def __new__(cls, edge_runs, edge_offsets, run_to_edge):
        return super().__new__(cls, (edge_runs, edge_offsets, run_to_edge))

    @property
    def edge_runs(self): return self[0]

    @property
    def edge_offsets(self): return self[1]

    @property
    def run_to_edge(self): return self[2]

    @property
    def edge_count(self) -> int: return len(self[1]) - 1


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass(frozen=True)
class Spec:
    """Mirror of the reference SynthSpec (synth.hpp:38-55)."""
    pattern: int
    width: int
    height: int
    bands: int = 0
    cell: int = 0
    density: float = 0.0
    seed: int = 0

    @staticmethod
    def full(w, h): return Spec(FULL, w, h)
    @staticmethod
    def empty(w, h): return Spec(EMPTY, w, h)
    @staticmethod
    def frame(w, h): return Spec(FRAME, w, h)
    @staticmethod
    def hbands(w, h, k): return Spec(HBANDS, w, h, bands=k)
    @staticmethod
    def checker(w, h, cell): return Spec(CHECKER, w, h, cell=cell)
    @staticmethod
    def random(w, h, density, seed): return Spec(RANDOM, w, h, density=density, seed=seed)

    @property
    def stride(self) -> int:
        return (self.width + 7) // 8


class Oracle:
    """Our C restatement (oracle/ychg_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        L.yo_splitmix64_next.restype = ctypes.c_uint64
        L.yo_splitmix64_next.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        L.yo_synth.restype = ctypes.c_int
        L.yo_synth.argtypes = [ctypes.c_int] * 5 + [ctypes.c_double, ctypes.c_uint64, _u8p]
        L.yo_cut_vertex_counts.restype = None
        L.yo_cut_vertex_counts.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _i32p]
        L.yo_detect_boundary_columns.restype = ctypes.c_int64
        L.yo_detect_boundary_columns.argtypes = [_i32p, ctypes.c_int64, _i32p]
        L.yo_hyperedge_count.restype = ctypes.c_int64
        L.yo_hyperedge_count.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _i64p, _i64p]
        L.yo_pair_link_counts.restype = ctypes.c_int
        L.yo_pair_link_counts.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _i32p]
        L.yo_a7_links.restype = ctypes.c_int64
        L.yo_a7_links.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
        L.yo_profile.restype = ctypes.c_int64
        L.yo_profile.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _i32p, ctypes.c_int64, _i32p]
        L.yo_foreground_count.restype = ctypes.c_int64
        L.yo_decompose.restype = ctypes.c_int64
        L.yo_decompose.argtypes = [_i32p, _i32p, ctypes.c_int, _i32p, _u32p, _u32p]
        L.yo_foreground_count.argtypes = [_u8p, ctypes.c_int64]
        self.lib = L

    def splitmix64(self, seed: int, n: int) -> list[int]:
        st = ctypes.c_uint64(seed)
        return [self.lib.yo_splitmix64_next(ctypes.byref(st)) for _ in range(n)]

    def synth(self, spec: Spec) -> np.ndarray:
        """Packed image as a (height, stride) uint8 array (reference BinaryImage bytes)."""
        out = np.zeros((spec.height, spec.stride), dtype=np.uint8)
        rc = self.lib.yo_synth(spec.pattern, spec.width, spec.height, spec.bands, spec.cell,
                               spec.density, spec.seed, _ptr(out, _u8p))
        if rc != 0:
            raise ValueError(f"invalid synth spec {spec}")
        return out

    def counts(self, bits: np.ndarray, w: int) -> np.ndarray:
        h = bits.shape[0]
        bits = np.ascontiguousarray(bits)
        out = np.zeros(w, dtype=np.int32)
        if w > 0 and h > 0:
            self.lib.yo_cut_vertex_counts(_ptr(bits, _u8p), w, h, bits.shape[1], _ptr(out, _i32p))
        return out

    def boundaries(self, counts: np.ndarray) -> np.ndarray:
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        out = np.zeros(max(1, counts.size), dtype=np.int32)
        n = self.lib.yo_detect_boundary_columns(_ptr(counts, _i32p), counts.size, _ptr(out, _i32p))
        return out[:n].copy()

    def hyperedges(self, bits: np.ndarray, w: int) -> tuple[int, int, int]:
        """(hyperedges, total_runs, links)."""
        h = bits.shape[0]
        bits = np.ascontiguousarray(bits)
        tr, lk = ctypes.c_int64(0), ctypes.c_int64(0)
        stride = bits.shape[1] if bits.ndim == 2 and bits.shape[1] > 0 else 1
        he = self.lib.yo_hyperedge_count(_ptr(bits, _u8p), w, h, stride,
                                         ctypes.byref(tr), ctypes.byref(lk))
        if he < 0:
            raise MemoryError("oracle hyperedge_count allocation failed")
        return int(he), int(tr.value), int(lk.value)

    def profile(self, bits: np.ndarray, w: int) -> np.ndarray:
        """(n, 3) int32 runs {col, y_top, y_bot}, column-major (build_profile flattened)."""
        h = bits.shape[0]
        if w == 0 or h == 0:
            return np.zeros((0, 3), dtype=np.int32)
        bits = np.ascontiguousarray(bits)
        n = self.lib.yo_profile(_ptr(bits, _u8p), w, h, bits.shape[1], None, 0, None)
        out = np.zeros((max(n, 1), 3), dtype=np.int32)
        self.lib.yo_profile(_ptr(bits, _u8p), w, h, bits.shape[1], _ptr(out, _i32p), n, None)
        return out[:n]

    def decompose_profile(self, runs: np.ndarray, counts: np.ndarray) -> Decomposition:
        """decompose (hypergraph.cpp:94-170) of a flat column-major profile."""
        runs = np.ascontiguousarray(runs, dtype=np.int32).reshape(-1, 3)
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        n = runs.shape[0]
        er = np.zeros((max(n, 1), 3), dtype=np.int32)
        eo = np.zeros(n + 1, dtype=np.uint32)
        r2e = np.zeros(max(n, 1), dtype=np.uint32)
        e = self.lib.yo_decompose(_ptr(runs, _i32p) if n else None, _ptr(counts, _i32p), len(counts),
                                  _ptr(er, _i32p), _ptr(eo, _u32p), _ptr(r2e, _u32p))
        if e < 0:
            raise MemoryError("oracle decompose allocation failed")
        return Decomposition(er[:n], eo[: e + 1], r2e[:n])

    def decompose(self, bits: np.ndarray, w: int) -> Decomposition:
        h = bits.shape[0]
        runs = self.profile(bits, w)
        counts = np.bincount(runs[:, 0], minlength=w).astype(np.int32) if len(runs) else np.zeros(w, np.int32)
        return self.decompose_profile(runs, counts)

    def a7_links(self, bits: np.ndarray, w: int) -> int:
        """Link total by the streaming a7 rule (yo_a7_links, OpenMP over column pairs):
        independent of decompose's run lists, so it reaches 65536^2."""
        h = bits.shape[0]
        if w < 2 or h == 0:
            return 0
        bits = np.ascontiguousarray(bits)
        return int(self.lib.yo_a7_links(_ptr(bits, _u8p), w, h, bits.shape[1]))

    def pair_links(self, bits: np.ndarray, w: int) -> np.ndarray:
        h = bits.shape[0]
        out = np.zeros(max(w - 1, 0), dtype=np.int32)
        if w >= 2 and h > 0:
            bits = np.ascontiguousarray(bits)
            self.lib.yo_pair_link_counts(_ptr(bits, _u8p), w, h, bits.shape[1], _ptr(out, _i32p))
        return out


class Reference:
    """The unmodified reference, compiled by oracle/Makefile into oracle/_ref/."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it with `make -C oracle ref` "
                                    "in a container that has /root/reference")
        L = ctypes.CDLL(path)
        L.yr_last_error.restype = ctypes.c_char_p
        L.yr_synth.restype = ctypes.c_int
        L.yr_synth.argtypes = [ctypes.c_int] * 5 + [ctypes.c_double, ctypes.c_uint64, _u8p]
        L.yr_splitmix64.restype = ctypes.c_uint64
        L.yr_splitmix64.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.yr_image_create.restype = ctypes.c_void_p
        L.yr_image_create.argtypes = [_u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
        L.yr_image_synth.restype = ctypes.c_void_p
        L.yr_image_synth.argtypes = [ctypes.c_int] * 5 + [ctypes.c_double, ctypes.c_uint64]
        L.yr_image_destroy.restype = None
        L.yr_image_destroy.argtypes = [ctypes.c_void_p]
        L.yr_image_bytes.restype = ctypes.c_void_p
        L.yr_image_bytes.argtypes = [ctypes.c_void_p]
        L.yr_counts.restype = ctypes.c_int
        L.yr_counts.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _i32p]
        L.yr_column_runs.restype = ctypes.c_int64
        L.yr_column_runs.argtypes = [ctypes.c_void_p, ctypes.c_int, _i32p, ctypes.c_int64]
        L.yr_boundaries.restype = ctypes.c_int64
        L.yr_boundaries.argtypes = [_i32p, ctypes.c_int64, _i32p]
        L.yr_hyperedges.restype = ctypes.c_int64
        L.yr_hyperedges.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.yr_profile.restype = ctypes.c_int64
        L.yr_profile.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _i32p, ctypes.c_int64]
        L.yr_load_pnm.restype = ctypes.c_int
        L.yr_load_pnm.argtypes = [_u8p, ctypes.c_int64, ctypes.c_int, _u8p, ctypes.c_int64, _i32p, _i32p, _i64p]
        L.yr_decompose.restype = ctypes.c_int64
        L.yr_decompose.argtypes = [ctypes.c_void_p, _i32p, ctypes.c_int64, _u32p, ctypes.c_int64, _u32p, _i64p]
        L.yr_time_path.restype = ctypes.c_int
        L.yr_time_path.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, _i64p, _i32p, _i64p, _i64p]
        self.lib = L

    def last_error(self) -> str:
        return self.lib.yr_last_error().decode()

    def synth(self, spec: Spec) -> np.ndarray:
        out = np.zeros((spec.height, spec.stride), dtype=np.uint8)
        rc = self.lib.yr_synth(spec.pattern, spec.width, spec.height, spec.bands, spec.cell,
                               spec.density, spec.seed, _ptr(out, _u8p))
        if rc != 0:
            raise ValueError(self.last_error())
        return out

    def load_pnm(self, data: bytes, threshold: int = 128):
        """load_pnm by the reference: ("ok", bits (h, stride) uint8, w, h) or
        ("parse", message, offset) / ("invalid", message) / ("error", message)."""
        buf = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        w, h, off = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int64(0)
        rc = self.lib.yr_load_pnm(_ptr(buf, _u8p), len(data), threshold, None, 0, ctypes.byref(w), ctypes.byref(h),
                                  ctypes.byref(off))
        if rc == -4:
            return ("parse", self.last_error(), off.value)
        if rc == -1:
            return ("invalid", self.last_error())
        if rc != 0:
            return ("error", self.last_error())
        stride = (w.value + 7) // 8
        out = np.zeros((max(h.value, 1), max(stride, 1)), dtype=np.uint8)
        self.lib.yr_load_pnm(_ptr(buf, _u8p), len(data), threshold, _ptr(out, _u8p), out.size, ctypes.byref(w),
                             ctypes.byref(h), ctypes.byref(off))
        return ("ok", out[: h.value, :stride], w.value, h.value)

    def image(self, bits: np.ndarray, w: int) -> "RefImage":
        bits = np.ascontiguousarray(bits)
        h = bits.shape[0]
        stride = bits.shape[1] if h > 0 else 0
        handle = self.lib.yr_image_create(_ptr(bits, _u8p) if bits.size else None, w, h, stride)
        if not handle:
            raise RuntimeError(self.last_error())
        return RefImage(self, handle, w, h)

    def image_synth(self, spec: Spec) -> "RefImage":
        handle = self.lib.yr_image_synth(spec.pattern, spec.width, spec.height, spec.bands,
                                         spec.cell, spec.density, spec.seed)
        if not handle:
            raise ValueError(self.last_error())
        return RefImage(self, handle, spec.width, spec.height)

    def boundaries(self, counts: np.ndarray) -> np.ndarray:
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        out = np.zeros(max(1, counts.size), dtype=np.int32)
        n = self.lib.yr_boundaries(_ptr(counts, _i32p), counts.size, _ptr(out, _i32p))
        return out[:n].copy()


class RefImage:
    def __init__(self, ref: Reference, handle, w: int, h: int):
        self.ref, self.handle, self.width, self.height = ref, handle, w, h

    def __del__(self):
        if getattr(self, "handle", None):
            self.ref.lib.yr_image_destroy(self.handle)
            self.handle = None

    def bytes(self) -> np.ndarray:
        stride = (self.width + 7) // 8
        n = stride * self.height
        if n == 0:
            return np.zeros((self.height, stride), dtype=np.uint8)
        p = self.ref.lib.yr_image_bytes(self.handle)
        return np.ctypeslib.as_array(ctypes.cast(p, _u8p), shape=(n,)).reshape(
            self.height, stride).copy()

    def counts(self, kind: int = 0, threads: int = 1) -> np.ndarray:
        out = np.zeros(max(1, self.width), dtype=np.int32)
        rc = self.ref.lib.yr_counts(self.handle, kind, threads, _ptr(out, _i32p))
        if rc == -1:
            raise ValueError(self.ref.last_error())
        if rc != 0:
            raise RuntimeError(self.ref.last_error())
        return out[: self.width].copy()

    def profile(self, kind: int = 0, threads: int = 1) -> np.ndarray:
        n = self.ref.lib.yr_profile(self.handle, kind, threads, None, 0)
        if n < 0:
            raise RuntimeError(self.ref.last_error())
        out = np.zeros((max(n, 1), 3), dtype=np.int32)
        self.ref.lib.yr_profile(self.handle, kind, threads, _ptr(out, _i32p), n)
        return out[:n]

    def column_runs(self, col: int) -> np.ndarray:
        """column_runs(img, col) by the reference: (n, 3) int32; ValueError(what()) when it throws."""
        n = self.ref.lib.yr_column_runs(self.handle, int(col), None, 0)
        if n < 0:
            raise ValueError(self.ref.last_error())
        out = np.zeros((max(n, 1), 3), dtype=np.int32)
        self.ref.lib.yr_column_runs(self.handle, int(col), _ptr(out, _i32p), n)
        return out[:n]

    def hyperedges(self, kind: int = 0, threads: int = 1) -> int:
        v = self.ref.lib.yr_hyperedges(self.handle, kind, threads)
        if v < 0:
            raise RuntimeError(self.ref.last_error())
        return int(v)

    def decompose(self) -> Decomposition:
        """decompose(build_profile(img)) by the reference (hypergraph.cpp:94-170)."""
        n = ctypes.c_int64(0)
        e = self.ref.lib.yr_decompose(self.handle, None, 0, None, 0, None, ctypes.byref(n))
        if e < 0:
            raise RuntimeError(self.ref.last_error())
        nr = n.value
        er = np.zeros((max(nr, 1), 3), dtype=np.int32)
        eo = np.zeros(e + 1, dtype=np.uint32)
        r2e = np.zeros(max(nr, 1), dtype=np.uint32)
        self.ref.lib.yr_decompose(self.handle, _ptr(er, _i32p), nr, _ptr(eo, _u32p), e + 1, _ptr(r2e, _u32p),
                                  ctypes.byref(n))
        return Decomposition(er[:nr], eo, r2e[:nr])

    def time_path(self, kind: int, threads: int, warmup: int, reps: int,
                  with_hyperedges: bool) -> dict:
        ns = np.zeros(reps, dtype=np.int64)
        counts = np.zeros(max(1, self.width), dtype=np.int32)
        nb, he = ctypes.c_int64(0), ctypes.c_int64(0)
        rc = self.ref.lib.yr_time_path(self.handle, kind, threads, warmup, reps,
                                       int(with_hyperedges), _ptr(ns, _i64p),
                                       _ptr(counts, _i32p), ctypes.byref(nb), ctypes.byref(he))
        if rc != 0:
            raise RuntimeError(self.ref.last_error())
        return {"ns": ns.tolist(), "counts": counts[: self.width], "n_boundaries": int(nb.value),
                "hyperedges": int(he.value)}


def random_corpus(count: int) -> list[tuple[str, Spec]]:
    """corpus.hpp:22-35: W,H in [1,64] from Splitmix64(9000+i), densities cycle, seed 40000+i."""
    dens = [0.1, 0.3, 0.5, 0.7, 0.9]
    out = []
    for i in range(count):
        st = [9000 + i]

        def nxt():
            st[0] = (st[0] + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
            z = st[0]
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
            return z ^ (z >> 31)

        w = 1 + nxt() % 64
        h = 1 + nxt() % 64
        out.append((f"random#{i}", Spec.random(w, h, dens[i % 5], 40000 + i)))
    return out


def pattern_corpus() -> list[tuple[str, Spec]]:
    """corpus.hpp:38-58: every pattern at 19 geometries."""
    geoms = [(1, 1), (2, 2), (3, 3), (4, 4), (5, 5), (6, 6), (7, 7), (8, 8), (12, 12), (16, 16),
             (24, 24), (31, 31), (32, 32), (8, 3), (3, 8), (32, 5), (5, 32), (1, 7), (7, 1)]
    out = []
    for w, h in geoms:
        d = f"{w}x{h}"
        out.append((f"full {d}", Spec.full(w, h)))
        out.append((f"empty {d}", Spec.empty(w, h)))
        out.append((f"frame {d}", Spec.frame(w, h)))
        for k in range(1, 6):
            if k <= h // 2:
                out.append((f"hbands({k}) {d}", Spec.hbands(w, h, k)))
        for cell in range(1, 4):
            out.append((f"checker({cell}) {d}", Spec.checker(w, h, cell)))
    return out


def full_corpus() -> list[tuple[str, Spec]]:
    """corpus.hpp:61-66: 1000 random + patterns = 1170 images."""
    return random_corpus(1000) + pattern_corpus()


def branch_example() -> np.ndarray:
    """corpus.hpp:70-75: 2x7, col 0 runs [0,1],[3,6]; col 1 runs [0,4],[6,6]."""
    img = np.zeros((7, 1), dtype=np.uint8)
    for y in (0, 1, 3, 4, 5, 6):
        img[y, 0] |= 0x80
    for y in (0, 1, 2, 3, 4, 6):
        img[y, 0] |= 0x40
    return img


def a7_links(bits: np.ndarray, w: int) -> int:
    """Streaming restatement of the link count, vectorised over
    column pairs with numpy.  Used to cross-check the per-row rule the GPU kernel
    implements against the decompose() restatement above."""
    h = bits.shape[0]
    if w < 2 or h == 0:
        return 0
    px = np.unpackbits(bits, axis=1)[:, :w].astype(bool)  # (h, w), MSB-first
    a_all, b_all = px[:, :-1], px[:, 1:]
    npairs = w - 1
    n = np.zeros(npairs, dtype=np.int64)  # runs in the open component (saturating at 3)
    pa = np.zeros(npairs, dtype=bool)
    pb = np.zeros(npairs, dtype=bool)
    links = 0
    for y in range(h + 1):
        if y < h:
            a, b = a_all[y], b_all[y]
        else:
            a = b = np.zeros(npairs, dtype=bool)
        cont = (a & pa) | (b & pb)
        ended = ~cont & (pa | pb)
        links += int(np.count_nonzero(ended & (n == 2)))
        new = (a & ~pa).astype(np.int64) + (b & ~pb).astype(np.int64)
        n = np.where(cont, np.minimum(n + new, 3), new)
        pa, pb = a, b
    return links
