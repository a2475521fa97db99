"""Graph500-style RMAT generation on the GPU (mirror of delegate_bfs.rmat).

Same names, arguments and errors as the reference module (rmat.py:1-208).
Generation runs in libdbfs (counter-based SplitMix64 draws, bit-exact with
rmat.py:107-150).  ``build_rmat_graph`` returns an :class:`RmatEdgeList`
whose arrays are generated lazily: ``partition_graph`` builds the partition
straight on the device from the parameters, so at scale >= 24 the edge list
never crosses PCIe.  Edge-list files (rmat.py:211-286): the packed binary
"DEL1" format goes through numpy; the text format is parsed and written by
libdbfs's host code (``dbfs_edges_parse_text`` / ``dbfs_edges_write_text``)
with the reference's line rules and errors.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib

BINARY_MAGIC = b"DEL1"
DESK_SCALE_CAP = 24
DEFAULT_EDGE_FACTOR = 16
DEFAULT_QUADS = (0.57, 0.19, 0.19, 0.05)


class ResourceError(ValueError):
    """Requested instance exceeds the configured desk-scale cap (rmat.py:31-32)."""


class FormatError(ValueError):
    """Malformed edge-list file (rmat.py:35-36)."""


@dataclass(frozen=True)
class RmatParams:
    """rmat.py:39-69 (same validation; scale_cap defaults to the reference's 24)."""

    scale: int
    edge_factor: int = DEFAULT_EDGE_FACTOR
    a: float = DEFAULT_QUADS[0]
    b: float = DEFAULT_QUADS[1]
    c: float = DEFAULT_QUADS[2]
    d_quad: float = DEFAULT_QUADS[3]
    seed: int = 0
    scale_cap: int = DESK_SCALE_CAP
    # This build only: Feistel relabeling after hash_randomize_vertices.  The
    # reference hash keeps an id's low bits a function of its low bits, so the
    # owners v mod p inherit RMAT's degree skew (p=8: heaviest worker 2.75x the
    # mean edges); scrambled ids balance workers.  Off = the reference graph.
    scramble: bool = False

    def __post_init__(self):
        if self.scale < 0:
            raise ValueError(f"scale must be >= 0, got {self.scale}")
        if self.edge_factor < 1:
            raise ValueError(f"edge_factor must be >= 1, got {self.edge_factor}")
        total = self.a + self.b + self.c + self.d_quad
        if abs(total - 1.0) > 1e-9:
            raise ValueError(f"quadrant probabilities sum to {total}, expected 1")
        if self.scale > self.scale_cap:
            raise ResourceError(f"scale {self.scale} exceeds desk-scale cap {self.scale_cap}")

    @property
    def n(self) -> int:
        return 1 << self.scale

    @property
    def num_edges(self) -> int:
        return self.n * self.edge_factor

    def to_c(self, randomize=True, symmetrize=True) -> _lib.RmatParamsC:
        p = _lib.RmatParamsC()
        p.scale = self.scale
        p.randomize = int(randomize)
        p.symmetrize = int(symmetrize)
        p.scramble = int(bool(self.scramble))
        p.edge_factor = self.edge_factor
        p.a, p.b, p.c = self.a, self.b, self.c
        p.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        return p


class EdgeList:
    """Flat directed edge set with 64-bit global vertex ids (rmat.py:72-104)."""

    def __init__(self, src, dst, n: int, symmetric: bool = False):
        self._src = np.asarray(src, dtype=np.int64)
        self._dst = np.asarray(dst, dtype=np.int64)
        self.n = int(n)
        self.symmetric = symmetric
        if self._src.shape != self._dst.shape:
            raise ValueError("src/dst length mismatch")

    @property
    def src(self) -> np.ndarray:
        return self._src

    @src.setter
    def src(self, v):
        self._src = np.asarray(v, dtype=np.int64)

    @property
    def dst(self) -> np.ndarray:
        return self._dst

    @dst.setter
    def dst(self, v):
        self._dst = np.asarray(v, dtype=np.int64)

    @property
    def m(self) -> int:
        return len(self.src)

    def edge_multiset(self):
        order = np.lexsort((self.dst, self.src))
        return self.src[order], self.dst[order]

    def __eq__(self, other):
        if not isinstance(other, EdgeList):
            return NotImplemented
        return (self.n == other.n and self.m == other.m and bool(np.array_equal(self.src, other.src))
                and bool(np.array_equal(self.dst, other.dst)))


class RmatEdgeList(EdgeList):
    """An RMAT edge list described by its parameters; arrays are generated on
    the device on first access (bit-exact with build_rmat_graph)."""

    def __init__(self, params: RmatParams, randomize: bool, symmetrize_: bool):
        self.params = params
        self.randomize = randomize
        self.n = params.n
        self.symmetric = symmetrize_
        self._m = params.num_edges * (2 if symmetrize_ else 1)
        self._arrays = None

    def _materialize(self):
        if self._arrays is None:
            src, dst = _generate(self.params, 0, self._m, self.randomize, self.symmetric)
            self._arrays = (src, dst)
        return self._arrays

    @property
    def src(self):
        return self._materialize()[0]

    @property
    def dst(self):
        return self._materialize()[1]

    @property
    def m(self) -> int:
        return self._m


def _generate(params: RmatParams, begin, end, randomize, symmetrize_, ctx=None):
    ctx = ctx or _lib.default_context()
    src = np.empty(end - begin, dtype=np.int64)
    dst = np.empty(end - begin, dtype=np.int64)
    cp = params.to_c(randomize, symmetrize_)
    _lib.check(_lib.load().dbfs_rmat_generate(ctx.handle, ctypes.byref(cp), begin, end,
                                              src.ctypes.data_as(_lib.vp), dst.ctypes.data_as(_lib.vp)),
               "rmat_generate")
    return src, dst


def generate_rmat(params: RmatParams) -> EdgeList:
    """2^scale * edge_factor directed RMAT edges, generated on the GPU (rmat.py:125-150)."""
    if params.scale == 0:
        z = np.zeros(params.num_edges, dtype=np.int64)
        return EdgeList(z, z.copy(), n=params.n, symmetric=False)
    src, dst = _generate(params, 0, params.num_edges, False, False)
    return EdgeList(src, dst, n=params.n, symmetric=False)


def hash_randomize_vertices(g: EdgeList, seed: int | None) -> EdgeList:
    """Bijective relabelling mod n (rmat.py:153-182), computed on the GPU."""
    if g.n == 0 or seed is None:
        return EdgeList(g.src.copy(), g.dst.copy(), g.n, g.symmetric)
    if g.n & (g.n - 1):
        raise ValueError(f"n={g.n} is not a power of two; hashing undefined")
    ctx = _lib.default_context()
    ids = np.ascontiguousarray(np.concatenate([g.src, g.dst]), dtype=np.int64)
    out = np.empty_like(ids)
    _lib.check(_lib.load().dbfs_hash_vertices(ctx.handle, g.n, seed & 0xFFFFFFFFFFFFFFFF,
                                              ids.ctypes.data_as(_lib.vp), out.ctypes.data_as(_lib.vp),
                                              len(ids)), "hash_vertices")
    return EdgeList(out[:g.m].copy(), out[g.m:].copy(), g.n, g.symmetric)


def symmetrize(g: EdgeList) -> EdgeList:
    """Append the reverse of every edge (rmat.py:185-189)."""
    if isinstance(g, RmatEdgeList) and not g.symmetric:
        return RmatEdgeList(g.params, g.randomize, True)
    src = np.concatenate([g.src, g.dst])
    dst = np.concatenate([g.dst, g.src])
    return EdgeList(src, dst, g.n, symmetric=True)


def is_symmetric(g: EdgeList) -> bool:
    a = g.edge_multiset()
    b = EdgeList(g.dst, g.src, g.n).edge_multiset()
    return np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def build_rmat_graph(params: RmatParams, randomize: bool = True, do_symmetrize: bool = True) -> EdgeList:
    """generate -> hash-randomize -> edge-double (rmat.py:200-208), lazily on the GPU."""
    if params.scale == 0:
        g = generate_rmat(params)
        if randomize:
            g = hash_randomize_vertices(g, params.seed)
        return symmetrize(g) if do_symmetrize else g
    return RmatEdgeList(params, randomize, do_symmetrize)


def save_edge_list(g: EdgeList, path, fmt: str = "binary") -> None:
    """Write ``g`` as packed binary ("DEL1", <Q n, then <u8 (src, dst) pairs) or as
    text ("# n <n>" then "u v" lines) -- rmat.py:211-229."""
    path = os.fspath(path)
    if fmt == "binary":
        pairs = np.empty((g.m, 2), dtype="<u8")
        pairs[:, 0] = g.src
        pairs[:, 1] = g.dst
        with open(path, "wb") as f:
            f.write(BINARY_MAGIC)
            f.write(struct.pack("<Q", g.n))
            f.write(pairs.tobytes())
    elif fmt == "text":
        src = np.ascontiguousarray(g.src, dtype=np.int64)
        dst = np.ascontiguousarray(g.dst, dtype=np.int64)
        _lib.check(_lib.load().dbfs_edges_write_text(path.encode(), int(g.n), src.ctypes.data_as(_lib.vp),
                                                     dst.ctypes.data_as(_lib.vp), len(src)), "edges_write_text")
    else:
        raise ValueError(f"unknown format {fmt!r}")


def _parse_text(path: str):
    L = _lib.load()
    with open(path, "rb") as f:
        data = f.read()
    if not data:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), None
    cap = _lib.i64()
    _lib.check(L.dbfs_edges_text_capacity(data, len(data), ctypes.byref(cap)))
    src = np.empty(cap.value, dtype=np.int64)
    dst = np.empty(cap.value, dtype=np.int64)
    m, hn = _lib.i64(), _lib.i64()
    try:
        _lib.check(L.dbfs_edges_parse_text(data, len(data), cap.value, src.ctypes.data_as(_lib.vp),
                                           dst.ctypes.data_as(_lib.vp), ctypes.byref(m), ctypes.byref(hn)),
                   "edges_parse_text")
    except FormatError as exc:
        raise FormatError(f"{path}:{exc}") from None
    return src[:m.value].copy(), dst[:m.value].copy(), (hn.value if hn.value >= 0 else None)


def load_edge_list(path, fmt: str = "auto") -> EdgeList:
    """Load a text ("u v" per line, '#' comments) or packed binary edge list
    (rmat.py:232-286).  n defaults to 1 + max id; the binary header and the text
    "# n <count>" comment override it.  Errors: FormatError (truncated binary,
    malformed line "<path>:<line>: ...", id overflow, id out of range)."""
    path = os.fspath(path)
    if fmt == "auto":
        with open(path, "rb") as f:
            fmt = "binary" if f.read(4) == BINARY_MAGIC else "text"
    if fmt == "binary":
        with open(path, "rb") as f:
            magic = f.read(4)
            header_n = None
            if magic == BINARY_MAGIC:
                header_n = struct.unpack("<Q", f.read(8))[0]
                body = f.read()
            else:
                body = magic + f.read()
        if len(body) % 16:
            raise FormatError(f"{path}: truncated binary edge list")
        pairs = np.frombuffer(body, dtype="<u8").reshape(-1, 2)
        if pairs.size and pairs.max() >= np.uint64(1 << 62):
            raise FormatError(f"{path}: vertex id overflow")
        src = pairs[:, 0].astype(np.int64)
        dst = pairs[:, 1].astype(np.int64)
    elif fmt == "text":
        src, dst, header_n = _parse_text(path)
    else:
        raise ValueError(f"unknown format {fmt!r}")
    if header_n is not None:
        n = int(header_n)
    else:
        n = int(max(src.max(initial=-1), dst.max(initial=-1))) + 1
    if len(src) and (src.min() < 0 or dst.min() < 0 or src.max() >= n or dst.max() >= n):
        raise FormatError(f"{path}: vertex id out of range [0, {n})")
    return EdgeList(src, dst, n=n)
