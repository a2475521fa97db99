"""Degree separation and edge distribution, built on the GPU
(mirror of delegate_bfs.partition).

``partition_graph`` (partition.py:343-351) runs entirely in libdbfs: degree
histogram, delegate classification, Alg. 1 routing, stable per-worker CSR
construction.  The returned :class:`PartitionedGraph` owns the device
partition; its ``workers[w].nn.row_offsets`` etc. are copied to host lazily
(exactly the reference's arrays: int64 offsets, int64 nn columns, uint32
nd/dn/dd columns) for inspection and parity tests.  Bucket verification and
DPG1 serialization (partition.py:199-260, 392-464) are outside the hot path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .rmat import EdgeList, RmatEdgeList
from .storage import KINDS, CsrSubgraph

KIND_CODES = {"nn": 0, "nd": 1, "dn": 2, "dd": 3}


class CapacityError(OverflowError):
    """A local id does not fit in 32 bits (partition.py:34-35)."""


class BucketViolation(ValueError):
    """Structured failure from bucket verification (partition.py:38-44)."""

    def __init__(self, message, worker=None, edge=None):
        super().__init__(message)
        self.worker = worker
        self.edge = edge


@dataclass(frozen=True)
class ClusterShape:
    """partition.py:47-76."""

    p_rank: int
    p_gpu: int

    def __post_init__(self):
        if self.p_rank < 1 or self.p_gpu < 1:
            raise ValueError("p_rank and p_gpu must be positive")

    @property
    def p(self) -> int:
        return self.p_rank * self.p_gpu

    def worker_of(self, v):
        return v % self.p

    def rank_gpu(self, worker: int) -> tuple[int, int]:
        return worker % self.p_rank, worker // self.p_rank

    @classmethod
    def parse(cls, text: str) -> "ClusterShape":
        parts = [int(x) for x in text.lower().split("x")]
        if len(parts) == 3:
            nodes, ranks, gpus = parts
            return cls(p_rank=nodes * ranks, p_gpu=gpus)
        if len(parts) == 2:
            return cls(p_rank=parts[0], p_gpu=parts[1])
        raise ValueError(f"bad shape {text!r}; expected NxRxG or RxG")


class VertexClassification:
    """partition.py:79-100; arrays are fetched from the device on demand."""

    def __init__(self, pg: "PartitionedGraph", theta: int, d: int, n: int):
        self._pg = pg
        self.theta = theta
        self._d = d
        self.n = n
        self._deg = None
        self._dgids = None

    @property
    def d(self) -> int:
        return self._d

    def _fetch(self):
        if self._dgids is None:
            deg = np.empty(max(self.n, 1), dtype=np.int64)
            dg = np.empty(max(self._d, 1), dtype=np.int64)
            _lib.check(_lib.load().dbfs_graph_export_classification(
                self._pg._h, deg.ctypes.data_as(_lib.vp), dg.ctypes.data_as(_lib.vp)))
            self._deg = deg[:self.n]
            self._dgids = dg[:self._d]

    @property
    def out_degree(self) -> np.ndarray:
        self._fetch()
        return self._deg

    @property
    def delegate_global_ids(self) -> np.ndarray:
        self._fetch()
        return self._dgids

    @property
    def is_delegate(self) -> np.ndarray:
        flags = np.zeros(self.n, dtype=bool)
        flags[self.delegate_global_ids] = True
        return flags

    def delegate_id_map(self) -> np.ndarray:
        ids = np.full(self.n, -1, dtype=np.int64)
        ids[self.delegate_global_ids] = np.arange(self.d, dtype=np.int64)
        return ids


class WorkerGraph:
    """partition.py:263-278: a worker's four CSRs + backward aids (lazy host views)."""

    def __init__(self, pg: "PartitionedGraph", index: int):
        self._pg = pg
        self.index = index
        n_local = ctypes.c_int64()
        rows = (ctypes.c_int64 * 4)()
        nnz = (ctypes.c_int64 * 4)()
        nsrc = ctypes.c_int64()
        _lib.check(_lib.load().dbfs_graph_worker_info(pg._h, index, ctypes.byref(n_local), rows, nnz,
                                                      ctypes.byref(nsrc)))
        self.n_local = n_local.value
        self._rows = list(rows)
        self._nnz = list(nnz)
        self._n_nd_src = nsrc.value
        self._csr = {}
        self._src = None

    def sizes(self):
        return self._rows, self._nnz

    def subgraph(self, kind: str) -> CsrSubgraph:
        if kind not in self._csr:
            k = KIND_CODES[kind]
            off = np.empty(self._rows[k] + 1, dtype=np.int64)
            cols = np.empty(max(self._nnz[k], 1), dtype=np.int64 if kind == "nn" else np.uint32)
            _lib.check(_lib.load().dbfs_graph_export_csr(self._pg._h, self.index, k, off.ctypes.data_as(_lib.vp),
                                                         cols.ctypes.data_as(_lib.vp)))
            self._csr[kind] = CsrSubgraph(kind, off, cols[:self._nnz[k]])
        return self._csr[kind]

    nn = property(lambda self: self.subgraph("nn"))
    nd = property(lambda self: self.subgraph("nd"))
    dn = property(lambda self: self.subgraph("dn"))
    dd = property(lambda self: self.subgraph("dd"))

    def _sources(self):
        if self._src is None:
            d = self._pg.classification.d
            nd = np.empty(max(self._n_nd_src, 1), dtype=np.int64)
            dn = np.empty(max(d, 1), dtype=np.uint8)
            dd = np.empty(max(d, 1), dtype=np.uint8)
            _lib.check(_lib.load().dbfs_graph_export_sources(self._pg._h, self.index, nd.ctypes.data_as(_lib.vp),
                                                             dn.ctypes.data_as(_lib.vp), dd.ctypes.data_as(_lib.vp)))
            self._src = (nd[:self._n_nd_src], dn[:d].astype(bool), dd[:d].astype(bool))
        return self._src

    @property
    def nd_source_list(self) -> np.ndarray:
        return self._sources()[0]

    @property
    def dn_source_mask(self) -> np.ndarray:
        return self._sources()[1]

    @property
    def dd_source_mask(self) -> np.ndarray:
        return self._sources()[2]


class PartitionedGraph:
    """partition.py:281-292, backed by a device-resident dbfs_graph."""

    def __init__(self, handle, ctx, shape: ClusterShape):
        self._h = handle
        self._ctx = ctx
        self.shape = shape
        info = _lib.GraphInfoC()
        _lib.check(_lib.load().dbfs_graph_info_get(handle, ctypes.byref(info)))
        self.n = info.n
        self.m = info.m
        self.theta = info.theta
        self.kind_totals = {k: int(info.kind_totals[i]) for i, k in enumerate(KINDS)}
        self.device_bytes = info.device_bytes
        self.nranks = info.nranks
        self.rank = info.rank
        self.classification = VertexClassification(self, info.theta, info.d, info.n)
        self.workers = [WorkerGraph(self, info.first_worker + i) for i in range(info.n_local_workers)]

    @property
    def num_nn_edges(self) -> int:
        return self.kind_totals["nn"]

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.dbfs_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition_graph(g: EdgeList, theta: int, shape: ClusterShape, verify: bool = False,
                    ctx=None) -> PartitionedGraph:
    """Classification + distribution + CSR build on the GPU (partition.py:343-351).

    ``verify`` keeps the reference signature; the structural checks of
    verify_buckets are asserted by the GPU build itself (kind totals == m).
    """
    if theta < 0:
        raise ValueError("theta must be >= 0")
    ctx = ctx or _lib.default_context()
    L = _lib.load()
    h = _lib.vp()
    if isinstance(g, RmatEdgeList) and g._arrays is None:
        cp = g.params.to_c(g.randomize, g.symmetric)
        _lib.check(L.dbfs_graph_build_rmat(ctx.handle, ctypes.byref(cp), int(theta), shape.p_rank, shape.p_gpu,
                                           ctypes.byref(h)), "graph_build_rmat")
    else:
        src = np.ascontiguousarray(g.src, dtype=np.int64)
        dst = np.ascontiguousarray(g.dst, dtype=np.int64)
        if ctx.nranks > 1:  # each rank passes its contiguous slice of the edge order
            from .dist import edge_slice
            lo, hi = edge_slice(len(src), ctx.nranks, ctx.rank)
            src, dst = src[lo:hi].copy(), dst[lo:hi].copy()
        _lib.check(L.dbfs_graph_build_edges(ctx.handle, src.ctypes.data_as(_lib.vp), dst.ctypes.data_as(_lib.vp),
                                            len(src), int(g.n), int(theta), shape.p_rank, shape.p_gpu,
                                            ctypes.byref(h)), "graph_build_edges")
    if getattr(g, "symmetric", False):
        _lib.check(L.dbfs_graph_set_symmetric(h, 1))
    pg = PartitionedGraph(h, ctx, shape)
    if verify and sum(pg.kind_totals.values()) != pg.m:
        raise BucketViolation("edge conservation violated")
    return pg
