"""Degree separation and edge distribution, built on the GPU
(mirror of delegate_bfs.partition).

``partition_graph`` (partition.py:343-351) runs entirely in libdbfs: degree
histogram, delegate classification, Alg. 1 routing, stable per-worker CSR
construction.  The returned :class:`PartitionedGraph` owns the device
partition; its ``workers[w].nn.row_offsets`` etc. are copied to host lazily
(exactly the reference's arrays: int64 offsets, int64 nn columns, uint32
nd/dn/dd columns) for inspection and parity tests.

DPG1 files (partition.py:392-464): ``save_partitioned_graph`` writes the
device partition byte-identically to the reference's writer;
``load_partitioned_graph`` turns the files back into a device partition by
replaying each worker's CSR entries as edges through the GPU build (see its
docstring for why that reproduces the stored arrays exactly).
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .rmat import EdgeList, RmatEdgeList
from .storage import KINDS, CsrSubgraph

KIND_CODES = {"nn": 0, "nd": 1, "dn": 2, "dd": 3}
DPG_MAGIC = b"DPG1"
DPG_VERSION = 1
_DPG_HEADER = "<IQQIIqQIQ"  # version, n, m, p_rank, p_gpu, theta, d, worker, n_local


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
            _lib.release(_lib._lib.dbfs_graph_free, self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition_graph(g: EdgeList, theta: int, shape: ClusterShape, verify: bool = False,
                    ctx=None, devices="auto") -> PartitionedGraph:
    """Classification + distribution + CSR build on the GPU (partition.py:343-351).

    ``verify`` keeps the reference signature; the structural checks of
    verify_buckets are asserted by the GPU build itself (kind totals == m).

    A shape of p > 1 workers goes on p GPUs of this process when that many
    are visible and the graph has >= 2^20 vertices (``devices="auto"``; a
    list picks the GPUs for any size): worker w on GPU w, one host thread per
    GPU, the peer engine over NVLink (``group.py``).
    Otherwise -- one GPU, ``devices=None``, ``DBFS_DEVICE_GROUP=0``, or a
    torchrun rank's context -- the p workers are simulated on one device, as
    the reference simulates them in one process.
    """
    if theta < 0:
        raise ValueError("theta must be >= 0")
    if ctx is None and shape.p > 1 and not (_lib._default_ctx is not None and _lib._default_ctx.nranks > 1):
        from .group import group_for, partition_group
        grp = group_for(shape.p, devices, int(g.n))
        if grp is not None:
            pg = partition_group(g, theta, shape, grp)
            if verify and sum(pg.kind_totals.values()) != pg.m:
                raise BucketViolation("edge conservation violated")
            return pg
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


def upload_partitioned_graph(ref_pg, ctx=None, symmetric: bool = False, shape: ClusterShape | None = None,
                             theta: int | None = None) -> PartitionedGraph:
    """A partition built elsewhere -- the reference's own PartitionedGraph
    (partition.py:263-292, from its partition_graph or load_partitioned_graph)
    or any object with the same fields -- onto the device as is
    (``dbfs_graph_upload_partitioned``): no edge list, no rebuild; every row
    keeps its neighbour order.  ``symmetric`` declares that every edge's
    reverse is present (build_rmat_graph with symmetrize): it enables the
    executor's pull / counting-push substitutions, so only set it when true.
    ``shape`` / ``theta`` default to the object's ``shape`` and
    ``classification.theta``."""
    shape = shape or ref_pg.shape
    cls = ref_pg.classification
    theta = int(cls.theta if theta is None else theta)
    n, m, p = int(ref_pg.n), int(ref_pg.m), shape.p
    if len(ref_pg.workers) != p:
        raise ValueError(f"{len(ref_pg.workers)} workers for a {p}-worker shape")
    dg = np.ascontiguousarray(cls.delegate_global_ids, dtype=np.int64)
    deg = getattr(cls, "out_degree", None)
    if deg is None:  # e.g. a partition loaded from DPG1 files: degrees from the rows
        deg = np.zeros(n, dtype=np.int64)
        for w in sorted(ref_pg.workers, key=lambda x: x.index):
            for k in KINDS:
                csr = w.subgraph(k)
                lens = np.diff(np.asarray(csr.row_offsets, dtype=np.int64))
                rows = (np.arange(len(lens), dtype=np.int64) * p + w.index) if k in ("nn", "nd") else dg[:len(lens)]
                np.add.at(deg, rows, lens)
    deg = np.ascontiguousarray(deg, dtype=np.int64)
    keep, offs, cols = [], [], []
    for w in sorted(ref_pg.workers, key=lambda x: x.index):
        for k in KINDS:
            csr = w.subgraph(k)
            o = np.ascontiguousarray(csr.row_offsets, dtype=np.int64)
            c = np.ascontiguousarray(csr.col_indices, dtype=np.int64 if k == "nn" else np.uint32)
            keep += [o, c]
            offs.append(o.ctypes.data)
            cols.append(c.ctypes.data)
    ctx = ctx or _lib.default_context()
    h = _lib.vp()
    off_arr = (_lib.vp * len(offs))(*offs)
    col_arr = (_lib.vp * len(cols))(*cols)
    _lib.check(_lib.load().dbfs_graph_upload_partitioned(
        ctx.handle, n, m, theta, shape.p_rank, shape.p_gpu, len(dg), dg.ctypes.data_as(_lib.vp),
        deg.ctypes.data_as(_lib.vp), off_arr, col_arr, int(bool(symmetric)), ctypes.byref(h)), "upload_partitioned")
    del keep
    return PartitionedGraph(h, ctx, shape)


# ---------------------------------------------------------------------------
# DPG1 serialization (partition.py:380-464)
# ---------------------------------------------------------------------------

def _put_array(f, arr: np.ndarray, dtype) -> None:
    data = np.ascontiguousarray(arr, dtype=dtype)
    f.write(struct.pack("<Q", len(data)))
    f.write(data.tobytes())


def _get_array(f, dtype, name: str) -> np.ndarray:
    head = f.read(8)
    if len(head) != 8:
        raise ValueError(f"{name}: truncated file")
    (count,) = struct.unpack("<Q", head)
    item = np.dtype(dtype).itemsize
    body = f.read(count * item)
    if len(body) != count * item:
        raise ValueError(f"{name}: truncated file")
    return np.frombuffer(body, dtype=dtype).copy()


def save_partitioned_graph(pg: PartitionedGraph, directory) -> None:
    """One DPG1 file per worker, ``worker_{index:05d}.dpg`` (partition.py:392-421).

    Little-endian: magic "DPG1", then u32 version, u64 n, u64 m, u32 p_rank,
    u32 p_gpu, i64 theta, u64 d, u32 worker, u64 n_local; the nn/nd/dn/dd CSRs
    (u64-counted int64 offsets, u64-counted columns: int64 for nn, uint32
    otherwise); the delegate global ids (int64), the nd source list (int64) and
    the dn/dd source masks (np.packbits, u64-counted bytes).  The arrays come
    from the device partition (dbfs_graph_export_*); a distributed partition
    writes the workers of this rank (rank r writes worker r).
    """
    directory = os.fspath(directory)
    os.makedirs(directory, exist_ok=True)
    cls = pg.classification
    for w in pg.workers:
        path = os.path.join(directory, f"worker_{w.index:05d}.dpg")
        with open(path, "wb") as f:
            f.write(DPG_MAGIC)
            f.write(struct.pack(_DPG_HEADER, DPG_VERSION, pg.n, pg.m, pg.shape.p_rank, pg.shape.p_gpu,
                                cls.theta, cls.d, w.index, w.n_local))
            for kind in KINDS:
                csr = w.subgraph(kind)
                _put_array(f, csr.row_offsets, np.int64)
                _put_array(f, csr.col_indices, np.int64 if kind == "nn" else np.uint32)
            _put_array(f, cls.delegate_global_ids, np.int64)
            _put_array(f, w.nd_source_list, np.int64)
            _put_array(f, np.packbits(w.dn_source_mask), np.uint8)
            _put_array(f, np.packbits(w.dd_source_mask), np.uint8)


@dataclass
class _DpgWorker:
    index: int
    n_local: int
    header: tuple
    csr: dict
    del_gid: np.ndarray
    nd_sources: np.ndarray
    dn_mask: np.ndarray
    dd_mask: np.ndarray


def _read_dpg(path: str) -> _DpgWorker:
    name = os.path.basename(path)
    with open(path, "rb") as f:
        if f.read(4) != DPG_MAGIC:
            raise ValueError(f"{name}: bad magic")
        raw = f.read(struct.calcsize(_DPG_HEADER))
        if len(raw) != struct.calcsize(_DPG_HEADER):
            raise ValueError(f"{name}: truncated file")
        version, n, m, p_rank, p_gpu, theta, d, index, n_local = struct.unpack(_DPG_HEADER, raw)
        if version != DPG_VERSION:
            raise ValueError(f"{name}: unsupported version {version}")
        csr = {}
        for kind in KINDS:
            off = _get_array(f, np.int64, name)
            cols = _get_array(f, np.int64 if kind == "nn" else np.uint32, name)
            csr[kind] = CsrSubgraph(kind, off, cols)
        del_gid = _get_array(f, np.int64, name)
        nd_sources = _get_array(f, np.int64, name)
        dn_mask = np.unpackbits(_get_array(f, np.uint8, name))[:d].astype(bool)
        dd_mask = np.unpackbits(_get_array(f, np.uint8, name))[:d].astype(bool)
    return _DpgWorker(index, n_local, (n, m, p_rank, p_gpu, theta, d), csr, del_gid, nd_sources, dn_mask, dd_mask)


def _worker_edges(wf: _DpgWorker, p: int) -> tuple[np.ndarray, np.ndarray]:
    """A worker's CSR entries as global (src, dst) pairs, kinds nn, nd, dn, dd, rows
    ascending, each row's columns in stored order (partition.py:319-326 inverted)."""
    w, gid = wf.index, wf.del_gid
    srcs, dsts = [], []
    for kind in KINDS:
        c = wf.csr[kind]
        rows = np.repeat(np.arange(c.num_rows, dtype=np.int64), np.diff(c.row_offsets))
        cols = c.col_indices.astype(np.int64)
        if kind in ("nn", "nd"):
            srcs.append(rows * p + w)
        else:
            srcs.append(gid[rows])
        if kind == "nn":
            dsts.append(cols)
        elif kind == "dn":
            dsts.append(cols * p + w)
        else:
            dsts.append(gid[cols])
    return np.concatenate(srcs), np.concatenate(dsts)


def load_partitioned_graph(directory, symmetric: bool | None = None, verify: bool = False,
                           ctx=None) -> PartitionedGraph:
    """Read DPG1 worker files back into a device partition (partition.py:424-464).

    In one process with ``symmetric`` given, the files' CSR arrays are
    uploaded as they are (``upload_partitioned_graph``).  Otherwise (a
    distributed context, or ``symmetric=None``, which checks the edge
    multiset on the host) every worker's CSR entries are replayed as global (src, dst) edges --
    workers in index order, kinds nn, nd, dn, dd, rows ascending, columns in
    stored order -- and fed to the GPU build (``dbfs_graph_build_edges``) with
    the stored theta and shape.  That edge list is the partition's own edge
    multiset, so degrees, the delegate set and Alg. 1 routing are the same; the
    build's stable (worker, kind, row) grouping keeps every row's stored column
    order, so the device CSRs equal the files' arrays.  The stored d, kind
    sizes and (with ``verify``) every array are checked against the rebuilt
    partition (ValueError on a mismatch).  In a distributed context (one
    worker per rank) rank r reads and builds from ``worker_r`` only.

    ``symmetric`` declares that every edge's reverse is present (it enables the
    executor's pull substitution); None checks the edge multiset on
    the host (single-process loads only).
    """
    directory = os.fspath(directory)
    files = sorted(f for f in os.listdir(directory) if f.endswith(".dpg"))
    if not files:
        raise FileNotFoundError(f"no .dpg worker files in {directory}")
    ctx = ctx or _lib.default_context()
    if ctx.nranks > 1:
        mine = [f for f in files if f == f"worker_{ctx.rank:05d}.dpg"]
        if len(files) != ctx.nranks or not mine:
            raise ValueError(f"{directory}: a distributed load needs one worker file per rank "
                             f"({len(files)} files, {ctx.nranks} ranks)")
        files = mine
    wfs = [_read_dpg(os.path.join(directory, f)) for f in files]
    n, m, p_rank, p_gpu, theta, d = wfs[0].header
    for wf in wfs[1:]:
        if wf.header != wfs[0].header:
            raise ValueError(f"{directory}: worker headers disagree")
    shape = ClusterShape(p_rank=p_rank, p_gpu=p_gpu)
    if ctx.nranks == 1 and sorted(wf.index for wf in wfs) != list(range(shape.p)):
        raise ValueError(f"{directory}: expected workers 0..{shape.p - 1}")
    wfs.sort(key=lambda wf: wf.index)
    if ctx.nranks == 1 and symmetric is not None:
        # single process: the files' arrays go to the device as they are
        from types import SimpleNamespace
        ref = SimpleNamespace(
            shape=shape, n=n, m=m,
            classification=SimpleNamespace(theta=theta, out_degree=None, delegate_global_ids=wfs[0].del_gid),
            workers=[SimpleNamespace(index=wf.index, subgraph=(lambda k, wf=wf: wf.csr[k])) for wf in wfs])
        pg = upload_partitioned_graph(ref, ctx=ctx, symmetric=bool(symmetric))
    else:
        parts = [_worker_edges(wf, shape.p) for wf in wfs]
        src = np.concatenate([a for a, _ in parts]) if parts else np.zeros(0, np.int64)
        dst = np.concatenate([b for _, b in parts]) if parts else np.zeros(0, np.int64)
        if symmetric is None:
            symmetric = _is_symmetric(src, dst, n, ctx)
        L = _lib.load()
        h = _lib.vp()
        _lib.check(L.dbfs_graph_build_edges(ctx.handle, src.ctypes.data_as(_lib.vp), dst.ctypes.data_as(_lib.vp),
                                            len(src), int(n), int(theta), p_rank, p_gpu, ctypes.byref(h)),
                   "graph_build_edges")
        if symmetric:
            _lib.check(L.dbfs_graph_set_symmetric(h, 1))
        pg = PartitionedGraph(h, ctx, shape)
    if pg.m != m or pg.classification.d != d:
        raise ValueError(f"{directory}: rebuilt partition disagrees with the files (m {pg.m} vs {m}, "
                         f"d {pg.classification.d} vs {d})")
    for wf, wg in zip(wfs, pg.workers):
        rows, nnz = wg.sizes()
        for k, kind in enumerate(KINDS):
            c = wf.csr[kind]
            if rows[k] != c.num_rows or nnz[k] != c.num_edges:
                raise ValueError(f"worker {wf.index} {kind}: rebuilt CSR size differs from the file")
        if verify:
            for kind in KINDS:
                a, b = wf.csr[kind], wg.subgraph(kind)
                if not (np.array_equal(a.row_offsets, b.row_offsets)
                        and np.array_equal(a.col_indices, b.col_indices)):
                    raise ValueError(f"worker {wf.index} {kind}: rebuilt CSR differs from the file")
            if not (np.array_equal(wf.del_gid, pg.classification.delegate_global_ids)
                    and np.array_equal(wf.nd_sources, wg.nd_source_list)
                    and np.array_equal(wf.dn_mask, wg.dn_source_mask)
                    and np.array_equal(wf.dd_mask, wg.dd_source_mask)):
                raise ValueError(f"worker {wf.index}: rebuilt source lists differ from the file")
    return pg


def _is_symmetric(src: np.ndarray, dst: np.ndarray, n: int, ctx) -> bool:
    """Edge multiset closed under reversal.  A distributed load holds one
    worker's edges per rank, and Alg. 1 may place an nn edge and its reverse on
    different workers, so there the answer is False unless the caller declares
    the graph symmetric."""
    if n > (1 << 32) or ctx.nranks > 1:
        return False
    fwd = np.sort((src.astype(np.uint64) << np.uint64(32)) | dst.astype(np.uint64))
    rev = np.sort((dst.astype(np.uint64) << np.uint64(32)) | src.astype(np.uint64))
    return bool(np.array_equal(fwd, rev))
