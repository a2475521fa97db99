"""CPU parity oracle for the delegate-BFS hot path -- TEST INFRASTRUCTURE ONLY.

This package wraps ``oracle/dbfs_oracle.c``, a C restatement of the reference
package ``delegate_bfs`` (rmat.py, partition.py, engine.py, traversal.py,
comm.py; see the file header for line-level citations).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may import
it, and only as the checker.  The product (``paper_1803_03922_b200``) never
imports it and has no CPU fallback.

The oracle is pinned against the reference by ``tests/golden`` (fixtures made
by ``tests/golden/make_golden.py`` from the reference itself) and, when
``/root/reference`` exists, by live comparisons in ``tests/``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
KINDS = ("nn", "nd", "dn", "dd")
DO_KINDS = ("dd", "dn", "nd")
_lib = None

i64 = ctypes.c_int64
u64 = ctypes.c_uint64
c_int = ctypes.c_int
c_double = ctypes.c_double
vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile liboracle.so in place (gcc, pthreads)."""
    src = os.path.join(_HERE, "dbfs_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
    return _LIB_PATH


class OrcOpts(ctypes.Structure):
    _fields_ = [("mode", c_int), ("source", i64), ("f0", c_double * 4), ("f1", c_double * 4),
                ("allow_switch_back", c_int), ("local_all2all", c_int), ("uniquify", c_int)]


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = ctypes.CDLL(_LIB_PATH)
    sig = {
        "orc_rmat_edges": (c_int, [c_int, i64, c_double, c_double, c_double, u64, c_int, c_int, i64, i64, vp, vp]),
        "orc_hash_vertices": (c_int, [i64, u64, vp, vp, i64]),
        "orc_rmat_summary": (c_int, [c_int, i64, c_double, c_double, c_double, u64, c_int, i64, vp,
                                     ctypes.POINTER(i64), vp]),
        "orc_partition": (c_int, [vp, vp, i64, i64, i64, c_int, c_int, ctypes.POINTER(vp)]),
        "orc_partition_rmat": (c_int, [c_int, i64, c_double, c_double, c_double, u64, i64, c_int, c_int, ctypes.POINTER(vp)]),
        "orc_partition_rmat_flags": (c_int, [c_int, i64, c_double, c_double, c_double, u64, c_int, i64, c_int, c_int,
                                             ctypes.POINTER(vp)]),
        "orc_graph_free": (None, [vp]),
        "orc_graph_new": (vp, [i64, i64, i64, c_int, c_int, i64, vp]),
        "orc_graph_set_csr": (c_int, [vp, c_int, c_int, i64, vp, vp]),
        "orc_graph_finalize": (c_int, [vp]),
        "orc_graph_n": (i64, [vp]), "orc_graph_m": (i64, [vp]), "orc_graph_d": (i64, [vp]),
        "orc_graph_p": (c_int, [vp]), "orc_graph_kind_total": (i64, [vp, c_int]),
        "orc_graph_degrees": (vp, [vp]), "orc_graph_delegates": (vp, [vp]),
        "orc_graph_n_local": (i64, [vp, c_int]),
        "orc_graph_csr_rows": (i64, [vp, c_int, c_int]), "orc_graph_csr_nnz": (i64, [vp, c_int, c_int]),
        "orc_graph_csr_off": (vp, [vp, c_int, c_int]), "orc_graph_csr_cols": (vp, [vp, c_int, c_int]),
        "orc_graph_n_nd_src": (i64, [vp, c_int]), "orc_graph_nd_src": (vp, [vp, c_int]),
        "orc_graph_dn_mask": (vp, [vp, c_int]), "orc_graph_dd_mask": (vp, [vp, c_int]),
        "orc_run_bfs": (c_int, [vp, ctypes.POINTER(OrcOpts), ctypes.POINTER(vp)]),
        "orc_run_free": (None, [vp]),
        "orc_run_levels": (vp, [vp]), "orc_run_iterations": (i64, [vp]),
        "orc_run_insp": (i64, [vp, c_int, c_int]), "orc_run_b_measured": (c_double, [vp]),
        "orc_run_dirs": (vp, [vp]), "orc_run_it_insp": (vp, [vp]), "orc_run_it_fv": (vp, [vp]),
        "orc_run_it_bv": (vp, [vp]), "orc_run_mask_bytes": (vp, [vp]),
        "orc_run_normal_bytes": (vp, [vp]), "orc_run_messages": (vp, [vp]), "orc_run_pairs": (vp, [vp]),
        "orc_bv": (c_double, [i64, i64, i64]),
        "orc_decide": (c_int, [c_int, i64, c_double, c_double, c_double, c_int]),
        "orc_bfs_levels_edges": (c_int, [vp, vp, i64, i64, i64, vp]),
        "orc_min_parents": (c_int, [vp, vp, i64, i64, i64, vp, vp]),
        "orc_validate": (c_int, [vp, vp, i64, i64, i64, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class OracleError(RuntimeError):
    pass


_ERRS = {1: ValueError, 2: ValueError, 3: OverflowError, 4: MemoryError}


def _check(rc, what):
    if rc:
        raise _ERRS.get(rc, OracleError)(f"oracle {what} failed (code {rc})")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(vp)


def _view(ptr, count, dtype):
    if count == 0:
        return np.empty(0, dtype=dtype)
    buf = (ctypes.c_char * (count * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count).copy()


# ---------------------------------------------------------------- generation

def rmat_edges(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=0, randomize=True,
               symmetrize=True, begin=0, end=None, scramble=False):
    """Edges [begin, end) of build_rmat_graph (rmat.py:125-208); ``scramble``
    adds this build's Feistel relabeling after the reference hash."""
    m0 = (1 << scale) * edge_factor
    m = 2 * m0 if symmetrize else m0
    end = m if end is None else end
    src = np.empty(end - begin, dtype=np.int64)
    dst = np.empty(end - begin, dtype=np.int64)
    _check(lib().orc_rmat_edges(scale, edge_factor, a, b, c, seed & (2**64 - 1),
                                int(bool(randomize)) | (2 if scramble else 0),
                                int(symmetrize), begin, end, _ptr(src), _ptr(dst)), "rmat")
    return src, dst


def rmat_summary(scale, theta, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=0, scramble=False):
    """(out-degree uint32[n], d, kind totals) of build_rmat_graph(params) with
    threshold theta, streamed from the counter-based generator (no edge list is
    stored, so scales 26-30 fit the host): partition.py:103-117 and the kind
    totals of partition.py:312-318."""
    n = 1 << scale
    deg = np.empty(n, dtype=np.uint32)
    d = i64()
    kinds = np.zeros(4, dtype=np.int64)
    _check(lib().orc_rmat_summary(scale, edge_factor, a, b, c, seed & (2**64 - 1), 3 if scramble else 1, theta,
                                  _ptr(deg), ctypes.byref(d), _ptr(kinds)), "rmat_summary")
    return deg, int(d.value), {k: int(kinds[i]) for i, k in enumerate(KINDS)}


def hash_vertices(n, seed, ids):
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty_like(ids)
    _check(lib().orc_hash_vertices(n, seed & (2**64 - 1), _ptr(ids), _ptr(out), len(ids)), "hash")
    return out


# ----------------------------------------------------------------- partition

class OracleCsr:
    def __init__(self, kind, row_offsets, col_indices):
        self.kind, self.row_offsets, self.col_indices = kind, row_offsets, col_indices


class OracleWorker:
    pass


class OracleGraph:
    """Partitioned graph with the reference PartitionedGraph's fields."""

    def __init__(self, handle, load_arrays=True):
        self._h = handle
        L = lib()
        self.n = L.orc_graph_n(handle)
        self.m = L.orc_graph_m(handle)
        self.d = L.orc_graph_d(handle)
        self.p = L.orc_graph_p(handle)
        self.kind_totals = {k: L.orc_graph_kind_total(handle, i) for i, k in enumerate(KINDS)}
        self.workers = []
        if not load_arrays:
            return
        self.degrees = _view(L.orc_graph_degrees(handle), self.n, np.int64)
        self.delegate_global_ids = _view(L.orc_graph_delegates(handle), self.d, np.int64)
        for w in range(self.p):
            W = OracleWorker()
            W.index = w
            W.n_local = L.orc_graph_n_local(handle, w)
            for ki, k in enumerate(KINDS):
                rows = L.orc_graph_csr_rows(handle, w, ki)
                nnz = L.orc_graph_csr_nnz(handle, w, ki)
                off = _view(L.orc_graph_csr_off(handle, w, ki), rows + 1, np.int64)
                cols = _view(L.orc_graph_csr_cols(handle, w, ki), nnz, np.int64 if k == "nn" else np.uint32)
                setattr(W, k, OracleCsr(k, off, cols))
            W.nd_source_list = _view(L.orc_graph_nd_src(handle, w), L.orc_graph_n_nd_src(handle, w), np.int64)
            W.dn_source_mask = _view(L.orc_graph_dn_mask(handle, w), self.d, np.uint8).astype(bool)
            W.dd_source_mask = _view(L.orc_graph_dd_mask(handle, w), self.d, np.uint8).astype(bool)
            self.workers.append(W)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_graph_free(self._h)
            self._h = None


def partition(src, dst, n, theta, p_rank=1, p_gpu=1) -> OracleGraph:
    """partition_graph (partition.py:343-351)."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    h = vp()
    _check(lib().orc_partition(_ptr(src), _ptr(dst), len(src), n, theta, p_rank, p_gpu,
                               ctypes.byref(h)), "partition")
    return OracleGraph(h)


def partition_rmat(scale, theta, p_rank=1, p_gpu=1, edge_factor=16, a=0.57, b=0.19, c=0.19,
                   seed=0, load_arrays=True, scramble=False) -> OracleGraph:
    h = vp()
    _check(lib().orc_partition_rmat_flags(scale, edge_factor, a, b, c, seed & (2**64 - 1), 3 if scramble else 1, theta,
                                    p_rank, p_gpu, ctypes.byref(h)), "partition_rmat")
    return OracleGraph(h, load_arrays=load_arrays)


def from_partition(pg) -> OracleGraph:
    """Oracle graph over an existing partition object exposing the reference
    PartitionedGraph fields (e.g. the GPU one, exported to host)."""
    L = lib()
    dg = np.ascontiguousarray(pg.classification.delegate_global_ids, dtype=np.int64)
    h = L.orc_graph_new(pg.n, pg.m, int(pg.classification.theta), pg.shape.p_rank, pg.shape.p_gpu,
                        int(pg.classification.d), _ptr(dg))
    for w in pg.workers:
        for ki, k in enumerate(KINDS):
            csr = w.subgraph(k)
            off = np.ascontiguousarray(csr.row_offsets, dtype=np.int64)
            cols = np.ascontiguousarray(csr.col_indices, dtype=np.int64 if k == "nn" else np.uint32)
            _check(L.orc_graph_set_csr(h, w.index, ki, len(off) - 1, _ptr(off), _ptr(cols)), "set_csr")
    L.orc_graph_finalize(h)
    return OracleGraph(vp(h), load_arrays=False)


# ----------------------------------------------------------------------- BFS

_DEF_F0 = {"dd": 0.5, "dn": 0.05, "nd": 1e-7}
_DEF_F1 = {"dd": 0.0, "dn": 0.0, "nd": 0.0}


def run_bfs(g: OracleGraph, source, mode="dobfs", factor0=None, factor1=None,
            allow_switch_back=True, local_all2all=False, uniquify=False) -> dict:
    """run_bfs (engine.py:98-330); returns BfsRun.to_dict() fields + levels."""
    f0 = dict(_DEF_F0, **(factor0 or {}))
    f1 = dict(_DEF_F1, **(factor1 or {}))
    o = OrcOpts()
    o.mode = {"bfs": 0, "dobfs": 1}[mode]
    o.source = int(source)
    for i, k in enumerate(KINDS):
        o.f0[i] = float(f0.get(k, 0.0))
        o.f1[i] = float(f1.get(k, 0.0))
    o.allow_switch_back = int(allow_switch_back)
    o.local_all2all = int(local_all2all)
    o.uniquify = int(uniquify)
    L = lib()
    h = vp()
    _check(L.orc_run_bfs(g._h, ctypes.byref(o), ctypes.byref(h)), "run_bfs")
    try:
        it = L.orc_run_iterations(h)
        p = g.p
        levels = _view(L.orc_run_levels(h), g.n, np.int32)
        dirs = _view(L.orc_run_dirs(h), it * p * 4, np.int8).reshape(it, p, 4)
        ins = _view(L.orc_run_it_insp(h), it * 4, np.int64).reshape(it, 4)
        fv = _view(L.orc_run_it_fv(h), it * 4, np.int64).reshape(it, 4)
        bv = _view(L.orc_run_it_bv(h), it * p * 4, np.float64).reshape(it, p, 4)
        mb = _view(L.orc_run_mask_bytes(h), it, np.float64)
        nb = _view(L.orc_run_normal_bytes(h), it, np.int64)
        msg = _view(L.orc_run_messages(h), it, np.int64)
        pairs = _view(L.orc_run_pairs(h), it, np.int64)
        per_it = []
        for i in range(it):
            per_it.append({
                "iteration": i,
                "directions": {k: ["forward" if dirs[i, w, ki] == 0 else "backward" for w in range(p)]
                               for ki, k in enumerate(KINDS)},
                "inspections": {k: int(ins[i, ki]) for ki, k in enumerate(KINDS)},
                "fv": {k: int(fv[i, ki]) for ki, k in enumerate(KINDS)},
                "bv": {k: [None if not math.isfinite(bv[i, w, KINDS.index(k)]) else float(bv[i, w, KINDS.index(k)])
                           for w in range(p)] for k in DO_KINDS},
                "mask_bytes": float(mb[i]),
                "normal_bytes": int(nb[i]),
            })
        insp = {k: {"forward": L.orc_run_insp(h, ki, 0), "backward": L.orc_run_insp(h, ki, 1)}
                for ki, k in enumerate(KINDS)}
        comm = {
            "mask_bytes": [float(x) for x in mb],
            "normal_bytes": [int(x) for x in nb],
            "message_count": [int(x) for x in msg],
            "pair_count": [int(x) for x in pairs],
        }
        comm["total_mask_bytes"] = sum(comm["mask_bytes"])
        comm["total_normal_bytes"] = sum(comm["normal_bytes"])
        comm["s_prime"] = sum(1 for b in comm["mask_bytes"] if b > 0)
        return {
            "levels": levels,
            "iterations": int(it),
            "per_iteration": per_it,
            "inspections": insp,
            "total_inspections": sum(v["forward"] + v["backward"] for v in insp.values()),
            "comm": comm,
            "b_measured": L.orc_run_b_measured(h),
            "levels_digest": levels_digest(levels),
        }
    finally:
        L.orc_run_free(h)


def levels_digest(levels) -> str:
    """engine.py:81-83."""
    import hashlib
    data = np.ascontiguousarray(levels, dtype="<i4").tobytes()
    return hashlib.blake2b(data, digest_size=8).hexdigest()


def bv(u, q, s):
    return lib().orc_bv(u, q, s)


def decide(direction, fv, bv_value, f0, f1, allow_back=True):
    return lib().orc_decide(direction, fv, bv_value, f0, f1, int(allow_back))


def bfs_levels(src, dst, n, source):
    """oracle.bfs_levels (oracle.py:36-53), without the 2^20 cap."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    out = np.empty(n, dtype=np.int32)
    _check(lib().orc_bfs_levels_edges(_ptr(src), _ptr(dst), len(src), n, source, _ptr(out)), "bfs_levels")
    return out


def min_parents(src, dst, n, root, levels):
    """SURVEY A19 min-ID parent rule (no reference counterpart)."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    levels = np.ascontiguousarray(levels, dtype=np.int32)
    out = np.empty(n, dtype=np.int64)
    _check(lib().orc_min_parents(_ptr(src), _ptr(dst), len(src), n, root, _ptr(levels), _ptr(out)),
           "min_parents")
    return out


def validate(src, dst, n, root, levels, parents) -> int:
    """SURVEY A20 certificate; 0 = valid, else bitmask of failed checks."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    levels = np.ascontiguousarray(levels, dtype=np.int32)
    parents = np.ascontiguousarray(parents, dtype=np.int64)
    return lib().orc_validate(_ptr(src), _ptr(dst), len(src), n, root, _ptr(levels), _ptr(parents))
