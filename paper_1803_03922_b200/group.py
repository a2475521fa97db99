"""One worker per GPU inside one process: the reference's ``ClusterShape``
partition (partition.py:47-76) spread over P visible GPUs by the drop-in
``partition_graph`` call itself (engine.py:149-164 runs those p workers in one
process; here they run on P devices).

Each worker w is GPU w, driven by host thread w with its own libdbfs context;
the contexts share one NCCL communicator (``dbfs_ctx_init_local_group``) and
map each other's arrays by device pointer with peer access over NVLink, so a
BFS is the same persistent peer engine a torchrun job runs (one launch per
GPU, delegate masks OR-ed from peer memory, normal records stored into the
owner's inbox), and the graph build is the distributed build (degree
all-reduce, edge all-to-all).  Calls into the C library release the GIL, so
the P threads run concurrently; collectives meet inside NCCL.

Results follow the reference API: ``run_bfs`` returns the whole level array
and ``per_iteration`` / ``comm_stats`` summed over the P workers exactly as
the reference sums its simulated workers.
"""

from __future__ import annotations

import ctypes
import math
import os
from concurrent.futures import FIRST_EXCEPTION, ThreadPoolExecutor, wait

import numpy as np

from . import _lib

KINDS = ("nn", "nd", "dn", "dd")
DO_KINDS = ("dd", "dn", "nd")


class DeviceGroup:
    """P contexts (devices[r] for rank r) with a shared NCCL communicator."""

    def __init__(self, devices):
        self.devices = [int(d) for d in devices]
        self.size = len(self.devices)
        if self.size < 2 or len(set(self.devices)) != self.size:
            raise ValueError("a device group needs >= 2 distinct devices")
        self.broken = False
        self._pool = ThreadPoolExecutor(max_workers=self.size, thread_name_prefix="dbfs-gpu")
        self.ctxs = [_lib.Context(d) for d in self.devices]
        uid = _lib.nccl_unique_id()
        self.map(lambda r: self.ctxs[r].init_local_group(uid, self.size, r))

    def map(self, fn):
        """fn(rank) on every rank's thread concurrently; results in rank order.
        If a rank fails, the others may wait in a collective for it forever:
        the group's communicators are aborted (pending collectives return),
        the group is retired and the first error is raised."""
        if self.broken:
            raise RuntimeError("this device group was aborted after an error; partition the graph again")
        with _lib.group_call():  # finalizers on rank threads must not free (and sync) GPU memory meanwhile
            futs = [self._pool.submit(fn, r) for r in range(self.size)]
            done, pending = wait(futs, return_when=FIRST_EXCEPTION)
            return self._collect(futs, done, pending)

    def _collect(self, futs, done, pending):
        failed = [f for f in done if f.exception() is not None]
        if failed:
            self.broken = True
            _groups.pop(tuple(self.devices), None)
            for c in self.ctxs:
                _lib.load().dbfs_ctx_abort(c.handle)
            wait(pending, timeout=60)
            raise failed[0].exception()
        return [f.result() for f in futs]


_groups: dict[tuple, DeviceGroup] = {}


# "auto" spreads a partition over GPUs from this many vertices on (scale 20):
# below it one device finishes a BFS in microseconds and the group's host
# threads and collectives would cost more than they save
AUTO_MIN_VERTICES = 1 << 20


def group_for(p: int, devices=None, n: int = 1 << 62) -> DeviceGroup | None:
    """The device group a p-worker partition of an n-vertex graph runs on, or
    None (simulated workers on one device).  ``devices``: "auto" (default)
    uses GPUs 0..p-1 when at least p are visible and n >= 2^20
    (``DBFS_DEVICE_GROUP=0`` keeps one device); a list names the devices;
    None/"single" keeps one device."""
    if devices in (None, "single") or p < 2:
        return None
    if devices == "auto":
        if (os.environ.get("DBFS_DEVICE_GROUP", "1") == "0" or _lib.device_count() < p or p > 64
                or n < AUTO_MIN_VERTICES):
            return None
        devices = list(range(p))
    devices = [int(d) for d in devices]
    if len(devices) != p:
        raise ValueError(f"ClusterShape has {p} workers but {len(devices)} devices were given")
    key = tuple(devices)
    if key not in _groups:
        _groups[key] = DeviceGroup(devices)
    return _groups[key]


class GroupPartitionedGraph:
    """PartitionedGraph (partition.py:281-292) whose worker w lives on GPU w."""

    def __init__(self, group: DeviceGroup, parts, shape):
        self.group = group
        self.parts = parts           # one single-worker PartitionedGraph per rank
        self.shape = shape
        p0 = parts[0]
        self.n, self.m, self.theta = p0.n, p0.m, p0.theta
        self.kind_totals = dict(p0.kind_totals)
        self.device_bytes = sum(pt.device_bytes for pt in parts)
        self.nranks, self.rank = 1, 0  # one process
        self.classification = p0.classification
        self.workers = [pt.workers[0] for pt in parts]

    @property
    def num_nn_edges(self) -> int:
        return self.kind_totals["nn"]

    @property
    def handle(self):
        raise TypeError("a device-group partition has one handle per GPU (see .parts)")

    def close(self):
        for pt in getattr(self, "parts", []):
            pt.close()


def partition_group(g, theta: int, shape, group: DeviceGroup) -> GroupPartitionedGraph:
    from .partition import partition_graph
    parts = group.map(lambda r: partition_graph(g, theta, shape, ctx=group.ctxs[r], devices=None))
    return GroupPartitionedGraph(group, parts, shape)


# ------------------------------------------------------------------- BFS API

def run_bfs(pg: GroupPartitionedGraph, opts):
    """engine.run_bfs on the device group: every rank runs the collective BFS;
    levels / parents come from rank 0 (assembled over NVLink), the records of
    all ranks are merged into the reference's per-iteration view."""
    import time

    from .engine import BfsRun, _bfs_raw, compute_teps, levels_digest
    t0 = time.perf_counter()
    n = pg.n
    if not (0 <= opts.source < n):
        raise ValueError(f"source {opts.source} out of range [0, {n})")
    outs = [(np.empty(n, dtype=np.int32), np.empty(n, dtype=np.int64) if opts.parents else None)
            for _ in range(pg.group.size)]
    sts = pg.group.map(lambda r: _bfs_raw(pg.parts[r], opts, outs[r][0], outs[r][1]))
    elapsed = time.perf_counter() - t0
    st = sts[0]
    levels, parents = outs[0]
    per_it, comm = merged_iterations(pg, int(st.iterations), opts.local_all2all)
    comm.wire_bytes = int(sum(s.wire_bytes for s in sts))
    insp = {k: {"forward": int(st.inspections[i][0]), "backward": int(st.inspections[i][1])}
            for i, k in enumerate(KINDS)}
    return BfsRun(levels=levels, iterations=int(st.iterations), per_iteration=per_it, inspections=insp,
                  comm_stats=comm, b_measured=float(st.b_measured), elapsed=elapsed,
                  teps=compute_teps(pg.m, elapsed), levels_digest=levels_digest(levels), parents=parents,
                  device_ms=float(max(s.device_ms for s in sts)),
                  kernel_launches=int(sum(s.kernel_launches for s in sts)))


def merged_iterations(pg: GroupPartitionedGraph, iterations: int, la: bool):
    """BfsRun.per_iteration + CommStats over all ranks' records (engine.py:291-302,
    comm.py:75-197): counters summed, directions / BV of worker w from rank w,
    the mask bytes of the (replicated) delegate finds, messages from the send
    matrix (regrouped per node with local_all2all)."""
    from .comm import CommStats
    from .traversal import BACKWARD, FORWARD
    L = _lib.load()
    p, P = pg.shape.p, pg.group.size
    recs, comm = [], CommStats()
    rec = _lib.IterationC()
    dirs = np.zeros(p * 4, dtype=np.int8)
    bv = np.zeros(p * 4, dtype=np.float64)
    sends = np.zeros(p, dtype=np.int64)
    for it in range(iterations):
        insp = np.zeros(4, dtype=np.int64)
        fv = np.zeros(4, dtype=np.int64)
        d_all = np.zeros((p, 4), dtype=np.int8)
        b_all = np.zeros((p, 4), dtype=np.float64)
        matrix = np.zeros((p, p), dtype=np.int64)
        normal = messages = 0
        mask = 0.0
        pairs = 0
        truncated = False
        for r in range(P):
            h = pg.parts[r].handle
            rc = L.dbfs_bfs_iteration(h, it, ctypes.byref(rec), dirs.ctypes.data_as(_lib.vp),
                                      bv.ctypes.data_as(_lib.vp))
            if rc == _lib.DBFS_ERANGE:
                truncated = True
                break
            _lib.check(rc)
            _lib.check(L.dbfs_bfs_iteration_sends(h, it, sends.ctypes.data_as(_lib.vp)))
            w = pg.workers[r].index
            insp += np.array(rec.inspections[:], dtype=np.int64)
            fv += np.array(rec.fv[:], dtype=np.int64)
            d_all[w] = dirs.reshape(p, 4)[w]
            b_all[w] = bv.reshape(p, 4)[w]
            matrix[w] = sends
            normal += int(rec.normal_bytes)
            messages += int(rec.message_count)
            if r == 0:
                mask, pairs = float(rec.mask_bytes), int(rec.pair_count)
        if truncated:
            break
        if la:
            pr = pg.shape.p_rank
            seen = set()
            for s in range(p):
                for o in range(p):
                    if matrix[s, o] > 0:
                        seen.add(((s % pr) + pr * (o // pr), o))
            messages = len(seen)
        recs.append({
            "iteration": it,
            "directions": {k: [FORWARD if d_all[w, i] == 0 else BACKWARD for w in range(p)]
                           for i, k in enumerate(KINDS)},
            "inspections": {k: int(insp[i]) for i, k in enumerate(KINDS)},
            "fv": {k: int(fv[i]) for i, k in enumerate(KINDS)},
            "bv": {k: [None if not math.isfinite(b_all[w, KINDS.index(k)]) else float(b_all[w, KINDS.index(k)])
                       for w in range(p)] for k in DO_KINDS},
            "mask_bytes": mask,
            "normal_bytes": normal,
        })
        comm.mask_bytes.append(mask)
        comm.normal_bytes.append(normal)
        comm.message_count.append(messages)
        comm.pair_count.append(pairs)
    return recs, comm


def bfs(pg: GroupPartitionedGraph, root: int, opts):
    from .engine import _bfs_raw
    n = pg.n
    outs = [(np.empty(n, dtype=np.int32), np.empty(n, dtype=np.int64)) for _ in range(pg.group.size)]
    sts = pg.group.map(lambda r: _bfs_raw(pg.parts[r], opts, outs[r][0], outs[r][1]))
    return outs[0][0], outs[0][1], sts[0]


def bfs_batch(pg: GroupPartitionedGraph, roots, outs, **kw):
    """Rank 0 receives every root's outputs; the other ranks take part in the
    collective traversals and assemblies only."""
    from .engine import bfs_batch as one
    if kw.get("parents") == "min":  # checked here: a rank failing in C would abort the whole group
        raise ValueError("min-ID parents are not available in multi-GPU batches; use bfs(pg, root, parents='min')")
    kw = dict(kw)
    compact = kw.pop("compact", None)
    stats = kw.pop("stats", False)
    kw.pop("local", None)
    compact = True if compact is None else bool(compact)  # one decision for all ranks (collective re-runs)
    res = pg.group.map(lambda r: one(pg.parts[r], roots, outs=outs if r == 0 else [(None, None)] * len(roots),
                                     compact=compact, stats=True, local=False, **kw))
    o0, st0 = res[0]
    return (o0, st0) if stats else o0


def validate(pg: GroupPartitionedGraph, root: int, levels, parents) -> int:
    from .engine import validate_bfs_tree
    return pg.group.map(lambda r: validate_bfs_tree(pg.parts[r], root, levels, parents))[0]


def min_parents(pg: GroupPartitionedGraph):
    from .engine import min_parents as one
    return pg.group.map(lambda r: one(pg.parts[r]))[0]
