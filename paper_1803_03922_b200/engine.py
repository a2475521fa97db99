"""BFS driver API (mirror of delegate_bfs.engine) over the libdbfs GPU engine.

``run_bfs(pg, BfsOptions)`` has the reference's signature and result type
(engine.py:98-330): identical ``levels``, ``iterations``, ``per_iteration``
records, ``inspections``, ``comm_stats`` and ``levels_digest``.  Timing
(``elapsed``/``teps``) is the wall clock of the call, like the reference;
``device_ms`` adds the CUDA-event time of the traversal alone.

New on top of the reference: ``bfs(pg, root)`` returns
(depth, parent) like Graph500, and ``validate_bfs_tree`` runs the O(m)
certificate on the GPU.
"""

from __future__ import annotations

import ctypes
import dataclasses
import hashlib
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, traversal
from .comm import CommStats
from .partition import PartitionedGraph
from .traversal import BACKWARD, DO_KINDS, FORWARD

MODES = ("bfs", "dobfs")
KINDS = ("nn", "nd", "dn", "dd")
PARENT_MODES = {None: 0, "none": 0, "any": 1, "min": 2}
ENGINES = {"auto": 0, "host": 1, "persistent": 2, "peer": 3}
# executor: "reported" runs the reference's directions; "cost" may pull a
# FORWARD-reported kind or push a BACKWARD-reported one (counters recovered
# exactly) when cheaper; "push" pushes every BACKWARD-reported kind
# it can (tests of the counter recovery)
EXEC_POLICIES = {"reported": 0, "cost": 1, "push": 2}


class EmptyReportError(RuntimeError):
    """Every benchmark run was discarded (S <= 1)."""


@dataclass
class BfsOptions:
    """engine.py:33-46, plus ``parents`` / ``engine`` switches of this build."""

    mode: str = "dobfs"
    source: int = 0
    factor0: dict = field(default_factory=lambda: dict(traversal.DEFAULT_FACTOR0))
    factor1: dict = field(default_factory=lambda: dict(traversal.DEFAULT_FACTOR1))
    local_all2all: bool = False
    uniquify: bool = False
    allow_switch_back: bool = True
    seed: int = 0
    parents: str | None = "any"
    engine: str = "auto"
    exec_policy: str = "cost"

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.parents not in PARENT_MODES:
            raise ValueError(f"parents must be one of {list(PARENT_MODES)}")
        if self.engine not in ENGINES:
            raise ValueError(f"engine must be one of {list(ENGINES)}")
        if self.exec_policy not in EXEC_POLICIES:
            raise ValueError(f"exec_policy must be one of {list(EXEC_POLICIES)}")

    def to_c(self) -> _lib.BfsOptionsC:
        o = _lib.BfsOptionsC()
        o.mode = MODES.index(self.mode)
        o.allow_switch_back = int(self.allow_switch_back)
        o.source = int(self.source)
        for i, k in enumerate(KINDS):
            o.factor0[i] = float(self.factor0.get(k, 0.0)) if k != "nn" else 0.0
            o.factor1[i] = float(self.factor1.get(k, 0.0)) if k != "nn" else 0.0
        o.local_all2all = int(self.local_all2all)
        o.uniquify = int(self.uniquify)
        o.parent_mode = PARENT_MODES[self.parents]
        o.engine = ENGINES[self.engine]
        o.record_iterations = 1
        o.exec_policy = EXEC_POLICIES[self.exec_policy]
        return o


@dataclass
class BfsRun:
    levels: np.ndarray
    iterations: int
    per_iteration: list
    inspections: dict
    comm_stats: CommStats
    b_measured: float
    elapsed: float
    teps: float
    levels_digest: str
    m_prime: int | None = None
    parents: np.ndarray | None = None
    device_ms: float = 0.0
    kernel_launches: int = 0

    @property
    def total_inspections(self) -> int:
        return sum(v["forward"] + v["backward"] for v in self.inspections.values())

    def to_dict(self) -> dict:
        return {
            "iterations": self.iterations,
            "per_iteration": self.per_iteration,
            "inspections": self.inspections,
            "total_inspections": self.total_inspections,
            "comm": self.comm_stats.to_dict(),
            "b_measured": self.b_measured,
            "m_prime": self.m_prime,
            "elapsed": self.elapsed,
            "teps": self.teps,
            "levels_digest": self.levels_digest,
        }


def levels_digest(levels: np.ndarray) -> str:
    """blake2b-8 over little-endian int32 levels (engine.py:81-83)."""
    data = np.ascontiguousarray(levels, dtype="<i4").tobytes()
    return hashlib.blake2b(data, digest_size=8).hexdigest()


def compute_teps(m: int, elapsed: float) -> float:
    """(m/2)/elapsed (engine.py:86-90)."""
    if elapsed <= 0:
        raise ValueError("elapsed must be positive")
    return (m / 2) / elapsed


def _bfs_raw(pg: PartitionedGraph, opts: BfsOptions, levels_out, parents_out):
    st = _lib.RunStatsC()
    o = opts.to_c()
    lv = levels_out.ctypes.data_as(_lib.vp) if levels_out is not None else None
    pa = parents_out.ctypes.data_as(_lib.vp) if parents_out is not None else None
    _lib.check(_lib.load().dbfs_bfs(pg.handle, ctypes.byref(o), lv, pa, ctypes.byref(st)), "bfs")
    return st


def _per_iteration(pg: PartitionedGraph, iterations: int):
    """BfsRun.per_iteration + CommStats from the device records (engine.py:291-302)."""
    L = _lib.load()
    p = pg.shape.p
    recs, comm = [], CommStats()
    rec = _lib.IterationC()
    dirs = np.zeros(p * 4, dtype=np.int8)
    bv = np.zeros(p * 4, dtype=np.float64)
    for it in range(iterations):
        rc = L.dbfs_bfs_iteration(pg.handle, it, ctypes.byref(rec), dirs.ctypes.data_as(_lib.vp),
                                  bv.ctypes.data_as(_lib.vp))
        if rc == _lib.DBFS_ERANGE:  # truncated record buffer
            break
        _lib.check(rc)
        d = dirs.reshape(p, 4)
        b = bv.reshape(p, 4)
        recs.append({
            "iteration": it,
            "directions": {k: [FORWARD if d[w, i] == 0 else BACKWARD for w in range(p)] for i, k in enumerate(KINDS)},
            "inspections": {k: int(rec.inspections[i]) for i, k in enumerate(KINDS)},
            "fv": {k: int(rec.fv[i]) for i, k in enumerate(KINDS)},
            "bv": {k: [None if not math.isfinite(b[w, KINDS.index(k)]) else float(b[w, KINDS.index(k)])
                       for w in range(p)] for k in DO_KINDS},
            "mask_bytes": float(rec.mask_bytes),
            "normal_bytes": int(rec.normal_bytes),
        })
        comm.measured_time_s += float(rec.comm_us) * 1e-6
        comm.mask_bytes.append(float(rec.mask_bytes))
        comm.normal_bytes.append(int(rec.normal_bytes))
        comm.message_count.append(int(rec.message_count))
        comm.pair_count.append(int(rec.pair_count))
    return recs, comm


def _group(pg):
    from .group import GroupPartitionedGraph
    return isinstance(pg, GroupPartitionedGraph)


def run_bfs(pg: PartitionedGraph, opts: BfsOptions) -> BfsRun:
    """One BFS/DOBFS on the GPU with the reference's result (engine.py:98-330)."""
    if _group(pg):
        from . import group
        return group.run_bfs(pg, opts)
    t0 = time.perf_counter()
    n = pg.n
    if not (0 <= opts.source < n):
        raise ValueError(f"source {opts.source} out of range [0, {n})")
    levels = np.empty(n, dtype=np.int32)
    parents = np.empty(n, dtype=np.int64) if opts.parents else None
    st = _bfs_raw(pg, opts, levels, parents)  # parents="min": the C side replaces the tree by the min-ID one
    elapsed = time.perf_counter() - t0
    per_it, comm = _per_iteration(pg, st.iterations)
    comm.wire_bytes = int(st.wire_bytes)
    insp = {k: {"forward": int(st.inspections[i][0]), "backward": int(st.inspections[i][1])}
            for i, k in enumerate(KINDS)}
    return BfsRun(levels=levels, iterations=int(st.iterations), per_iteration=per_it, inspections=insp,
                  comm_stats=comm, b_measured=float(st.b_measured), elapsed=elapsed,
                  teps=compute_teps(pg.m, elapsed), levels_digest=levels_digest(levels), parents=parents,
                  device_ms=float(st.device_ms), kernel_launches=int(st.kernel_launches))


def _run_entry(s, iterations, teps, total_insp, mask_bytes, normal_bytes, s_prime, digest):
    return {"source": s, "iterations": iterations, "teps": teps, "total_inspections": total_insp,
            "mask_bytes": mask_bytes, "normal_bytes": normal_bytes, "s_prime": s_prime, "levels_digest": digest}


def _share_digests(pg, digests):
    """Rank 0's 8-byte digests to every rank (an NCCL sum with zeros elsewhere)."""
    vals = np.array([int(d, 16) if d is not None else 0 for d in digests], dtype=np.uint64).view(np.int64)
    _lib.check(_lib.load().dbfs_ctx_allreduce_sum_i64(pg._ctx.handle, vals.ctypes.data_as(_lib.vp), len(vals)))
    return [f"{int(v):016x}" for v in vals.view(np.uint64)]


def benchmark(pg: PartitionedGraph, sources, opts: BfsOptions) -> dict:
    """Per-source runs, discard S <= 1, geometric-mean TEPS (engine.py:333-364);
    the Graph500 harmonic mean is reported beside it.

    One process owning the whole graph runs the sources as a pipelined batch
    (``dbfs_bfs_batch``): every root's levels reach host memory (the depth
    travels as int8 and is widened on the host's cores while later roots
    traverse), its iteration records give the same inspections / mask bytes /
    normal bytes / S' as ``run_bfs``, and digests are taken after the call
    (the reference, too, hashes outside its timed region).  Runs are
    pipelined, so a per-run wall clock does not exist: a run's ``teps`` uses
    its device-timed traversal, and the report adds ``wall_s`` (the batch
    calls, host copies included) and ``e2e_teps`` over all runs.  With one
    worker per GPU (torchrun) every rank receives the whole level array of
    every root (assembled over NVLink) and the per-rank counters are summed
    over ranks after the call.  The host-loop engine runs ``run_bfs`` per
    source."""
    sources = [int(s) for s in sources]
    for s in sources:
        if not (0 <= s < pg.n):
            raise ValueError(f"source {s} out of range [0, {pg.n})")
    entries, t_total, d2h = [], 0.0, 0
    if opts.engine == "host":
        for s in sources:
            run = run_bfs(pg, dataclasses.replace(opts, source=s))
            t_total += run.elapsed
            entries.append((run.iterations, _run_entry(s, run.iterations, run.teps, run.total_inspections,
                                                       run.comm_stats.total_mask_bytes,
                                                       run.comm_stats.total_normal_bytes,
                                                       run.comm_stats.s_prime, run.levels_digest)))
    else:
        n = pg.n
        # one worker per GPU (torchrun): rank 0 receives every root's levels (the
        # other ranks take part in the traversals only, so a host widens one copy)
        # and shares its digests with the ranks over NCCL
        receiver = pg.nranks == 1 or pg.rank == 0
        chunk = max(1, min(len(sources), (8 << 30) // max(4 * n, 1)))  # <= 8 GiB of host levels per call
        # host level arrays: page-locked, kept with the graph and reused by later
        # calls (pageable pages are faulted in -- or NUMA-migrated -- while the
        # host widens the depths inside the call)
        held = getattr(pg, "_benchmark_levels", None)
        if receiver and (held is None or len(held) < chunk or held[0].array.size != n):
            pg._benchmark_levels = None
            held = [_lib.pinned_empty(n, np.int32) for _ in range(chunk)]
            pg._benchmark_levels = held
        bufs = [h.array for h in held] if receiver else [None] * chunk
        for c0 in range(0, len(sources), chunk):
            roots = sources[c0:c0 + chunk]
            t0 = time.perf_counter()
            outs, sts = bfs_batch(pg, roots, outs=[(bufs[i], None) for i in range(len(roots))], mode=opts.mode,
                                  parents=opts.parents, stats=True, options=opts, accounting=True,
                                  compact=True if pg.nranks > 1 else None)
            t_total += time.perf_counter() - t0
            d2h += sum(int(st.d2h_bytes) for st in sts)
            digests = [None] * len(roots)
            if receiver:
                from concurrent.futures import ThreadPoolExecutor  # digests after the timed call (hashlib drops the GIL)
                with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
                    digests = list(ex.map(levels_digest, bufs[:len(roots)]))
            if pg.nranks > 1:
                digests = _share_digests(pg, digests)
            for i, (s, st) in enumerate(zip(roots, sts)):
                if not st.accounting_valid:  # records truncated (deep BFS): exact stats from a single run
                    run = run_bfs(pg, dataclasses.replace(opts, source=s))
                    entries.append((run.iterations, _run_entry(
                        s, run.iterations, run.teps, run.total_inspections, run.comm_stats.total_mask_bytes,
                        run.comm_stats.total_normal_bytes, run.comm_stats.s_prime, run.levels_digest)))
                    continue
                it = int(st.iterations)
                total = sum(int(st.inspections[k][0]) + int(st.inspections[k][1]) for k in range(4))
                teps = compute_teps(pg.m, max(st.device_ms, 1e-6) / 1e3)
                entries.append((it, _run_entry(s, it, teps, total, float(st.total_mask_bytes),
                                               int(st.total_normal_bytes), int(st.s_prime), digests[i])))
    runs = [e for it, e in entries if it > 1]
    if not runs:
        raise EmptyReportError("all runs discarded (every source trivial)")
    teps = np.array([r["teps"] for r in runs])
    geomean = float(np.exp(np.log(teps).mean()))
    harmonic = float(len(teps) / np.sum(1.0 / teps))
    return {
        "num_runs": len(runs),
        "num_discarded": len(sources) - len(runs),
        "geomean_teps": geomean,
        "harmonic_teps": harmonic,
        "wall_s": t_total,
        "e2e_teps": len(sources) * (pg.m / 2) / t_total if t_total > 0 else 0.0,
        "d2h_bytes": d2h,  # device -> host bytes of the batch calls (this process)
        "runs": runs,
    }


def bfs(pg: PartitionedGraph, root: int, parents: str = "any", mode: str = "dobfs", out=None,
        stats: bool = False):
    """Graph500-style BFS: (depth int32[n], parent int64[n]).  ``parents="min"``
    gives the deterministic min-ID tree.  ``out=(levels, parents)``
    writes into caller buffers (e.g. pinned, see ``_lib.pinned_empty``);
    ``stats=True`` also returns the C run-stats struct."""
    if not (0 <= root < pg.n):
        raise ValueError(f"source {root} out of range [0, {pg.n})")
    if parents not in ("any", "min"):
        raise ValueError("parents must be 'any' or 'min'")
    opts = BfsOptions(mode=mode, source=int(root), parents=parents)
    if _group(pg):
        from . import group
        lv, pa, st = group.bfs(pg, root, opts)
        if out is not None:
            out[0][:pg.n] = lv
            out[1][:pg.n] = pa
            lv, pa = out
        return (lv, pa, st) if stats else (lv, pa)
    if out is None:
        levels = np.empty(pg.n, dtype=np.int32)
        par = np.empty(pg.n, dtype=np.int64)
    else:
        levels, par = out
        _check_host_array(levels, np.int32, pg.n, "levels")
        _check_host_array(par, np.int64, pg.n, "parents")
    st = _bfs_raw(pg, opts, levels, par)
    return (levels, par, st) if stats else (levels, par)


def _check_host_array(a, dtype, n: int, what: str):
    """Caller buffers handed to the C side as raw pointers: right dtype, >= n
    entries, C-contiguous (the library writes 4n / 8n bytes)."""
    if not isinstance(a, np.ndarray) or a.dtype != dtype or a.size < n or not a.flags.c_contiguous:
        raise ValueError(f"{what} must be a contiguous {np.dtype(dtype).name} array of >= {n} entries")


def bfs_batch(pg: PartitionedGraph, roots, outs=None, mode: str = "dobfs", parents: str | None = "any",
              stats: bool = False, local: bool = False, compact: bool | None = None,
              options: BfsOptions | None = None, accounting: bool = False):
    """Graph500's multi-root loop in one call (``dbfs_bfs_batch``): returns one
    (depth, parent) pair per root.  The device-to-host copy of root k runs on a
    separate stream while root k+1 traverses, so PCIe time hides behind the
    BFS.  ``outs`` is a list of (levels int32, parents int64) host arrays of
    ``batch_output_count(pg, local)`` entries (pinned for the overlap, see
    ``_lib.pinned_empty``); entries may repeat, e.g. two buffer pairs used
    alternately, in which case each root's result is in its pair until root
    k+2 overwrites it.  ``local=True`` in a distributed run gives each rank
    only the vertices it owns (entry i = vertex rank + i*world), the
    distributed Graph500 result.  ``compact`` sends the depth as int8 over
    PCIe (9 instead of 12 bytes per vertex; parents go straight into ``outs``)
    and widens it on the host's cores while later roots traverse (identical
    results; a root with a depth >= 127 is re-run with full arrays).  None:
    on for a single process, off when ranks share the host (their widening
    competes for it); ``DBFS_COMPACT=0/1`` overrides.  Per-iteration records
    are not kept; ``accounting=True`` (single process) keeps each root's
    records long enough to fill its run stats with the reference's
    inspections and CommStats totals (``accounting_valid``).  ``options``
    supplies the other BfsOptions fields (factors, executor, ...).
    ``stats=True`` also returns the per-root C run-stats structs."""
    if parents not in PARENT_MODES:
        raise ValueError(f"parents must be one of {list(PARENT_MODES)}")
    roots = np.ascontiguousarray([int(r) for r in roots], dtype=np.int64)
    for r in roots:
        if not (0 <= r < pg.n):
            raise ValueError(f"source {r} out of range [0, {pg.n})")
    count = len(roots)
    if _group(pg):
        from . import group
        if outs is None:
            outs = [(np.empty(pg.n, dtype=np.int32), np.empty(pg.n, dtype=np.int64) if parents else None)
                    for _ in range(count)]
        return group.bfs_batch(pg, list(roots), outs, mode=mode, parents=parents, stats=stats, compact=compact,
                               options=options, accounting=accounting)
    nout = batch_output_count(pg, local)
    if outs is None:
        outs = [(np.empty(nout, dtype=np.int32), np.empty(nout, dtype=np.int64) if parents else None)
                for _ in range(count)]
    if len(outs) != count:
        raise ValueError("outs must hold one (levels, parents) pair per root")
    for lv, pa in outs:
        if lv is not None and (lv.dtype != np.int32 or lv.size < nout or not lv.flags.c_contiguous):
            raise ValueError(f"levels buffers must be contiguous int32[{nout}]")
        if pa is not None and (pa.dtype != np.int64 or pa.size < nout or not pa.flags.c_contiguous):
            raise ValueError(f"parents buffers must be contiguous int64[{nout}]")
    if compact is None:
        env = os.environ.get("DBFS_COMPACT")
        compact = (env == "1") if env in ("0", "1") else pg.nranks <= 1
    lv_ptrs = (_lib.vp * max(count, 1))(*[lv.ctypes.data if lv is not None else None for lv, _ in outs])
    pa_ptrs = (_lib.vp * max(count, 1))(*[pa.ctypes.data if pa is not None else None for _, pa in outs])
    st = (_lib.RunStatsC * max(count, 1))()
    base = options if options is not None else BfsOptions()
    opts = dataclasses.replace(base, mode=mode, source=int(roots[0]) if count else 0, parents=parents).to_c()
    opts.record_iterations = int(bool(accounting))
    _lib.check(_lib.load().dbfs_bfs_batch(pg.handle, ctypes.byref(opts), roots.ctypes.data_as(_lib.vp), count,
                                          lv_ptrs, pa_ptrs if parents and any(pa is not None for _, pa in outs) else None,
                                          int(bool(local)), int(bool(compact)),
                                          st), "bfs_batch")
    return (outs, list(st)[:count]) if stats else outs


def batch_output_count(pg: PartitionedGraph, local: bool = False) -> int:
    """Entries per output array of ``bfs_batch``: n, or this rank's own vertex
    count when ``local`` in a distributed run."""
    if _group(pg):
        return pg.n
    c = ctypes.c_int64()
    _lib.check(_lib.load().dbfs_bfs_batch_output_count(pg.handle, int(bool(local)), ctypes.byref(c)))
    return int(c.value)


def bfs_device(pg: PartitionedGraph, root: int, mode: str = "dobfs", parents: str | None = "any",
               exec_policy: str = "cost"):
    """One BFS leaving depth/parents in device memory (for timing); returns run stats."""
    if _group(pg):
        o = BfsOptions(mode=mode, source=int(root), parents=parents, exec_policy=exec_policy)
        return pg.group.map(lambda r: _bfs_raw(pg.parts[r], o, None, None))[0]
    return _bfs_raw(pg, BfsOptions(mode=mode, source=int(root), parents=parents, exec_policy=exec_policy), None, None)


def min_parents(pg: PartitionedGraph) -> np.ndarray:
    """Min-ID parents of the last BFS, computed on the GPU."""
    if _group(pg):
        from . import group
        return group.min_parents(pg)
    out = np.empty(pg.n, dtype=np.int64)
    _lib.check(_lib.load().dbfs_min_parents(pg.handle, out.ctypes.data_as(_lib.vp)), "min_parents")
    return out


def validate_bfs_tree(pg: PartitionedGraph, root: int, levels=None, parents=None) -> int:
    """Graph500 certificate on the GPU.  0 = valid, else a bitmask:
    1 root, 2 edge spans > 1 level, 4 reached-unreached edge, 8 parent level,
    16 tree edge not in E, 32 parent of unreached / missing parent."""
    if not (0 <= root < pg.n):
        raise ValueError(f"root {root} out of range [0, {pg.n})")
    if _group(pg):
        from . import group
        return group.validate(pg, root, levels, parents)
    rep = ctypes.c_int32()
    lva = pa_ = None
    if levels is not None:
        lva = np.ascontiguousarray(levels, dtype=np.int32)
        if lva.ndim != 1 or lva.size != pg.n:
            raise ValueError(f"levels must hold exactly n = {pg.n} entries")
    if parents is not None:
        pa_ = np.ascontiguousarray(parents, dtype=np.int64)
        if pa_.ndim != 1 or pa_.size != pg.n:
            raise ValueError(f"parents must hold exactly n = {pg.n} entries")
    lv = lva.ctypes.data_as(_lib.vp) if lva is not None else None
    pa = pa_.ctypes.data_as(_lib.vp) if pa_ is not None else None
    _lib.check(_lib.load().dbfs_validate(pg.handle, int(root), lv, pa, ctypes.byref(rep)), "validate")
    del lva, pa_  # the converted copies live until the call returned
    return int(rep.value)
