"""ctypes binding of libdbfs.so (include/dbfs.h) and device-context handling.

The shared object is built in-tree (``paper_1803_03922_b200/libdbfs.so``).
There is no CPU fallback: if the library or a CUDA device is missing, every
entry point that needs the GPU raises :class:`DeviceUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DBFS_LIB", os.path.join(_HERE, "libdbfs.so"))

i32, i64, u64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
vp = ctypes.c_void_p

DBFS_OK, DBFS_EINVAL, DBFS_ERANGE, DBFS_ECAPACITY, DBFS_ERESOURCE = 0, 1, 2, 3, 4
DBFS_ENOMEM, DBFS_ECUDA, DBFS_ENCCL, DBFS_EROUTING, DBFS_ESTRUCT = 5, 6, 7, 8, 9
DBFS_ETIMEOUT, DBFS_EINTERNAL, DBFS_EFORMAT, DBFS_EIO = 10, 11, 12, 13

KIND_INDEX = {"nn": 0, "nd": 1, "dn": 2, "dd": 3}


class DeviceUnavailable(RuntimeError):
    """libdbfs.so or a CUDA device is missing; the product has no CPU path."""


class DbfsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class RmatParamsC(ctypes.Structure):
    _fields_ = [("scale", i32), ("randomize", i32), ("symmetrize", i32), ("scramble", i32),
                ("edge_factor", i64), ("a", dbl), ("b", dbl), ("c", dbl), ("seed", u64)]


class GraphInfoC(ctypes.Structure):
    _fields_ = [("n", i64), ("m", i64), ("d", i64), ("theta", i64),
                ("p_rank", i32), ("p_gpu", i32), ("p", i32), ("nranks", i32), ("rank", i32),
                ("n_local_workers", i32), ("first_worker", i32), ("_pad", i32),
                ("kind_totals", i64 * 4), ("device_bytes", i64)]


class BfsOptionsC(ctypes.Structure):
    _fields_ = [("mode", i32), ("allow_switch_back", i32), ("source", i64),
                ("factor0", dbl * 4), ("factor1", dbl * 4),
                ("local_all2all", i32), ("uniquify", i32), ("parent_mode", i32), ("engine", i32),
                ("record_iterations", i32), ("exec_policy", i32)]


class RunStatsC(ctypes.Structure):
    _fields_ = [("iterations", i64), ("inspections", (i64 * 2) * 4), ("b_measured", dbl),
                ("device_ms", dbl), ("reached", i64), ("kernel_launches", i64), ("wire_bytes", i64),
                ("h2d_bytes", i64), ("d2h_bytes", i64), ("rows_touched", i64), ("init_us", dbl), ("work_inspections", i64),
                ("per_iteration_truncated", i32), ("engine_used", i32),
                ("total_mask_bytes", dbl), ("total_normal_bytes", i64), ("s_prime", i64),
                ("accounting_valid", i32), ("_pad", i32)]


class IterationC(ctypes.Structure):
    _fields_ = [("iteration", i64), ("inspections", i64 * 4), ("fv", i64 * 4), ("mask_bytes", dbl),
                ("normal_bytes", i64), ("message_count", i64), ("pair_count", i64),
                ("frontier_normals", i64), ("frontier_delegates", i64), ("work", i64 * 4), ("exec_dirs", i32 * 4),
                ("task_avg_us", dbl * 8), ("task_max_us", dbl * 8), ("visit_us", dbl), ("finish_us", dbl),
                ("sync_us", dbl * 4), ("comm_us", dbl)]


P = ctypes.POINTER
# Every symbol declared in include/dbfs.h with its argtypes (tests check the
# library exports exactly these).
SIGNATURES = {
    "dbfs_last_error": (ctypes.c_char_p, []),
    "dbfs_abi_version": (i32, []),
    "dbfs_device_count": (i32, [P(i32)]),
    "dbfs_kernel_launch_counter": (i64, []),
    "dbfs_host_alloc": (i32, [i64, P(vp)]),
    "dbfs_host_free": (i32, [vp]),
    "dbfs_ctx_flush_l2": (i32, [vp]),
    "dbfs_ctx_create": (i32, [i32, P(vp)]),
    "dbfs_ctx_destroy": (i32, [vp]),
    "dbfs_nccl_unique_id": (i32, [vp, i64]),
    "dbfs_ctx_init_dist": (i32, [vp, vp, i64, i32, i32]),
    "dbfs_ctx_barrier": (i32, [vp]),
    "dbfs_ctx_allreduce_max_f64": (i32, [vp, vp, i64]),
    "dbfs_ctx_allreduce_sum_i64": (i32, [vp, vp, i64]),
    "dbfs_rmat_generate": (i32, [vp, P(RmatParamsC), i64, i64, vp, vp]),
    "dbfs_hash_vertices": (i32, [vp, i64, u64, vp, vp, i64]),
    "dbfs_graph_build_rmat": (i32, [vp, P(RmatParamsC), i64, i32, i32, P(vp)]),
    "dbfs_graph_build_edges": (i32, [vp, vp, vp, i64, i64, i64, i32, i32, P(vp)]),
    "dbfs_graph_free": (i32, [vp]),
    "dbfs_graph_set_symmetric": (i32, [vp, i32]),
    "dbfs_graph_info_get": (i32, [vp, P(GraphInfoC)]),
    "dbfs_graph_worker_info": (i32, [vp, i32, P(i64), vp, vp, P(i64)]),
    "dbfs_graph_export_csr": (i32, [vp, i32, i32, vp, vp]),
    "dbfs_graph_export_sources": (i32, [vp, i32, vp, vp, vp]),
    "dbfs_graph_export_classification": (i32, [vp, vp, vp]),
    "dbfs_bfs": (i32, [vp, P(BfsOptionsC), vp, vp, P(RunStatsC)]),
    "dbfs_fetch_result": (i32, [vp, vp, vp]),
    "dbfs_bfs_batch": (i32, [vp, P(BfsOptionsC), vp, i64, vp, vp, i32, i32, vp]),
    "dbfs_bfs_batch_output_count": (i32, [vp, i32, P(i64)]),
    "dbfs_bfs_iteration": (i32, [vp, i64, P(IterationC), vp, vp]),
    "dbfs_min_parents": (i32, [vp, vp]),
    "dbfs_bfs_iteration_sends": (i32, [vp, i64, vp]),
    "dbfs_ctx_init_local_group": (i32, [vp, vp, i64, i32, i32]),
    "dbfs_ctx_abort": (i32, [vp]),
    "dbfs_graph_nvls_active": (i32, [vp]),
    "dbfs_graph_upload_partitioned": (i32, [vp, i64, i64, i64, i32, i32, i64, vp, vp, vp, vp, i32, P(vp)]),
    "dbfs_validate": (i32, [vp, i64, vp, vp, P(i32)]),
    "dbfs_edges_text_capacity": (i32, [vp, i64, P(i64)]),
    "dbfs_edges_parse_text": (i32, [vp, i64, i64, vp, vp, P(i64), P(i64)]),
    "dbfs_edges_write_text": (i32, [ctypes.c_char_p, i64, vp, vp, i64]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libdbfs.so (raises DeviceUnavailable when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailable(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc, what="dbfs"):
    """Map a dbfs_status onto the reference's exception types."""
    if rc == DBFS_OK:
        return
    msg = load().dbfs_last_error().decode(errors="replace") or what
    from .partition import CapacityError
    from .rmat import FormatError, ResourceError
    from .comm import RoutingError, StructuralError
    if rc in (DBFS_EINVAL, DBFS_ERANGE):
        raise ValueError(msg)
    if rc == DBFS_ECAPACITY:
        raise CapacityError(msg)
    if rc == DBFS_ERESOURCE:
        raise ResourceError(msg)
    if rc == DBFS_EROUTING:
        raise RoutingError(msg)
    if rc == DBFS_ESTRUCT:
        raise StructuralError(msg)
    if rc == DBFS_ENOMEM:
        raise MemoryError(msg)
    if rc == DBFS_EFORMAT:
        raise FormatError(msg)
    if rc == DBFS_EIO:
        raise OSError(msg)
    raise DbfsError(rc, msg)


def device_count() -> int:
    n = i32(0)
    check(load().dbfs_device_count(ctypes.byref(n)))
    return int(n.value)


class Context:
    """One CUDA device + stream (+ optional NCCL communicator) in libdbfs."""

    def __init__(self, device: int = 0):
        L = load()
        if device_count() <= device:
            raise DeviceUnavailable("no CUDA device visible: the B200 engine has no CPU fallback")
        h = vp()
        check(L.dbfs_ctx_create(int(device), ctypes.byref(h)), "ctx_create")
        self._h = h
        self.device = device
        self.nranks = 1
        self.rank = 0

    @property
    def handle(self):
        return self._h

    def init_dist(self, uid: bytes, nranks: int, rank: int):
        buf = ctypes.create_string_buffer(uid, len(uid))
        check(load().dbfs_ctx_init_dist(self._h, buf, len(uid), nranks, rank), "init_dist")
        self.nranks, self.rank = nranks, rank

    def init_local_group(self, uid: bytes, nranks: int, rank: int):
        """Rank `rank` of a one-process device group (dbfs_ctx_init_local_group)."""
        buf = ctypes.create_string_buffer(uid, len(uid))
        check(load().dbfs_ctx_init_local_group(self._h, buf, len(uid), nranks, rank), "init_local_group")
        self.nranks, self.rank = nranks, rank

    def barrier(self):
        check(load().dbfs_ctx_barrier(self._h))

    def flush_l2(self):
        check(load().dbfs_ctx_flush_l2(self._h))

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            release(_lib.dbfs_ctx_destroy, self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context() -> Context:
    """The process-wide context: LOCAL_RANK's device (or 0)."""
    global _default_ctx
    if _default_ctx is None:
        dev = int(os.environ.get("DBFS_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        _default_ctx = Context(dev)
    return _default_ctx


def set_default_context(ctx: Context):
    global _default_ctx
    _default_ctx = ctx


# Releases of device / pinned memory synchronise the GPU(s).  A finalizer can
# run on whatever thread the garbage collector happens to run on -- including
# a device-group rank thread (group.py) while the other ranks wait for it in a
# collective, which would then never finish.  Finalizers therefore release
# immediately only on the main thread outside device-group calls; otherwise
# the release is queued and done at the next safe point (drain_releases).
_deferred = []
_deferred_lock = threading.Lock()
_group_depth = 0  # device-group calls in flight (main thread waits inside them)


def release(fn, handle):
    """Call fn(handle) now if that cannot stall a device group, else later."""
    if threading.current_thread() is threading.main_thread() and _group_depth == 0:
        fn(handle)
    else:
        with _deferred_lock:
            _deferred.append((fn, handle))


def drain_releases():
    """Run the queued releases (main thread, no device-group call in flight)."""
    while True:
        with _deferred_lock:
            if not _deferred:
                return
            items = list(_deferred)
            _deferred.clear()
        for fn, handle in items:
            try:
                fn(handle)
            except Exception:
                pass


class group_call:
    """Context manager around a device-group call (see release)."""

    def __enter__(self):
        global _group_depth
        drain_releases()
        _group_depth += 1

    def __exit__(self, *exc):
        global _group_depth
        _group_depth -= 1
        if _group_depth == 0:
            drain_releases()
        return False


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(load().dbfs_nccl_unique_id(buf, 128), "nccl_unique_id")
    return buf.raw


def kernel_launches() -> int:
    return int(load().dbfs_kernel_launch_counter())


class PinnedArray:
    """A numpy array over page-locked host memory (cudaHostAlloc) for fast D2H."""

    def __init__(self, count, dtype):
        import numpy as np
        self.dtype = np.dtype(dtype)
        nbytes = max(int(count) * self.dtype.itemsize, 1)
        p = vp()
        check(load().dbfs_host_alloc(nbytes, ctypes.byref(p)), "host_alloc")
        self._p = p
        buf = (ctypes.c_char * nbytes).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(count))

    def __del__(self):
        try:
            if self._p and _lib is not None:
                release(_lib.dbfs_host_free, self._p)
                self._p = None
        except Exception:
            pass


def pinned_empty(count, dtype):
    """Page-locked numpy array; keep the returned holder alive while using .array."""
    return PinnedArray(count, dtype)
