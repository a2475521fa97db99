"""Per-level breakdown of device BFS time (visit / finish phases), frontier
sizes, directions and inspections.  Usage: python tools/level_profile.py [scale] [roots] [mode]"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_03922_b200 as api  # noqa: E402
from paper_1803_03922_b200 import _lib  # noqa: E402
from paper_1803_03922_b200.engine import bfs_device  # noqa: E402
from bench import graph500_roots  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mode = sys.argv[3] if len(sys.argv) > 3 else "dobfs"
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40)), 16, api.ClusterShape(1, 1))
roots = graph500_roots(pg.classification.out_degree, 64)
print(f"scale {scale} n {pg.n} m {pg.m} d {pg.classification.d} kinds {pg.kind_totals}")
L = _lib.load()
for r in roots[:nroots]:
    for _ in range(2):
        st = bfs_device(pg, r, mode=mode)
    print(f"root {r}: device {st.device_ms:.3f} ms  init {st.init_us:.1f} us  iterations {st.iterations} "
          f"insp {[list(x) for x in st.inspections]}")
    rec = _lib.IterationC()
    dirs = np.zeros(4, dtype=np.int8)
    for it in range(st.iterations):
        L.dbfs_bfs_iteration(pg.handle, it, ctypes.byref(rec), dirs.ctypes.data_as(_lib.vp), None)
        print(f"  L{it}: V {rec.visit_us:8.1f} us  F {rec.finish_us:7.1f} us  front n={rec.frontier_normals:9d} "
              f"d={rec.frontier_delegates:8d}  dirs {''.join('FB'[x] for x in dirs)}  "
              f"exec {''.join('FBP'[x] for x in rec.exec_dirs)}  work {list(rec.work)}  "
              f"sync {[round(x, 1) for x in rec.sync_us]}")
        names = ["T1n", "T2dn", "T2dd", "T4dn", "T5nd", "T6dd", "F1d", "F3n"]
        print("       tasks avg/max us: " + "  ".join(f"{nm} {rec.task_avg_us[i]:.0f}/{rec.task_max_us[i]:.0f}"
                                                   for i, nm in enumerate(names) if rec.task_max_us[i] > 1))
# raw pinned D2H bandwidth
n = pg.n
lv = _lib.pinned_empty(n, np.int32); pa = _lib.pinned_empty(n, np.int64)
t = time.perf_counter()
for _ in range(5):
    api.bfs(pg, roots[0], out=(lv.array, pa.array))
dt = (time.perf_counter() - t) / 5
print(f"e2e bfs() with pinned outputs: {dt*1e3:.2f} ms/step ({12*n/dt/1e9:.1f} GB/s incl. BFS)")
