"""Per-task timers for one root under option variants (needs the timers build via DBFS_LIB)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1803_03922_b200 as api
from paper_1803_03922_b200 import _lib
from paper_1803_03922_b200.engine import BfsOptions, _bfs_raw
from bench import graph500_roots
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=24, scale_cap=40)), 16, api.ClusterShape(1, 1))
roots = graph500_roots(pg.classification.out_degree, 8)
L = _lib.load()
names = ["T1n", "T2dn", "T2dd", "T4dn", "T5nd", "T6dd", "F1d", "F3n"]
for label, kw in [("parents", dict(parents="any")), ("no-parents", dict(parents=None)),
                  ("reported", dict(parents="any", exec_policy="reported"))]:
    for _ in range(2):
        st = _bfs_raw(pg, BfsOptions(source=roots[0], **kw), None, None)
    print(f"== {label}: device {st.device_ms:.3f} ms")
    rec = _lib.IterationC()
    for it in range(st.iterations):
        L.dbfs_bfs_iteration(pg.handle, it, ctypes.byref(rec), None, None)
        print(f"  L{it} V {rec.visit_us:6.1f} F {rec.finish_us:6.1f} | " +
              " ".join(f"{nm} {rec.task_avg_us[i]:.0f}/{rec.task_max_us[i]:.0f}" for i, nm in enumerate(names)
                       if rec.task_max_us[i] > 5))
