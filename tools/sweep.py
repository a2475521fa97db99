"""Average device ms over roots for the current DBFS_LIB (variant sweep)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1803_03922_b200 as api
from paper_1803_03922_b200.engine import bfs_device
from bench import graph500_roots
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40)), 16, api.ClusterShape(1, 1))
roots = graph500_roots(pg.classification.out_degree, 16)
out = []
for mode in ("dobfs", "bfs"):
    bfs_device(pg, roots[0], mode=mode)
    t = [bfs_device(pg, r, mode=mode).device_ms for r in roots]
    out.append(f"{mode}: mean {np.mean(t):.3f} ms  hmean-GTEPS {len(t)*pg.m/2/(sum(t)/1e3)/1e9:.1f}")
print(os.path.basename(os.environ.get("DBFS_LIB", "libdbfs.so")), " | ".join(out))
