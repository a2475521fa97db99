"""DBFS_TRACE of one BFS in a device group: python tools/group_trace.py <gpus> <scale> <trace path>
(the trace goes to <trace path>.<rank>; summarise with tools/trace_summary.py)."""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_1803_03922_b200 as api
from paper_1803_03922_b200.engine import _bfs_raw
from bench import graph500_roots
P = int(sys.argv[1]); scale = int(sys.argv[2])
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40, scramble=True)), 16,
                         api.ClusterShape(1, P), devices=list(range(P)))
roots = graph500_roots(pg.classification.out_degree, 64)
o = api.BfsOptions(source=roots[0])
for _ in range(2): pg.group.map(lambda k: _bfs_raw(pg.parts[k], o, None, None))
os.environ["DBFS_TRACE"] = sys.argv[3]
sts = pg.group.map(lambda k: _bfs_raw(pg.parts[k], o, None, None))
print("device ms", [s.device_ms for s in sts])
