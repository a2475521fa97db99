"""Host-loop engine on one s24 root so ncu can profile each level's k_visit / k_finish launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_03922_b200 as api
from paper_1803_03922_b200.engine import BfsOptions, _bfs_raw
from bench import graph500_roots
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40)), 16, api.ClusterShape(1, 1))
roots = graph500_roots(pg.classification.out_degree, 8)
st = _bfs_raw(pg, BfsOptions(source=roots[0], engine="host"), None, None)
print("iterations", st.iterations, "ms", st.device_ms)
