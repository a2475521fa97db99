"""ncu driver: ER (uniform quadrants) scale 24, Theta 64 (all-nn), a few DOBFS roots on one GPU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_03922_b200 as api
from paper_1803_03922_b200.engine import bfs_device
from bench import graph500_roots
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40, a=0.25, b=0.25, c=0.25,
                                                             d_quad=0.25, scramble=True)), 64, api.ClusterShape(1, 1))
roots = graph500_roots(pg.classification.out_degree, 8)
for r in roots[:3]:
    st = bfs_device(pg, r, mode="dobfs")
    print(r, st.device_ms, st.iterations)
