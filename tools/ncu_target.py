"""Small driver for ncu: build an RMAT graph (reference labels, Theta 16) and run
a few BFS roots (device-resident results).

  python tools/ncu_target.py [scale] [mode] [roots]

The first BFS also builds the executor's aids (dd rows by degree, twin
positions), so a capture of the build kernels (k_rs_*, k_route, k_twin_fill,
...) and of k_bfs_persistent can come from the same command."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_03922_b200 as api
from paper_1803_03922_b200.engine import bfs_device
from bench import graph500_roots
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
mode = sys.argv[2] if len(sys.argv) > 2 else "dobfs"
nroots = int(sys.argv[3]) if len(sys.argv) > 3 else 4
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40)), 16, api.ClusterShape(1, 1))
roots = graph500_roots(pg.classification.out_degree, 8)
for r in roots[:nroots]:
    st = bfs_device(pg, r, mode=mode)
    print(r, st.device_ms)
