"""e2e A/B of bfs_batch transfer forms on one GPU (s24, 64 roots, two pinned buffer pairs)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_03922_b200 as api
from paper_1803_03922_b200 import _lib
from bench import graph500_roots
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=24, scramble=True)), 16, api.ClusterShape(1, 1))
roots = graph500_roots(pg.classification.out_degree, 64)
n = pg.n
pairs = [(_lib.pinned_empty(n, np.int32), _lib.pinned_empty(n, np.int64)) for _ in range(2)]
outs = [(pairs[i % 2][0].array, pairs[i % 2][1].array) for i in range(64)]
for compact in (False, True, False, True):
    api.bfs_batch(pg, roots[:4], outs=outs[:4], compact=compact)
    t = time.perf_counter()
    api.bfs_batch(pg, roots, outs=outs, compact=compact)
    dt = time.perf_counter() - t
    print("compact", compact, "e2e GTEPS", round(64 * (pg.m / 2) / dt / 1e9, 2), flush=True)
