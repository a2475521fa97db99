#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_b.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_b.log
cat > /tmp/e2e_ab.py <<'PY'
import sys, time, numpy as np
sys.path.insert(0, ".")
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
PY
timeout 600 python /tmp/e2e_ab.py; nproc
