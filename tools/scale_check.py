"""Larger / other configs on one GPU: build time, memory, BFS time, certificate."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1803_03922_b200 as api
from paper_1803_03922_b200.engine import bfs_device
from bench import graph500_roots, suggested_theta

def run(scale, mode="dobfs", quads=None, theta=None, roots=8):
    kw = dict(a=quads[0], b=quads[1], c=quads[2], d_quad=quads[3]) if quads else {}
    p = api.RmatParams(scale=scale, scale_cap=40, **kw)
    th = theta if theta is not None else suggested_theta(scale)
    t0 = time.time()
    pg = api.partition_graph(api.build_rmat_graph(p), th, api.ClusterShape(1, 1))
    bt = time.time() - t0
    rs = graph500_roots(pg.classification.out_degree, roots)
    bfs_device(pg, rs[0], mode=mode)
    ts = []
    for r in rs:
        st = bfs_device(pg, r, mode=mode)
        ts.append(st.device_ms)
    bad = api.validate_bfs_tree(pg, rs[0])
    g = len(ts) * pg.m / 2 / (sum(ts) / 1e3) / 1e9
    print(f"s{scale} {'ER' if quads else 'RMAT'} theta={th} {mode}: build {bt:.1f}s d={pg.classification.d} "
          f"kinds={pg.kind_totals} dev_bytes={pg.device_bytes/1e9:.1f}GB  mean {np.mean(ts):.3f} ms  "
          f"hmean {g:.1f} GTEPS  certificate {bad}", flush=True)
    del pg

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("er", "all"):
    import oracle as O
    # parity of the ER path at s18 against the oracle
    pq = (0.25, 0.25, 0.25, 0.25)
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=18, a=.25, b=.25, c=.25, d_quad=.25)), 64,
                             api.ClusterShape(1, 1))
    og = O.partition_rmat(18, 64, a=.25, b=.25, c=.25)
    for r in (3, 999):
        for mode in ("bfs", "dobfs"):
            got = api.run_bfs(pg, api.BfsOptions(source=r, mode=mode)).to_dict()
            ref = O.run_bfs(og, r, mode=mode)
            ok = all(got[k] == ref[k] for k in ("iterations", "per_iteration", "inspections", "levels_digest"))
            print(f"ER s18 {mode} root {r}: parity {'OK' if ok else 'MISMATCH'}", flush=True)
    del pg
    run(22, "bfs", quads=pq, theta=64)
    run(22, "dobfs", quads=pq, theta=64)
if which in ("big", "all"):
    run(24, "bfs")
    run(26, "dobfs")
    run(26, "bfs", roots=4)
    run(27, "dobfs", roots=4)
