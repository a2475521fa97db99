"""Single-process multi-GPU (device group) timing: one worker per GPU inside
one process through the reference API, with the delegate-mask OR read from the
peers (default) or reduced in the NVSwitch (DBFS_NVLS=1).

  python tools/group_bench.py <gpus> <scale> [mode] [scramble]

Prints harmonic-mean GTEPS over the 64 Graph500 roots (device time = max over
the GPUs of each BFS, L2 flushed before every BFS) and the F-phase times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1803_03922_b200 as api
from paper_1803_03922_b200 import _lib
from paper_1803_03922_b200.engine import bfs_device
from bench import graph500_roots, suggested_theta

P = int(sys.argv[1]); scale = int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "dobfs"
scramble = len(sys.argv) > 4 and sys.argv[4] == "scramble"
theta = suggested_theta(scale)
t0 = time.perf_counter()
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40, scramble=scramble)), theta,
                         api.ClusterShape(1, P), devices=list(range(P)))
build = time.perf_counter() - t0
roots = graph500_roots(pg.classification.out_degree, 64)
for r in roots[:4]:
    bfs_device(pg, r, mode=mode)
ms = []
for r in roots:
    pg.group.map(lambda k: pg.group.ctxs[k].flush_l2())
    sts = pg.group.map(lambda k: __import__("paper_1803_03922_b200.engine", fromlist=["_bfs_raw"])._bfs_raw(
        pg.parts[k], api.BfsOptions(mode=mode, source=r), None, None))
    ms.append(max(s.device_ms for s in sts))
nvls = [_lib.load().dbfs_graph_nvls_active(pt.handle) for pt in pg.parts]  # set up by the first BFS
gteps = len(ms) * (pg.m / 2) / (sum(ms) / 1e3) / 1e9
print(f"P={P} scale={scale} theta={theta} mode={mode} scramble={scramble} nvls={nvls} build {build:.1f}s "
      f"harmonic {gteps:.1f} GTEPS, {np.mean(ms):.3f} ms per BFS")
run = api.run_bfs(pg, api.BfsOptions(mode=mode, source=roots[0]))
print("levels:", run.iterations, "mask bytes", run.comm_stats.total_mask_bytes, "normal bytes",
      run.comm_stats.total_normal_bytes)
pg.close()
