"""Per-level timing of the multi-GPU engines (torchrun, one process per GPU).

  torchrun --nproc-per-node N tools/dist_levels.py [base_scale] [roots] [engines]
"""
import ctypes, datetime, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch.distributed as tdist

import paper_1803_03922_b200 as api
from paper_1803_03922_b200 import _lib
from paper_1803_03922_b200.dist import env_world, init_nccl_context, weak_scale
from paper_1803_03922_b200.engine import BfsOptions, _bfs_raw
from bench import graph500_roots

base = int(sys.argv[1]) if len(sys.argv) > 1 else 24
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 2
engines = sys.argv[3].split(",") if len(sys.argv) > 3 else ["peer", "host"]
er = "er" in sys.argv[4:]
theta = int(sys.argv[5]) if len(sys.argv) > 5 else 16
mode = sys.argv[6] if len(sys.argv) > 6 else "dobfs"
world, rank, local = env_world()
tdist.init_process_group("gloo", timeout=datetime.timedelta(minutes=10))
ctx = _lib.Context(local)
_lib.set_default_context(ctx)
init_nccl_context(ctx, tdist)
scale = weak_scale(base, world)
Q = dict(a=0.25, b=0.25, c=0.25, d_quad=0.25) if er else {}
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40, scramble=True, **Q)), theta,
                         api.ClusterShape(1, world), ctx=ctx)
roots = graph500_roots(pg.classification.out_degree, 64)[:nroots]
L = _lib.load()
names = ["T1n", "T2dn", "T2dd", "T4dn", "T5nd", "T6dd", "F1d", "F3n"]
out = []
for eng in engines:
    for r in roots:
        for _ in range(3):
            lv = np.empty(pg.n, dtype=np.int32)
            st = _bfs_raw(pg, BfsOptions(source=int(r), engine=eng, mode=mode), lv, None)
        ms = [None] * world
        tdist.all_gather_object(ms, st.device_ms)
        lines = [f"[{eng}:{st.engine_used}] rank {rank} root {r}: device {st.device_ms:.3f} ms (max {max(ms):.3f}) "
                 f"iters {st.iterations}"]
        rec = _lib.IterationC()
        dirs = np.zeros(4 * world, dtype=np.int8)
        for it in range(st.iterations):
            L.dbfs_bfs_iteration(pg.handle, it, ctypes.byref(rec), dirs.ctypes.data_as(_lib.vp), None)
            lines.append(f"  L{it}: V {rec.visit_us:8.1f} F {rec.finish_us:7.1f} us  n={rec.frontier_normals:9d} "
                         f"d={rec.frontier_delegates:8d} exec {''.join('FBP'[x] for x in rec.exec_dirs)} "
                         f"insp {list(rec.inspections)} work {list(rec.work)} nbytes {rec.normal_bytes} "
                         f"sync {[round(x, 1) for x in rec.sync_us]}")
            if max(rec.task_max_us) > 1:
                lines.append("       tasks avg/max us: " + "  ".join(
                    f"{nm} {rec.task_avg_us[i]:.0f}/{rec.task_max_us[i]:.0f}" for i, nm in enumerate(names)
                    if rec.task_max_us[i] > 1))
        out.append("\n".join(lines))
allout = [None] * world
tdist.all_gather_object(allout, out)
if rank == 0:
    print(f"scale {scale} on {world} GPUs: n {pg.n} m {pg.m} d {pg.classification.d} kinds {pg.kind_totals}")
    for i in range(len(out)):
        for rk in range(world):
            print(allout[rk][i])
tdist.barrier()
tdist.destroy_process_group()
