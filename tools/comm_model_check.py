"""Cost model (cost_model.py:61-78) against measured
communication, one process per GPU:

  torchrun --nproc-per-node N tools/comm_model_check.py [base_scale] [roots]

For each root: the delegate model's volume / time bound (g = 1 / 900 GB/s),
the reference accounting of the run (mask + normal bytes), the bytes the GPUs
actually moved, and -- with the NCCL level loop (engine="host"), where the
exchange is a separate step -- its measured device time per BFS and per level
(CUDA events around each level's mask all-gather and record all-to-all).  The
peer engine fuses the exchange into the traversal (no separate time)."""
import datetime, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed as tdist

import paper_1803_03922_b200 as api
from paper_1803_03922_b200 import _lib
from paper_1803_03922_b200.cost_model import delegate_comm_check
from paper_1803_03922_b200.dist import env_world, init_nccl_context, weak_scale
from bench import graph500_roots

base = int(sys.argv[1]) if len(sys.argv) > 1 else 22
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 4
world, rank, local = env_world()
tdist.init_process_group("gloo", timeout=datetime.timedelta(minutes=10))
ctx = _lib.Context(local)
_lib.set_default_context(ctx)
init_nccl_context(ctx, tdist)
scale = weak_scale(base, world)
pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=40, scramble=True)), 16,
                         api.ClusterShape(1, world), ctx=ctx)
rows = []
for r in graph500_roots(pg.classification.out_degree, 64)[:nroots]:
    api.run_bfs(pg, api.BfsOptions(source=r, engine="host"))
    run = api.run_bfs(pg, api.BfsOptions(source=r, engine="host"))
    c = delegate_comm_check(pg, run)
    c["root"] = r
    rows.append(c)
allrows = [None] * world
tdist.all_gather_object(allrows, rows)
if rank == 0:
    print(f"scale {scale} on {world} GPUs (NCCL level loop), theta 16, scrambled labels")
    for i in range(len(rows)):
        per = [allrows[k][i] for k in range(world)]
        c = per[0]
        tmax = max(x["measured_time_s"] for x in per)
        print(json.dumps({"root": c["root"], "iterations": c["iterations"], "s_prime": c["s_prime"],
                          "model_volume_B": c["model_volume"], "model_time_us": round(c["model_time_s"] * 1e6, 2),
                          "accounted_B": c["accounted"], "wire_B_rank0": c["wire_bytes"],
                          "wire_time_us_at_900GBps_rank0": round(c["wire_time_s_at_g"] * 1e6, 2),
                          "measured_exchange_us_max_rank": round(tmax * 1e6, 1),
                          "within_bound": c["within_bound"]}))
tdist.barrier()
tdist.destroy_process_group()
