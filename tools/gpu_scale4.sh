#!/bin/bash
# 4-GPU box: default-config bench at N = 1, 2, 4 (weak from s24), BFS strong s26 at 4, per-level profile at 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s_n1.json 2> gpurun_out/s_n1.err; echo "n1 rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > gpurun_out/s_n$N.json 2> gpurun_out/s_n$N.err; echo "n$N rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --mode bfs --scale 26 --scaling strong > gpurun_out/bfs26_n4.json 2> gpurun_out/bfs26_n4.err; echo "bfs26 rc=$?"
for N in 1 2 4; do python -c "
import json,sys; d=json.load(open('gpurun_out/s_n$N.json')); print($N, d['value'], d['e2e']['value'], d['ms_per_step'], d['config']['workload'])"; done
python -c "
import json,sys; d=json.load(open('gpurun_out/bfs26_n4.json')); print(d['value'], d['e2e']['value'], d['config']['workload'])"
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/dist_levels.py 24 1 peer > gpurun_out/dist_levels_n4.txt 2>&1; echo "lv rc=$?"
grep -i error gpurun_out/*.err | head
