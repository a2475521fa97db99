#!/bin/bash
# 4-GPU box: e2e of bfs_batch compact vs full, at 1 GPU, and the N = 2 / 4 bench lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc; python -c "import os; print(os.cpu_count(), len(os.sched_getaffinity(0)))"
timeout 600 python tools/e2e_ab.py
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tools/dist_check.py 18 > gpurun_out/dist18_4.log 2>&1; echo "dist18x4 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent" gpurun_out/dist18_4.log | head -5
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --no-alt-labeling > gpurun_out/s_n$N.json 2> gpurun_out/s_n$N.err; echo "n$N rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/s_n$N.json')); print($N, d['value'], d['e2e']['value'], d['e2e']['per_call_bfs'])"
done
