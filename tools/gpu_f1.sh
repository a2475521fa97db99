#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tools/dist_check.py 18 > gpurun_out/dist18_4.log 2>&1; echo "dist18x4 rc=$?"; grep -E "DIST|FAIL|mismatch" gpurun_out/dist18_4.log | head -5; tail -2 gpurun_out/dist18_4.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --no-alt-labeling > gpurun_out/s_n$N.json 2> gpurun_out/s_n$N.err; echo "n$N rc=$?"
python -c "
import json,sys; d=json.load(open('gpurun_out/s_n$N.json')); print($N, d['value'], d['e2e']['value'], d['ms_per_step'], d['config']['workload'])"
done
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/dist_levels.py 24 1 peer > gpurun_out/dist_levels_n4.txt 2>&1; echo "lv rc=$?"
grep -A16 "rank 0 root" gpurun_out/dist_levels_n4.txt | head -17
