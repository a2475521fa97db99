#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tools/dist_check.py 18 > gpurun_out/dist18_4.log 2>&1; echo "dist18x4 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent" gpurun_out/dist18_4.log | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tools/dist_check.py 17 - er > gpurun_out/dist17er_4.log 2>&1; echo "dist17er x4 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent" gpurun_out/dist17er_4.log | head -5
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 tools/dist_levels.py 25 1 peer er 64 bfs > gpurun_out/er_levels_n4.txt 2>&1; echo "lv4 rc=$?"
grep "device" gpurun_out/er_levels_n4.txt | head -4
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --no-alt-labeling > gpurun_out/s_n$N.json 2> gpurun_out/s_n$N.err; echo "n$N rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/s_n$N.json')); print($N, d['value'], d['e2e']['value'])"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29574 bench.py --gpus 4 --no-alt-labeling --graph er --mode bfs --scale 28 --scaling strong --theta 64 --steps 16 > gpurun_out/er28_4.json 2> gpurun_out/er28_4.err; echo "er4 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/er28_4.json')); print(d['value'], d['e2e']['value'], d['ms_per_step'])"
