#!/bin/bash
# 4-GPU box: GPU test suite, 4-rank dist check, bench N = 1, 2, 4, per-level profile at 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_all.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tests/dist_check_worker.py 18 > gpurun_out/dist18_4.log 2>&1; echo "dist18x4 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent" gpurun_out/dist18_4.log | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tests/dist_check_worker.py 17 > gpurun_out/dist17_2.log 2>&1; echo "dist17x2 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent" gpurun_out/dist17_2.log | head -5
timeout 600 python bench.py --no-alt-labeling > gpurun_out/s_n1.json 2> gpurun_out/s_n1.err; echo "n1 rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --no-alt-labeling > gpurun_out/s_n$N.json 2> gpurun_out/s_n$N.err; echo "n$N rc=$?"
done
for N in 1 2 4; do python -c "
import json,sys; d=json.load(open('gpurun_out/s_n$N.json')); print($N, d['value'], d['e2e']['value'], d['ms_per_step'], d['config']['workload'])"; done
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/dist_levels.py 24 1 peer > gpurun_out/dist_levels_n4.txt 2>&1; echo "lv rc=$?"
grep -A16 "rank 0 root" gpurun_out/dist_levels_n4.txt | head -17
