#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for N in 2 4; do
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N tools/dist_levels.py 25 1 peer er 64 bfs > gpurun_out/er_levels_n$N.txt 2>&1; echo "lv$N rc=$?"
grep -A22 "rank 0 root" gpurun_out/er_levels_n$N.txt | head -24
done
