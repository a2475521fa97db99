#!/bin/bash
N=${1:-2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 tools/dist_check.py 18 > gpurun_out/peer_check_n$N.log 2>&1; echo "check rc=$?"; grep -E "DIST|disagree|rror" gpurun_out/peer_check_n$N.log | head
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 tools/dist_levels.py 24 1 peer > gpurun_out/dist_levels_n$N.txt 2>&1; echo "rc=$?"
grep -v "^\*\*\*\|OMP_NUM" gpurun_out/dist_levels_n$N.txt | head -c 9000
