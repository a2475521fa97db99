#!/bin/bash
N=${1:-2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_peer.sh $N 18 24
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 tools/dist_levels.py 24 1 peer,host > gpurun_out/dist_levels_n$N.txt 2>&1; echo "rc=$?"
head -c 12000 gpurun_out/dist_levels_n$N.txt
