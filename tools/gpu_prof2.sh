#!/bin/bash
# fresh per-level profiles: single GPU s24 dobfs, and 2-GPU peer engine (s25)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/levels_s24_dobfs.txt 2>&1; echo "lv rc=$?"; head -30 gpurun_out/levels_s24_dobfs.txt
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/dist_levels.py 24 1 peer > gpurun_out/dist_levels_n2.txt 2>&1; echo "rc=$?"
head -c 8000 gpurun_out/dist_levels_n2.txt
