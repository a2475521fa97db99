#!/bin/bash
# launch list of the default bench command + one full capture of the BFS kernel (each after its plain run exits 0)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-alt-labeling > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-alt-labeling > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/ncu_target.py 24 dobfs > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bfs_persistent -s 1 -c 1 -o gpurun_out/prof_bfs_r01 python tools/ncu_target.py 24 dobfs > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/prof_bfs_r01.ncu-rep
