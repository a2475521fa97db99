cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 python bench.py --steps 4 --warmup 1 --no-cpu-baseline --no-alt-labeling > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 1 --no-cpu-baseline --no-alt-labeling > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/ncu_target.py 24 dobfs > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bfs_persistent -s 1 -c 1 -o gpurun_out/prof_bfs_r01 python tools/ncu_target.py 24 dobfs > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
