#!/bin/bash
# ncu evidence (one GPU; each capture only after its plain run exited 0):
# full captures of k_bfs_persistent (s24 DOBFS, s26 top-down BFS) and of the
# build kernels, plus the launch list of the bench command; summarised by
# tools/summarize_ncu.py gpurun_out/ncu profiles/<round>.
cd $GRAFT_REPO_ROOT; O=gpurun_out/ncu; mkdir -p $O
timeout 300 python tools/ncu_target.py 24 dobfs > $O/plain24.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bfs_persistent -s 1 -c 1 -o $O/bfs_s24 python tools/ncu_target.py 24 dobfs > $O/ncu_s24.log 2>&1; echo "s24 rc=$?"
timeout 300 python tools/ncu_target.py 26 bfs 2 > $O/plain26.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_bfs_persistent -s 1 -c 1 -o $O/bfs_s26_bfs python tools/ncu_target.py 26 bfs 2 > $O/ncu_s26.log 2>&1; echo "s26 rc=$?"
for k in k_rs_scatter k_route k_twin_fill k_rs_hist k_degree k_gather_cols; do
  timeout 900 ncu --set full --clock-control none -k regex:$k -c 1 -o $O/build_$k python tools/ncu_target.py 24 dobfs 1 > $O/ncu_$k.log 2>&1; echo "$k rc=$?"
done
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-series > $O/bench_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-series > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
