#!/bin/bash
# single-GPU: bench line, per-level profile with task timers, GPU test suite
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "n1 rc=$?"; cat gpurun_out/bench_n1.json; tail -3 gpurun_out/bench_n1.err
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python tools/level_profile.py 24 2 dobfs > gpurun_out/levels_s24_dobfs.txt 2>&1; echo "lv rc=$?"; head -40 gpurun_out/levels_s24_dobfs.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
