#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_s24.json 2> gpurun_out/bench_s24.err; echo "b rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s24.json')); print(d['value'], d['e2e']['value'], d['cpu_baseline'])"; tail -2 gpurun_out/bench_s24.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json; nproc; free -g | head -2
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/levels_s24_dobfs.txt 2>&1; echo "lv rc=$?"; head -40 gpurun_out/levels_s24_dobfs.txt
