#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_twin.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/t_twin.log
timeout 900 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "b1 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench1.json')); print(d['value'], d['e2e']['value'], d['roofline'], d['executed_inspections_mean'])"; tail -3 gpurun_out/bench1.err
DBFS_NO_TWINS=1 timeout 900 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/bench1nt.json 2> gpurun_out/bench1nt.err; echo "b1nt rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench1nt.json')); print(d['value'], d['e2e']['value'], d['build_s'])"
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/levels_s24_dobfs.txt 2>&1; echo "lv rc=$?"; head -40 gpurun_out/levels_s24_dobfs.txt
