#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_all.log
for v in 0 1 0 1 0 1; do
if [ $v = 1 ]; then export DBFS_NO_HEADS=1; else unset DBFS_NO_HEADS; fi
timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "no_heads=$v rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'], d['executed_inspections_mean'])"
done
unset DBFS_NO_HEADS
rm -f gpurun_out/trace1.txt
DBFS_TRACE=$PWD/gpurun_out/trace1.txt timeout 300 python tools/level_profile.py 24 1 dobfs > gpurun_out/lv_trace.txt 2>&1; echo "lv rc=$?"
python tools/trace_summary.py gpurun_out/trace1.txt 2>/dev/null | tail -8
