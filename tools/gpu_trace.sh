#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
rm -f gpurun_out/trace1.txt
DBFS_TRACE=$PWD/gpurun_out/trace1.txt timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/lv_trace.txt 2>&1; echo "lv rc=$?"
python tools/trace_summary.py gpurun_out/trace1.txt | head -40
grep -v tasks gpurun_out/lv_trace.txt | head -18
