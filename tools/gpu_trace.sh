#!/bin/bash
# DBFS_TRACE block phase timestamps: s24 DOBFS on one GPU, s25 in a 2-GPU device group (needs gpurun --gpus 2)
cd $GRAFT_REPO_ROOT; O=gpurun_out/trace; mkdir -p $O; rm -f $O/*.txt*
DBFS_TRACE=$PWD/$O/s24.txt timeout 300 python tools/level_profile.py 24 1 dobfs > $O/lv24.txt 2>&1
python tools/trace_summary.py $O/s24.txt | tail -8
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  timeout 600 python tools/group_trace.py 2 25 $PWD/$O/group2.txt > /dev/null 2>&1 || true
  python tools/trace_summary.py $O/group2.txt.0 2>/dev/null | tail -10
fi
