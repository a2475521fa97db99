#!/bin/bash
# A/B of block shape / occupancy variants of libdbfs (same bench command)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in libdbfs.so libdbfs_bt1024.so libdbfs_bt512m2.so libdbfs.so; do
DBFS_LIB=$PWD/paper_1803_03922_b200/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling --steps 64 > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$lib rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done
