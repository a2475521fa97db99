#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for t in 32 1000000000 8 32 1000000000 8; do
DBFS_PULL_DYN_MIN=$t timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "pull_dyn_min=$t rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done
