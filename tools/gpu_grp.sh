#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_all.log
for grp in 1 4 8 1 4 8; do
DBFS_CHUNK_GRP=$grp timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "grp=$grp rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done
