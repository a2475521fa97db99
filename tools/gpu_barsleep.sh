#!/bin/bash
# A/B of the grid-barrier poll sleep (DBFS_BAR_SLEEP ns; default build = 64), s24 DOBFS bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in 64 0 16 256; do
if [ $v = 64 ]; then lib=paper_1803_03922_b200/libdbfs.so; else lib=paper_1803_03922_b200/libdbfs_s$v.so; fi
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "sleep=$v rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done; done
