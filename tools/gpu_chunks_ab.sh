#!/bin/bash
# A/B of compile-time chunk / unroll tunables (DBFS_CWD, DBFS_CWN, DBFS_UNR), s24 DOBFS bench; "base" = default build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in base cwd4 cwd16 cwd32 cwn16 unr2 unr8; do
if [ $v = base ]; then lib=paper_1803_03922_b200/libdbfs.so; else lib=paper_1803_03922_b200/libdbfs_$v.so; fi
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$v rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done; done
