#!/bin/bash
# A/B of the push unroll per push kind: DBFS_ROWS_UNR (nn/nd row pushes) / DBFS_LIST_UNR (dn/dd delegate-list pushes)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in rows2 list2; do
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_$v.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${v}_tests.log 2>&1; echo "$v tests rc=$?"; tail -1 gpurun_out/${v}_tests.log
done
for rep in 1 2; do for v in base rows2 list2; do
if [ $v = base ]; then lib=paper_1803_03922_b200/libdbfs.so; else lib=paper_1803_03922_b200/libdbfs_$v.so; fi
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$v s24 dobfs rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling --mode bfs --scale 26 --scaling strong --steps 16 > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$v s26 bfs rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done; done
