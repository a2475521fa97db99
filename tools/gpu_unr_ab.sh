#!/bin/bash
# A/B of the push unroll DBFS_UNR (default build = 4): s24 DOBFS and s26 top-down BFS; GPU suite on UNR=2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_unr2.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/unr2_tests.log 2>&1; echo "unr2 tests rc=$?"; tail -1 gpurun_out/unr2_tests.log
for rep in 1 2; do for v in base unr1 unr2 unr3; do
if [ $v = base ]; then lib=paper_1803_03922_b200/libdbfs.so; else lib=paper_1803_03922_b200/libdbfs_$v.so; fi
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$v s24 dobfs rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling --mode bfs --scale 26 --scaling strong --steps 16 > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$v s26 bfs rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done; done
