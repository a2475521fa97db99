#!/bin/bash
# A/B of a push-step change: libdbfs_base.so (previous build) vs the current build; GPU suite on the current build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/guard_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/guard_tests.log
for rep in 1 2; do for v in base new; do
if [ $v = new ]; then lib=paper_1803_03922_b200/libdbfs.so; else lib=paper_1803_03922_b200/libdbfs_base.so; fi
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$v s24 dobfs rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling --mode bfs --scale 26 --scaling strong --steps 16 > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "$v s26 bfs rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done; done
