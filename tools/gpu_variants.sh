#!/bin/bash
# bench the default build and compile-time variants (libdbfs_v*.so), interleaved, twice
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for lib in paper_1803_03922_b200/libdbfs.so paper_1803_03922_b200/libdbfs_v*.so; do
  DBFS_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['mode'], d['value'], d['ms_per_step'])"
done; done
