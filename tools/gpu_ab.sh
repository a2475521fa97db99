#!/bin/bash
# A/B of an environment toggle: bench lines with VAR=0 and VAR=1, alternating
VAR=${1:-DBFS_DEGREE_IDS}; shift
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in 0 1; do
  env $VAR=$v timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', d['config']['mode'], d['value'], d['ms_per_step'], d['e2e']['value'])"
done; done
