#!/bin/bash
# bench lines for several values of one environment variable ("default" = unset)
VAR=$1; VALS=$2; shift 2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in $VALS; do
  if [ "$v" = "default" ]; then E=""; else E="$VAR=$v"; fi
  env $E timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', d['config']['mode'], d['value'], d['ms_per_step'])"
done; done
