#!/bin/bash
# 2-GPU A/B of an env toggle on the default bench and on ER theta=64 (all-nn)
VAR=${1:-DBFS_NO_SEND_FILTER}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for args in "" "--graph er --theta 64 --scale 25 --scaling strong --steps 16"; do
for v in ${ORDER:-0 1}; do
  if [ $v = 1 ]; then E="$VAR=1"; else E=""; fi
  env $E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 100)) bench.py --gpus 2 --no-alt-labeling $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$v', d['config']['workload'][:40], d['value'], d['ms_per_step'])"
done; done
