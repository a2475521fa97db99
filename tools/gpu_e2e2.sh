#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 0 1 0 1; do
DBFS_COMPACT=$c timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --no-alt-labeling --steps 32 > gpurun_out/s_n2.json 2> gpurun_out/s_n2.err; echo "compact=$c rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/s_n2.json')); print('   ', d['value'], d['e2e']['value'])"
done
