#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for t in 1 0 1 0; do
DBFS_F3_DYN=$t timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "f3_dyn=$t rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('   ', d['value'], d['ms_per_step'])"
done
for t in 1 0; do
DBFS_F3_DYN=$t timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --no-alt-labeling --steps 32 > gpurun_out/ab2.json 2> gpurun_out/ab2.err; echo "n2 f3_dyn=$t rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ab2.json')); print('   ', d['value'], d['ms_per_step'])"
done
