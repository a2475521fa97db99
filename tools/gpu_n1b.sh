#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final
timeout 900 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err; echo "n1 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/final/bench_n1.json')); print(d['value'], d['e2e'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 > gpurun_out/final/bench_n2.json 2> gpurun_out/final/bench_n2.err; echo "n2 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/final/bench_n2.json')); print(d['value'], d['e2e']['value'])"
