#!/bin/bash
# default-config bench at N GPUs (weak: 24 + log2 N) and the paper setup (27 + log2 N)
N=${1:-2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "rc=$?"; cat gpurun_out/bench_n$N.json
timeout 1000 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus $N --scale 27 > gpurun_out/weak27_n$N.json 2> gpurun_out/weak27_n$N.err; echo "rc=$?"; cat gpurun_out/weak27_n$N.json
grep -i "error" gpurun_out/bench_n$N.err gpurun_out/weak27_n$N.err | head -5
