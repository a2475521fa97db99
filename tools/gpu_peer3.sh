#!/bin/bash
N=${1:-2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "n1 rc=$?"; cat gpurun_out/bench_n1.json
bash tools/gpu_peer2.sh $N
