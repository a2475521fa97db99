#!/bin/bash
# paper headline setup: RMAT DOBFS weak scaling from scale 27 (1 GPU) -> 27 + log2 N
N=${1:-1}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ "$N" = "1" ]; then
  timeout 900 python bench.py --scale 27 --no-cpu-baseline > gpurun_out/weak27_n1.json 2> gpurun_out/weak27_n1.err; echo "rc=$?"
else
  timeout 1000 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N --scale 27 > gpurun_out/weak27_n$N.json 2> gpurun_out/weak27_n$N.err; echo "rc=$?"
fi
cat gpurun_out/weak27_n$N.json; grep -v "^\*\*\*\|OMP_NUM" gpurun_out/weak27_n$N.err | tail -5
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
