#!/bin/bash
# BASELINE configs[2] (s26 top-down BFS strong scaling) and configs[4] (ER s28 BFS) at N GPUs
N=${1:-1}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() {  # name, args...
  local name=$1; shift
  if [ "$N" = "1" ]; then
    timeout 900 python bench.py --no-cpu-baseline --no-alt-labeling "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 100)) bench.py --gpus $N --no-alt-labeling "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err
  fi
  echo "$name rc=$?"; python -c "import json,sys; d=json.loads(open('gpurun_out/$name.json').read().strip().splitlines()[-1]); print(d['config']['workload'], d['value'], d['ms_per_step'], d['e2e']['value'], d.get('worker_edges_max_over_mean'))" 2>&1 | tail -1
  grep -i "error" gpurun_out/$name.err | head -3
}
run bfs26_n$N --mode bfs --scale 26 --scaling strong --steps 16
if [ "$N" != "1" ]; then run er28_n$N --graph er --mode bfs --scale 28 --scaling strong --steps 16; fi
run er24_n$N --graph er --mode bfs --scale 24 --scaling weak --steps 16
run er24d_n$N --graph er --mode dobfs --scale 24 --scaling weak --steps 16
