#!/bin/bash
# results table refresh on a 4-GPU box: BFS strong s26 (1/2/4), ER s28 BFS (2/4), paper setup s27/s28/s29 (1/2/4)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/cfg
run() {  # name N args...
  local name=$1 N=$2; shift 2
  if [ "$N" = 1 ]; then timeout 900 python bench.py --no-cpu-baseline --no-alt-labeling "$@" > gpurun_out/cfg/$name.json 2> gpurun_out/cfg/$name.err
  else timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --no-alt-labeling "$@" > gpurun_out/cfg/$name.json 2> gpurun_out/cfg/$name.err; fi
  echo "$name rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/cfg/$name.json')); print('  ', d['value'], d['e2e']['value'], d['ms_per_step'], d['config']['workload'])" 2>/dev/null
}
run s26_4gpu_peer 4 --steps 64
run bfs_s26_1gpu 1 --mode bfs --scale 26 --scaling strong --steps 16
run bfs_s26_2gpu 2 --mode bfs --scale 26 --scaling strong --steps 16
run bfs_s26_4gpu 4 --mode bfs --scale 26 --scaling strong --steps 16
run er_s28_bfs_2gpu 2 --graph er --mode bfs --scale 28 --scaling strong --theta 64 --steps 16
run er_s28_bfs_4gpu 4 --graph er --mode bfs --scale 28 --scaling strong --theta 64 --steps 16
run s27_1gpu 1 --scale 27 --steps 32
run s28_2gpu 2 --scale 27 --steps 32
run s29_4gpu 4 --scale 27 --steps 32
run er_s24_dobfs_1gpu 1 --graph er --scale 24 --steps 32
run er_s25_dobfs_2gpu 2 --graph er --steps 32
run er_s26_dobfs_4gpu 4 --graph er --steps 32
run er_s24_bfs_1gpu 1 --graph er --mode bfs --scale 24 --steps 16
run er_s25_bfs_2gpu 2 --graph er --mode bfs --steps 16
run er_s26_bfs_4gpu 4 --graph er --mode bfs --steps 16
