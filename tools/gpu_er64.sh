#!/bin/bash
# ER (uniform quadrants) scale 28, Theta = 64 pinned (d ~ 0, all-nn: the record exchange dominates)
N=${1:-2}; S=${2:-28}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for mode in bfs dobfs; do
  name=er${S}t64_${mode}_n$N
  if [ "$N" = "1" ]; then
    timeout 900 python bench.py --no-cpu-baseline --no-alt-labeling --graph er --theta 64 --mode $mode --scale $S --scaling strong --steps 16 > gpurun_out/$name.json 2> gpurun_out/$name.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 100)) bench.py --gpus $N --no-alt-labeling --graph er --theta 64 --mode $mode --scale $S --scaling strong --steps 16 > gpurun_out/$name.json 2> gpurun_out/$name.err
  fi
  echo "$name rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/$name.json').read().strip().splitlines()[-1]); print(d['config']['workload'], d['value'], d['ms_per_step'], d['e2e']['value'], d['graph']['d'], d['graph']['kind_totals'])" 2>&1 | tail -1
  grep -i "error\|certif" gpurun_out/$name.err | head -3
done
