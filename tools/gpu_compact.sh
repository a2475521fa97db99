#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_all.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tools/dist_check.py 17 > gpurun_out/dist17_2.log 2>&1; echo "dist17x2 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent|Error" gpurun_out/dist17_2.log | head -5
timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "b1 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench1.json')); print(d['value'], d['e2e'])"; tail -2 gpurun_out/bench1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --no-alt-labeling > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "n2 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench2.json')); print(d['value'], d['e2e']['value'], d['e2e']['d2h_bytes_per_step'])"; nproc
