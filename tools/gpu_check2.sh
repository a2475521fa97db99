#!/bin/bash
# 2-GPU box: distributed check (engines, policies, bfs_batch, DPG1 round trip) and the N=2 bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tools/dist_check.py 17 > gpurun_out/dist17_2.log 2>&1; echo "dist17x2 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent|Error" gpurun_out/dist17_2.log | head -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --no-alt-labeling --steps 16 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "n2 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench2.json')); print(d['value'], d['e2e']['value'], d.get('comm'))"; tail -2 gpurun_out/bench2.err
