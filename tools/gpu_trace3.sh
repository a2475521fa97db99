#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_all.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tests/dist_check_worker.py 17 > gpurun_out/dist17_2.log 2>&1; echo "dist17x2 rc=$?"; grep -E "PASS|FAIL|differ|inconsistent" gpurun_out/dist17_2.log | head -5
rm -f gpurun_out/trace1.txt
DBFS_TRACE=$PWD/gpurun_out/trace1.txt timeout 300 python tools/level_profile.py 24 1 dobfs > gpurun_out/lv_trace.txt 2>&1; echo "lv rc=$?"
python tools/trace_summary.py gpurun_out/trace1.txt 2>/dev/null | tail -8
timeout 600 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "b1 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench1.json')); print(d['value'], d['e2e']['value'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --no-alt-labeling > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "n2 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench2.json')); print(d['value'], d['e2e']['value'])"
