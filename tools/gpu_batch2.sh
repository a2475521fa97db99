#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_batch.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_batch.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_batch.log
timeout 900 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "b1 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench1.json')); print(d['value'], d['e2e'])"; tail -3 gpurun_out/bench1.err
