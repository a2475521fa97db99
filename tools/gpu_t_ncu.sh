#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_all.log
timeout 600 python bench.py > gpurun_out/bench_s24.json 2> gpurun_out/bench_s24.err; echo "b rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s24.json')); print(d['value'], d['e2e'], d['roofline'])"
bash tools/gpu_ncu3.sh
