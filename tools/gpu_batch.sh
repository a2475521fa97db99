#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_batch.py tests/test_cli.py tests/test_io.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t_batch.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_batch.log
timeout 900 python bench.py --no-cpu-baseline --no-alt-labeling > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "b1 rc=$?"; cat gpurun_out/bench1.json; tail -3 gpurun_out/bench1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --no-alt-labeling > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "b2 rc=$?"; cat gpurun_out/bench2.json; tail -3 gpurun_out/bench2.err
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/dist_levels.py 24 1 peer > gpurun_out/dist_levels_n2.txt 2>&1; echo "rc=$?"
grep "device" gpurun_out/dist_levels_n2.txt
