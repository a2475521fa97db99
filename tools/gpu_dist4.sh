cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tools/dist_check.py 18 > gpurun_out/dist18_4.log 2>&1; echo "dist18x4 rc=$?"; grep -E "root|DIST|built" gpurun_out/dist18_4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --steps 16 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench4 rc=$?"; cut -c1-700 gpurun_out/bench_n4.json; tail -3 gpurun_out/bench_n4.err
