cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --scale 20 --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s20.json 2> gpurun_out/bench_s20.err; echo "s20 rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_s24.json 2> gpurun_out/bench_s24.err; echo "s24 rc=$?"
cat gpurun_out/bench_s20.json gpurun_out/bench_s24.json; tail -5 gpurun_out/bench_s20.err gpurun_out/bench_s24.err
