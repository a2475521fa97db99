# correctness first, then per-level profile of both occupancy variants, then the bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
if grep -q "passed" gpurun_out/gpu_tests.log && ! grep -q "failed" gpurun_out/gpu_tests.log; then
  timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/lv_b2.txt 2>&1
  DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_b3.so timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/lv_b3.txt 2>&1
  timeout 300 python tools/level_profile.py 24 1 bfs > gpurun_out/lv_b2_bfs.txt 2>&1
  DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_b3.so timeout 300 python tools/level_profile.py 24 1 bfs > gpurun_out/lv_b3_bfs.txt 2>&1
  cat gpurun_out/lv_b2.txt gpurun_out/lv_b3.txt gpurun_out/lv_b2_bfs.txt gpurun_out/lv_b3_bfs.txt
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
fi
