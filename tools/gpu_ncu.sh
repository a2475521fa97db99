cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/lv.txt 2>&1; cat gpurun_out/lv.txt
timeout 300 python tools/ncu_target.py 24 dobfs > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bfs_persistent -s 1 -c 1 -o gpurun_out/prof_bfs python tools/ncu_target.py 24 dobfs > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
