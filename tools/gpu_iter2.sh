cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python tools/level_profile.py 24 2 dobfs > gpurun_out/lv.txt 2>&1; cat gpurun_out/lv.txt
timeout 300 python tools/sweep.py 24
