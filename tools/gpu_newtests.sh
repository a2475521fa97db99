cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_io.py tests/test_cli.py -m gpu -q -p no:cacheprovider > gpurun_out/gpu_newtests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/gpu_newtests.log
