cd $GRAFT_REPO_ROOT
timeout 600 python tools/level_profile.py 24 3 dobfs > gpurun_out/levels_s24_dobfs.txt 2>&1; echo "rc=$?"
timeout 600 python tools/level_profile.py 24 2 bfs > gpurun_out/levels_s24_bfs.txt 2>&1; echo "rc=$?"
cat gpurun_out/levels_s24_dobfs.txt gpurun_out/levels_s24_bfs.txt
