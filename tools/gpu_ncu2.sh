cd $GRAFT_REPO_ROOT
timeout 300 python tools/ncu_levels.py 24 > gpurun_out/ncu2_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_visit -c 7 -o gpurun_out/prof_visit python tools/ncu_levels.py 24 > gpurun_out/ncu2.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu2.log; cat gpurun_out/ncu2_plain.log
