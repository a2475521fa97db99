cd $GRAFT_REPO_ROOT
for lib in paper_1803_03922_b200/libdbfs*.so; do DBFS_LIB=$PWD/$lib timeout 300 python tools/sweep.py 24 2>&1 | tail -1; done
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 300 python tools/level_profile.py 24 1 dobfs 2>&1 | head -20
DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 300 python tools/level_profile.py 24 1 bfs 2>&1 | head -20
