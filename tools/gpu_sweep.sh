cd $GRAFT_REPO_ROOT
for lib in paper_1803_03922_b200/libdbfs*.so; do DBFS_LIB=$PWD/$lib timeout 300 python tools/sweep.py 24 2>&1 | tail -1; done
