cd $GRAFT_REPO_ROOT; DBFS_LIB=$PWD/paper_1803_03922_b200/libdbfs_timers.so timeout 300 python tools/variant_profile.py
