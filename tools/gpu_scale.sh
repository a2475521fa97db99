cd $GRAFT_REPO_ROOT
timeout 1500 python tools/scale_check.py all 2>&1 | grep -v Warning | tail -20
