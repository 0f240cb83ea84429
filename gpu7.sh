cd $GRAFT_REPO_ROOT
timeout 600 python dbg4.py 2>&1 | tail -20
