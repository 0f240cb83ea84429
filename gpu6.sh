cd $GRAFT_REPO_ROOT
timeout 600 python dbg3.py 2>&1 | tail -40
