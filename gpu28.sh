cd $GRAFT_REPO_ROOT
timeout 600 python tools/ablate_step.py 2>&1 | tail -8
