cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_timeline.py 2>&1 | tail -24
timeout 300 python tools/gemm_timeline.py --full-step 2>&1 | tail -8
