cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_timeline.py --detail 2>&1 | grep -E "launch|slow|fast"
