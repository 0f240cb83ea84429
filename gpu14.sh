cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf -k linear 2>&1 | grep -E "FAILED|passed|failed" | tail -10
