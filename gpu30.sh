cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest_full.log; grep FAILED gpurun_out/pytest_full.log | head
