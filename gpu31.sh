cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dist.py -m gpu -q -rf -k "tp2 or two_stage" > gpurun_out/pytest_dist2.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest_dist2.log; grep -E "FAILED|Error" gpurun_out/pytest_dist2.log | head -5
