cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_2gpu.log 2>&1; echo rc=$?
grep -E "FAILED|Error|error|assert" gpurun_out/pytest_2gpu.log | head -20
