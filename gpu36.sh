cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "deferred or norms" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -1
timeout 600 python tools/ablate_step.py 2>&1 | grep -E "none|norms"
