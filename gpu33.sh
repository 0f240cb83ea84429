cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "linear" 2>&1 | tail -1
timeout 600 python tools/prefill_gemm_bench.py
