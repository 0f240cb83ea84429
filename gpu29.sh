cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "decode" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -2
timeout 600 python tools/ablate_step.py 2>&1 | head -2
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b13.json 2>/dev/null
tail -1 gpurun_out/b13.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], d['prefill_ms'], r['gemm_ms_per_step'])"
