cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k linear 2>&1 | tail -1
timeout 300 python tools/gemm_timeline.py --detail 2>&1 | grep -E "mean|total|launch"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b9.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b9.json')); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], r['gemm_ms_per_step'], {k:v['GBps'] for k,v in r['per_shape'].items()})"
