cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b11.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b11.json')); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], r['gemm_ms_per_step'])"
