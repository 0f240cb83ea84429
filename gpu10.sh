cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "linear" 2>&1 | tail -2
for c in 1 2; do
HX_SK_CTAS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench5_$c.json 2> gpurun_out/bench5_$c.err; echo bench $c rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench5_$c.json')); print('ctas',$c, d['value'], d['p50_decode_step_ms'], d['roofline']['achieved'], d['roofline']['gemm_ms_per_step'])"
done
