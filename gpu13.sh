cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed|Error|error" | tail -10
HX_ATTN_MMA_MIN_G=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k decode 2>&1 | tail -2
for g in 2 1; do
HX_ATTN_MMA_MIN_G=$g timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_$g.json 2> gpurun_out/bench7_$g.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench7_$g.json')); print('mma min G',$g, d['value'], d['p50_decode_step_ms'], d['prefill_ms'])"
done
