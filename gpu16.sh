cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -1
for c in 1 0; do
HX_MAX_CARVEOUT=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench8_$c.json 2> gpurun_out/bench8_$c.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench8_$c.json')); print('carveout',$c, d['value'], d['p50_decode_step_ms'], d['roofline']['gemm_ms_per_step'], d['roofline']['per_shape'])"
done
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_decode5.csv python tools/profile_decode.py > gpurun_out/ncu6.log 2>&1
echo ncu rc=$?
