cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b12.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b12.json')); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], d['prefill_ms'], r['gemm_ms_per_step'])"
timeout 300 python tools/profile_decode.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --nvtx --nvtx-include "decode/" --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_decode6.csv python tools/profile_decode.py > gpurun_out/ncu7.log 2>&1
echo ncu rc=$?
