#!/bin/bash
# A/B of one env knob: kernel test subset, 7B bench and 70B TP=4 / 13B TP=2 shard timelines per setting.
# usage: KNOB=HX_DEFER_QKV VALUES="0 1" TESTS="-k deferred_qkv" gpurun --timeout 1500 -- bash tools/gpu_ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -rf $TESTS > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log; fi
for v in $VALUES; do
  env $KNOB=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${KNOB}_$v.json 2>/dev/null
  tail -1 gpurun_out/ab_${KNOB}_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$KNOB=$v 7B', d['value'], d['p50_decode_step_ms'], d['step_roofline']['frac'])"
  env $KNOB=$v timeout 300 python tools/gemm_timeline.py llama2-70b --tp=4 --layers=20 --full-step > gpurun_out/ab_tl70_${KNOB}_$v.txt 2>&1; echo "$KNOB=$v 70B tp4 shard"; tail -5 gpurun_out/ab_tl70_${KNOB}_$v.txt
done
