#!/bin/bash
# persistent tcgen05 prefill attention (default) vs one CTA per item (HX_PREFILL_TC_P=0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pfa
O=gpurun_out/pfa
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -rf -k "prefill_attention_tcgen05 or tcgen05_prefill or two_layers" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for v in 1 0 1 0; do
  HX_PREFILL_TC_P=$v timeout 300 python tools/attn_prefill_bench.py > $O/bench_$v.txt 2>&1; echo "HX_PREFILL_TC_P=$v"; grep "tcgen05 " $O/bench_$v.txt
done
for v in 1 0; do
  HX_PREFILL_TC_P=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/b_$v.json 2> $O/b_$v.err
  tail -1 $O/b_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('HX_PREFILL_TC_P=$v 7B prefill_ms', d['prefill_ms'], 'e2e', d['e2e']['value'])" || tail -3 $O/b_$v.err
done
