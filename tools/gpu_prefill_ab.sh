#!/bin/bash
# Prefill GEMM: persistent (default) vs per-tile kernel (HX_GEMM_PERSISTENT=0), one process per setting.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pf
O=gpurun_out/pf
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -rf -k "linear_bf16 or tcgen05_prefill or two_layers or c2" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
for v in 1 0 1 0; do
  HX_GEMM_PERSISTENT=$v timeout 600 python tools/prefill_gemm_bench.py $SEL > $O/gemm_$v.txt 2>&1; echo "HX_GEMM_PERSISTENT=$v"; cat $O/gemm_$v.txt
done
for v in 1 0; do
  HX_GEMM_PERSISTENT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$v.json 2>/dev/null
  tail -1 $O/bench_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('HX_GEMM_PERSISTENT=$v 7B prefill_ms', d['prefill_ms'], 'e2e', d['e2e']['value'], 'decode', d['value'])"
done
