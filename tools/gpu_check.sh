#!/bin/bash
# GPU-box check used for the round numbers: gpu tests, step ablation, 1-GPU bench.
# usage: gpurun --timeout 1500 -- bash tools/gpu_check.sh
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; tail -1 gpurun_out/pytest_gpu.log; grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head -8
timeout 600 python tools/ablate_step.py 2>&1 | grep -E "^none|all-but|norms|attn"
timeout 300 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_n1.json 2>/dev/null
tail -1 gpurun_out/bench_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['p50_decode_step_ms'], d['prefill_ms'], r['gemm_ms_per_step'], d['e2e']['value'], r['frac'])"
