#!/bin/bash
# 1-GPU check: gpu test suite (single-GPU part) + smoke + N=1 bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
O=gpurun_out/c1
timeout 1500 python -m pytest tests -m gpu -q -rfs ${K:+-k "$K"} > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?"
tail -1 $O/bench_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('N=1', d['value'], 'p50', d['p50_decode_step_ms'], 'frac', d['step_roofline']['frac'], 'gemm frac', r['frac'], 'prefill', d['prefill_ms'], 'e2e', d['e2e']['value'])"
