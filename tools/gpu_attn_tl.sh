#!/bin/bash
# decode-attention transition timelines (real context) + parity + 1-GPU bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/atl
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 | tee gpurun_out/atl/pytest.txt
python tools/attn_timeline.py llama2-70b --tp=4 2>&1 | tee gpurun_out/atl/tp4.txt
python tools/attn_timeline.py llama2-70b --tp=2 2>&1 | tee gpurun_out/atl/tp2.txt
python tools/attn_timeline.py llama2-7b 2>&1 | tee gpurun_out/atl/7b.txt
python tools/attn_bench.py 2>&1 | tee gpurun_out/atl/attn_bench.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/atl/bench.json 2> gpurun_out/atl/bench.err
tail -1 gpurun_out/atl/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d.get('p50_step_ms'), d['e2e']['value'], d['roofline']['frac'])"
