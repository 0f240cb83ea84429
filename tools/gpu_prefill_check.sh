#!/bin/bash
# prefill check: N=2 70B [1,1] and C3 [2,1] (micro-batched), N=1 7B (one-shot)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pfc
for spec in "n2 2" "c3asym 3 --workload c3-asym"; do
  set -- $spec; tag=$1; n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n --steps 2 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/pfc/$tag.json 2> gpurun_out/pfc/$tag.err
  echo "$tag: $(tail -1 gpurun_out/pfc/$tag.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill_ms', d['prefill_ms'], 'value', d['value'], 'e2e', d['e2e']['value'])")"
done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pfc/n1.json 2>/dev/null
echo "n1: $(tail -1 gpurun_out/pfc/n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill_ms', d['prefill_ms'], 'value', d['value'], 'e2e', d['e2e']['value'])")"
