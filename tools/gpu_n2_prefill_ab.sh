#!/bin/bash
# N=2 (70B [1,1]) prefill: persistent prefill GEMM / attention on vs off, one process per setting, same box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/n2ab
for spec in "X=1" "HX_GEMM_PERSISTENT=0" "HX_PREFILL_TC_P=0" "X=1"; do
  env $spec timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/n2ab/b.json 2> gpurun_out/n2ab/b.err
  echo "$spec: $(tail -1 gpurun_out/n2ab/b.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill_ms', d['prefill_ms'], 'value', d['value'], 'e2e', d['e2e']['value'])")"
done
